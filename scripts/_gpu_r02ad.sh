timeout 1500 python -m pytest tests/test_gpu_sharded.py -q -rf -x 2>&1 | tail -30
