timeout 900 python -m pytest tests/test_gpu_gemm.py -q -x 2>&1 | tail -2
timeout 600 python scripts/ubench_dgemm.py 2>&1 | tail -6
