for i in 1 2 3; do timeout 600 python -m pytest tests/test_gpu_sharded.py tests/test_gpu_pml.py -q -rf -x -k "sharded or world or loopback" 2>&1 | tail -2; echo "run $i rc=$?"; done
