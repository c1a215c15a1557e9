mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_sharded.py tests/test_gpu_gemm.py -q -x 2>&1 | tail -3
timeout 600 python scripts/time_driver.py 3 4:2 2>&1 | tail -2
timeout 1500 bash scripts/driver_launches.sh 4:2 gpurun_out/r02h_cfg4_launches.csv; echo ncu4=$?
timeout 900 bash scripts/driver_launches.sh 3 gpurun_out/r02h_cfg3_launches.csv; echo ncu3=$?
