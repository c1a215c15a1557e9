mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_gemm.py tests/test_gpu_qr.py tests/test_gpu_propagator.py -q -x -k "gemm or qr or transfer" 2>&1 | tail -3
timeout 600 python scripts/ubench_dgemm.py 2>&1 | tail -6
timeout 600 python scripts/time_driver.py 3 4:2 2>&1 | tail -2
timeout 1500 bash scripts/driver_launches.sh 4:2 gpurun_out/r02i_cfg4_launches.csv; echo ncu4=$?
timeout 900 bash scripts/driver_launches.sh 3 gpurun_out/r02i_cfg3_launches.csv; echo ncu3=$?
