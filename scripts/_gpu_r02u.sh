# round-2 call U: two-panel TSQR, streaming pair sums, prefetching Fourier y pass — parity + timing
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_qr.py tests/test_gpu_path.py tests/test_gpu_configs.py tests/test_gpu_propagator.py tests/test_gpu_golden.py tests/test_gpu_race_stress.py -q -x -rf --durations=5 > gpurun_out/r02u_tests.log 2>&1; echo tests_rc=$?
tail -12 gpurun_out/r02u_tests.log
timeout 900 python scripts/time_driver.py 3 3 4:3 4:3 2>&1 | tail -3 | python -c "
import json,sys
for l in sys.stdin:
    d=json.loads(l); print(d['cfg'], 'it', d['iteration_ms'], 'proc', d['procrustes_ms'], 'sweep', d['sweep_ms'], 'fin', d['finalize_ms'], 'par', d['parallel_ms'])"
python scripts/time_driver.py 4:2 > /dev/null 2>&1 && timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02u_cfg4_launches.csv python scripts/time_driver.py 4:2 > /dev/null 2>&1; echo ncu=$?
python scripts/launch_table.py gpurun_out/r02u_cfg4_launches.csv 16
