# round-2 call AA: row-sharded update_svd — loopback worlds 2/3/4 bitwise, config parity, timing
mkdir -p gpurun_out
timeout 1800 python -m pytest tests/test_gpu_sharded.py tests/test_gpu_configs.py tests/test_gpu_path.py tests/test_gpu_qr.py tests/test_gpu_race_stress.py -q -x -rf --durations=5 > gpurun_out/r02aa_tests.log 2>&1; echo tests_rc=$?
tail -12 gpurun_out/r02aa_tests.log
timeout 900 python scripts/time_driver.py 2 2 3 3 4:3 4:3 2>&1 | python -c "
import json,sys
rows=[json.loads(l) for l in sys.stdin if l.startswith('{')]
for d in rows[1::2]: print(d['cfg'], 'it', d['iteration_ms'], 'proc', d['procrustes_ms'], 'sweep', d['sweep_ms'], 'fin', d['finalize_ms'])"
