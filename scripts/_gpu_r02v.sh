# round-2 call V: fused one-GPU large-corrector sweep step (bitwise vs the sharded path) + timing
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_sharded.py tests/test_gpu_configs.py -q -x -rf > gpurun_out/r02v_tests.log 2>&1; echo tests_rc=$?
tail -4 gpurun_out/r02v_tests.log
timeout 900 python scripts/time_driver.py 4:3 4:3 2>&1 | tail -1 | python -c "
import json,sys
for l in sys.stdin:
    d=json.loads(l); print(d['cfg'], 'it', d['iteration_ms'], 'proc', d['procrustes_ms'], 'sweep', d['sweep_ms'], 'fin', d['finalize_ms'], 'par', d['parallel_ms'])"
