# round-2 session-5 call AC: k_nan_where per slice with early exit: driver tests + cfg3/cfg4 timing
python -m pytest tests/test_gpu_path.py tests/test_gpu_sharded.py tests/test_gpu_golden.py -x -q 2>&1 | tail -3
python scripts/time_driver.py 3 4 2>&1 | python -c "
import sys, json
for l in sys.stdin:
    try: d = json.loads(l)
    except Exception: continue
    print(d['cfg'], 'iteration_ms', d['iteration_ms'], 'parallel_ms', d['parallel_ms'][-3:], 'sweep', d['sweep_ms'][-3:], 'fin', d['finalize_ms'][-3:])
"
