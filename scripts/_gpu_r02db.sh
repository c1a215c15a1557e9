# round-2 session-5 call AB: periodic driver's fine stage reads cur directly (no state copy): driver tests + timing
python -m pytest tests/test_gpu_path.py tests/test_gpu_configs.py tests/test_gpu_sharded.py tests/test_gpu_refsuite.py tests/test_gpu_golden.py -x -q 2>&1 | tail -3
python scripts/time_driver.py 3 4 2>&1 | python -c "
import sys, json
for l in sys.stdin:
    try: d = json.loads(l)
    except Exception: continue
    print(d['cfg'], 'iteration_ms', d['iteration_ms'], 'parallel_ms', d['parallel_ms'])
"
