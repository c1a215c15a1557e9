# round-2 session-5 call AI: periodic theta driver reserves its rank-sized buffers: driver tests + cold cfg4 runs
python -m pytest tests/test_gpu_path.py tests/test_gpu_configs.py tests/test_gpu_sharded.py -x -q 2>&1 | tail -2
for i in 1 2 3; do python scripts/time_driver.py 4 2>&1 | python -c "
import sys, json
for l in sys.stdin:
    try: d = json.loads(l)
    except Exception: continue
    print(d['cfg'], 'iteration_ms', d['iteration_ms'])
"; done
