mkdir -p gpurun_out
python scripts/prof_fft_y.py 16; python scripts/prof_fft_y.py 16
timeout 600 python -m pytest tests/test_gpu_propagator.py -q -x -k transfer 2>&1 | tail -2
timeout 900 python scripts/time_driver.py 4:2 4:2 2>&1 | tail -1 | python -c "
import json,sys
for l in sys.stdin:
    d=json.loads(l); print(d['cfg'], 'it', d['iteration_ms'], 'fin', d['finalize_ms'])"
