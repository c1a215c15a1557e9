# round-2 session-4 call E: lane-aware row blocks: parity + cfg5 sweep through the bench
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_propagator.py tests/test_gpu_fullrow.py tests/test_gpu_bench_plans.py -q -x -rf 2>&1 | tail -3
timeout 1200 python bench.py --no-e2e --no-parareal --no-pml --no-cpu --steps 3 > gpurun_out/r02be_bench.json 2> gpurun_out/r02be_bench.err; echo rc=$?
python - <<'PY'
import json
d=json.loads(open('gpurun_out/r02be_bench.json').read().strip().splitlines()[-1])
print(d['value'], d['roofline']['frac'], d['roofline']['kernel'])
for s in d['cfg5_sweep']: print(s['grid'], s['batch'], round(s['updates_per_s']/1e9), round(s['frac_binding'],3), s['plan'])
PY
python scripts/time_driver.py 3 | cut -c1-400
