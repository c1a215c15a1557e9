mkdir -p gpurun_out
timeout 2400 python -m pytest tests -q -m gpu > gpurun_out/r02g_tests.log 2>&1; echo tests_rc=$?
tail -15 gpurun_out/r02g_tests.log
timeout 900 python bench.py --no-sweep > gpurun_out/r02g_bench.json 2> gpurun_out/r02g_bench.err; echo bench_rc=$?
tail -c 400 gpurun_out/r02g_bench.err
python - <<'PY'
import json
d=json.loads(open('gpurun_out/r02g_bench.json').read().splitlines()[-1])
print({k:d[k] for k in ('value','ms_per_step','parity') if k in d}); print(d['roofline']['kernel'], d['roofline']['frac'])
print({k:v for k,v in d.items() if k.startswith('s_per')})
for k,v in d['parareal'].items(): print(k, v['phase_ms_median'], v['final_energy_error'])
print(d.get('cpu_baseline_parareal')); print(d.get('cfg4_pml'))
PY
