# round-2 call R: race stress tests, the default bench line (theta-PML section included)
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_race_stress.py tests/test_gpu_pml.py -q -rf --durations=8 > gpurun_out/r02r_tests.log 2>&1; echo tests_rc=$?
tail -14 gpurun_out/r02r_tests.log
timeout 1500 python bench.py > gpurun_out/r02r_bench.json 2> gpurun_out/r02r_bench.err; echo bench_rc=$?
tail -c 400 gpurun_out/r02r_bench.err
python - <<'PY'
import json
d=json.loads(open('gpurun_out/r02r_bench.json').read().splitlines()[-1])
print({k:d[k] for k in ('value','ms_per_step','e2e','clocks') if k in d}); print(d['roofline']['frac'], d['roofline']['fp64']['frac'])
print({k:v for k,v in d.items() if k.startswith('s_per')})
for k,v in d.get('parareal',{}).items(): print(k, v.get('phase_ms_median'))
print(d.get('cfg4_pml'))
print(d.get('cpu_baseline')); print(d.get('cpu_baseline_parareal'))
PY
