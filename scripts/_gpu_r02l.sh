# round-2 re-entry: full GPU suite + default bench line at HEAD
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv
timeout 2400 python -m pytest tests -q -m gpu -rf > gpurun_out/r02l_tests.log 2>&1; echo tests_rc=$?
tail -15 gpurun_out/r02l_tests.log
timeout 1200 python bench.py > gpurun_out/r02l_bench.json 2> gpurun_out/r02l_bench.err; echo bench_rc=$?
tail -c 600 gpurun_out/r02l_bench.err
python - <<'PY'
import json
d=json.loads(open('gpurun_out/r02l_bench.json').read().splitlines()[-1])
print({k:d[k] for k in ('value','ms_per_step','parity','e2e','clocks') if k in d}); print(d['roofline'])
print({k:v for k,v in d.items() if k.startswith('s_per')})
for k,v in d.get('parareal',{}).items(): print(k, v.get('phase_ms_median'), v.get('final_energy_error'))
print(d.get('cfg5_sweep'))
print(d.get('cfg4_pml'))
PY
