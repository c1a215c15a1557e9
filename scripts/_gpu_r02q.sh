# round-2 call Q: k_wave2 register-prefetch variants (4, 5) vs the cp.async ring (0); DGEMM after the
# staging fix + transposed short-m route; Procrustes timeline (PTB_PROF) on configs 1 and 4
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_gemm.py -q -x 2>&1 | tail -2
timeout 600 python scripts/ubench_dgemm.py > gpurun_out/r02q_dgemm.jsonl 2>&1; echo dgemm=$?
cat gpurun_out/r02q_dgemm.jsonl
for v in 0 4 5; do
  if [ $v != 0 ]; then export PTB_LIB=$PWD/paratime_b200/_ab/libparatime_b200_ring$v.so; fi
  timeout 900 python bench.py --no-parareal --no-pml --no-cpu --no-e2e --steps 5 > gpurun_out/r02q_bench_ring$v.json 2> gpurun_out/r02q_bench_ring$v.err; echo bench_ring$v=$?
  python - $v <<'PY'
import json,sys
d=json.loads(open(f'gpurun_out/r02q_bench_ring{sys.argv[1]}.json').read().splitlines()[-1])
print('ring', sys.argv[1], '%.3e' % d['value'], round(d['roofline']['frac'], 3), d.get('parity',{}).get('ok'))
for r in d.get('cfg5_sweep',[]): print('  ', r['grid'], r['batch'], '%.3e'%r['updates_per_s'], round(r['frac_binding'],3), r['plan'])
PY
done
unset PTB_LIB
PTB_PROF=1 timeout 900 python scripts/time_driver.py 1:3 4:3 > gpurun_out/r02q_prof.log 2>&1; echo prof=$?
grep -v "^\[ptb prof\] finalize\|combine" gpurun_out/r02q_prof.log | tail -120
