# round-2 call N: theta-PML + DGEMM (DMMA/DFMA) tests, DGEMM micro-benchmark, k_wave2 ring variants 0-3
# on the cfg5 sweep, parareal phase times with the DMMA and DFMA GEMMs
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_pml.py tests/test_gpu_gemm.py -q -x -rf --durations=10 > gpurun_out/r02n_tests.log 2>&1; echo tests_rc=$?
tail -15 gpurun_out/r02n_tests.log
timeout 600 python scripts/ubench_dgemm.py > gpurun_out/r02n_dgemm.jsonl 2>&1; echo dgemm=$?
cat gpurun_out/r02n_dgemm.jsonl
for v in 0 1 2 3; do
  if [ $v != 0 ]; then export PTB_LIB=$PWD/paratime_b200/_ab/libparatime_b200_ring$v.so; fi
  timeout 900 python bench.py --no-parareal --no-pml --no-cpu --no-e2e --steps 5 > gpurun_out/r02n_bench_ring$v.json 2> gpurun_out/r02n_bench_ring$v.err; echo bench_ring$v=$?
  python - $v <<'PY'
import json,sys
d=json.loads(open(f'gpurun_out/r02n_bench_ring{sys.argv[1]}.json').read().splitlines()[-1])
print('ring', sys.argv[1], '%.3e' % d['value'], round(d['roofline']['frac'], 3))
for r in d.get('cfg5_sweep',[]): print('  ', r['grid'], r['batch'], '%.3e'%r['updates_per_s'], round(r['frac_binding'],3), r['plan'])
PY
done
unset PTB_LIB
for g in dmma dfma; do
  echo "== PTB_DGEMM=$g"; PTB_DGEMM=$g timeout 900 python scripts/time_driver.py 3 4 2>&1 | tail -4
done
