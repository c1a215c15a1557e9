# round-2 call M: bulk-copy k_wave2 ring + theta with the absorbing layer (parity), A/B vs the
# cp.async ring on the cfg5 sweep, hand-written DGEMM vs cuBLAS DMMA on the corrector shapes
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_pml.py tests/test_gpu_bench_plans.py tests/test_gpu_propagator.py tests/test_gpu_fullrow.py -q -x -rf --durations=25 > gpurun_out/r02m_tests.log 2>&1; echo tests_rc=$?
tail -40 gpurun_out/r02m_tests.log
for v in bulk cpasync; do
  if [ $v = cpasync ]; then export PTB_LIB=$PWD/paratime_b200/_ab/libparatime_b200_cpasync.so; fi
  timeout 900 python bench.py --no-parareal --no-pml --no-cpu --no-e2e --steps 5 > gpurun_out/r02m_bench_$v.json 2> gpurun_out/r02m_bench_$v.err; echo bench_$v=$?
  python - $v <<'PY'
import json,sys
d=json.loads(open(f'gpurun_out/r02m_bench_{sys.argv[1]}.json').read().splitlines()[-1])
print(sys.argv[1], d['value'], d['roofline']['frac'], d.get('parity'))
for r in d.get('cfg5_sweep',[]): print('  ', r['grid'], r['batch'], '%.3e'%r['updates_per_s'], round(r['frac_binding'],3), r['plan'])
PY
done
unset PTB_LIB
timeout 600 python scripts/ubench_dgemm.py > gpurun_out/r02m_dgemm.jsonl 2>&1; echo dgemm=$?
cat gpurun_out/r02m_dgemm.jsonl
