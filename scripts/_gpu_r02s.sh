# round-2 call S: theta-PML with uncorrected auxiliary fields + the k_wave2 interior of the PML pass
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_pml.py -q -rf > gpurun_out/r02s_tests.log 2>&1; echo tests_rc=$?
tail -6 gpurun_out/r02s_tests.log
for w in 1 0; do
PTB_PML_WAVE=$w timeout 1500 python bench.py --no-sweep --no-parareal --no-cpu --no-e2e --steps 3 > gpurun_out/r02s_bench_w$w.json 2> gpurun_out/r02s_bench_w$w.err; echo bench_rc=$?
python - $w <<'PY'
import json,sys
d=json.loads(open(f'gpurun_out/r02s_bench_w{sys.argv[1]}.json').read().splitlines()[-1])
print(sys.argv[1], json.dumps(d.get('cfg4_pml')))
PY
done
