# round-2 GPU call A: new parity tests, bench line, sanitizer
mkdir -p gpurun_out
nvidia-smi --query-gpu=clocks.sm,clocks.max.sm,power.draw --format=csv
timeout 1500 python -m pytest tests/test_gpu_bench_plans.py tests/test_gpu_configs.py -x -q -rA > gpurun_out/r02a_tests.log 2>&1; echo tests_rc=$?
tail -30 gpurun_out/r02a_tests.log
timeout 900 python bench.py > gpurun_out/r02a_bench.json 2> gpurun_out/r02a_bench.err; echo bench_rc=$?
tail -c 600 gpurun_out/r02a_bench.err
python -c "import json;d=json.loads(open('gpurun_out/r02a_bench.json').read().splitlines()[-1]);print({k:d[k] for k in ('value','ms_per_step','parity','e2e') if k in d}); print(d['roofline']['kernel'], d['roofline']['frac']); print({k:v for k,v in d.items() if k.startswith('s_per')})"
