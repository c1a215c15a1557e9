# round-2 session-5: full GPU suite + default bench line
python -m pytest tests -m gpu -x -q --durations=15 > gpurun_out/r02d_gpu_suite.log 2>&1; echo suite rc=$?
tail -4 gpurun_out/r02d_gpu_suite.log
python bench.py > gpurun_out/r02d_bench.json 2> gpurun_out/r02d_bench.err; echo bench rc=$?
tail -c 600 gpurun_out/r02d_bench.json
