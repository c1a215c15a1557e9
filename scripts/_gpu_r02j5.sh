# round-2 session-5: final full GPU suite + default bench line
python -m pytest tests -m gpu -x -q --durations=10 > gpurun_out/r02j_gpu_suite.log 2>&1; echo suite rc=$?
tail -3 gpurun_out/r02j_gpu_suite.log
python bench.py > gpurun_out/r02j_bench.json 2> gpurun_out/r02j_bench.err; echo bench rc=$?
tail -c 400 gpurun_out/r02j_bench.json
