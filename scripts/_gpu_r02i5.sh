# round-2 session-5: last full GPU suite + smoke of the round (after the theta clamp-check change)
python -m pytest tests -m gpu -x -q --durations=5 > gpurun_out/r02i_gpu_suite.log 2>&1; echo suite rc=$?
tail -3 gpurun_out/r02i_gpu_suite.log
python __graft_entry__.py smoke 2>&1 | tail -1
python bench.py --no-sweep --no-cpu --steps 3 --e2e-steps 1 > gpurun_out/r02i_bench_short.json 2> gpurun_out/r02i_bench_short.err; echo bench rc=$?
tail -c 300 gpurun_out/r02i_bench_short.json
