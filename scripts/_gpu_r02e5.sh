# round-2 session-5: full GPU suite after the paired two-panel QR + smoke
python -m pytest tests -m gpu -x -q --durations=10 > gpurun_out/r02e_gpu_suite.log 2>&1; echo suite rc=$?
tail -4 gpurun_out/r02e_gpu_suite.log
python __graft_entry__.py smoke 2>&1 | tail -2
