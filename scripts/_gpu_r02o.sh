# round-2 call O: the full GPU suite with per-test durations (round-1 suite + round-2 additions)
mkdir -p gpurun_out
timeout 3300 python -m pytest tests -q -m gpu -rf --timeout=1200 --durations=60 > gpurun_out/r02o_tests.log 2>&1; echo tests_rc=$?
tail -75 gpurun_out/r02o_tests.log
