mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_configs.py -q -s -rA > gpurun_out/r02b_tests.log 2>&1; echo tests_rc=$?
grep -E "iterate energy|error-table|passed|failed|Error" gpurun_out/r02b_tests.log | head -30
