# round-2 session-5 call AA: out-of-place layered fine stage (no state copy): PML tests + theta timing
python -m pytest tests/test_gpu_pml.py -x -q 2>&1 | tail -3
python scripts/time_pml_theta.py 6 2>&1 | tail -1
