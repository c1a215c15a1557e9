# round-2 session-5 call P: frame path band kernels on two streams: PML tests + theta timing
python -m pytest tests/test_gpu_pml.py -x -q 2>&1 | tail -3
python scripts/time_pml_theta.py 4 2>&1 | tail -1
python scripts/time_pml.py 2>&1 | tail -4
