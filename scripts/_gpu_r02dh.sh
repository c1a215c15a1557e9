# round-2 session-5 call AH: reserved rank-sized buffers incl. the Lambda-dagger planes: PML tests + 6 cold theta runs
python -m pytest tests/test_gpu_pml.py -x -q 2>&1 | tail -2
for i in 1 2 3 4 5 6; do python scripts/time_pml_theta.py 8 2>&1 | tail -1; done
