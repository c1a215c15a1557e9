# round-2 session-5 call AF: buffers reserved at driver start: PML tests + 4 cold theta runs (stalls?) + remaining slow allocations
python -m pytest tests/test_gpu_pml.py -x -q 2>&1 | tail -2
for i in 1 2 3 4; do python scripts/time_pml_theta.py 8 2>&1 | tail -1; done
PTB_PROF=1 python scripts/time_pml_theta.py 8 2>&1 | awk '/DeviceBuffer/ && $(NF-1)+0 > 20 {print}' | tail
