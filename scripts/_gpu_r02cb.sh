# round-2 session-5 call B: PML layer kernel with the per-pass 1/(1+hd sg) plane; PML tests
python scripts/time_pml.py
python -m pytest tests/test_gpu_pml.py -x -q 2>&1 | tail -5
