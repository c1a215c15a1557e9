# round-2 session-5 call A: PML band tiles on the lane stream (overlap with the interior wavefront) A/B + PML tests
for L in 0 1; do
  echo "== PTB_PML_LANES=$L"
  PTB_PML_LANES=$L python scripts/time_pml.py
done
python -m pytest tests/test_gpu_pml.py -x -q 2>&1 | tail -5
