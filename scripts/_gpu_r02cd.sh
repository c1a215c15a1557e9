# round-2 session-5 call D: PML super-pass (8-step interior + two 4-step band passes) A/B + PML tests
for L in 0 1; do
  echo "== PTB_PML_SUPER=$L"
  PTB_PML_SUPER=$L python scripts/time_pml.py
done
python -m pytest tests/test_gpu_pml.py -x -q 2>&1 | tail -8
