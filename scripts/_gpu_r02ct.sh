# round-2 session-5 call T: do the sporadic iteration stalls come from lazy module loading?
for i in 1 2 3; do echo "EAGER $(CUDA_MODULE_LOADING=EAGER python scripts/time_pml_theta.py 6 2>&1 | tail -1)"; done
for i in 1 2; do echo "LAZY  $(python scripts/time_pml_theta.py 6 2>&1 | tail -1)"; done
