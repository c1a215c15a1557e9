# round-2 session-5 call S: theta-with-layer iteration times, band streams on/off, 3 runs each (K = 6)
for L in 1 0 1 0 1 0; do echo "LANES=$L $(PTB_PML_LANES=$L python scripts/time_pml_theta.py 6 2>&1 | tail -1)"; done
