# round-2 session-5 call Q: theta-with-layer phase timeline, band streams on/off
for L in 1 0; do echo "== PTB_PML_LANES=$L"; PTB_PML_LANES=$L PTB_PROF=1 python scripts/time_pml_theta.py 3 2>&1 | grep "pml theta\|iteration_ms" | tail -7; done
