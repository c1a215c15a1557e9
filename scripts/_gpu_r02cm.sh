# round-2 session-5 call M: phase timeline of theta parareal with the layer on config 4
PTB_PROF=1 python scripts/time_pml_theta.py 3 2>&1 | grep -v "jacobi\|qr2\|svd:\|update" | tail -30
