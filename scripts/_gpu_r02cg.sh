# round-2 session-5 call G: host timeline of cfg4's two-panel QR (PTB_PROF=1), 3 iterations
PTB_PROF=1 python scripts/time_driver.py 4:3 2>&1 | grep -v "^\[ptb prof\] jacobi" | tail -60
