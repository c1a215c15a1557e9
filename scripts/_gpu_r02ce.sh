# round-2 session-5 call E: host timeline (PTB_PROF=1) of the cfg4 and cfg3 iterations
PTB_PROF=1 python scripts/time_driver.py 4:2 2>&1 | grep -v "^\[ptb prof\] jacobi" | tail -80
echo ==== cfg3
PTB_PROF=1 python scripts/time_driver.py 3:2 2>&1 | grep -v "^\[ptb prof\] jacobi" | tail -60
