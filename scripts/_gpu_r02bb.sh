# round-2 session-4 call B: cfg3/cfg4 phase timings with the two-lane K1 + Procrustes host timeline
mkdir -p gpurun_out
python scripts/time_driver.py 3 4
PTB_PROF=1 python scripts/time_driver.py 4:4 2>&1 | tail -150
