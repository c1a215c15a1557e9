# round-2 session-5 call AG: what still stalls at iteration 5 (PTB_PROF: slow allocations and marks > 60 ms)
for i in 1 2 3 4; do echo "== run $i"; PTB_PROF=1 python scripts/time_pml_theta.py 6 2>&1 | grep -v "jacobi " | awk '/DeviceBuffer/ {print} /ptb prof/ && !/DeviceBuffer/ && $(NF-1)+0 > 60 && !/parallel stage/ {print} /iteration_ms/ {print}' | tail -14; done
