# round-2 session-5 call U: which PTB_PROF mark absorbs the sporadic stalls (5 runs, marks > 60 ms)
for i in 1 2 3 4 5; do echo "== run $i"; PTB_PROF=1 python scripts/time_pml_theta.py 5 2>&1 | grep -v "jacobi " | awk '/ptb prof/ && $(NF-1)+0 > 60 && !/parallel stage/ {print} /iteration_ms/ {print}'; done
