# round-2 session-5 call R: theta-with-layer full PTB_PROF timeline with band streams (K = 4), twice
for i in 1 2; do PTB_PROF=1 python scripts/time_pml_theta.py 4 2>&1 | grep -v "jacobi " | tail -75 > gpurun_out/r02cr_$i.log; tail -1 gpurun_out/r02cr_$i.log; done
