# round-2 session-5 call V: sporadic stalls — cold vs warm buffers (the driver run 3 times in one process), 2 processes
for i in 1 2; do echo "== process $i"; python scripts/time_pml_theta.py 6 3 2>&1 | tail -3; done
