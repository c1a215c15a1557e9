# round-2 session-5 call O: launch list of theta-with-layer iterations (serial reference skipped)
ncu --metrics gpu__time_duration.sum --clock-control none --launch-skip 24500 -c 8000 --csv --log-file gpurun_out/r02co_pml_theta.csv python scripts/time_pml_theta.py 2 > /dev/null 2>&1
python scripts/launch_table.py gpurun_out/r02co_pml_theta.csv 45 > gpurun_out/r02co_pml_theta.md
