# round-2 session-5 call N: theta with the layer: px/py combine skipped; PML tests; launch list of 2 iterations
python -m pytest tests/test_gpu_pml.py -x -q 2>&1 | tail -3
python scripts/time_pml_theta.py 4 2>&1 | tail -1
ncu --metrics gpu__time_duration.sum --clock-control none -c 12000 --csv --log-file gpurun_out/r02cn_pml_theta.csv python scripts/time_pml_theta.py 2 > /dev/null 2>&1
python scripts/launch_table.py gpurun_out/r02cn_pml_theta.csv 45 > gpurun_out/r02cn_pml_theta.md
