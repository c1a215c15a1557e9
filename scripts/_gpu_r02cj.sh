# round-2 session-5 call J: launch lists of the cfg1 and cfg2 drivers
bash scripts/driver_launches.sh 1 gpurun_out/r02cj_cfg1.csv
bash scripts/driver_launches.sh 2 gpurun_out/r02cj_cfg2.csv
python scripts/launch_table.py gpurun_out/r02cj_cfg1.csv 40 > gpurun_out/r02cj_cfg1.md
python scripts/launch_table.py gpurun_out/r02cj_cfg2.csv 40 > gpurun_out/r02cj_cfg2.md
