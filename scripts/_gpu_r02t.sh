# round-2 call T: ncu evidence — launch lists of the cfg4 (K=2) and cfg3 drivers, one --set full
# capture of the headline kernel (k_wave2, 4096^2 x 64) and of the DMMA GEMM
mkdir -p gpurun_out
python scripts/time_driver.py 4:2 > gpurun_out/r02t_plain4.log 2>&1 && \
  timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02t_cfg4_launches.csv python scripts/time_driver.py 4:2 > /dev/null 2>&1; echo ncu4=$?
python scripts/time_driver.py 3 > gpurun_out/r02t_plain3.log 2>&1 && \
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02t_cfg3_launches.csv python scripts/time_driver.py 3 > /dev/null 2>&1; echo ncu3=$?
python scripts/prof_prop.py 4096 64 1 > gpurun_out/r02t_plainK1.log 2>&1 && \
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_wave2 -s 8 -c 1 -o gpurun_out/r02t_k1 python scripts/prof_prop.py 4096 64 1 > gpurun_out/r02t_ncuK1.log 2>&1; echo ncuK1=$?
python scripts/ubench_dgemm.py > gpurun_out/r02t_plaingemm.log 2>&1 && \
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_dgemm_mma -s 2 -c 1 -o gpurun_out/r02t_dmma python scripts/ubench_dgemm.py > gpurun_out/r02t_ncugemm.log 2>&1; echo ncugemm=$?
python scripts/launch_table.py gpurun_out/r02t_cfg4_launches.csv 25
python scripts/launch_table.py gpurun_out/r02t_cfg3_launches.csv 25
