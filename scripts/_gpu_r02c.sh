mkdir -p gpurun_out
timeout 900 python scripts/diag_procrustes.py 3 3 > gpurun_out/r02c_diag3.log 2>&1; echo rc=$?
tail -8 gpurun_out/r02c_diag3.log
timeout 900 python scripts/diag_procrustes.py 2 3 > gpurun_out/r02c_diag2.log 2>&1; echo rc=$?
tail -5 gpurun_out/r02c_diag2.log
