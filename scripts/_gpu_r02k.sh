mkdir -p gpurun_out
timeout 900 ncu --set full --import-source on -k regex:k_dgemm --launch-skip 2 --launch-count 1 -o gpurun_out/r02_gemm_nn python scripts/ubench_dgemm.py > gpurun_out/r02k.log 2>&1; echo rc=$?
tail -3 gpurun_out/r02k.log
