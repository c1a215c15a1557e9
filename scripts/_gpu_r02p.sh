# round-2 call P: compute-sanitizer racecheck (ONE tool per call) over the mbarrier / st.async /
# DSMEM / grid-barrier kernels (scripts/sanitize_kernels.py); summary to gpurun_out/r02p_racecheck.log
mkdir -p gpurun_out
timeout 600 python scripts/sanitize_kernels.py > gpurun_out/r02p_plain.log 2>&1; echo plain_rc=$?
tail -3 gpurun_out/r02p_plain.log
timeout 1500 compute-sanitizer --tool racecheck --racecheck-report all \
  --kernel-name kernel_regex='k_cluster|k_wave2|k_jacobi|k_qr|k_tsqr|k_wy' \
  python scripts/sanitize_kernels.py > gpurun_out/r02p_racecheck.log 2>&1; echo racecheck_rc=$?
tail -25 gpurun_out/r02p_racecheck.log
