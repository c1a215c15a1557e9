# round-2 call X: ncu of the Fourier y pass (config 4 combine shape) and of the PML layer kernel
mkdir -p gpurun_out
python scripts/prof_fft_y.py 16 > gpurun_out/r02x_plain_ffty.log 2>&1 && cat gpurun_out/r02x_plain_ffty.log && \
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_fourier_fft_y -s 4 -c 1 -o gpurun_out/r02x_ffty python scripts/prof_fft_y.py 16 > gpurun_out/r02x_ncu1.log 2>&1; echo ncu1=$?
python scripts/time_pml.py > gpurun_out/r02x_plain_pml.log 2>&1 && tail -3 gpurun_out/r02x_plain_pml.log && \
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_pml -s 2 -c 1 -o gpurun_out/r02x_pml python scripts/time_pml.py > gpurun_out/r02x_ncu2.log 2>&1; echo ncu2=$?
