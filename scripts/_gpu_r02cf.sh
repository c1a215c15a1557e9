# round-2 session-5 call F: per-grid ncu counters of the fine propagator (cfg5 grids, batch 64, FAST)
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active,l1tex__throughput.avg.pct_of_peak_sustained_active,l1tex__data_pipe_lsu_wavefronts_mem_shared.sum,sm__warps_active.avg.pct_of_peak_sustained_active,smsp__issue_active.avg.pct_of_peak_sustained_active,gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed,launch__registers_per_thread,launch__grid_size,launch__block_size,smsp__inst_executed.sum
for g in 128 256 512 1024 2048 4096; do
  skip=8; [ $g = 128 ] && skip=1
  ncu --metrics $M --clock-control none -k regex:'k_wave2|k_cluster' -s $skip -c 1 --csv --log-file gpurun_out/r02cf_k1_$g.csv python scripts/prof_prop.py $g 64 2 > gpurun_out/r02cf_$g.log 2>&1
  tail -1 gpurun_out/r02cf_$g.log
done
