# round-2 session-4 call A: two-lane chunk loop + bulk ring on W=256 full-row strips: parity + A/B timing
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_propagator.py tests/test_gpu_fullrow.py tests/test_gpu_bench_plans.py tests/test_gpu_pml.py -q -x -rf 2>&1 | tail -3
for L in 1 0; do
  echo "== PTB_LANES=$L"
  PTB_LANES=$L python scripts/prof_prop.py 4096 512 2
  PTB_LANES=$L python scripts/prof_prop.py 4096 64 3
  PTB_LANES=$L python scripts/prof_prop.py 2048 128 3
  PTB_LANES=$L python scripts/prof_prop.py 2048 64 3
  PTB_LANES=$L python scripts/prof_prop.py 1024 64 5
done
echo "== lanes + DIV=2"
PTB_WAVE_DIV=2 python scripts/prof_prop.py 4096 512 2
PTB_WAVE_DIV=2 python scripts/prof_prop.py 2048 128 3
echo "== lanes from 2^24 points"
PTB_LANE_MIN_POINTS=16777216 python scripts/prof_prop.py 1024 64 5
PTB_LANE_MIN_POINTS=16777216 python scripts/prof_prop.py 512 64 5
PTB_LANE_MIN_POINTS=4194304 python scripts/prof_prop.py 512 64 5
PTB_LANE_MIN_POINTS=4194304 python scripts/prof_prop.py 256 64 5
python scripts/prof_prop.py 512 64 5
python scripts/prof_prop.py 256 64 5
