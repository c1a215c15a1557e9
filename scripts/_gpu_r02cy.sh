# round-2 session-5 call Y: lane chunk size (PTB_SCRATCH_MIB) on the large-batch cfg5 points
for M in 16384 4096 2048 1024 512; do
  echo "== PTB_SCRATCH_MIB=$M"
  for c in "1024 512 3" "512 512 3" "2048 128 3" "256 512 5"; do
    PTB_SCRATCH_MIB=$M python scripts/prof_prop.py $c
  done
done
