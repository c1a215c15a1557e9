# round-2 session-5 call X: ring refill issued at the end of the iteration (A/B build) vs the product
for L in "" paratime_b200/_ab/libparatime_b200_late.so; do
  echo "== PTB_LIB=$L"
  for c in "4096 64 3" "2048 64 3" "1024 64 5" "512 64 8" "512 512 3" "256 64 10"; do
    PTB_LIB=$L python scripts/prof_prop.py $c
  done
done
