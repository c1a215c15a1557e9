# round-2 session-4 call F: k_wave2 CTA order (strips fastest vs slices fastest) A/B
for O in 1 0; do
  echo "== PTB_WAVE_ORDER=$O"
  for c in "4096 512 2" "4096 64 3" "2048 128 3" "2048 64 3" "1024 64 5" "1024 512 3"; do
    PTB_WAVE_ORDER=$O python scripts/prof_prop.py $c
  done
done
