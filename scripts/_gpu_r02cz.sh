# round-2 session-5 call Z: 1024^2 x 512: row blocks / strip width overrides
for E in "" "PTB_WAVE_DIV=2" "PTB_WAVE_DIV=4" "PTB_WAVE_W=96" "PTB_WAVE_W=128" "PTB_WAVE_W=96 PTB_WAVE_DIV=2" "PTB_WAVE_W=256"; do
  echo "== $E: $(env $E python scripts/prof_prop.py 1024 512 3)"
done
