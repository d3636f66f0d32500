# One-shot call A/B: current phase policy vs the old fixed four phases
# ((W+3)/4 words per phase, forced with PBSA_PACKED_PHASE_WORDS).  Run under gpurun.
for spec in "512 G81 4" "1024 G81 8" "2048 G81 16" "4096 G81 32" "4096 G55 32" "1024 G55 8" "4096 G67 32"; do
  set -- $spec
  echo "== $2 x $1 new"; python tools/experiments/oneshot_time.py $1 $2 | tail -2
  echo "== $2 x $1 old (phase words $3)"; PBSA_PACKED_PHASE_WORDS=$3 python tools/experiments/oneshot_time.py $1 $2 | tail -2
done
