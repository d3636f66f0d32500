# phase widths of the N-GPU shard sizes (G81 x 1024 / 512 trials)
for spec in "1024 0 16 11 8" "512 0 8 6 4"; do
  set -- $spec; T=$1; shift
  for pw in "$@"; do echo -n "T=$T pw=$pw "; PBSA_PACKED_PHASE_WORDS=$pw timeout 100 python tools/timing_run.py G81 0,0,0 $T 1000 | cut -c44-140; done
done
