# phase-width sweep of the replayed sweep on the C5 x 4096 rows, chunk balancing on/off
for bal in 1 0; do
for spec in "G60 0 26 32 43" "G67 0 20 26 32" "G77 13 19 26" "G55 0 43 64" "G81 13"; do
  set -- $spec; g=$1; shift
  for pw in "$@"; do
    echo -n "bal=$bal $g pw=$pw "; PBSA_BALANCE_CHUNKS=$bal PBSA_PACKED_PHASE_WORDS=$pw timeout 100 python tools/timing_run.py $g 0,0,0 4096 1000 | cut -c30-60
  done
done
done
for g in G55 G60 G81; do echo -n "bal=1 $g x1024 "; timeout 100 python tools/timing_run.py $g 0,0,0 1024 1000 | cut -c30-60; echo -n "bal=0 $g x1024 "; PBSA_BALANCE_CHUNKS=0 timeout 100 python tools/timing_run.py $g 0,0,0 1024 1000 | cut -c30-60; done
