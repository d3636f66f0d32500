# L = 4 at 9 blocks: launch shapes for G55 / G60
for spec in "G60 4096 43 0" "G60 4096 43 1" "G60 4096 32 0" "G55 4096 64 1" "G55 4096 64 0" "G55 4096 0 0" "G60 1024 0 0" "G55 1024 0 0"; do
  set -- $spec
  echo -n "$1 x $2 pw=$3 bal=$4: "; PBSA_PACKED_PHASE_WORDS=$3 PBSA_BALANCE_CHUNKS=$4 timeout 100 python tools/timing_run.py $1 0,0,0 $2 1000 | cut -c40-110
done
