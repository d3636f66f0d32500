# resident plain / varied-profile kernel: cluster size
for spec in "G1 0,0,0 1024" "G1 0.5,0,0 1024" "G22 0,0,0 1024" "G47 0,0,0 1024" "G1 0,0,0 100"; do
  set -- $spec
  for cs in 0 2 8; do
    echo -n "$1 $2 x$3 cs=$cs: "; if [ $cs = 0 ]; then unset PBSA_RESIDENT_CS; else export PBSA_RESIDENT_CS=$cs; fi
    timeout 100 python tools/timing_run.py $1 $2 $3 1000 | cut -c40-80
  done; unset PBSA_RESIDENT_CS
done
