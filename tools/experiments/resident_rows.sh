# resident-kernel rows (C1, C2 lam/delta, C5 small) and TApSA resident
for k in 1 2; do
  for args in "G1 0,0,0 100" "G1 0,0,0 1024" "G1 1.0,0,0 1024" "G22 0,0,0 1024" "G47 0,0,0 1024" "G1 0,0,0 100 philox" "G1 1.0,0,0 1024 philox"; do
    set -- $args; echo "$args: $(timeout 100 python tools/timing_run.py $1 $2 $3 1000 $4 2>/dev/null | cut -c1-100 | tail -1)"
  done
done
