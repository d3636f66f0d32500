# bucket kernel launch shape: warps per word and chains (BASELINE C3 rows)
for g in "G81 200" "G55 500"; do set -- $g
  for wpw in 0 48 140 200; do
    echo -n "wpw=$wpw "; if [ $wpw = 0 ]; then unset PBSA_WARPS_PER_WORD; else export PBSA_WARPS_PER_WORD=$wpw; fi
    timeout 100 python tools/timing_run.py $1 0.5,0.5,0.5 4096 $2 | cut -c1-120
  done; unset PBSA_WARPS_PER_WORD
  for ch in 2 8; do echo -n "chains=$ch "; PBSA_PACKED_CHAINS=$ch timeout 100 python tools/timing_run.py $1 0.5,0.5,0.5 4096 $2 | cut -c1-120; done
done
