# C5 x 1024 rows: chains and warps per word
for g in G55 G60 G48; do
  for ch in 0 16 32; do echo -n "$g chains=$ch "; if [ $ch = 0 ]; then unset PBSA_PACKED_CHAINS; else export PBSA_PACKED_CHAINS=$ch; fi; timeout 100 python tools/timing_run.py $g 0,0,0 1024 1000 | cut -c44-130; done; unset PBSA_PACKED_CHAINS
  for w in 80 40; do echo -n "$g wpw=$w "; PBSA_WARPS_PER_WORD=$w timeout 100 python tools/timing_run.py $g 0,0,0 1024 1000 | cut -c44-130; done
done
