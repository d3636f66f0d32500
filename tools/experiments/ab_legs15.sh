# resident_timing vs the period-bucket kernel at the word-count boundary
for spec in "G1 0,0,0.5 4096" "G1 0,0,0.5 2048" "G47 0.5,0.5,0.5 4096" "G22 0.5,0.5,0.5 2048" "G22 0.5,0.5,0.5 1024" "G47 0.5,0.5,0.5 2048"; do
  set -- $spec
  for r in 1 0; do echo -n "res=$r "; PBSA_RESIDENT=$r timeout 100 python tools/timing_run.py $1 $2 $3 300 | cut -c1-80; done
done
