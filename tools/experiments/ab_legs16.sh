# resident cluster kernels vs the launched sweep, plain rule
for spec in "G1 100" "G1 1024" "G47 1024" "G22 1024" "G1 2048" "G22 2048"; do
  set -- $spec
  for r in 1 0; do echo -n "res=$r "; PBSA_RESIDENT=$r timeout 100 python tools/timing_run.py $1 0,0,0 $2 1000 | cut -c1-80; done
done
