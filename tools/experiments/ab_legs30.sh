# resident_timing knobs on C2 sigma_nu (G1 x 1024)
for env in "X=0" "PBSA_RESIDENT_CS=2" "PBSA_RESIDENT_CS=8" "PBSA_RES_SPLIT=0" "PBSA_RES_PROF=0"; do
  echo -n "$env: "; env $env timeout 100 python tools/timing_run.py G1 0,0,0.5 1024 300 | cut -c40-140
done
