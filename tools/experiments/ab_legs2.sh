for spec in "G55 4096" "G60 4096" "G1 4096"; do
  set -- $spec
  echo "$(timeout 100 python tools/timing_run.py $1 0,0,0 $2 1000 | cut -c1-64) | $(PBSA_CTA_FLUSH=0 timeout 100 python tools/timing_run.py $1 0,0,0 $2 1000 | cut -c52-64) (no cta flush)"
done
