# launched timing kernel: 8-bit profile codes vs the fp16 pair (C3 rows)
for g in G55 G81; do
  for p in 1 0; do
    echo "$g C3 prof8=$p: $(PBSA_PROF8=$p timeout 300 python tools/timing_run.py $g 0.5,0.5,0.5 4096 1000 2>&1 | cut -c1-110 | tail -1)"
  done
done
for p in 1 0; do
  echo "G81 sigma_nu=1 x1024 prof8=$p: $(PBSA_PROF8=$p timeout 300 python tools/timing_run.py G81 0,0,1.0 1024 1000 2>&1 | cut -c1-110 | tail -1)"
done
