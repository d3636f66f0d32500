# resident cluster size / residency sweep for the timing-spread and TApSA rows
for cs in 2 4 8 16; do
  echo "G1 sigma_nu=0.5 x1024 CS=$cs: $(PBSA_RESIDENT_CS=$cs timeout 120 python tools/timing_run.py G1 0,0,0.5 1024 1000 2>&1 | cut -c1-150 | tail -1)"
  echo "G1 sigma_nu=1.0 x1024 CS=$cs: $(PBSA_RESIDENT_CS=$cs timeout 120 python tools/timing_run.py G1 0,0,1.0 1024 1000 2>&1 | cut -c1-150 | tail -1)"
done
for cs in 1 2 4; do
  echo "G22 C3 x4096 CS=$cs: $(PBSA_RESIDENT_CS=$cs timeout 200 python tools/timing_run.py G22 0.5,0.5,0.5 4096 1000 2>&1 | cut -c1-150 | tail -1)"
done
for cs in 1 2; do
  echo "G55 C3 x4096 resident CS=$cs: $(PBSA_RESIDENT=1 PBSA_RESIDENT_CS=$cs timeout 200 python tools/timing_run.py G55 0.5,0.5,0.5 4096 1000 2>&1 | cut -c1-150 | tail -1)"
done
timeout 300 python tools/experiments/tapsa_ab.py G1:4096:4 G22:4096:4 G47:4096:4 G1:4096:8 2>&1
