# small-batch resident rows (C1, C2, C5 small) with and without the two-lane split
for sp in 1 0; do
  echo "split=$sp"
  PBSA_RES_SPLIT=$sp python tools/timing_run.py G1 0,0,0 100 1000 | cut -c1-120
  PBSA_RES_SPLIT=$sp python tools/timing_run.py G1 1.0,0,0 1024 1000 | cut -c1-120
  PBSA_RES_SPLIT=$sp python tools/timing_run.py G1 0,0,0 1024 1000 | cut -c1-120
  PBSA_RES_SPLIT=$sp python tools/timing_run.py G22 0,0,0 1024 1000 | cut -c1-120
  PBSA_RES_SPLIT=$sp python tools/timing_run.py G1 0,0,0.5 1024 1000 | cut -c1-120
done
