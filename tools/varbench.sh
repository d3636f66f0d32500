# resident multi-cycle sweep vs launched sweeps
run() { timeout 300 python tools/general_bench.py "$@" 1000; }
for g in "G1 psa 0,0,0 100" "G1 psa 0,0,0 1024" "G47 psa 0,0,0 1024" "G22 psa 0,0,0 1024" "G22 psa 0,0,0 4096" "G1 tapsa 0,0,0 1024" "G1 spsa 0,0,0 1024"; do
  run $g
  PBSA_RESIDENT=1 PBSA_RESIDENT_CS=4 run $g
done
run G81 psa 0,0,0 4096
run G1 psa 0.5,0.5,0.5 1024
