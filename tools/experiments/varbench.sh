# resident uniform variability
run() { timeout 300 python tools/experiments/general_bench.py "$@" 1000; }
run G1 psa 0.5,0,0 1024
PBSA_RESIDENT=0 run G1 psa 0.5,0,0 1024
run G1 psa 0,1.0,0 1024
run G22 psa 0.5,0.5,0 1024
PBSA_RESIDENT=0 run G22 psa 0.5,0.5,0 1024
run G22 psa 0.5,0.5,0.5 4096
