# development timing of the variability paths (BASELINE C2/C3 shapes)
run() { timeout 300 python tools/general_bench.py "$@" 1000; }
run G81 psa 0.5,0.5,0.5 4096
run G55 psa 0.5,0.5,0.5 4096
run G22 psa 0.5,0.5,0.5 4096
run G1 psa 0,0,0.5 1024
run G1 psa 0.5,0,0 1024
run G1 psa 0,0,0 1024
run G22 psa 0,0,0 1024
run G55 psa 0,0,0 4096
run G81 psa 0,0,0 4096
run G81 psa 0.5,0.5,0 4096
