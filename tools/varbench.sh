# development timing of the packed variability path (BASELINE C2/C3 shapes)
run() { timeout 300 python tools/general_bench.py "$@" 1000; }
run G81 psa 0.5,0.5,0 4096
PBSA_PACKED_CACHE=0 run G81 psa 0.5,0.5,0 4096
PBSA_PACKED_PHASE_WORDS=20 run G81 psa 0.5,0.5,0 4096
PBSA_PACKED_PHASE_WORDS=6 run G81 psa 0.5,0.5,0 4096
run G22 psa 0.5,0.5,0 4096
run G22 psa 0.5,0.5,0.5 4096
