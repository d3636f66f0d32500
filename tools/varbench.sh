# development timing of the packed path phase policy (BASELINE C3/C5 shapes)
run() { timeout 300 python tools/general_bench.py "$@" 1000; }
run G81 psa 0,0,0 1024
run G55 psa 0,0,0 1024
run G1 psa 0,0,0 1024
run G55 psa 0,0,0 4096
PBSA_PACKED_PHASE_WORDS=0 run G55 psa 0,0,0 4096
run G22 psa 0,0,0 4096
PBSA_PACKED_PHASE_WORDS=0 run G22 psa 0,0,0 4096
run G81 psa 0,0,0 4096
run G81 psa 0,0,0 2048
PBSA_PACKED_PHASE_WORDS=0 run G81 psa 0,0,0 2048
