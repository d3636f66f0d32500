# development timing of the packed rules (SpSA / TApSA)
run() { timeout 300 python tools/general_bench.py "$@" 1000; }
run G81 spsa 0,0,0 4096
run G55 spsa 0,0,0 4096
run G1 spsa 0,0,0 1024
run G81 tapsa 0,0,0 4096
PBSA_PACKED_PHASE_WORDS=0 PBSA_PACKED_CHAINS=4 run G81 tapsa 0,0,0 4096
run G55 tapsa 0,0,0 4096
