# development timing of the packed rules (SpSA / TApSA)
run() { timeout 300 python tools/general_bench.py "$@" 1000; }
run G81 spsa 0,0,0 4096
run G55 spsa 0,0,0 4096
run G81 tapsa 0,0,0 4096
run G22 tapsa 0,0,0 4096
run G1 tapsa 0,0,0 1024
