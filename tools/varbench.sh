# development timing of the packed rules (TApSA)
run() { timeout 300 python tools/general_bench.py "$@" 1000; }
run G1 tapsa 0,0,0 1024
run G22 tapsa 0,0,0 4096
run G81 tapsa 0,0,0 4096
run G55 tapsa 0,0,0 4096
