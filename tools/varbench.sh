# resident sweeps
run() { timeout 300 python tools/general_bench.py "$@" 1000; }
for g in "G1 psa 0,0,0.5 1024" "G22 psa 0.5,0.5,0.5 1024" "G1 psa 0,0,0.5 100" "G1 psa 0,0,0 1024" "G1 psa 0,0,0 100" "G47 psa 0,0,0 1024"; do
  run $g
done
