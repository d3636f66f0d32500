for cfg in "G1 psa 0.5,0,0 1024" "G1 psa 0,0.5,0 1024" "G1 psa 0,0,0.5 1024" "G1 psa 0.5,0.5,0.5 1024" "G22 psa 0.5,0.5,0.5 4096" "G55 psa 0.5,0.5,0.5 4096" "G81 psa 0.5,0.5,0.5 4096" "G81 psa 0.5,0.5,0 4096"; do
  set -- $cfg
  timeout 300 python tools/general_bench.py $1 $2 $3 $4 1000
  PBSA_PACKED_VAR=0 timeout 300 python tools/general_bench.py $1 $2 $3 $4 1000
done
