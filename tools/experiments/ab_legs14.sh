# G81 x 4096 phase width around the model's pick, final build
for pw in 13 10 16 19 26; do echo -n "pw=$pw "; PBSA_PACKED_PHASE_WORDS=$pw timeout 100 python tools/timing_run.py G81 0,0,0 4096 1000 | cut -c44-130; done
for wpw in 316 160 212; do echo -n "wpw=$wpw "; PBSA_WARPS_PER_WORD=$wpw timeout 100 python tools/timing_run.py G81 0,0,0 4096 1000 | cut -c44-130; done
