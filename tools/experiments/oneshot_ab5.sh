# One-shot G81 at the N=2/N=4 shard sizes: phase width sweep.  Run under gpurun.
for pw in 32 16 11; do echo "== 1024 pw $pw"; PBSA_PACKED_PHASE_WORDS=$pw python tools/experiments/oneshot_time.py 1024 G81 | tail -2; done
for pw in 64 32 22 16; do echo "== 2048 pw $pw"; PBSA_PACKED_PHASE_WORDS=$pw python tools/experiments/oneshot_time.py 2048 G81 | tail -2; done
