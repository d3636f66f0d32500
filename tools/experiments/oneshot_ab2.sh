# One-shot G81 x 4096: pipelined phase width / chains sweep.  Run under gpurun.
for pw in 32 16 13; do for ch in 1 2 4; do
  echo "== phase words $pw chains $ch"
  PBSA_PACKED_PHASE_WORDS=$pw PBSA_PACKED_CHAINS=$ch python tools/experiments/oneshot_time.py 4096 G81 | tail -2
done; done
echo "== PBSA_PIPELINE=0 (graph)"; PBSA_PIPELINE=0 python tools/experiments/oneshot_time.py 4096 G81 | tail -2
