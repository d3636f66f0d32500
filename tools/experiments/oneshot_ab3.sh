# One-shot G81 x 4096: phase widths around the L2 size, and the hash cache off.  Run under gpurun.
for pw in 20 26 43; do
  echo "== phase words $pw"; PBSA_PACKED_PHASE_WORDS=$pw python tools/experiments/oneshot_time.py 4096 G81 | tail -2
done
for pw in 32 64; do
  echo "== phase words $pw cache off"; PBSA_PACKED_CACHE=0 PBSA_PACKED_PHASE_WORDS=$pw python tools/experiments/oneshot_time.py 4096 G81 | tail -2
done
echo "== default"; python tools/experiments/oneshot_time.py 4096 G81 | tail -2
