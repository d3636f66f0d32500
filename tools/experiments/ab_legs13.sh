# 1-D vs 2-D grid of the launched sweeps (PBSA_GRID2D)
for v in 0 1; do
  echo "grid2d=$v"; export PBSA_GRID2D=$v
  timeout 300 python bench.py --steps 5 --no-var-leg --no-cpu-baseline --no-philox-leg --e2e-steps 1 | python -c "import sys,json; d=json.loads(sys.stdin.read()); print('C4 %.4g' % d['value'])"
  bash tools/experiments/ab_legs9.sh
done
