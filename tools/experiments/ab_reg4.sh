# A/B of the degree-4 gather fast path (PBSA_REG4=0 disables it)
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
for r in 1 0; do
PBSA_REG4=$r timeout 300 python bench.py --no-cpu-baseline --e2e-steps 1 --steps 3 2>&1 | python -c "import sys,json; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('reg4=$r', 'replay %.4g' % d['value'], 'frac %.3f' % d['roofline']['frac'], 'philox %.4g' % d['philox']['value'], d['clocks'])"
done
