# quick check: GPU tests + replay/philox bench line (3 steps)
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -1
for k in 1 2; do
timeout 300 python bench.py --no-cpu-baseline --e2e-steps 1 --steps 3 "$@" 2>&1 | python -c "import sys,json; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('replay %.4g' % d['value'], 'frac %.3f' % d['roofline']['frac'], 'e2e %.4g' % d['e2e']['value'], 'philox %.4g' % d['philox']['value'], d['clocks'])"
done
