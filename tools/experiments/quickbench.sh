#!/bin/bash
# quick GPU check used during development: parity tests + short bench
timeout 600 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
python bench.py --steps 3 --warmup 2 --e2e-steps 1 --no-cpu-baseline "$@" 2>&1 | python -c "import sys,json; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('value %.4g ms/step %.2f kernel_ms %.4f frac %.3f clocks %s' % (d['value'], d['ms_per_step'], d['roofline']['kernel_ms_mean'], d['roofline']['frac'], d['clocks']))"
