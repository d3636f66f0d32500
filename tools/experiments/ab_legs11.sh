# hash-cache layout A/B (c1 = y_hi * M1L cached or not): the cached sweeps
timeout 200 python bench.py --steps 5 --no-philox-leg --no-var-leg --no-cpu-baseline --e2e-steps 1 | python -c "import sys,json; d=json.loads(sys.stdin.read()); print('C4 %.4g' % d['value'], d['clocks']['sm_mhz'])"
timeout 100 python tools/timing_run.py G55 0,0,0 4096 1000 | cut -c1-60
timeout 100 python tools/timing_run.py G1 0,0,0 4096 1000 | cut -c1-60
timeout 100 python tools/timing_run.py G81 0,0,0 4096 300 replay tapsa | cut -c1-60
timeout 100 python tools/timing_run.py G81 0.5,0.5,0 4096 300 | cut -c1-60
