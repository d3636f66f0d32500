# next chunk's neighbour words loaded half-way through the decisions (PBSA_NB_AHEAD)
timeout 200 python bench.py --steps 5 --no-var-leg --no-cpu-baseline --no-philox-leg --e2e-steps 1 | python -c "import sys,json; d=json.loads(sys.stdin.read()); print('C4 %.4g' % d['value'])"
timeout 100 python tools/timing_run.py G81 0,0,0 1024 1000 | cut -c40-70
timeout 100 python tools/timing_run.py G67 0,0,0 4096 1000 | cut -c40-70
