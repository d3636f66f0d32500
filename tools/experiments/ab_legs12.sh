# threshold addressing A/B (PRMT of byte counts vs nibble shifts)
timeout 200 python bench.py --steps 5 --no-var-leg --no-cpu-baseline --e2e-steps 1 | python -c "import sys,json; d=json.loads(sys.stdin.read()); print('C4 %.4g philox %.4g' % (d['value'], d['philox']['value']), d['clocks']['sm_mhz'])"
timeout 100 python tools/timing_run.py G55 0,0,0 4096 1000 | cut -c1-60
timeout 100 python tools/timing_run.py G55 0,0,0 4096 1000 philox | cut -c1-60
timeout 100 python tools/timing_run.py G81 0,0,0 1024 1000 | cut -c1-60
