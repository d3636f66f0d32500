# trial-pair cache tiles with pair loads in every consumer
timeout 200 python bench.py --steps 5 --no-var-leg --no-cpu-baseline --e2e-steps 1 | python -c "import sys,json; d=json.loads(sys.stdin.read()); print('C4 %.4g philox %.4g' % (d['value'], d['philox']['value']))"
timeout 100 python tools/timing_run.py G81 0,0,0 1024 1000 | cut -c40-70
timeout 100 python tools/timing_run.py G55 0,0,0 4096 1000 | cut -c40-70
timeout 100 python tools/timing_run.py G81 0,0,0 4096 300 replay tapsa | cut -c40-70
timeout 100 python tools/timing_run.py G81 0,0,0 4096 300 replay spsa | cut -c40-70
timeout 100 python tools/timing_run.py G81 0.5,0.5,0 4096 300 | cut -c40-70
timeout 100 python tools/timing_run.py G1 0,0,0 1024 1000 | cut -c40-70
timeout 100 python tools/timing_run.py G1 0.5,0,0 1024 1000 | cut -c40-70
