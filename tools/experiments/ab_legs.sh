# one line per workload (tools/ab_libs.sh runs this per library variant)
timeout 200 python bench.py --steps 5 --no-philox-leg --no-var-leg --no-cpu-baseline --e2e-steps 1 | python -c "import sys,json; d=json.loads(sys.stdin.read()); print('C4', '%.4g' % d['value'], d['clocks']['sm_mhz'])"
for spec in "G67 1024" "G55 1024" "G60 1024" "G22 4096" "G1 4096" "G55 4096"; do
  set -- $spec
  timeout 100 python tools/timing_run.py $1 0,0,0 $2 1000 | cut -c1-72
done
