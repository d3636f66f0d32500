# L1 prefetch of the hash-cache tiles at the final build (PBSA_CACHE_PREFETCH=0/1)
for pf in 1 0 1 0; do
  echo -n "prefetch=$pf "; PBSA_CACHE_PREFETCH=$pf timeout 200 python bench.py --steps 5 --no-var-leg --no-cpu-baseline --no-philox-leg --e2e-steps 1 | python -c "import sys,json; d=json.loads(sys.stdin.read()); print('C4 %.4g' % d['value'])"
  PBSA_CACHE_PREFETCH=$pf timeout 100 python tools/timing_run.py G81 0,0,0 1024 1000 | cut -c40-70
done
