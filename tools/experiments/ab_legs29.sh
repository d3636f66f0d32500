# chains per phase and PDL at the current build (C4)
for env in "X=0" "PBSA_PACKED_CHAINS=7" "PBSA_PACKED_CHAINS=4" "PBSA_PDL=0"; do
  echo -n "$env: "; env $env timeout 200 python bench.py --steps 5 --no-var-leg --no-cpu-baseline --no-philox-leg --e2e-steps 1 | python -c "import sys,json; d=json.loads(sys.stdin.read()); print('C4 %.4g' % d['value'])"
done
