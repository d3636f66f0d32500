for lib in libpbsa.so libpbsa_mb3.so libpbsa_mb5.so; do
PBSA_LIB=$PWD/paper_2601_14476_b200/_lib/$lib timeout 300 python bench.py --no-cpu-baseline --e2e-steps 1 --steps 3 2>&1 | python -c "import sys,json; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$lib', 'replay %.4g' % d['value'], 'philox %.4g' % d['philox']['value'], d['clocks'])"
done
python bench.py --rng philox --steps 2 --warmup 3 --cycles 20 --e2e-steps 1 --no-cpu-baseline --no-philox-leg > gpurun_out/b20_phx.json 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file gpurun_out/launches_philox.csv python bench.py --rng philox --steps 2 --warmup 3 --cycles 20 --e2e-steps 1 --no-cpu-baseline --no-philox-leg > gpurun_out/ncu_l.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:packed_sweep --launch-skip 15 --launch-count 1 -o gpurun_out/r01_sweep_philox python bench.py --rng philox --steps 1 --warmup 0 --cycles 20 --e2e-steps 1 --no-cpu-baseline --no-philox-leg > gpurun_out/ncu_f.log 2>&1
ls -la gpurun_out
