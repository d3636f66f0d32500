# Round-1 profiling recipe (run under gpurun): bench lines, ncu launch list, and
# one ncu --set full capture of a steady-state phased update sweep.
# Application replay keeps the L2 state each launch really sees (kernel replay
# restores memory between passes, which evicts the phase's L2-resident cache).
set -x
MODE=${1:-all}
if [ "$MODE" = all ]; then
python bench.py > gpurun_out/bench_n1.json 2> gpurun_out/bench_n1.err
python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_ref.json 2>&1
python bench.py --steps 2 --warmup 3 --cycles 20 --e2e-steps 1 --no-cpu-baseline > gpurun_out/b20.json 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 3 --cycles 20 --e2e-steps 1 --no-cpu-baseline > gpurun_out/ncu1.log 2>&1
fi
PBSA_PACKED_CHAINS=1 python bench.py --steps 1 --warmup 0 --cycles 20 --e2e-steps 1 --no-cpu-baseline > gpurun_out/b20c1.json 2>&1 && \
PBSA_PACKED_CHAINS=1 timeout 1500 ncu --set full --replay-mode application --clock-control none --cache-control none --import-source on -k regex:packed_sweep --launch-skip 15 --launch-count 1 -o gpurun_out/r01_sweep_phase_app python bench.py --steps 1 --warmup 0 --cycles 20 --e2e-steps 1 --no-cpu-baseline > gpurun_out/ncu2.log 2>&1
ls -la gpurun_out
