# Round-2 profiling recipe (run under gpurun, one GPU): the ncu launch list of
# the bench command, a steady-state --set full capture of the headline sweep
# (application replay keeps each phase's L2-resident hash cache, which kernel
# replay would evict) and of the timing-spread bucket kernel (BASELINE C3).
set -x
mkdir -p gpurun_out
python bench.py --steps 2 --warmup 3 --cycles 20 --e2e-steps 1 --no-cpu-baseline --no-var-leg > gpurun_out/r02_b20.json 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 5000 --csv --log-file gpurun_out/r02_launches.csv \
  python bench.py --steps 2 --warmup 3 --cycles 20 --e2e-steps 1 --no-cpu-baseline --no-var-leg > gpurun_out/r02_ncu_list.log 2>&1
python tools/headline_run.py 20 > gpurun_out/r02_hr.log 2>&1 && \
PBSA_PACKED_CHAINS=1 timeout 1200 ncu --set full --replay-mode application --clock-control none --cache-control none \
  --import-source on -k regex:packed_sweep --launch-skip 15 --launch-count 1 -o gpurun_out/r02_sweep_phase_app \
  python tools/headline_run.py 20 > gpurun_out/r02_ncu_sweep.log 2>&1
python tools/headline_run.py 30 G55 0.5,0.5,0.5 > gpurun_out/r02_hr_c3.log 2>&1 && \
PBSA_PACKED_CHAINS=1 timeout 900 ncu --set full --clock-control none --cache-control none --import-source on \
  -k regex:packed_sweep_bucket --launch-skip 121 --launch-count 1 -o gpurun_out/r02_bucket_g55 \
  python tools/headline_run.py 30 G55 0.5,0.5,0.5 > gpurun_out/r02_ncu_bucket.log 2>&1
ls -la gpurun_out | tail -20
