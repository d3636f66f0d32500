# end-of-round measurement pass (run under gpurun): GPU suite, smoke, bench lines,
# config table, one ncu capture of the resident TApSA kernel
mkdir -p gpurun_out/final
timeout 1200 python -m pytest tests -m gpu -q > gpurun_out/final/gpu_tests.log 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/final/smoke.log 2>&1
timeout 600 python bench.py > gpurun_out/final/bench_n1.json 2> gpurun_out/final/bench_n1.err
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/final/bench_ref.json 2>&1
timeout 1500 python tools/config_table.py --tag r01 > gpurun_out/final/configs.log 2>&1
cp profiles/r01_configs.* gpurun_out/final/
timeout 400 ncu --set full --clock-control none --import-source on -k regex:resident_sweep --launch-count 1 \
  -o gpurun_out/final/r01_resident_tapsa_g1 python tools/experiments/tapsa_ab.py G1:100:4 > gpurun_out/final/ncu_tapsa.log 2>&1
ls -la gpurun_out/final
