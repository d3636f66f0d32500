# blocks per SM of the cached plain sweep for L = 4 and L = 7 at the current build
timeout 100 python tools/timing_run.py G55 0,0,0 4096 1000 | cut -c40-70
timeout 100 python tools/timing_run.py G60 0,0,0 4096 1000 | cut -c40-70
timeout 100 python tools/timing_run.py G55 0,0,0 1024 1000 | cut -c40-70
timeout 100 python tools/timing_run.py G1 0,0,0 4096 1000 | cut -c40-70
timeout 100 python tools/timing_run.py G22 0,0,0 4096 1000 | cut -c40-70
