# masked 8-entry tail batch in the neighbour gather (PBSA_MASKED_TAIL)
timeout 100 python tools/timing_run.py G55 0,0,0 1024 1000 | cut -c40-70
timeout 100 python tools/timing_run.py G60 0,0,0 1024 1000 | cut -c40-70
timeout 100 python tools/timing_run.py G55 0,0,0 4096 1000 | cut -c40-70
timeout 100 python tools/timing_run.py G60 0,0,0 4096 1000 | cut -c40-70
timeout 100 python tools/timing_run.py G55 0.5,0.5,0.5 4096 300 | cut -c40-70
timeout 100 python tools/timing_run.py G22 0.5,0.5,0.5 4096 300 | cut -c40-70
timeout 100 python tools/timing_run.py G22 0,0,0 4096 1000 | cut -c40-70
timeout 100 python tools/timing_run.py G1 0,0,0 1024 1000 | cut -c40-70
timeout 100 python tools/timing_run.py G1 0,0,0.5 1024 300 | cut -c40-70
