timeout 100 python tools/timing_run.py G81 0,0,0 4096 300 replay tapsa | cut -c40-70
timeout 100 python tools/timing_run.py G1 0,0,0 4096 300 replay tapsa | cut -c40-70
timeout 100 python tools/timing_run.py G55 0,0,0 4096 300 replay tapsa | cut -c40-70
