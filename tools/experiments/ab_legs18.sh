timeout 100 python tools/timing_run.py G81 0,0,0 4096 1000 replay tapsa | cut -c1-70
timeout 100 python tools/timing_run.py G1 0,0,0 1024 1000 replay spsa | cut -c1-70
timeout 100 python tools/timing_run.py G81 0,0,0 4096 1000 | cut -c1-70
timeout 100 python tools/timing_run.py G81 0,0,0 1024 1000 | cut -c1-70
