# min-blocks A/B of the Philox and TApSA / varied-profile sweeps
timeout 100 python tools/timing_run.py G81 0,0,0 4096 1000 philox | cut -c1-70
timeout 100 python tools/timing_run.py G81 0.5,0.5,0 4096 300 | cut -c1-70
timeout 100 python tools/timing_run.py G81 0.5,0.5,0 4096 300 philox | cut -c1-70
timeout 100 python tools/timing_run.py G81 0,0,0 4096 300 replay tapsa | cut -c1-70
timeout 100 python tools/timing_run.py G81 0,0,0 4096 300 philox tapsa | cut -c1-70
timeout 100 python tools/timing_run.py G55 0,0,0 4096 300 philox | cut -c1-70
timeout 100 python tools/timing_run.py G1 0,0,0 4096 300 philox | cut -c1-70
