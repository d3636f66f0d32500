# resident timing kernel: double-buffered divisor masks written before the cluster barrier
timeout 100 python tools/timing_run.py G1 0,0,0.5 1024 300 | cut -c40-70
timeout 100 python tools/timing_run.py G1 0,0,1.0 1024 300 | cut -c40-70
timeout 100 python tools/timing_run.py G22 0.5,0.5,0.5 1024 300 | cut -c40-70
