# bucket kernel staging size / blocks per SM (BASELINE C3 rows)
timeout 100 python tools/timing_run.py G81 0.5,0.5,0.5 4096 200 | cut -c1-70
timeout 100 python tools/timing_run.py G55 0.5,0.5,0.5 4096 500 | cut -c1-70
