# default launch shape (choose_phases) at every shard size
for T in 4096 2048 1024 512; do
for g in G48 G55 G60 G67 G77 G81; do
  timeout 100 python tools/timing_run.py $g 0,0,0 $T 1000 | cut -c1-100
done; done
