# default launch shape (choose_phases) on the C5 rows
for T in 4096 2048 1024; do
for g in G48 G55 G60 G67 G77 G81; do
  timeout 100 python tools/timing_run.py $g 0,0,0 $T 1000 | cut -c1-110
done; done
