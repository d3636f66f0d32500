# One rank's shard of the C4 job (G81, 4096 trials, strong scaling) timed on
# one B200: at N GPUs each rank anneals 4096/N trials with no data-path
# exchange, so the N-GPU job time is the max over ranks
# of this shard time plus the end-of-run NCCL reduce.  Run under gpurun.
set -x
for N in 1 2 4 8; do
  T=$((4096 / N))
  timeout 600 python bench.py --trials $T --steps 5 --warmup 3 --no-cpu-baseline \
    > gpurun_out/shard_n$N.json 2> gpurun_out/shard_n$N.err
done
ls -la gpurun_out
