"""Per-rank cost of the N-GPU job on one B200: the shard of rank N-1 (4096/N
trials of G81, global seeds) through the bench Plan (device) and through the
one-shot C-ABI call with page-locked outputs (e2e, warm plan).
    python tools/shard_e2e.py [1 2 4 8]"""
import sys
import time
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402
from paper_2601_14476_b200 import _native, benchmarks, streams  # noqa: E402
from paper_2601_14476_b200.annealer import derive_schedule  # noqa: E402
from paper_2601_14476_b200.distributed import shard_range  # noqa: E402
from paper_2601_14476_b200.model import maxcut_to_ising  # noqa: E402

g, _ = benchmarks.load("G81")
m = maxcut_to_ising(g)
sch = derive_schedule(m, 1000, 10)
for N in [int(x) for x in sys.argv[1:]] or [1, 2, 4, 8]:
    lo, hi = shard_range(4096, N - 1, N)
    b = _native.Batch(m, sch, streams.run_keys(streams.trial_seeds(0, hi)[lo:hi]), graph=g, first_trial=lo)
    plan = _native.Plan(b)
    plan.run()
    dev = min(plan.run() for _ in range(3))
    plan.close()
    pinned = {k: torch.empty(v.shape, dtype=getattr(torch, str(v.dtype)), pin_memory=True).numpy()
              for k, v in b.alloc_outputs().items()}
    _native.anneal_batch(b, out=pinned)
    e2e = []
    for _ in range(3):
        t0 = time.perf_counter()
        _native.anneal_batch(b, out=pinned)
        e2e.append(1e3 * (time.perf_counter() - t0))
    _native.plan_cache_clear()
    ups = (hi - lo) * g.n * 1000
    print(f"N={N} shard {hi - lo} trials: device {dev:.2f} ms ({ups / dev / 1e9:.3g} T upd/s per rank, "
          f"x{N} = {N * ups / dev / 1e9:.3g}), e2e {min(e2e):.2f} ms ({N * ups / min(e2e) / 1e9:.3g} T upd/s job)",
          flush=True)
