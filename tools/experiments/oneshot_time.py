"""Wall and device time of the one-shot C-ABI call (pinned outputs), graph x T
(usage: oneshot_time.py [T] [graph])."""
import sys, time
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[2]))
import torch
from paper_2601_14476_b200 import _native, benchmarks, streams
from paper_2601_14476_b200.annealer import derive_schedule
from paper_2601_14476_b200.model import maxcut_to_ising
T = int(sys.argv[1]) if len(sys.argv) > 1 else 4096
G = sys.argv[2] if len(sys.argv) > 2 else "G81"
g, _ = benchmarks.load(G)
m = maxcut_to_ising(g)
b = _native.Batch(m, derive_schedule(m, 1000, 10), streams.run_keys(streams.trial_seeds(0, T)), graph=g)
pinned = {k: torch.empty(v.shape, dtype=getattr(torch, str(v.dtype)), pin_memory=True).numpy()
          for k, v in b.alloc_outputs().items()}
for rep in range(4):
    t0 = time.perf_counter()
    out, ms = _native.anneal_batch(b, out=pinned)
    print(f"one-shot {G} T={T}: wall {1e3 * (time.perf_counter() - t0):.1f} ms, device {ms:.1f} ms", flush=True)
