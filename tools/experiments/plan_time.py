"""Device time of one G81 x T plan run (phases/chains via PBSA_* env vars)."""
import sys, time
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[2]))
from paper_2601_14476_b200 import _native, benchmarks, streams
from paper_2601_14476_b200.annealer import derive_schedule
from paper_2601_14476_b200.model import maxcut_to_ising
T = int(sys.argv[1]) if len(sys.argv) > 1 else 4096
rng = sys.argv[2] if len(sys.argv) > 2 else "replay"
g, _ = benchmarks.load("G81")
m = maxcut_to_ising(g)
b = _native.Batch(m, derive_schedule(m, 1000, 10), streams.run_keys(streams.trial_seeds(0, T)), graph=g,
                  rng=rng, rng_seed=streams.native_seed(0))
t0 = time.perf_counter(); plan = _native.Plan(b); t1 = time.perf_counter()
ms = [plan.run() for _ in range(4)]
info = plan.info()
print(f"T={T} {rng}: create {1e3*(t1-t0):.0f} ms, device runs {[round(x,1) for x in ms]} ms, launches {info['launches']}")
