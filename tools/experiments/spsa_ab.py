"""SpSA device time, full-sector drive-index stores on/off (PBSA_SIDX_FULL)."""
import os
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[2]))
from paper_2601_14476_b200 import _native, benchmarks, streams
from paper_2601_14476_b200.annealer import derive_schedule
from paper_2601_14476_b200.model import maxcut_to_ising

for name, T in (("G81", 4096), ("G55", 4096), ("G1", 1024), ("G22", 4096)):
    g, _ = benchmarks.load(name)
    m = maxcut_to_ising(g)
    sch = derive_schedule(m, 1000, 10)
    keys = streams.run_keys(streams.trial_seeds(0, T))
    row = []
    for rng in ("replay", "philox"):
        for full in ("1", "0"):
            os.environ["PBSA_SIDX_FULL"] = full
            b = _native.Batch(m, sch, keys, graph=g, algo_code=2, alpha=1, p_stall=0.5, rng=rng,
                              rng_seed=streams.native_seed(0))
            plan = _native.Plan(b)
            ms = min(plan.run() for _ in range(2))
            plan.close()
            row.append(f"{rng}/full={full}: {ms:.1f}")
    print(f"SpSA {name} x {T}: " + "; ".join(row), flush=True)
