"""TApSA / SpSA on G81 x 4096: device time vs word-phase size (PBSA_PACKED_PHASE_WORDS)."""
import os
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[2]))
from paper_2601_14476_b200 import _native, benchmarks, streams
from paper_2601_14476_b200.annealer import derive_schedule
from paper_2601_14476_b200.model import maxcut_to_ising

g, _ = benchmarks.load("G81")
m = maxcut_to_ising(g)
sch = derive_schedule(m, 1000, 10)
T = 4096
keys = streams.run_keys(streams.trial_seeds(0, T))
for algo, alpha in ((1, 4), (2, 1)):
    for rng in ("replay", "philox"):
        row = []
        for pw in ("", "8", "13", "26", "128"):
            if pw:
                os.environ["PBSA_PACKED_PHASE_WORDS"] = pw
            else:
                os.environ.pop("PBSA_PACKED_PHASE_WORDS", None)
            b = _native.Batch(m, sch, keys, graph=g, algo_code=algo, alpha=alpha, p_stall=0.5, rng=rng,
                              rng_seed=streams.native_seed(0))
            plan = _native.Plan(b)
            ms = min(plan.run() for _ in range(2))
            plan.close()
            row.append(f"pw={pw or 'default'}: {ms:.1f}")
        print(f"algo={algo} {rng}: " + "; ".join(row), flush=True)
