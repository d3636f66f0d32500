"""Device time of TApSA plans, resident cluster kernel vs launched packed
sweep (PBSA_RESIDENT=1/0 is read at plan creation).

usage: python tools/experiments/tapsa_ab.py [GRAPH:TRIALS:ALPHA ...]
"""
import os
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[2]))
from paper_2601_14476_b200 import _native, benchmarks, streams
from paper_2601_14476_b200.annealer import derive_schedule
from paper_2601_14476_b200.model import maxcut_to_ising

cases = sys.argv[1:] or ["G1:100:4", "G1:1024:4", "G22:100:4", "G47:256:4", "G1:2048:8"]
for case in cases:
    name, T, alpha = case.split(":")
    T, alpha = int(T), int(alpha)
    g, _ = benchmarks.load(name)
    m = maxcut_to_ising(g)
    sch = derive_schedule(m, 1000, 10)
    keys = streams.run_keys(streams.trial_seeds(0, T))
    row = []
    for rng in ("replay", "philox"):
        for res in ("1", "0"):
            os.environ["PBSA_RESIDENT"] = res
            b = _native.Batch(m, sch, keys, graph=g, algo_code=1, alpha=alpha, rng=rng,
                              rng_seed=streams.native_seed(0))
            try:
                plan = _native.Plan(b)
            except Exception as e:  # noqa: BLE001
                row.append(f"{rng}/res={res}: {e}")
                continue
            kern = plan.info()["kernel"]
            ms = min(plan.run() for _ in range(3))
            plan.close()
            row.append(f"{rng}/{kern}: {ms:.2f} ms")
    print(f"{name} x {T} alpha={alpha}: " + "; ".join(row), flush=True)
