"""Wall time of engine.run_trials on BASELINE C3 with host (numpy) profiles
and replayed draws, with host profiles and Philox draws, and with native
(device-drawn) profiles:  python tools/native_profile_e2e.py [G81] [4096]"""
import dataclasses
import sys
import time
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2601_14476_b200 import benchmarks, engine  # noqa: E402
from paper_2601_14476_b200.annealer import Algorithm, AlgorithmConfig  # noqa: E402
from paper_2601_14476_b200.pbit import VariabilityConfig  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "G81"
T = int(sys.argv[2]) if len(sys.argv) > 2 else 4096
g, _ = benchmarks.load(name)
base = engine.ExperimentSpec(graph=name, algo=AlgorithmConfig(Algorithm.PSA),
                             variability=VariabilityConfig(0.5, 0.5, 0.5), cycles=1000, trials=T)
for label, spec in (("replay, host profiles", base),
                    ("philox, host profiles", dataclasses.replace(base, rng="philox")),
                    ("philox, native profiles", dataclasses.replace(base, rng="philox", native_profiles=True))):
    for rep in range(2):
        t0 = time.perf_counter()
        s = engine.run_trials(spec, {name: g})
        dt = time.perf_counter() - t0
    print(f"{name} x {T} C3 {label}: {dt * 1e3:.0f} ms wall (run_trials), mean cut {s.mean_cut:.1f}", flush=True)
