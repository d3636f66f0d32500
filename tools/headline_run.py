"""One run of the bench plan (G81 x 4096, replayed stream) or a C3 plan, for
ncu captures:  python tools/headline_run.py [cycles] [graph] [sigma] [trials]"""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2601_14476_b200 import _native, benchmarks, streams  # noqa: E402
from paper_2601_14476_b200.annealer import Algorithm, AlgorithmConfig, derive_schedule, profile_rows  # noqa: E402
from paper_2601_14476_b200.engine import ExperimentSpec, trial_profiles  # noqa: E402
from paper_2601_14476_b200.model import maxcut_to_ising  # noqa: E402
from paper_2601_14476_b200.pbit import VariabilityConfig  # noqa: E402

cyc = int(sys.argv[1]) if len(sys.argv) > 1 else 20
name = sys.argv[2] if len(sys.argv) > 2 else "G81"
sig = tuple(float(x) for x in sys.argv[3].split(",")) if len(sys.argv) > 3 else (0.0, 0.0, 0.0)
T = int(sys.argv[4]) if len(sys.argv) > 4 else 4096
g, _ = benchmarks.load(name)
m = maxcut_to_ising(g)
sch = derive_schedule(m, cyc, 10)
seeds = streams.trial_seeds(0, T)
spec = ExperimentSpec(graph=name, algo=AlgorithmConfig(Algorithm.PSA), variability=VariabilityConfig(*sig),
                      cycles=cyc, trials=T)
profs = trial_profiles(spec, m.n, seeds)
b = _native.Batch(m, sch, streams.run_keys(seeds), profile_rows=profile_rows(profs, m.n), graph=g)
plan = _native.Plan(b)
ms = plan.run()
print(name, sig, T, cyc, f"{ms:.2f} ms", plan.info(), plan.layout())
