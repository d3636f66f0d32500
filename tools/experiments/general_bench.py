"""Development timing of the GENERAL device path on the variability configs
(BASELINE C2/C3 shapes). Prints device ms and updates/s per config."""
import sys, time
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[2]))
import numpy as np
from paper_2601_14476_b200 import _native, benchmarks, streams
from paper_2601_14476_b200.annealer import Algorithm, AlgorithmConfig, derive_schedule, profile_rows
from paper_2601_14476_b200.engine import ExperimentSpec, trial_profiles
from paper_2601_14476_b200.model import maxcut_to_ising
from paper_2601_14476_b200.pbit import VariabilityConfig

def run(name, kind, sig, T, cycles=1000, alpha=4):
    g, _ = benchmarks.load(name)
    m = maxcut_to_ising(g)
    sch = derive_schedule(m, cycles, 10)
    spec = ExperimentSpec(graph=name, algo=AlgorithmConfig(kind, alpha=alpha), variability=VariabilityConfig(*sig), cycles=cycles, trials=T)
    seeds = streams.trial_seeds(0, T)
    t0 = time.perf_counter()
    profs = trial_profiles(spec, m.n, seeds)
    t1 = time.perf_counter()
    b = _native.Batch(m, sch, streams.run_keys(seeds), profile_rows=profile_rows(profs, m.n), graph=g,
                      algo_code=kind.code, alpha=spec.algo.kernel_alpha, p_stall=0.5)
    plan = _native.Plan(b)
    plan.run()
    ms = min(plan.run() for _ in range(2))
    s, best, ups = plan.summary()
    info = plan.info()
    print(f"{name} {kind.value} sigma={sig} T={T}: path={info['path']} device {ms:.1f} ms, "
          f"{ups/ms*1e3:.3g} upd/s, launches {info['launches']}, profile sampling {t1-t0:.2f} s, mean cut {s/T:.1f}", flush=True)

if __name__ == "__main__" and len(sys.argv) > 1:
    name, kind, sig, T, cyc = sys.argv[1:6]
    run(name, Algorithm(kind), tuple(float(x) for x in sig.split(",")), int(T), int(cyc))
elif __name__ == "__main__":
  for cfg in [("G1", Algorithm.PSA, (0.5, 0.5, 0.5), 1024), ("G1", Algorithm.PSA, (0, 0, 1.0), 1024),
            ("G1", Algorithm.TAPSA, (0, 0, 0), 1024), ("G1", Algorithm.SPSA, (0, 0, 0), 1024),
            ("G55", Algorithm.PSA, (0.5, 0.5, 0.5), 4096), ("G22", Algorithm.PSA, (0.5, 0.5, 0.5), 4096),
            ("G81", Algorithm.TAPSA, (0, 0, 0), 4096)]:
    run(*cfg)
