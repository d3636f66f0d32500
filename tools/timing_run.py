"""One short anneal of a timing-spread config (for ncu captures of
packed_sweep_timing):  python tools/timing_run.py G55 0.5,0.5,0.5 4096 20 [philox [tapsa|spsa]]"""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2601_14476_b200 import _native, benchmarks, streams  # noqa: E402
from paper_2601_14476_b200.annealer import Algorithm, AlgorithmConfig, derive_schedule, profile_rows  # noqa: E402
from paper_2601_14476_b200.engine import ExperimentSpec, trial_profiles  # noqa: E402
from paper_2601_14476_b200.model import maxcut_to_ising  # noqa: E402
from paper_2601_14476_b200.pbit import VariabilityConfig  # noqa: E402

name, sig, T, cyc = sys.argv[1], tuple(float(x) for x in sys.argv[2].split(",")), int(sys.argv[3]), int(sys.argv[4])
rng = sys.argv[5] if len(sys.argv) > 5 else "replay"
algo = Algorithm(sys.argv[6]) if len(sys.argv) > 6 else Algorithm.PSA
g, _ = benchmarks.load(name)
m = maxcut_to_ising(g)
sch = derive_schedule(m, cyc, 10)
spec = ExperimentSpec(graph=name, algo=AlgorithmConfig(algo), variability=VariabilityConfig(*sig),
                      cycles=cyc, trials=T)
seeds = streams.trial_seeds(0, T)
profs = trial_profiles(spec, m.n, seeds)
b = _native.Batch(m, sch, streams.run_keys(seeds), profile_rows=profile_rows(profs, m.n), graph=g,
                  algo_code=spec.algo.kind.code, alpha=spec.algo.alpha, p_stall=spec.algo.p_stall,
                  rng=rng, rng_seed=streams.native_seed(0))
plan = _native.Plan(b)
ms = plan.run()
ms = plan.run()
s, best, ups = plan.summary()
lay = plan.layout()
print(f"{name} {sig} T={T} cycles={cyc} {rng}: {ms:.2f} ms, {ups / ms * 1e3:.3g} upd/s, pw={lay['phase_words']} "
      f"chains={lay['chains']} wpw={lay['warps_per_word']} {plan.info()}")
