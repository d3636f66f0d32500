"""A/B of the timing-spread kernels on the BASELINE C2 sigma_nu / C3 rows.

    python tools/var_rows.py [--cycles 1000] [--modes default,res0,bucket0] [--rows all|c3|c2]

Each row x mode builds a fresh plan (the PBSA_* variables are read at plan
creation) and reports the device time of the second of two whole runs, the
kernel family and updates/s.  Prints one JSON object per line.
"""
import argparse
import json
import os
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2601_14476_b200 import _native, benchmarks, streams  # noqa: E402
from paper_2601_14476_b200.annealer import Algorithm, AlgorithmConfig, derive_schedule, profile_rows  # noqa: E402
from paper_2601_14476_b200.engine import ExperimentSpec, trial_profiles  # noqa: E402
from paper_2601_14476_b200.model import maxcut_to_ising  # noqa: E402
from paper_2601_14476_b200.pbit import VariabilityConfig  # noqa: E402

ROWS = {
    "c2": [("G1", (0.0, 0.0, 0.5), 1024), ("G1", (0.0, 0.0, 1.0), 1024)],
    "c3": [("G22", (0.5, 0.5, 0.5), 4096), ("G55", (0.5, 0.5, 0.5), 4096), ("G81", (0.5, 0.5, 0.5), 4096)],
}
MODES = {"default": {}, "res0": {"PBSA_RESIDENT": "0"}, "bucket0": {"PBSA_BUCKET": "0"},
         "res1": {"PBSA_RESIDENT": "1"}}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--cycles", type=int, default=1000)
    ap.add_argument("--modes", default="default,res0,bucket0")
    ap.add_argument("--rows", default="all")
    ap.add_argument("--rng", default="replay")
    args = ap.parse_args()
    rows = ROWS["c2"] + ROWS["c3"] if args.rows == "all" else ROWS[args.rows]
    for name, sig, T in rows:
        g, _ = benchmarks.load(name)
        m = maxcut_to_ising(g)
        sch = derive_schedule(m, args.cycles, 10)
        spec = ExperimentSpec(graph=name, algo=AlgorithmConfig(Algorithm.PSA),
                              variability=VariabilityConfig(*sig), cycles=args.cycles, trials=T)
        seeds = streams.trial_seeds(0, T)
        profs = trial_profiles(spec, m.n, seeds)
        b = _native.Batch(m, sch, streams.run_keys(seeds), profile_rows=profile_rows(profs, m.n),
                          graph=g, rng=args.rng, rng_seed=streams.native_seed(0))
        for mode in args.modes.split(","):
            env = MODES[mode]
            saved = {k: os.environ.get(k) for k in env}
            os.environ.update(env)
            try:
                plan = _native.Plan(b)
                plan.run()
                ms = plan.run()
                s, best, ups = plan.summary()
                info = plan.info()
                plan.close()
            finally:
                for k, v in saved.items():
                    if v is None:
                        os.environ.pop(k, None)
                    else:
                        os.environ[k] = v
            print(json.dumps(dict(graph=name, sigma=sig, trials=T, cycles=args.cycles, mode=mode,
                                  rng=args.rng, kernel=info["kernel"], ms=round(ms, 3),
                                  upd_s=ups / ms * 1e3, mean_cut=s / T, best=best,
                                  sweep_ms_mean=info["sweep_ms_mean"])), flush=True)


if __name__ == "__main__":
    main()
