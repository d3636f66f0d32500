"""Generate tests/golden/fullbatch.npz: per-trial digests of whole benchmark
batches at the sizes the BASELINE configs (and bench.py) run, from the ORACLE.

    python tests/golden/make_fullbatch.py [tag ...]

The oracle (oracle/psa_oracle.c) is pinned bit-for-bit to the reference by
tests/golden/bench.npz (make_golden.py, which imports the reference); the
reference itself would need ~1.5 h of numba time for the G81 batch alone, so
the whole batches come from the oracle, and the GPU tests
(tests/test_gpu_parity.py::test_full_batch_*) compare the CUDA path's exact
launch shapes against these digests trial by trial.  Inputs are drawn exactly
as engine.run_trials draws them (/root/reference/pkg/src/pbitsa/engine.py:101-116):
trial k has seed trial_seed(0, k) and profile default_rng(profile_seed(seed)).

Per config and trial: final cut, best cut, sum of the cut trace, sum of the
update counts, CRC32 of the final spins (int8 bytes) and CRC32 of the final
inputs (float64 bytes).
"""

from __future__ import annotations

import os
import sys
import time
import zlib
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))

from cases import bench_inputs  # noqa: E402
from oracle import oracle as orc  # noqa: E402
from paper_2601_14476_b200 import benchmarks  # noqa: E402
from paper_2601_14476_b200.annealer import Algorithm  # noqa: E402

OUT = Path(__file__).resolve().parent / "fullbatch.npz"

# tag -> (graph, sigmas, trials): BASELINE C4 (the bench workload), C3 and C2 sigma_nu
CONFIGS = {
    "c4_g81": ("G81", (0.0, 0.0, 0.0), 4096),
    "c3_g22": ("G22", (0.5, 0.5, 0.5), 4096),
    "c3_g55": ("G55", (0.5, 0.5, 0.5), 4096),
    "c2_g1_nu1": ("G1", (0.0, 0.0, 1.0), 1024),
}


def digest(out):
    T = out["spins"].shape[0]
    return {
        "final_cut": out["cut_trace"][:, -1].astype(np.int64),
        "best": np.asarray(out["best_cut"], np.int64),
        "cut_sum": out["cut_trace"].sum(axis=1).astype(np.int64),
        "counts_sum": out["counts"].sum(axis=1).astype(np.int64),
        "spins_crc": np.array([zlib.crc32(np.ascontiguousarray(out["spins"][t]).tobytes())
                               for t in range(T)], np.uint32),
        "inputs_crc": np.array([zlib.crc32(np.ascontiguousarray(out["inputs"][t]).tobytes())
                                for t in range(T)], np.uint32),
    }


def run(tag, chunk=256):
    name, sig, trials = CONFIGS[tag]
    graph = benchmarks.load(name)[0]
    parts = []
    t0 = time.time()
    for lo in range(0, trials, chunk):
        ks = list(range(lo, min(trials, lo + chunk)))
        model, sch, cfg, _, profs, keys = bench_inputs(graph, Algorithm.PSA, sig, ks)
        from paper_2601_14476_b200.pbit import VariabilityProfile
        out = orc.anneal_batch(model, sch, "psa", profs or VariabilityProfile.ideal(model.n), keys,
                               graph=graph, threads=os.cpu_count())
        parts.append(digest(out))
        print(f"{tag}: {ks[-1] + 1}/{trials} trials, {time.time() - t0:.0f} s", flush=True)
    return {k: np.concatenate([p[k] for p in parts]) for k in parts[0]}


def main():
    tags = sys.argv[1:] or list(CONFIGS)
    orc.build()
    data = dict(np.load(OUT)) if OUT.exists() else {}
    for tag in tags:
        for k, v in run(tag).items():
            data[f"{tag}_{k}"] = v
        np.savez_compressed(OUT, **data)


if __name__ == "__main__":
    main()
