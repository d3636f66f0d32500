"""Generate the golden fixtures in tests/golden/ from the REFERENCE package.

Run in the build container (the only place /root/reference exists):

    NUMBA_CACHE_DIR=/tmp/nc PYTHONPATH=/root/reference/pkg/src \
        python tests/golden/make_golden.py

It imports the reference ``pbitsa`` package and its test helpers
(``/root/reference/pkg/tests/analogs.py``, ``solvers.py``) and records their
outputs; nothing from the reference is copied into this repository.  The
fixtures pin the oracle (tests/test_oracle_golden.py) and, through it, the
CUDA path (tests/test_gpu_parity.py) to the reference's own behaviour.

Outputs:
  streams.json   hash KATs (/root/reference/pkg/tests/test_streams.py:26-45)
                 plus a (key, tag, a, b) grid evaluated by pbitsa.streams
  analogs.json   per-benchmark analog sizes, an edge-list digest (so the
                 repo's own analog generator is pinned) and the Metropolis
                 denominators of tests/solvers.reference_best_cut
  small.npz      14-node differential case of test_annealer.py:271-293:
                 all three rules x {ideal, varied} x seeds {0, 1}, full outputs
  bench.npz      benchmark-sized runs at cycles=1000 (G1/G22/G55/G81 analogs)
  acceptance.npz per-trial results of the reference's acceptance criteria 4, 5
                 and 7 (variability runs of all three rules); `make_golden.py
                 acceptance` regenerates only this file
"""

from __future__ import annotations

import hashlib
import json
import sys
from pathlib import Path

import numpy as np

REF_TESTS = Path("/root/reference/pkg/tests")
sys.path.insert(0, str(REF_TESTS))

import analogs  # noqa: E402  (reference test helper)
import solvers  # noqa: E402
from pbitsa import streams  # noqa: E402
from pbitsa.annealer import (  # noqa: E402
    Algorithm, AlgorithmConfig, derive_schedule, run_anneal)
from pbitsa.engine import ExperimentSpec, run_trials  # noqa: E402
from pbitsa.gset import to_graph  # noqa: E402
from pbitsa.model import MaxCutGraph, maxcut_to_ising  # noqa: E402
from pbitsa.pbit import VariabilityConfig, VariabilityProfile, sample_variability  # noqa: E402

OUT = Path(__file__).resolve().parent
CYCLES = 1000


def edge_digest(g) -> str:
    arr = np.stack([g.edge_i, g.edge_j, g.edge_w]).astype(np.int64)
    return hashlib.sha256(arr.tobytes()).hexdigest()


def make_streams() -> None:
    grid = []
    keys = [0, 1, 7, 2**31, 2**63, 2**64 - 1, 0xDEADBEEFCAFEBABE]
    for key in keys:
        for tag in (1, 2, 3, 4, 5, 6):
            for a in (0, 1, 13, 10**6, 2**40):
                for b in (0, 3, 999983):
                    grid.append([str(key), tag, str(a), b, str(streams.stream_u64(key, tag, a, b)),
                                 streams.uniform01(key, tag, a, b).hex()])
    data = {
        "mix64": {str(z): str(streams.mix64(z)) for z in (0, 1, 2**64 - 1, 0x123456789ABCDEF0)},
        "run_key": {str(s): str(streams.run_key(s)) for s in (0, 1, 12345, 2**64 - 1)},
        "trial_seed": [[b, k, str(streams.trial_seed(b, k))] for b in (0, 1) for k in range(8)],
        "profile_seed": {str(s): str(streams.profile_seed(s)) for s in (0, 12345)},
        "grid": grid,
    }
    (OUT / "streams.json").write_text(json.dumps(data, indent=0))


def make_analogs() -> dict:
    info = {}
    for name in analogs.BENCHMARKS:
        g = to_graph(analogs.make_analog(name))
        denom = solvers.reference_best_cut(g) if name in ("G1", "G22", "G55", "G81") else None
        info[name] = {"n": g.n, "m": g.m, "sha256": edge_digest(g), "total_weight": g.total_weight(),
                      "best_known_analog": denom}
        print(name, info[name], flush=True)
    (OUT / "analogs.json").write_text(json.dumps(info, indent=1))
    return info


def _small_graph() -> MaxCutGraph:
    # test_annealer.py:146-152 with (n=14, seed=9, weights=(-2,-1,1,2), p_edge=0.6)
    rng = np.random.default_rng(9)
    edges = [(i, j, int(rng.choice((-2, -1, 1, 2))))
             for i in range(14) for j in range(i + 1, 14) if rng.random() < 0.6]
    return MaxCutGraph.from_edges(14, edges)


def make_small() -> None:
    g = _small_graph()
    model = maxcut_to_ising(g)
    sch = derive_schedule(model, cycles=30, t_res=5)
    varied = sample_variability(VariabilityConfig(0.3, 0.5, 0.6, t_res=5), 14,
                                np.random.default_rng(6))
    ideal = VariabilityProfile.ideal(14, t_res=5)
    out = {"edges": np.stack([g.edge_i, g.edge_j, g.edge_w]),
           "schedule": np.array([sch.i0_min, sch.i0_max, sch.beta, sch.cycles, sch.t_res]),
           "var_lam": varied.lam, "var_delta": varied.delta, "var_period": varied.period}
    for pname, prof in (("ideal", ideal), ("varied", varied)):
        for kind in Algorithm:
            cfg = AlgorithmConfig(kind, alpha=3, p_stall=0.4)
            for seed in (0, 1):
                r = run_anneal(model, sch, cfg, prof, seed=seed, graph=g)
                p = f"{pname}_{kind.value}_{seed}_"
                out[p + "spins"] = r.final_state.spins
                out[p + "inputs"] = r.final_state.inputs
                out[p + "hist"] = r.final_state.ti_history
                out[p + "counts"] = r.update_counts
                out[p + "i0"] = r.i0_trace
                out[p + "energy"] = r.energy_trace
                out[p + "cut"] = r.cut_trace
                out[p + "best"] = np.array(r.best_cut)
    np.savez_compressed(OUT / "small.npz", **out)


def _profile(cfg: VariabilityConfig, n: int, k: int):
    seed = streams.trial_seed(0, k)
    return seed, sample_variability(cfg, n, np.random.default_rng(streams.profile_seed(seed)))


def make_bench() -> None:
    out = {}
    # (tag, graph, algo, sigma triple, trial indices recorded in full)
    cases = [
        ("g1_psa_s0", "G1", Algorithm.PSA, (0.0, 0.0, 0.0), [0, 1, 2, 3]),
        ("g1_psa_s5", "G1", Algorithm.PSA, (0.5, 0.5, 0.5), [0, 1]),
        ("g1_psa_nu1", "G1", Algorithm.PSA, (0.0, 0.0, 1.0), [0, 1]),
        ("g1_tapsa_s0", "G1", Algorithm.TAPSA, (0.0, 0.0, 0.0), [0, 1]),
        ("g1_spsa_s0", "G1", Algorithm.SPSA, (0.0, 0.0, 0.0), [0, 1]),
        ("g22_psa_s5", "G22", Algorithm.PSA, (0.5, 0.5, 0.5), [0, 1, 1024, 4095]),
        ("g55_psa_s5", "G55", Algorithm.PSA, (0.5, 0.5, 0.5), [0, 1, 1024, 4095]),
        ("g81_psa_s0", "G81", Algorithm.PSA, (0.0, 0.0, 0.0), [0, 1, 2047, 4095]),
        ("g81_psa_s5", "G81", Algorithm.PSA, (0.5, 0.5, 0.5), [0]),
    ]
    graphs = {}
    for tag, name, kind, sig, trials in cases:
        if name not in graphs:
            graphs[name] = to_graph(analogs.make_analog(name))
        g = graphs[name]
        model = maxcut_to_ising(g)
        sch = derive_schedule(model, CYCLES, 10)
        cfg = VariabilityConfig(*sig)
        algo = AlgorithmConfig(kind)
        for k in trials:
            seed, prof = _profile(cfg, g.n, k)
            r = run_anneal(model, sch, algo, prof, seed, graph=g)
            p = f"{tag}_{k}_"
            out[p + "spins"] = r.final_state.spins
            out[p + "cut"] = r.cut_trace.astype(np.int32)
            out[p + "best"] = np.array(r.best_cut)
            out[p + "counts_sum"] = np.array(int(r.update_counts.sum()))
            out[p + "inputs"] = r.final_state.inputs
            if k == 0:
                out[p + "lam3"] = prof.lam[:3]
                out[p + "delta3"] = prof.delta[:3]
                out[p + "period8"] = prof.period[:8]
        print(tag, "done", flush=True)
    # 100-trial summaries on G1 at sigma = 0 (acceptance criterion 3 numbers,
    # /root/reference/pkg/test_output.txt:148)
    for kind in Algorithm:
        spec = ExperimentSpec(graph="G1", algo=AlgorithmConfig(kind), cycles=CYCLES, trials=100,
                              base_seed=0, threads=8)
        s = run_trials(spec, {"G1": graphs["G1"]})
        out[f"g1_{kind.value}_s0_final_cuts100"] = np.array([r.final_cut for r in s.results])
        out[f"g1_{kind.value}_s0_best_cuts100"] = np.array([r.best_cut for r in s.results])
        print(kind.value, "summary mean", s.mean_cut, flush=True)
    np.savez_compressed(OUT / "bench.npz", **out)


def make_acceptance() -> None:
    """Per-trial results behind the reference's acceptance criteria 4, 5 and 7
    (/root/reference/pkg/tests/test_acceptance.py:156-230): the variability
    runs of the plain, time-averaged and stalled rules."""
    from pbitsa.engine import sweep
    out = {}
    g1 = to_graph(analogs.make_analog("G1"))
    # criterion 4: plain rule, sigma_nu in {0, 1}, 50 trials
    for sn in (0.0, 1.0):
        spec = ExperimentSpec(graph="G1", algo=AlgorithmConfig(Algorithm.PSA),
                              variability=VariabilityConfig(sigma_nu=sn, t_res=10),
                              cycles=CYCLES, trials=50, base_seed=0, threads=8)
        s = run_trials(spec, {"G1": g1})
        out[f"c4_nu{sn:g}_final_cuts"] = np.array([r.final_cut for r in s.results])
        print("criterion 4", sn, s.mean_cut, flush=True)
    # criterion 5: time-averaged rule (alpha 4), sweep sigma_delta in {0, 0.5, 1}, 100 trials
    spec = ExperimentSpec(graph="G1", algo=AlgorithmConfig(Algorithm.TAPSA, alpha=4),
                          cycles=CYCLES, trials=100, base_seed=0, threads=8)
    for v, s in zip((0.0, 0.5, 1.0), sweep(spec, "sigma_delta", [0.0, 0.5, 1.0], {"G1": g1})):
        out[f"c5_delta{v:g}_final_cuts"] = np.array([r.final_cut for r in s.results])
        print("criterion 5", v, s.mean_cut, flush=True)
    # criterion 7 specs (120 cycles, 6 trials, seed 2): full cut traces
    for name, kind, sig in (("G1", Algorithm.PSA, (0.0, 0.0, 0.3)),
                            ("G47", Algorithm.TAPSA, (0.5, 0.0, 0.0)),
                            ("G48", Algorithm.SPSA, (0.0, 0.5, 0.0))):
        g = to_graph(analogs.make_analog(name))
        spec = ExperimentSpec(graph=name, algo=AlgorithmConfig(kind), cycles=120, trials=6,
                              base_seed=2, variability=VariabilityConfig(*sig), threads=2)
        s = run_trials(spec, {name: g})
        out[f"c7_{name}_{kind.value}_cut_traces"] = np.stack([r.cut_trace for r in s.results])
        out[f"c7_{name}_{kind.value}_energy_traces"] = np.stack([r.energy_trace for r in s.results])
        print("criterion 7", name, kind.value, s.mean_cut, flush=True)
    np.savez_compressed(OUT / "acceptance.npz", **out)


if __name__ == "__main__":
    if sys.argv[1:] == ["acceptance"]:
        make_acceptance()
        raise SystemExit
    make_streams()
    make_small()
    make_analogs()
    make_bench()
    make_acceptance()
