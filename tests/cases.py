"""Shared case builders for the parity tests (mirrors the reference's own
test cases: /root/reference/pkg/tests/test_annealer.py:146-152, 271-293 and
the benchmark configs of BASELINE.json)."""

from __future__ import annotations

import numpy as np

from paper_2601_14476_b200 import streams
from paper_2601_14476_b200.annealer import Algorithm, AlgorithmConfig, derive_schedule
from paper_2601_14476_b200.model import MaxCutGraph, maxcut_to_ising
from paper_2601_14476_b200.pbit import VariabilityConfig, VariabilityProfile, sample_variability


def random_graph(n, seed, weights=(-1, 1), p_edge=0.5):
    rng = np.random.default_rng(seed)
    edges = [(i, j, int(rng.choice(weights)))
             for i in range(n) for j in range(i + 1, n) if rng.random() < p_edge]
    if not edges:
        edges = [(0, 1, 1)]
    return MaxCutGraph.from_edges(n, edges)


def small_case():
    """The 14-node differential case of test_annealer.py:271-293."""
    g = random_graph(14, 9, (-2, -1, 1, 2), 0.6)
    model = maxcut_to_ising(g)
    sch = derive_schedule(model, cycles=30, t_res=5)
    varied = sample_variability(VariabilityConfig(0.3, 0.5, 0.6, t_res=5), 14,
                                np.random.default_rng(6))
    return g, model, sch, {"ideal": VariabilityProfile.ideal(14, t_res=5), "varied": varied}


# bench.npz tags -> (graph, rule, sigmas, recorded trial indices)
BENCH_CASES = {
    "g1_psa_s0": ("G1", Algorithm.PSA, (0.0, 0.0, 0.0), [0, 1, 2, 3]),
    "g1_psa_s5": ("G1", Algorithm.PSA, (0.5, 0.5, 0.5), [0, 1]),
    "g1_psa_nu1": ("G1", Algorithm.PSA, (0.0, 0.0, 1.0), [0, 1]),
    "g1_tapsa_s0": ("G1", Algorithm.TAPSA, (0.0, 0.0, 0.0), [0, 1]),
    "g1_spsa_s0": ("G1", Algorithm.SPSA, (0.0, 0.0, 0.0), [0, 1]),
    "g22_psa_s5": ("G22", Algorithm.PSA, (0.5, 0.5, 0.5), [0, 1, 1024, 4095]),
    "g55_psa_s5": ("G55", Algorithm.PSA, (0.5, 0.5, 0.5), [0, 1, 1024, 4095]),
    "g81_psa_s0": ("G81", Algorithm.PSA, (0.0, 0.0, 0.0), [0, 1, 2047, 4095]),
    "g81_psa_s5": ("G81", Algorithm.PSA, (0.5, 0.5, 0.5), [0]),
}


def bench_inputs(graph, kind, sig, trials, cycles=1000):
    """(model, schedule, algo cfg, seeds, profiles or None, keys) for given
    global trial indices, drawn exactly like engine.run_trials."""
    model = maxcut_to_ising(graph)
    sch = derive_schedule(model, cycles, 10)
    cfg = VariabilityConfig(*sig)
    seeds = [streams.trial_seed(0, k) for k in trials]
    if cfg.is_ideal:
        profs = None
    else:
        profs = [sample_variability(cfg, graph.n, np.random.default_rng(streams.profile_seed(s)))
                 for s in seeds]
    keys = [streams.run_key(s) for s in seeds]
    return model, sch, AlgorithmConfig(kind), seeds, profs, keys
