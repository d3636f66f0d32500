"""Host-side API mirror: same names, validation and arithmetic as the
reference package (patterns of /root/reference/pkg/tests/test_streams.py,
test_model.py, test_pbit.py, test_gset.py, test_annealer.py:43-67 and
test_engine.py:101-159).  No GPU needed."""

from __future__ import annotations

import io
import itertools
import math
import statistics

import numpy as np
import pytest

import paper_2601_14476_b200 as pb
from paper_2601_14476_b200 import benchmarks, streams
from paper_2601_14476_b200.annealer import AlgorithmConfig, Algorithm, AnnealSchedule, derive_schedule
from paper_2601_14476_b200.engine import SWEEP_AXES, ExperimentSpec, summarize

REFERENCE_ALL = [
    "Algorithm", "AlgorithmConfig", "AnnealSchedule", "AnnealerState", "ExperimentSpec",
    "ExperimentSummary", "GsetFile", "GsetParseError", "IsingModel", "MaxCutGraph", "TraceRecord",
    "TrialResult", "VariabilityConfig", "VariabilityProfile", "bundled_best_known",
    "compute_raw_input", "cut_value", "derive_schedule", "energy", "load_best_known",
    "load_best_known_path", "local_field", "maxcut_to_ising", "next_input_psa", "next_input_spsa",
    "next_input_tapsa", "parse_gset", "parse_gset_path", "pbit_update", "random_state",
    "run_anneal", "run_trials", "sample_variability", "serialize_gset", "summarize", "sweep",
    "to_graph"]


def test_public_api_matches_reference_names():
    assert sorted(pb.__all__) == sorted(REFERENCE_ALL)
    for name in REFERENCE_ALL:
        assert hasattr(pb, name)


# ---------------------------------------------------------------- streams

def test_stream_kats(golden_streams):
    assert streams.mix64(1) == 0x10A81D8AD3D870A3
    assert streams.mix64(2**64 - 1) == 0x76D4311972CA5AB3
    assert streams.stream_u64(42, 3, 7, 123) == 0xB71C3C338A17B8FA
    assert streams.stream_u64(2**64 - 1, 6, 0, 0) == 0x7C21402D9AC96F99
    assert streams.uniform01(0, 2, 0, 0) == 0.004799147651941116
    assert streams.run_key(0) == 0x9D9A85784BF1C21D
    assert streams.trial_seed(0, 1) == 0xDA28150A69217582
    assert streams.profile_seed(12345) == 0xB62E0384700FB443
    for key, tag, a, b, want, u in golden_streams["grid"]:
        assert streams.stream_u64(int(key), tag, int(a), b) == int(want)
        assert streams.uniform01(int(key), tag, int(a), b) == float.fromhex(u)
    for b, k, want in golden_streams["trial_seed"]:
        assert streams.trial_seed(b, k) == int(want)
    with pytest.raises(ValueError):
        streams.trial_seed(0, -1)


def test_vectorised_key_helpers_match_scalar():
    seeds = streams.trial_seeds(7, 50)
    assert seeds == [streams.trial_seed(7, k) for k in range(50)]
    assert streams.trial_seeds(7, 10, 40) == seeds[40:]
    keys = streams.run_keys(seeds)
    assert [int(k) for k in keys] == [streams.run_key(s) for s in seeds]


# ------------------------------------------------------------------ model

def _all_states(n):
    return ((np.arange(2 ** n)[:, None] >> np.arange(n)) & 1).astype(np.int8) * 2 - 1


def test_energy_cut_identity_exhaustive():
    rng = np.random.default_rng(0)
    for _ in range(20):
        n = int(rng.integers(2, 9))
        edges = [(i, j, int(rng.choice([-2, -1, 1, 3]))) for i, j in itertools.combinations(range(n), 2)
                 if rng.random() < 0.6] or [(0, 1, 1)]
        g = pb.MaxCutGraph.from_edges(n, edges)
        m = pb.maxcut_to_ising(g)
        for s in _all_states(n):
            assert 2 * pb.cut_value(g, s) - g.total_weight() == pytest.approx(-pb.energy(m, s))


def test_csr_is_symmetric_sorted_and_complete():
    g = pb.MaxCutGraph.from_edges(6, [(0, 3, 1), (1, 2, -1), (4, 5, 2), (0, 1, 1), (2, 5, 1)])
    m = pb.maxcut_to_ising(g)
    for i in range(6):
        cols = m.indices[m.indptr[i]:m.indptr[i + 1]]
        assert list(cols) == sorted(cols)
    dense = np.zeros((6, 6))
    for i in range(6):
        for k in range(m.indptr[i], m.indptr[i + 1]):
            dense[i, m.indices[k]] = m.values[k]
    assert np.array_equal(dense, dense.T)
    assert np.count_nonzero(dense) == 2 * g.m


def test_local_field_and_raw_input():
    m = pb.IsingModel.from_edges(3, [(0, 1, 1.0), (1, 2, -2.0)], h=[0.5, -1.0, 2.0])
    s = np.array([1, -1, 1], dtype=np.int8)
    assert pb.compute_raw_input(m, s, 1) == -1.0 + 1.0 - 2.0
    assert pb.local_field(m, s, 0) == 0.5 - 1.0


def test_model_validation():
    with pytest.raises(ValueError, match="self-loop"):
        pb.MaxCutGraph.from_edges(3, [(1, 1, 1)])
    with pytest.raises(ValueError, match="duplicate"):
        pb.MaxCutGraph.from_edges(3, [(0, 1, 1), (1, 0, 1)])
    with pytest.raises(ValueError, match="out of range"):
        pb.MaxCutGraph.from_edges(3, [(0, 3, 1)])
    with pytest.raises(ValueError, match="finite"):
        pb.IsingModel.from_edges(2, [(0, 1, float("nan"))])
    with pytest.raises(ValueError):
        pb.cut_value(pb.MaxCutGraph.from_edges(2, [(0, 1, 1)]), np.array([1, 0]))


# ------------------------------------------------------------------- pbit

def test_pbit_rule_and_sampler():
    assert pb.pbit_update(0.0, 0.0) == 1            # sign(0) = +1
    assert pb.pbit_update(-100.0, -0.5) == -1
    cfg = pb.VariabilityConfig(0.3, 0.4, 0.5)
    prof = pb.sample_variability(cfg, 1000, np.random.default_rng(5))
    rng = np.random.default_rng(5)
    lam = 1.0 + 0.3 * rng.standard_normal(1000)
    delta = 0.4 * rng.standard_normal(1000)
    nu = 0.5 * rng.standard_normal(1000)
    assert np.array_equal(prof.lam, lam) and np.array_equal(prof.delta, delta)
    assert np.array_equal(prof.period, np.maximum(1, np.rint(10 * (1 + nu))).astype(np.int64))
    ideal = pb.sample_variability(pb.VariabilityConfig(), 50, np.random.default_rng(1))
    assert ideal.is_ideal() and pb.VariabilityProfile.ideal(50).is_ideal()
    with pytest.raises(ValueError):
        pb.VariabilityConfig(sigma_nu=-1)


# ------------------------------------------------------------------- gset

def test_gset_round_trip_and_errors():
    text = "3 2\n1 2 1\n2 3 -1\n"
    gf = pb.parse_gset(io.StringIO(text), name="x")
    assert (gf.n, gf.m, gf.edges) == (3, 2, [(1, 2, 1), (2, 3, -1)])
    assert pb.serialize_gset(gf) == text
    g = pb.to_graph(gf)
    assert g.edge_list() == [(0, 1, 1), (1, 2, -1)]
    for bad, line in [("", 1), ("3\n", 1), ("3 1\n1 1 1\n", 2), ("3 2\n1 2 1\n", 2),
                      ("3 1\n1 4 1\n", 2), ("3 1\n1 2 x\n", 2)]:
        with pytest.raises(pb.GsetParseError) as e:
            pb.parse_gset(io.StringIO(bad))
        assert e.value.line == line
    reg = pb.bundled_best_known()
    assert reg["G1"] == 11624 and reg["G81"] == 14030
    with pytest.raises(ValueError, match="duplicate"):
        pb.load_best_known(["G1 1", "G1 2"])


def test_analog_generator_is_pinned_to_reference(golden_analogs):
    import hashlib
    for name, info in golden_analogs.items():
        g = pb.to_graph(benchmarks.make_analog(name))
        digest = hashlib.sha256(np.stack([g.edge_i, g.edge_j, g.edge_w]).astype(np.int64).tobytes())
        assert (g.n, g.m) == (info["n"], info["m"])
        assert digest.hexdigest() == info["sha256"], name
        if info["best_known_analog"]:
            assert benchmarks.ANALOG_BEST_KNOWN[name] == info["best_known_analog"]


# --------------------------------------------------------------- schedule

def test_schedule_closed_forms():
    tri = pb.maxcut_to_ising(pb.MaxCutGraph.from_edges(3, [(0, 1, 1), (1, 2, 1), (0, 2, 1)]))
    sch = derive_schedule(tri, cycles=3)
    assert sch.i0_min == pytest.approx(0.15, rel=1e-12) and sch.beta == pytest.approx(0.1, rel=1e-12)
    path = pb.maxcut_to_ising(pb.MaxCutGraph.from_edges(3, [(0, 1, 2), (1, 2, -3)]))
    assert derive_schedule(path, 5).i0_min == pytest.approx(0.9 / (10 + 2 * math.sqrt(19)), rel=1e-12)
    seq = AnnealSchedule(0.2, 20.0, 0.01 ** (1 / 7), 8, 10).i0_sequence()
    assert seq[0] == 0.2 and abs(seq[-1] - 20) / 20 <= 1e-9 and np.all(np.diff(seq) > 0)
    with pytest.raises(ValueError, match="zero"):
        derive_schedule(pb.maxcut_to_ising(pb.MaxCutGraph.from_edges(3, [(0, 1, 0)])), 10)
    with pytest.raises(ValueError, match="beta"):
        AnnealSchedule(i0_min=0.1, i0_max=10.0, beta=0.9, cycles=4, t_res=10)


def test_input_rules_and_config_validation():
    assert pb.next_input_psa(3.0, 0.5) == 1.5
    assert pb.next_input_tapsa([1.0, 3.0], 2.0) == 4.0
    assert pb.next_input_spsa(7.0, 3.0, 2.0, 0.49, 0.5) == 7.0
    assert pb.next_input_spsa(7.0, 3.0, 2.0, 0.50, 0.5) == 6.0
    with pytest.raises(ValueError):
        pb.next_input_tapsa([], 1.0)
    with pytest.raises(ValueError):
        AlgorithmConfig(Algorithm.TAPSA, alpha=0)
    assert AlgorithmConfig(Algorithm.TAPSA, alpha=3).kernel_alpha == 3
    assert AlgorithmConfig(Algorithm.SPSA, alpha=3).kernel_alpha == 1


# ----------------------------------------------------------------- engine

def test_spec_summary_and_sweep_validation():
    with pytest.raises(ValueError):
        ExperimentSpec(graph="g", algo=AlgorithmConfig(Algorithm.PSA), cycles=1)
    with pytest.raises(ValueError):
        ExperimentSpec(graph="g", algo=AlgorithmConfig(Algorithm.PSA), trials=0)
    assert SWEEP_AXES == ("sigma_lambda", "sigma_delta", "sigma_nu")

    class R:
        def __init__(self, c, e):
            self.final_cut, self.final_energy = c, e
    rs = [R(c, -c) for c in (10, 12, 15, 9)]
    s = summarize(rs, best_known=20)
    assert s.mean_cut == pytest.approx(statistics.fmean([10, 12, 15, 9]))
    assert s.std_cut == pytest.approx(statistics.stdev([10, 12, 15, 9]))
    assert s.normalized_mean_cut == pytest.approx(s.mean_cut / 20)
    assert summarize(rs[:1]).std_cut == 0.0
    with pytest.raises(ValueError, match="finite and positive"):
        summarize(rs, best_known=-1)
    spec = ExperimentSpec(graph="g", algo=AlgorithmConfig(Algorithm.PSA))
    with pytest.raises(ValueError, match="axis"):
        pb.sweep(spec, "cycles", [1.0], {})
    with pytest.raises(KeyError, match="unknown graph"):
        pb.run_trials(spec, {})


def test_parallel_profile_sampling_is_reentrant():
    """Concurrent sample_profiles calls (run_trials_devices runs one per device
    thread) each fill their own buffers: identical to sequential calls and to
    the reference's one-trial-at-a-time draws (engine.py:107-112)."""
    from concurrent.futures import ThreadPoolExecutor

    from paper_2601_14476_b200 import streams
    from paper_2601_14476_b200.pbit import VariabilityConfig, sample_variability
    from paper_2601_14476_b200.profiles import sample_profiles
    cfg = VariabilityConfig(0.5, 0.5, 0.5)
    seed_sets = [streams.trial_seeds(b, 900) for b in (0, 5, 9)]
    seq = [sample_profiles(cfg, 5000, s) for s in seed_sets]
    with ThreadPoolExecutor(3) as ex:
        par = list(ex.map(lambda s: sample_profiles(cfg, 5000, s), seed_sets))
    for a, b in zip(seq, par):
        for x, y in zip(a, b):
            assert np.array_equal(x, y)
    for k in (0, 899):
        p = sample_variability(cfg, 5000, np.random.default_rng(streams.profile_seed(seed_sets[1][k])))
        assert np.array_equal(par[1][0][k], p.lam) and np.array_equal(par[1][2][k], p.period)
