"""CUDA path vs the reference (golden fixtures) and the oracle, bit-for-bit.

Every test here calls the product through the C ABI (libpbsa.so via the
package API) on a real GPU.  Bar: spins, cut traces, update counts, inputs,
histories, best cuts and i0 traces are bit-identical; energies are compared
exactly too (they are integer sums for every integer-weight case, and the
fp64 case keeps the reference's accumulation order).
"""

from __future__ import annotations

import dataclasses
import math

import numpy as np
import pytest

from cases import BENCH_CASES, bench_inputs, random_graph, small_case
from paper_2601_14476_b200 import _native, engine, streams
from paper_2601_14476_b200.annealer import (Algorithm, AlgorithmConfig, AnnealSchedule,
                                            derive_schedule, profile_rows, run_anneal)
from paper_2601_14476_b200.model import IsingModel, maxcut_to_ising
from paper_2601_14476_b200.pbit import VariabilityConfig, VariabilityProfile, sample_variability

pytestmark = pytest.mark.gpu

M64 = (1 << 64) - 1


def _batch(model, sch, cfg, keys, profs, graph):
    b = _native.Batch(model, sch, keys, profile_rows=profile_rows(profs, model.n), graph=graph,
                      algo_code=cfg.kind.code, alpha=cfg.kernel_alpha, p_stall=cfg.p_stall)
    return _native.anneal_batch(b)[0]


def test_device_hash_matches_reference_kats(golden_streams):
    rows = golden_streams["grid"]
    keys = [int(r[0]) for r in rows]
    tags = [r[1] for r in rows]
    a = [int(r[2]) for r in rows]
    b = [r[3] for r in rows]
    got = _native.debug_stream_u64(keys, tags, a, b)
    assert [int(x) for x in got] == [int(r[4]) for r in rows]
    kat = _native.debug_stream_u64([42, 0], [3, 1], [7, 0], [123, 0])
    assert int(kat[0]) == 0xB71C3C338A17B8FA and int(kat[1]) == 0x9D9A85784BF1C21D


def test_device_tanh_matches_host_libm():
    rng = np.random.default_rng(5)
    x = np.concatenate([rng.uniform(-25, 25, 400_000), rng.uniform(-1.5, 1.5, 400_000),
                        rng.standard_normal(200_000) * 1e-9,
                        np.ldexp(rng.uniform(0.5, 1, 200_000), rng.integers(-60, 5, 200_000))])
    got = _native.debug_tanh(x)
    want = np.array([math.tanh(v) for v in x])
    assert np.array_equal(got.view(np.uint64), want.view(np.uint64))


@pytest.mark.parametrize("pname", ["ideal", "varied"])
@pytest.mark.parametrize("kind", list(Algorithm))
def test_small_case_matches_reference(golden_small, pname, kind):
    g, model, sch, profiles = small_case()
    cfg = AlgorithmConfig(kind, alpha=3, p_stall=0.4)
    for seed in (0, 1):
        r = run_anneal(model, sch, cfg, profiles[pname], seed=seed, graph=g)
        p = f"{pname}_{kind.value}_{seed}_"
        assert np.array_equal(r.final_state.spins, golden_small[p + "spins"])
        assert np.array_equal(r.final_state.inputs, golden_small[p + "inputs"])
        assert np.array_equal(r.final_state.ti_history, golden_small[p + "hist"])
        assert np.array_equal(r.update_counts, golden_small[p + "counts"])
        assert np.array_equal(r.i0_trace, golden_small[p + "i0"])
        assert np.array_equal(r.energy_trace, golden_small[p + "energy"])
        assert np.array_equal(r.cut_trace, golden_small[p + "cut"])
        assert r.best_cut == golden_small[p + "best"]


@pytest.mark.parametrize("tag", list(BENCH_CASES))
def test_benchmark_trials_match_reference(golden_bench, bench_graphs, tag):
    name, kind, sig, trials = BENCH_CASES[tag]
    graph = bench_graphs(name)
    model, sch, cfg, seeds, profs, keys = bench_inputs(graph, kind, sig, trials)
    out = _batch(model, sch, cfg, keys, profs, graph)
    for idx, k in enumerate(trials):
        p = f"{tag}_{k}_"
        assert np.array_equal(out["spins"][idx], golden_bench[p + "spins"]), p
        assert np.array_equal(out["cut_trace"][idx], golden_bench[p + "cut"]), p
        assert out["best_cut"][idx] == golden_bench[p + "best"], p
        assert out["counts"][idx].sum() == golden_bench[p + "counts_sum"], p
        assert np.array_equal(out["inputs"][idx], golden_bench[p + "inputs"]), p
        W = graph.total_weight()
        assert np.array_equal(out["energy_trace"][idx], W - 2.0 * out["cut_trace"][idx])


@pytest.mark.parametrize("kind", list(Algorithm))
def test_g1_hundred_trial_summaries_match_reference(golden_bench, bench_graphs, kind):
    # acceptance criterion 3 numbers (/root/reference/pkg/test_output.txt:148)
    spec = engine.ExperimentSpec(graph="G1", algo=AlgorithmConfig(kind), cycles=1000, trials=100)
    s = engine.run_trials(spec, {"G1": bench_graphs("G1")})
    assert np.array_equal([r.final_cut for r in s.results],
                          golden_bench[f"g1_{kind.value}_s0_final_cuts100"])
    assert np.array_equal([r.best_cut for r in s.results],
                          golden_bench[f"g1_{kind.value}_s0_best_cuts100"])
    want = {"psa": 0.0, "tapsa": 0.9973, "spsa": 0.7418}[kind.value]
    assert round(s.mean_cut / 11605, 4) == want


def _oracle_compare(oracle, model, sch, cfg, profs, keys, graph):
    got = _batch(model, sch, cfg, keys, profs, graph)
    ref_profs = profs if profs is not None else VariabilityProfile.ideal(model.n, sch.t_res)
    want = oracle.anneal_batch(model, sch, cfg.kind.value, ref_profs, keys, graph=graph,
                               alpha=cfg.kernel_alpha, p_stall=cfg.p_stall)
    for k in ("spins", "inputs", "hist", "counts", "i0_trace", "energy_trace", "best_cut"):
        assert np.array_equal(got[k], want[k]), k
    if graph is not None:
        assert np.array_equal(got["cut_trace"], want["cut_trace"])


@pytest.mark.parametrize("case", range(12))
def test_random_specs_match_oracle(oracle, case):
    # criterion-2-style random specs (test_acceptance.py:82-118), all rules
    rng = np.random.default_rng(7000 + case)
    n = int(rng.integers(4, 60))
    g = random_graph(n, int(rng.integers(0, 1 << 30)), weights=(-2, -1, 1, 2) if case % 2 else (-1, 1),
                     p_edge=float(rng.uniform(0.1, 0.8)))
    model = maxcut_to_ising(g)
    t_res = int(rng.choice([1, 3, 10]))
    sch = derive_schedule(model, cycles=int(rng.integers(5, 80)), t_res=t_res)
    kind = list(Algorithm)[case % 3]
    cfg = AlgorithmConfig(kind, alpha=int(rng.integers(1, 6)), p_stall=float(rng.uniform(0, 1)))
    T = int(rng.integers(1, 70))
    keys = [streams.run_key(int(rng.integers(0, 1 << 62))) for _ in range(T)]
    if case % 4 == 0:
        profs = None
    else:
        vc = VariabilityConfig(*(float(x) for x in rng.uniform(0, 0.8, 3)), t_res=t_res)
        profs = [sample_variability(vc, n, np.random.default_rng(int(rng.integers(0, 1 << 30))))
                 for _ in range(T)]
    _oracle_compare(oracle, model, sch, cfg, profs, keys, g)


def test_fractional_model_without_graph_matches_oracle(oracle):
    # non-integer couplings and fields, no graph: fp64 field/energy order path
    rng = np.random.default_rng(3)
    n = 25
    edges = [(i, j, float(rng.normal())) for i in range(n) for j in range(i + 1, n)
             if rng.random() < 0.3]
    model = IsingModel.from_edges(n, edges, h=rng.normal(size=n) * 0.3)
    sch = derive_schedule(model, cycles=40, t_res=4)
    for kind in Algorithm:
        cfg = AlgorithmConfig(kind, alpha=2, p_stall=0.3)
        keys = [streams.run_key(s) for s in range(9)]
        _oracle_compare(oracle, model, sch, cfg, None, keys, None)


def test_single_spin_bias_saturates_to_plus_one():
    # /root/reference/pkg/tests/test_annealer.py:182-190
    model = IsingModel.from_edges(1, [], h=[2.0])
    sch = AnnealSchedule(i0_min=0.5, i0_max=50.0, beta=0.01 ** (1.0 / 9.0), cycles=10, t_res=3)
    res = run_anneal(model, sch, AlgorithmConfig(Algorithm.PSA),
                     VariabilityProfile.ideal(1, t_res=3), seed=5)
    assert res.final_state.spins[0] == 1
    assert res.final_energy == -2.0
    assert res.cut_trace is None and res.final_cut is None and res.best_cut is None


def test_degenerate_rules_are_bitwise_plain_rule(bench_graphs):
    # alpha=1 TApSA and p=0 SpSA collapse onto pSA (criterion 2), on the packed path
    g = bench_graphs("G81")
    model = maxcut_to_ising(g)
    sch = derive_schedule(model, 60, 10)
    keys = [streams.run_key(s) for s in range(64)]
    base = _batch(model, sch, AlgorithmConfig(Algorithm.PSA), keys, None, g)
    for cfg in (AlgorithmConfig(Algorithm.TAPSA, alpha=1), AlgorithmConfig(Algorithm.SPSA, p_stall=0.0)):
        other = _batch(model, sch, cfg, keys, None, g)
        for k in ("spins", "cut_trace", "energy_trace", "counts", "inputs"):
            assert np.array_equal(base[k], other[k]), (cfg, k)


def test_full_size_g81_properties_and_shard_invariance(bench_graphs, golden_bench):
    """BASELINE config C4 at full size (4096 trials): recorded trials match the
    reference, E = W - 2 cut on every trace entry, and any trial split (the
    multi-GPU sharding) gives identical per-trial results."""
    g = bench_graphs("G81")
    spec = engine.ExperimentSpec(graph="G81", algo=AlgorithmConfig(Algorithm.PSA), cycles=1000,
                                 trials=4096)
    full, _ = engine.run_trial_range(spec, g, 0, 4096)
    half, _ = engine.run_trial_range(spec, g, 2048, 4096)
    for k in (0, 1, 2047, 4095):
        assert np.array_equal(full[k].cut_trace, golden_bench[f"g81_psa_s0_{k}_cut"])
        assert np.array_equal(full[k].final_state.spins, golden_bench[f"g81_psa_s0_{k}_spins"])
    for k in range(2048, 4096, 97):
        assert np.array_equal(full[k].final_state.spins, half[k - 2048].final_state.spins)
        assert np.array_equal(full[k].cut_trace, half[k - 2048].cut_trace)
    W = g.total_weight()
    for r in full[::256]:
        assert np.array_equal(r.energy_trace, W - 2.0 * r.cut_trace)
        assert r.best_cut == r.cut_trace.max()


def test_batched_sweep_is_paired_with_single_runs():
    # /root/reference/pkg/tests/test_engine.py:118-134: a sweep point equals the
    # standalone run at that sigma; here all varied points share one device batch
    g = random_graph(80, 14, p_edge=0.15)
    graphs = {"toy": g}
    spec = engine.ExperimentSpec(graph="toy", algo=AlgorithmConfig(Algorithm.TAPSA), cycles=80,
                                 trials=6)
    values = [0.0, 0.4, 0.7]
    sums = engine.sweep(spec, "sigma_delta", values, graphs, registry={"toy": 100})
    for v, s in zip(values, sums):
        alone = engine.run_trials(engine.ExperimentSpec(
            graph="toy", algo=AlgorithmConfig(Algorithm.TAPSA), cycles=80, trials=6,
            variability=VariabilityConfig(sigma_delta=v)), graphs, registry={"toy": 100})
        assert [r.final_cut for r in s.results] == [r.final_cut for r in alone.results]
        for a, b in zip(s.results, alone.results):
            assert np.array_equal(a.energy_trace, b.energy_trace)
            assert np.array_equal(a.final_state.spins, b.final_state.spins)
            assert np.array_equal(a.final_state.ti_history, b.final_state.ti_history)
        assert s.mean_cut == alone.mean_cut and s.std_cut == alone.std_cut
        assert s.normalized_mean_cut == alone.normalized_mean_cut


def test_philox_sweep_is_paired_with_single_runs(bench_graphs):
    """A native-stream sweep: every point equals its standalone run_trials (the
    Philox stream is indexed by global trial, so points are not batched)."""
    g = bench_graphs("G22")
    spec = engine.ExperimentSpec(graph="G22", algo=AlgorithmConfig(Algorithm.PSA), cycles=60,
                                 trials=40, rng="philox")
    values = [0.3, 0.6]
    sums = engine.sweep(spec, "sigma_nu", values, {"G22": g})
    for v, s in zip(values, sums):
        alone = engine.run_trials(dataclasses.replace(
            spec, variability=VariabilityConfig(sigma_nu=v)), {"G22": g})
        for a, b in zip(s.results, alone.results):
            assert np.array_equal(a.final_state.spins, b.final_state.spins)
            assert np.array_equal(a.cut_trace, b.cut_trace)


@pytest.mark.parametrize("name,p_stall,cycles", [("G81", 0.5, 150), ("G55", 0.3, 120),
                                                  ("G48", 1.0, 60), ("G22", 0.7, 80)])
def test_packed_spsa_matches_oracle(oracle, bench_graphs, name, p_stall, cycles):
    """Stalled rule on the packed path (per-p-bit drive index, two hashes per update)."""
    g = bench_graphs(name)
    model = maxcut_to_ising(g)
    sch = derive_schedule(model, cycles, 10)
    cfg = AlgorithmConfig(Algorithm.SPSA, p_stall=p_stall)
    keys = [streams.run_key(streams.trial_seed(5, k)) for k in range(5)]
    b = _native.Batch(model, sch, keys, graph=g, algo_code=cfg.kind.code, alpha=1, p_stall=p_stall)
    plan = _native.Plan(b)
    assert plan.info()["path"] == "packed"
    plan.run()
    got = plan.download()
    plan.close()
    want = oracle.anneal_batch(model, sch, "spsa", VariabilityProfile.ideal(model.n), keys, graph=g,
                               alpha=1, p_stall=p_stall)
    for k in ("spins", "inputs", "hist", "counts", "i0_trace", "energy_trace", "cut_trace", "best_cut"):
        assert np.array_equal(got[k], want[k]), k


@pytest.mark.parametrize("name,alpha,cycles", [("G81", 4, 200), ("G55", 4, 120), ("G48", 7, 150),
                                               ("G1", 4, 60), ("G22", 4, 80), ("G81", 8, 50),
                                               ("G1", 2, 40), ("G22", 11, 40)])
def test_packed_tapsa_matches_oracle(oracle, bench_graphs, name, alpha, cycles):
    """Time-averaged rule on the packed path (bit-sliced history ring)."""
    g = bench_graphs(name)
    model = maxcut_to_ising(g)
    sch = derive_schedule(model, cycles, 10)
    cfg = AlgorithmConfig(Algorithm.TAPSA, alpha=alpha)
    keys = [streams.run_key(streams.trial_seed(3, k)) for k in range(5)]
    b = _native.Batch(model, sch, keys, graph=g, algo_code=cfg.kind.code, alpha=cfg.kernel_alpha)
    plan = _native.Plan(b)
    assert plan.info()["path"] == "packed"
    plan.run()
    got = plan.download()
    plan.close()
    want = oracle.anneal_batch(model, sch, "tapsa", VariabilityProfile.ideal(model.n), keys, graph=g,
                               alpha=alpha)
    for k in ("spins", "inputs", "hist", "counts", "i0_trace", "energy_trace", "cut_trace", "best_cut"):
        assert np.array_equal(got[k], want[k]), k


@pytest.mark.parametrize("bucket", ["1", "0"])
@pytest.mark.parametrize("name,sig,trials,cycles,rng", [
    ("G81", (1.0, 1.0, 1.0), 128, 50, "replay"), ("G55", (0.5, 0.5, 0.5), 96, 60, "replay"),
    ("G60", (0.8, 0.2, 0.6), 64, 40, "replay"), ("G81", (0.5, 0.5, 0.5), 64, 40, "philox"),
    ("G48", (0.0, 2.0, 0.5), 64, 40, "replay"), ("G81", (0.0, 0.0, 0.5), 64, 40, "replay"),
    ("G1", (0.0, 0.0, 3.0), 45, 30, "replay"), ("G22", (0.5, 0.5, 2.0), 100, 30, "philox")])
def test_timing_kernel_wide_spreads_match_oracle(oracle, bench_graphs, monkeypatch, name, sig, trials,
                                                 cycles, rng, bucket):
    """The launched timing-spread kernels at wide spreads, replay and Philox:
    packed_sweep_bucket (period-sorted slots, the default) and, with
    PBSA_BUCKET=0, packed_sweep_timing (bit-sliced periods), both with the fp16
    profile pair and the slope-scaled prefilter margin; bit-identical to the
    oracle (sigma_nu 2-3: dozens of period classes, many dividing per sub-step)."""
    monkeypatch.setenv("PBSA_BUCKET", bucket)
    monkeypatch.setenv("PBSA_RESIDENT", "0")
    graph = bench_graphs(name)
    model = maxcut_to_ising(graph)
    sch = derive_schedule(model, cycles, 10)
    seeds = [streams.trial_seed(21, k) for k in range(trials)]
    profs = [sample_variability(VariabilityConfig(*sig), graph.n,
                                np.random.default_rng(streams.profile_seed(s))) for s in seeds]
    keys = [streams.run_key(s) for s in seeds]
    seed = 0x0DDB_A11_5EED
    b = _native.Batch(model, sch, keys, profile_rows=profile_rows(profs, model.n), graph=graph,
                      rng=rng, rng_seed=seed)
    plan = _native.Plan(b)
    assert plan.info()["kernel"] == ("packed_bucket" if bucket == "1" else "packed_timing"), plan.info()
    up, _ = plan.transfer_bytes()
    plan.run()
    got = plan.download()
    plan.close()
    assert up >= trials * graph.n * 4   # the fp16 pairs are counted in the upload
    extra = dict(rng="philox", rng_seed=seed) if rng == "philox" else {}
    want = oracle.anneal_batch(model, sch, "psa", profs, keys, graph=graph, **extra)
    for k in ("spins", "inputs", "counts", "i0_trace", "energy_trace", "cut_trace", "best_cut"):
        assert np.array_equal(got[k], want[k]), k


@pytest.mark.parametrize("name,alpha,trials,cycles,rng", [
    ("G1", 4, 100, 80, "replay"), ("G22", 11, 40, 40, "replay"), ("G47", 2, 64, 50, "replay"),
    ("G1", 8, 36, 60, "replay"), ("G1", 3, 40, 60, "philox"), ("G22", 4, 100, 40, "philox"),
    ("G1", 4, 8, 3, "replay")])
@pytest.mark.parametrize("resident", ["1", "0"])
def test_tapsa_resident_cluster_kernel_matches_oracle(oracle, bench_graphs, monkeypatch, name,
                                                      alpha, trials, cycles, rng, resident):
    """TApSA on the resident cluster kernel (resident_sweep<TAPSA>: the CTA's
    slice of the bit-sliced ring held in shared memory for the whole run,
    written back for the history output) and, forced off, on the launched
    packed sweep: both bit-identical to the oracle (cycles < alpha included)."""
    monkeypatch.setenv("PBSA_RESIDENT", resident)
    graph = bench_graphs(name)
    model = maxcut_to_ising(graph)
    sch = derive_schedule(model, cycles, 10)
    seed = 0x5EED_0000_7777
    keys = [streams.run_key(streams.trial_seed(0, k)) for k in range(trials)]
    b = _native.Batch(model, sch, keys, graph=graph, algo_code=1, alpha=alpha,
                      rng=rng, rng_seed=seed)
    plan = _native.Plan(b)
    info = plan.info()
    assert info["kernel"] == ("resident" if resident == "1" else "packed"), info
    plan.run()
    got = plan.download()
    plan.close()
    extra = dict(rng="philox", rng_seed=seed) if rng == "philox" else {}
    want = oracle.anneal_batch(model, sch, "tapsa", VariabilityProfile.ideal(model.n), keys,
                               graph=graph, alpha=alpha, **extra)
    for k in ("spins", "inputs", "hist", "counts", "i0_trace", "energy_trace", "cut_trace",
              "best_cut"):
        assert np.array_equal(got[k], want[k]), k


@pytest.mark.parametrize("name,sig,cycles,margin,force", [
    ("G81", (0.5, 0.0, 0.0), 120, None, None), ("G81", (0.0, 0.7, 0.0), 120, None, None),
    ("G55", (0.5, 0.5, 0.5), 60, None, None), ("G22", (1.0, 1.0, 0.0), 80, None, None),
    ("G1", (0.3, 0.4, 0.8), 40, None, None), ("G48", (0.0, 0.0, 1.0), 50, None, None),
    ("G55", (0.5, 0.5, 0.5), 30, "1e9", None), ("G1", (0.8, 0.3, 0.0), 30, "1e9", None),
    ("G48", (0.0, 0.0, 1.0), 30, "1e9", None),
    ("G55", (0.5, 0.5, 0.5), 60, None, "0"), ("G1", (0.3, 0.4, 0.8), 30, None, "0"),
    ("G55", (0.5, 0.5, 0.5), 30, "1e9", "0"), ("G22", (0.7, 0.2, 0.0), 30, None, "0")])
def test_variability_matches_oracle(oracle, bench_graphs, monkeypatch, name, sig, cycles, margin,
                                    force):
    """Per-trial variability profiles on the packed kernel (ALG=3 without a
    timing spread, ALG=4 with one) or, with PBSA_PACKED_VAR=0, on the
    active-list fast kernel; all use the fp32 sigmoid prefilter with an exact
    fp64/libm recheck, and margin 1e9 sends every update through the exact
    recheck, so both branches meet the oracle."""
    if margin is not None:
        monkeypatch.setenv("PBSA_VAR_MARGIN", margin)
    if force is not None:
        monkeypatch.setenv("PBSA_PACKED_VAR", force)
    want_path = "general" if force == "0" else "packed"
    g = bench_graphs(name)
    model = maxcut_to_ising(g)
    sch = derive_schedule(model, cycles, 10)
    T = 37
    seeds = [streams.trial_seed(11, k) for k in range(T)]
    vc = VariabilityConfig(*sig)
    profs = [sample_variability(vc, g.n, np.random.default_rng(streams.profile_seed(s))) for s in seeds]
    keys = [streams.run_key(s) for s in seeds]
    b = _native.Batch(model, sch, keys, profile_rows=profile_rows(profs, model.n), graph=g,
                      algo_code=Algorithm.PSA.code)
    plan = _native.Plan(b)
    assert plan.info()["path"] == want_path
    plan.run()
    got = plan.download()
    plan.close()
    want = oracle.anneal_batch(model, sch, "psa", profs, keys, graph=g)
    for k in ("spins", "inputs", "hist", "counts", "i0_trace", "energy_trace", "cut_trace", "best_cut"):
        assert np.array_equal(got[k], want[k]), k


@pytest.mark.parametrize("sig", [(0.6, 0.6, 0.6), (0.6, 0.6, 0.0), (0.0, 0.0, 0.7)])
def test_variability_paths_agree_with_shared_profile(bench_graphs, monkeypatch, sig):
    """One profile shared by all trials (profile_stride 0): the packed
    variability kernel, the active-list fast kernel and the original
    active-list kernel give the same bits."""
    g = bench_graphs("G22")
    model = maxcut_to_ising(g)
    sch = derive_schedule(model, 50, 10)
    prof = sample_variability(VariabilityConfig(*sig), g.n, np.random.default_rng(4))
    keys = [streams.run_key(s) for s in range(70)]
    outs = []
    for env in ({"PBSA_PACKED_VAR": "1"}, {"PBSA_PACKED_VAR": "0"},
                {"PBSA_PACKED_VAR": "0", "PBSA_ACTIVE_FAST": "0"}):
        for k, v in env.items():
            monkeypatch.setenv(k, v)
        b = _native.Batch(model, sch, keys, profile_rows=profile_rows(prof, model.n), graph=g,
                          algo_code=Algorithm.PSA.code)
        plan = _native.Plan(b)
        assert plan.info()["path"] == ("packed" if env["PBSA_PACKED_VAR"] == "1" else "general")
        plan.run()
        outs.append(plan.download())
        plan.close()
        for k in env:
            monkeypatch.delenv(k)
    for o in outs[1:]:
        for k in ("spins", "inputs", "hist", "counts", "energy_trace", "cut_trace", "best_cut"):
            assert np.array_equal(outs[0][k], o[k]), k


@pytest.mark.parametrize("t_res,sig_nu,want", [(40, 0.8, "packed"), (64, 3.0, "general"), (1, 0.0, "packed"),
                                                (3, 2.0, "packed")])
def test_variability_long_periods_and_many_divisors(oracle, t_res, sig_nu, want):
    """Long periods need all 8 bit planes and sub-steps with many dividing
    periods; a period >= 256 (after clamping to cycles * t_res) falls back to
    the general path. Non-multiple-of-32 node count and trial count."""
    g = random_graph(333, 21, weights=(-1, 1), p_edge=0.02)
    model = maxcut_to_ising(g)
    sch = derive_schedule(model, cycles=12, t_res=t_res)
    T = 45
    rng = np.random.default_rng(t_res)
    vc = VariabilityConfig(0.3, 0.3, sig_nu, t_res=t_res)
    profs = [sample_variability(vc, g.n, np.random.default_rng(int(rng.integers(1 << 30)))) for _ in range(T)]
    keys = [streams.run_key(int(rng.integers(1 << 62))) for _ in range(T)]
    b = _native.Batch(model, sch, keys, profile_rows=profile_rows(profs, model.n), graph=g,
                      algo_code=Algorithm.PSA.code)
    plan = _native.Plan(b)
    assert plan.info()["path"] == want
    plan.run()
    got = plan.download()
    plan.close()
    want_out = oracle.anneal_batch(model, sch, "psa", profs, keys, graph=g)
    for k in ("spins", "inputs", "hist", "counts", "i0_trace", "energy_trace", "cut_trace", "best_cut"):
        assert np.array_equal(got[k], want_out[k]), k


def test_concurrent_calls_from_threads_are_independent(bench_graphs):
    """The C ABI is reentrant (ctypes releases the GIL; every call owns its
    plan, stream and buffers), as the reference kernel is under the engine's
    thread pool (engine.py:122-123): concurrent calls equal sequential ones."""
    from concurrent.futures import ThreadPoolExecutor
    jobs = []
    for k, (name, sig) in enumerate([("G81", (0, 0, 0)), ("G55", (0.5, 0.5, 0.5)), ("G1", (0.4, 0, 0)),
                                     ("G22", (0, 0, 0)), ("G81", (0.3, 0.3, 0.3)), ("G48", (0, 0, 0))]):
        g = bench_graphs(name)
        model = maxcut_to_ising(g)
        sch = derive_schedule(model, 40, 10)
        seeds = [streams.trial_seed(k, j) for j in range(40)]
        vc = VariabilityConfig(*sig)
        profs = None if vc.is_ideal else [
            sample_variability(vc, g.n, np.random.default_rng(streams.profile_seed(s))) for s in seeds]
        jobs.append(_native.Batch(model, sch, [streams.run_key(s) for s in seeds],
                                  profile_rows=profile_rows(profs, model.n), graph=g,
                                  algo_code=Algorithm.PSA.code))
    seq = [_native.anneal_batch(b)[0] for b in jobs]
    with ThreadPoolExecutor(max_workers=len(jobs)) as ex:
        par = list(ex.map(lambda b: _native.anneal_batch(b)[0], jobs + jobs))
    for k, out in enumerate(par):
        for key in ("spins", "inputs", "counts", "energy_trace", "cut_trace", "best_cut"):
            assert np.array_equal(out[key], seq[k % len(jobs)][key]), (k, key)


def test_acceptance_criterion_4_timing_variability(golden_acceptance, bench_graphs):
    """/root/reference/pkg/tests/test_acceptance.py:156-172: pSA on G1 with
    sigma_nu = 1 beats sigma_nu = 0 by > 2 SE over 50 trials -- here every
    per-trial final cut equals the reference's."""
    g = bench_graphs("G1")
    means, ses = {}, {}
    for sn in (0.0, 1.0):
        spec = engine.ExperimentSpec(graph="G1", algo=AlgorithmConfig(Algorithm.PSA),
                                     variability=VariabilityConfig(sigma_nu=sn, t_res=10),
                                     cycles=1000, trials=50)
        s = engine.run_trials(spec, {"G1": g})
        assert np.array_equal([r.final_cut for r in s.results],
                              golden_acceptance[f"c4_nu{sn:g}_final_cuts"]), sn
        means[sn], ses[sn] = s.mean_cut, s.std_cut / math.sqrt(50)
    assert means[1.0] - means[0.0] > 2.0 * math.hypot(ses[1.0], ses[0.0])


def test_acceptance_criterion_5_offset_sweep_time_averaged(golden_acceptance, bench_graphs):
    """test_acceptance.py:173-187: TApSA (alpha 4) on G1 swept over
    sigma_delta in {0, 0.5, 1} (one device batch), 100 trials each: per-trial
    final cuts equal the reference's and the normalized means vary < 0.02."""
    g = bench_graphs("G1")
    spec = engine.ExperimentSpec(graph="G1", algo=AlgorithmConfig(Algorithm.TAPSA, alpha=4),
                                 cycles=1000, trials=100)
    sums = engine.sweep(spec, "sigma_delta", [0.0, 0.5, 1.0], {"G1": g})
    for v, s in zip((0.0, 0.5, 1.0), sums):
        assert np.array_equal([r.final_cut for r in s.results],
                              golden_acceptance[f"c5_delta{v:g}_final_cuts"]), v
    norms = [s.mean_cut / 11605 for s in sums]
    assert max(norms) - min(norms) < 0.02


@pytest.mark.parametrize("name,kind,sig", [("G1", Algorithm.PSA, (0.0, 0.0, 0.3)),
                                           ("G47", Algorithm.TAPSA, (0.5, 0.0, 0.0)),
                                           ("G48", Algorithm.SPSA, (0.0, 0.5, 0.0))])
def test_acceptance_criterion_7_specs(golden_acceptance, bench_graphs, name, kind, sig):
    """The three specs of test_acceptance.py:205-230 (120 cycles, 6 trials,
    seed 2): full cut and energy traces equal the reference's."""
    g = bench_graphs(name)
    spec = engine.ExperimentSpec(graph=name, algo=AlgorithmConfig(kind), cycles=120, trials=6,
                                 base_seed=2, variability=VariabilityConfig(*sig))
    s = engine.run_trials(spec, {name: g})
    assert np.array_equal(np.stack([r.cut_trace for r in s.results]),
                          golden_acceptance[f"c7_{name}_{kind.value}_cut_traces"])
    assert np.array_equal(np.stack([r.energy_trace for r in s.results]),
                          golden_acceptance[f"c7_{name}_{kind.value}_energy_traces"])


def test_acceptance_criteria_6_and_8_schedule_endpoints_and_largest_graph(bench_graphs):
    """test_acceptance.py:189-203 and 233-255: on every benchmark the recorded
    i0 sequence starts at i0_min, ends at i0_max (1e-9 relative) and increases;
    G81 TApSA (alpha 4) for one trial is well inside the 600 s budget."""
    import time
    from paper_2601_14476_b200 import benchmarks
    for name in benchmarks.BENCHMARKS:
        g = bench_graphs(name)
        model = maxcut_to_ising(g)
        sch = derive_schedule(model, cycles=1000)
        t0 = time.perf_counter()
        res = run_anneal(model, sch, AlgorithmConfig(Algorithm.TAPSA), VariabilityProfile.ideal(model.n),
                         seed=0, graph=g)
        elapsed = time.perf_counter() - t0
        assert res.i0_trace[0] == sch.i0_min, name
        assert abs(res.i0_trace[-1] - sch.i0_max) / sch.i0_max <= 1e-9, name
        assert np.all(np.diff(res.i0_trace) > 0), name
        if name == "G81":
            assert (g.n, g.m) == (20000, 40000) and elapsed < 600.0


# ------------------------------------------------------------ native Philox mode

def test_device_philox_matches_random123_kats_and_host():
    from test_native_abi import PHILOX_KATS
    ctr = np.array([c for c, _, _ in PHILOX_KATS], np.uint32)
    key = np.array([k for _, k, _ in PHILOX_KATS], np.uint32)
    got = _native.debug_philox(ctr, key)
    assert got.tolist() == [w for _, _, w in PHILOX_KATS]
    rng = np.random.default_rng(9)
    ctr = rng.integers(0, 2 ** 32, (5000, 4), dtype=np.uint64).astype(np.uint32)
    key = rng.integers(0, 2 ** 32, (5000, 2), dtype=np.uint64).astype(np.uint32)
    got = _native.debug_philox(ctr, key)
    for k in range(0, 5000, 97):
        assert got[k].tolist() == _native.philox_host(ctr[k].tolist(), key[k].tolist())


def _native_run(graph, trials, cycles, seed=0x1234_5678_9ABC_DEF0, first_trial=0, algo=0,
                alpha=1, p_stall=0.5, profs=None):
    model = maxcut_to_ising(graph)
    sch = derive_schedule(model, cycles, 10)
    keys = [streams.run_key(streams.trial_seed(0, first_trial + k)) for k in range(trials)]
    b = _native.Batch(model, sch, keys, graph=graph, algo_code=algo, alpha=alpha,
                      p_stall=p_stall, rng="philox", rng_seed=seed, first_trial=first_trial,
                      profile_rows=profile_rows(profs, model.n))
    return model, sch, keys, _native.anneal_batch(b)[0]


@pytest.mark.parametrize("name,sig,trials,cycles", [
    ("G81", (0.5, 0.5, 0.5), 64, 30), ("G55", (0.5, 0.5, 0.0), 64, 40),
    ("G1", (0.0, 0.0, 0.5), 40, 60), ("G22", (0.5, 0.5, 0.5), 36, 40),
    ("G1", (0.5, 0.5, 0.0), 40, 60)])
def test_philox_mode_with_variability_matches_oracle(oracle, bench_graphs, name, sig, trials,
                                                     cycles):
    """Varied profiles under the native stream: the sigmoid prefilter and the
    exact fp64 recheck on the Philox draw (packed_sweep ALG=5,
    packed_sweep_timing<L, NATIVE>, and the resident cluster kernels for the
    small G1 batches) against the oracle's Philox mode."""
    graph = bench_graphs(name)
    n = graph.n
    profs = [sample_variability(VariabilityConfig(*sig), n, np.random.default_rng(500 + k))
             for k in range(trials)]
    seed = 0xFEED_F00D_1234
    model, sch, keys, got = _native_run(graph, trials, cycles, seed, profs=profs)
    want = oracle.anneal_batch(model, sch, "psa", profs, keys, graph=graph, rng="philox",
                               rng_seed=seed)
    for k in ("spins", "inputs", "counts", "i0_trace", "energy_trace", "cut_trace", "best_cut"):
        assert np.array_equal(got[k], want[k]), k


@pytest.mark.parametrize("name,trials,cycles", [("G81", 96, 40), ("G55", 64, 60),
                                                ("G22", 40, 80), ("G1", 72, 100)])
def test_philox_mode_matches_oracle(oracle, bench_graphs, name, trials, cycles):
    graph = bench_graphs(name)
    seed = 0x1234_5678_9ABC_DEF0
    model, sch, keys, got = _native_run(graph, trials, cycles, seed)
    want = oracle.anneal_batch(model, sch, "psa", VariabilityProfile.ideal(model.n), keys,
                               graph=graph, rng="philox", rng_seed=seed)
    for k in ("spins", "inputs", "counts", "i0_trace", "energy_trace", "cut_trace", "best_cut"):
        assert np.array_equal(got[k], want[k]), k


def test_philox_mode_plain_rule_equivalents_and_shards(oracle, bench_graphs):
    """TApSA alpha=1 / SpSA p=0 are the plain rule; a shard starting at a
    multiple of 4 reproduces the same trials of the whole batch."""
    graph = bench_graphs("G81")
    _, _, _, whole = _native_run(graph, 128, 30)
    _, _, _, tail = _native_run(graph, 68, 30, first_trial=60)
    _, _, _, tap = _native_run(graph, 128, 30, algo=1, alpha=1)
    _, _, _, sps = _native_run(graph, 128, 30, algo=2, p_stall=0.0)
    for k in ("spins", "cut_trace", "energy_trace", "best_cut"):
        assert np.array_equal(whole[k][60:], tail[k]), k
        assert np.array_equal(whole[k], tap[k]), k
        assert np.array_equal(whole[k], sps[k]), k


def test_philox_mode_rejects_unsupported_inputs(bench_graphs):
    graph = bench_graphs("G1")
    prof = [sample_variability(VariabilityConfig(0.5, 0.5, 0.5), graph.n,
                               np.random.default_rng(k)) for k in range(8)]
    with pytest.raises(ValueError, match="philox"):   # TApSA with a varied profile: general path
        _native_run(graph, 8, 10, algo=1, alpha=3, profs=prof)
    g2 = random_graph(30, 5, (-2, -1, 1, 2), 0.3)     # |J| = 2: general path
    with pytest.raises(ValueError, match="philox"):
        _native_run(g2, 8, 10)
    with pytest.raises(ValueError, match="multiple of 4"):
        _native_run(graph, 8, 10, first_trial=2)


@pytest.mark.parametrize("name,algo,alpha,p_stall,trials,cycles", [
    ("G81", 1, 4, 0.5, 64, 30), ("G81", 2, 1, 0.4, 64, 30), ("G1", 1, 3, 0.5, 40, 60),
    ("G1", 2, 1, 0.5, 40, 60), ("G55", 1, 8, 0.5, 36, 40), ("G22", 2, 1, 1.0, 36, 40)])
def test_philox_mode_time_averaged_and_stalled_rules_match_oracle(oracle, bench_graphs, name, algo,
                                                                  alpha, p_stall, trials, cycles):
    """Native stream for the paper's TApSA and SpSA rules (packed_sweep ALG=6/7;
    SpSA's stall draw uses tag 4) against the oracle's Philox mode."""
    graph = bench_graphs(name)
    seed = 0xABCD_0123_4567
    model, sch, keys, got = _native_run(graph, trials, cycles, seed, algo=algo, alpha=alpha,
                                        p_stall=p_stall)
    want = oracle.anneal_batch(model, sch, ["psa", "tapsa", "spsa"][algo],
                               VariabilityProfile.ideal(model.n), keys, graph=graph, alpha=alpha,
                               p_stall=p_stall, rng="philox", rng_seed=seed)
    for k in ("spins", "inputs", "hist", "counts", "i0_trace", "energy_trace", "cut_trace",
              "best_cut"):
        assert np.array_equal(got[k], want[k]), k


@pytest.mark.parametrize("name,sig,trials,kind", [("G1", (0.0, 0.0, 0.5), 128, Algorithm.PSA),
                                                  ("G81", (0.5, 0.5, 0.5), 256, Algorithm.PSA),
                                                  ("G55", (1.0, 0.0, 0.0), 256, Algorithm.PSA),
                                                  ("G1", (0, 0, 0), 128, Algorithm.TAPSA),
                                                  ("G1", (0, 0, 0), 128, Algorithm.SPSA)])
def test_philox_cut_statistics_match_reference_with_variability(bench_graphs, golden_analogs,
                                                                name, sig, trials, kind):
    """The north_star statistical bar where the anneal works (the variability
    study, TApSA and SpSA; normalized cuts 0.4-0.999): mean final cut and mean
    per-trial best cut of the native stream within 0.5 % of the best-known cut
    of the replayed reference stream (which is bit-exact to the reference)."""
    graph = bench_graphs(name)
    best_known = golden_analogs[name]["best_known_analog"]
    spec = engine.ExperimentSpec(graph=name, algo=AlgorithmConfig(kind, alpha=4, p_stall=0.5),
                                 variability=VariabilityConfig(*sig), cycles=1000, trials=trials)
    rep = engine.run_trials(spec, {name: graph})
    nat = engine.run_trials(dataclasses.replace(spec, rng="philox"), {name: graph})
    assert abs(nat.mean_cut - rep.mean_cut) <= 0.005 * best_known, (nat.mean_cut, rep.mean_cut)
    b_rep = np.mean([r.best_cut for r in rep.results])
    b_nat = np.mean([r.best_cut for r in nat.results])
    assert abs(b_nat - b_rep) <= 0.005 * best_known, (b_nat, b_rep)
    assert nat.mean_cut > 0.3 * best_known  # a run that anneals, not the sigma = 0 degenerate case


def test_philox_cut_statistics_match_reference_stream(bench_graphs, golden_analogs):
    """north_star: with the native stream the distribution of the mean and the
    best cut over >= 100 trials matches the reference stream within 0.5 % of
    the best-known cut: the mean final cut and the mean per-trial best cut
    (the maximum over trials is an extreme value of a heavy tail for pSA at
    sigma = 0 and is not compared).  G81 analog 512 trials x 1000 cycles, G22 x 256."""
    for name, trials in (("G81", 512), ("G22", 256)):
        graph = bench_graphs(name)
        best_known = golden_analogs[name]["best_known_analog"]
        spec = engine.ExperimentSpec(graph=name, algo=AlgorithmConfig(Algorithm.PSA),
                                     cycles=1000, trials=trials)
        rep = engine.run_trials(spec, {name: graph})
        nat = engine.run_trials(dataclasses.replace(spec, rng="philox"),
                                {name: graph})
        best_rep = np.mean([r.best_cut for r in rep.results])
        best_nat = np.mean([r.best_cut for r in nat.results])
        assert abs(nat.mean_cut - rep.mean_cut) <= 0.005 * best_known, (name, nat.mean_cut, rep.mean_cut)
        assert abs(best_nat - best_rep) <= 0.005 * best_known, (name, best_nat, best_rep)


def test_variability_prefilter_is_exact_where_it_decides():
    """The fp16-profile prefilter of the timing kernels (var_prefilter) may only decide an update
    when every draw u 2^32 in [zh - 1, zh + 2) gives the reference's fp64
    decision r + tanh(lam (i0 raw + delta)) >= 0 (_kernels.py:149-152).
    Probed on 2M random and near-threshold inputs, including large |x|."""
    rng = np.random.default_rng(21)
    m = 2_000_000
    lam = 1.0 + rng.choice([0.1, 0.5, 1.0, 3.0], m) * rng.standard_normal(m)
    delta = rng.choice([0.0, 0.1, 0.5, 2.0], m) * rng.standard_normal(m)
    i0 = np.exp(rng.uniform(np.log(0.01), np.log(10.0), m))
    raw = rng.integers(-40, 41, m)
    x = lam * (i0 * raw + delta)
    tt = np.tanh(x)
    ustar = (1.0 - tt) / 2.0                  # +1 iff u >= u* (up to fp64 rounding)
    near = np.floor(ustar * 2.0 ** 32) + rng.integers(-3_000_000, 3_000_000, m)
    uni = rng.integers(0, 2 ** 32, m).astype(np.float64)
    is_uni = rng.random(m) < 0.3
    zh = np.where(is_uni, uni, near)
    zh = np.clip(zh, 1, 2 ** 32 - 3).astype(np.uint64).astype(np.uint32)
    code = _native.debug_var_prefilter(lam, delta, i0, raw, zh)
    decided = (code & 2) == 0
    # exact reference decision at both ends of the draw's interval (monotone in u)
    inp = i0 * raw
    for off in (-1.0, 1.999999):
        u = (zh.astype(np.float64) + off) * 2.0 ** -32
        r = 2.0 * u - 1.0
        ref = (r + np.tanh(lam * (inp + delta))) >= 0.0
        bad = decided & (ref != ((code & 1) == 1))
        assert not bad.any(), np.flatnonzero(bad)[:5]
    # random draws rarely need the recheck (here A reaches ~10^3, beyond the
    # benchmark range, and A > 256 always rechecks); the near-threshold probe
    # straddles the margin
    moderate = np.abs(lam) * np.abs(inp) + np.abs(lam * delta) < 64
    assert decided[is_uni & moderate].mean() > 0.99
    assert 0.05 < decided[~is_uni].mean() < 0.99


# ------------------------------------------------ engine invariances (test_engine.py)

@pytest.mark.parametrize("name,kind,sig", [("G81", Algorithm.PSA, (0, 0, 0)),
                                           ("G1", Algorithm.PSA, (0, 0, 0.5)),
                                           ("G55", Algorithm.TAPSA, (0, 0, 0)),
                                           ("G22", Algorithm.SPSA, (0.5, 0.5, 0.0))])
def test_rerun_identical_and_more_trials_never_perturb_earlier_ones(bench_graphs, name, kind, sig):
    """/root/reference/pkg/tests/test_engine.py:34-41 (rerun identical) and
    :57-62 (adding trials never perturbs the earlier ones) on the device paths:
    word padding, word phases and chains must not leak between trials."""
    graph = bench_graphs(name)
    base = engine.ExperimentSpec(graph=name, algo=AlgorithmConfig(kind, alpha=3, p_stall=0.4),
                                 variability=VariabilityConfig(*sig), cycles=40, trials=37)
    a = engine.run_trials(base, {name: graph})
    b = engine.run_trials(base, {name: graph})
    c = engine.run_trials(dataclasses.replace(base, trials=100), {name: graph})
    for ra, rb, rc in zip(a.results, b.results, c.results[:37]):
        assert np.array_equal(ra.final_state.spins, rb.final_state.spins)
        assert np.array_equal(ra.final_state.spins, rc.final_state.spins)
        assert np.array_equal(ra.cut_trace, rc.cut_trace)
        assert np.array_equal(ra.final_state.inputs, rc.final_state.inputs)
        assert np.array_equal(ra.update_counts, rc.update_counts)


def test_with_and_without_graph_same_dynamics(bench_graphs):
    """/root/reference/pkg/tests/test_annealer.py:216-230: the graph only adds
    the cut trace; spins, inputs and energies are the same without it."""
    g = bench_graphs("G22")
    model = maxcut_to_ising(g)
    sch = derive_schedule(model, 50, 10)
    for cfg in (AlgorithmConfig(Algorithm.PSA), AlgorithmConfig(Algorithm.TAPSA, alpha=4)):
        for prof in (VariabilityProfile.ideal(model.n),
                     sample_variability(VariabilityConfig(0.5, 0.5, 0.5), model.n,
                                        np.random.default_rng(4))):
            with_g = run_anneal(model, sch, cfg, prof, seed=11, graph=g)
            without = run_anneal(model, sch, cfg, prof, seed=11)
            assert np.array_equal(with_g.final_state.spins, without.final_state.spins)
            assert np.array_equal(with_g.energy_trace, without.energy_trace)
            assert np.array_equal(with_g.final_state.inputs, without.final_state.inputs)
            assert without.cut_trace is None and with_g.cut_trace is not None


@pytest.mark.parametrize("name,trials", [("G81", 600), ("G81", 1000), ("G81", 2600), ("G55", 3000)])
def test_pipelined_one_shot_equals_graph_run(bench_graphs, monkeypatch, name, trials):
    """The one-shot call of the plain rule runs pipelined (word phases launched
    directly, each phase's outputs copied back while the next anneals); its
    eight outputs equal the captured-graph run of the same batch, including a
    ragged last word (600 = 18.75 words) and ragged last phases (phases are at
    least two waves of word-warps: G81 16 words, G55 61 words; at most four)."""
    g = bench_graphs(name)
    model = maxcut_to_ising(g)
    sch = derive_schedule(model, 40, 10)
    keys = [streams.run_key(streams.trial_seed(0, k)) for k in range(trials)]
    b = _native.Batch(model, sch, keys, graph=g)
    piped, _ = _native.anneal_batch(b)
    monkeypatch.setenv("PBSA_PIPELINE", "0")
    plain, _ = _native.anneal_batch(b)
    for k in _native.OUT_ORDER:
        assert np.array_equal(piped[k], plain[k]), k


def test_device_list_fan_out_equals_single_call(bench_graphs):
    """distributed.run_trials_devices (one process, a device-ordinal list; here
    the one visible B200 listed twice, two concurrent plans) gives the
    single-call run_trials results trial by trial."""
    from paper_2601_14476_b200.distributed import run_trials_devices
    g = bench_graphs("G81")
    spec = engine.ExperimentSpec(graph="G81", algo=AlgorithmConfig(Algorithm.PSA), cycles=40,
                                 trials=300)
    one = engine.run_trials(spec, {"G81": g}, {"G81": 14004})
    two = run_trials_devices(spec, {"G81": g}, {"G81": 14004}, devices=[0, 0])
    assert len(two.results) == spec.trials
    for a, b in zip(one.results, two.results):
        assert np.array_equal(a.final_state.spins, b.final_state.spins)
        assert np.array_equal(a.cut_trace, b.cut_trace)
    assert one.mean_cut == two.mean_cut and one.std_cut == two.std_cut


# ------------------------------------ whole batches at the configured launch shapes

def _digest(spins, inputs, cut_trace, counts, best):
    import zlib
    T = spins.shape[0]
    return {"final_cut": cut_trace[:, -1].astype(np.int64),
            "best": np.asarray(best, np.int64),
            "cut_sum": cut_trace.sum(axis=1).astype(np.int64),
            "counts_sum": counts.sum(axis=1).astype(np.int64),
            "spins_crc": np.array([zlib.crc32(np.ascontiguousarray(spins[t]).tobytes())
                                   for t in range(T)], np.uint32),
            "inputs_crc": np.array([zlib.crc32(np.ascontiguousarray(inputs[t]).tobytes())
                                    for t in range(T)], np.uint32)}


def _check_digest(golden_full, tag, got):
    for k, v in got.items():
        want = golden_full[f"{tag}_{k}"]
        bad = np.flatnonzero(v != want)
        assert bad.size == 0, (tag, k, bad[:8])


def test_full_batch_bench_plan_matches_oracle(bench_graphs, golden_full, golden_bench):
    """The exact plan bench.py times (BASELINE C4: G81 x 4096 x 1000, replayed
    stream): word phases of 13 words in concurrent chains with the per-phase
    first-absorb cache, replayed as one CUDA graph.  Every trial's final cut,
    best cut, cut-trace sum, update count, final spins and inputs equal the
    oracle's (tests/golden/fullbatch.npz); the recorded reference trials match
    the reference's own outputs; the aggregate is the bench's quality line."""
    from paper_2601_14476_b200 import streams as st
    g = bench_graphs("G81")
    model = maxcut_to_ising(g)
    sch = derive_schedule(model, 1000, 10)
    b = _native.Batch(model, sch, st.run_keys(st.trial_seeds(0, 4096)), graph=g)
    plan = _native.Plan(b)
    lay = plan.layout()
    assert plan.info()["kernel"] == "packed"
    assert 0 < lay["phase_words"] < 128 and lay["chains"] > 1 and lay["hash_cache"], lay
    plan.run()
    cut_sum, best, updates = plan.summary()
    out = plan.download()
    plan.close()
    assert (cut_sum, best, updates) == (598190, 2164, 4096 * 20000 * 1000)
    _check_digest(golden_full, "c4_g81", _digest(out["spins"], out["inputs"], out["cut_trace"],
                                                  out["counts"], out["best_cut"]))
    for k in (0, 1, 2047, 4095):
        assert np.array_equal(out["spins"][k], golden_bench[f"g81_psa_s0_{k}_spins"])
        assert np.array_equal(out["cut_trace"][k], golden_bench[f"g81_psa_s0_{k}_cut"])


def test_full_batch_one_shot_call_matches_oracle(bench_graphs, golden_full):
    """The same batch through the one-shot C-ABI call (what run_trials and the
    bench's e2e leg use: pipelined word phases, outputs copied per phase)."""
    from paper_2601_14476_b200 import streams as st
    g = bench_graphs("G81")
    model = maxcut_to_ising(g)
    sch = derive_schedule(model, 1000, 10)
    b = _native.Batch(model, sch, st.run_keys(st.trial_seeds(0, 4096)), graph=g)
    out, _ = _native.anneal_batch(b)
    _check_digest(golden_full, "c4_g81", _digest(out["spins"], out["inputs"], out["cut_trace"],
                                                  out["counts"], out["best_cut"]))


@pytest.mark.parametrize("tag,name,sig,trials,env,kernel", [
    ("c3_g22", "G22", (0.5, 0.5, 0.5), 4096, {}, "packed_bucket"),
    ("c3_g22", "G22", (0.5, 0.5, 0.5), 4096, {"PBSA_RESIDENT": "1"}, "resident_timing"),
    ("c3_g55", "G55", (0.5, 0.5, 0.5), 4096, {}, "packed_bucket"),
    ("c3_g55", "G55", (0.5, 0.5, 0.5), 4096, {"PBSA_BUCKET": "0"}, "packed_timing"),
    ("c2_g1_nu1", "G1", (0.0, 0.0, 1.0), 1024, {}, "resident_timing"),
    ("c2_g1_nu1", "G1", (0.0, 0.0, 1.0), 1024, {"PBSA_RESIDENT": "0"}, "packed_bucket")])
def test_full_batch_variability_configs_match_oracle(bench_graphs, golden_full, golden_bench,
                                                     monkeypatch, tag, name, sig, trials, env,
                                                     kernel):
    """BASELINE C3 (G22 / G55 x 4096, sigma = 0.5^3) and C2's sigma_nu = 1 row
    (G1 x 1024) through engine.run_trials -- the reference's own entry point,
    per-trial seeds and profiles as /root/reference/pkg/src/pbitsa/engine.py:101-116
    -- on the kernel each config runs by default and on the alternative one:
    every trial equals the oracle's, and the trials the reference recorded
    (1024, 4095) equal the reference's outputs."""
    for k, v in env.items():
        monkeypatch.setenv(k, v)
    g = bench_graphs(name)
    model = maxcut_to_ising(g)
    sch = derive_schedule(model, 1000, 10)
    cfg = VariabilityConfig(*sig)
    from paper_2601_14476_b200 import streams as st
    seeds = st.trial_seeds(0, trials)
    from paper_2601_14476_b200.profiles import sample_profiles
    lam, delta, period = sample_profiles(cfg, model.n, seeds)
    b = _native.Batch(model, sch, st.run_keys(seeds), profile_rows=(lam, delta, period, model.n),
                      graph=g)
    plan = _native.Plan(b)
    assert plan.info()["kernel"] == kernel, plan.info()
    plan.close()
    spec = engine.ExperimentSpec(graph=name, algo=AlgorithmConfig(Algorithm.PSA),
                                 variability=cfg, cycles=1000, trials=trials)
    s = engine.run_trials(spec, {name: g})
    rs = s.results
    _check_digest(golden_full, tag, _digest(
        np.stack([r.final_state.spins for r in rs]), np.stack([r.final_state.inputs for r in rs]),
        np.stack([r.cut_trace for r in rs]), np.stack([r.update_counts for r in rs]),
        [r.best_cut for r in rs]))
    bench_tag = {"c3_g22": "g22_psa_s5", "c3_g55": "g55_psa_s5"}.get(tag)
    if bench_tag:
        for k in (1024, 4095):
            p = f"{bench_tag}_{k}_"
            assert np.array_equal(rs[k].final_state.spins, golden_bench[p + "spins"]), p
            assert np.array_equal(rs[k].cut_trace, golden_bench[p + "cut"]), p
            assert np.array_equal(rs[k].final_state.inputs, golden_bench[p + "inputs"]), p


@pytest.mark.parametrize("rng,sig,trials", [("replay", (0, 0, 0), 301), ("philox", (0, 0, 0), 300),
                                            ("replay", (0.5, 0.5, 0.5), 130)])
def test_run_trials_device_list_equals_one_device(bench_graphs, monkeypatch, rng, sig, trials):
    """engine.run_trials over a device-ordinal list (ExperimentSpec.devices or
    PBSA_DEVICES; the library shards the batch: pbsa_anneal_loop_batch_devices,
    4-aligned shards, one host thread and plan per shard) is trial-identical
    to one device -- here the one visible B200 listed several times."""
    g = bench_graphs("G81")
    base = engine.ExperimentSpec(graph="G81", algo=AlgorithmConfig(Algorithm.PSA), cycles=40,
                                 trials=trials, rng=rng, variability=VariabilityConfig(*sig))
    one = engine.run_trials(base, {"G81": g}, {"G81": 14004})
    three = engine.run_trials(dataclasses.replace(base, devices=(0, 0, 0)), {"G81": g}, {"G81": 14004})
    monkeypatch.setenv("PBSA_DEVICES", "0,0")
    env2 = engine.run_trials(base, {"G81": g}, {"G81": 14004})
    for other in (three, env2):
        assert len(other.results) == trials
        for a, b in zip(one.results, other.results):
            assert np.array_equal(a.final_state.spins, b.final_state.spins)
            assert np.array_equal(a.final_state.inputs, b.final_state.inputs)
            assert np.array_equal(a.cut_trace, b.cut_trace)
            assert np.array_equal(a.update_counts, b.update_counts)
        assert one.mean_cut == other.mean_cut and one.std_cut == other.std_cut


@pytest.mark.parametrize("name,trials,rng", [("G81", 600, "replay"), ("G55", 1000, "philox")])
def test_cached_one_shot_plan_equals_uncached(bench_graphs, monkeypatch, name, trials, rng):
    """One-shot calls with page-locked outputs reuse their plan (graph with the
    per-phase output copies) for the next call of the same shape: a second
    call with other per-trial keys and other output buffers, and a third with
    the first keys, equal fresh uncached calls (PBSA_PLAN_CACHE=0)."""
    import torch
    g = bench_graphs(name)
    model = maxcut_to_ising(g)
    sch = derive_schedule(model, 40, 10)
    seed = 0x1357_2468

    def batch(base):
        return _native.Batch(model, sch, streams.run_keys(streams.trial_seeds(base, trials)), graph=g,
                             rng=rng, rng_seed=seed)

    def pinned(b):
        return {k: torch.empty(v.shape, dtype=getattr(torch, str(v.dtype)), pin_memory=True).numpy()
                for k, v in b.alloc_outputs().items()}
    b1, b2 = batch(0), batch(7)
    A, B = pinned(b1), pinned(b1)
    _native.plan_cache_clear()
    r1 = {k: v.copy() for k, v in _native.anneal_batch(b1, out=A)[0].items()}
    r2 = {k: v.copy() for k, v in _native.anneal_batch(b2, out=B)[0].items()}
    r3 = {k: v.copy() for k, v in _native.anneal_batch(b1, out=B)[0].items()}
    monkeypatch.setenv("PBSA_PLAN_CACHE", "0")
    ref1, _ = _native.anneal_batch(b1)
    ref2, _ = _native.anneal_batch(b2)
    for k in _native.OUT_ORDER:
        assert np.array_equal(r1[k], ref1[k]), k
        assert np.array_equal(r2[k], ref2[k]), k
        assert np.array_equal(r3[k], ref1[k]), k
    _native.plan_cache_clear()


@pytest.mark.parametrize("sig", [(0.0, 0.0, 0.0), (0.4, 0.3, 0.6)])
def test_wide_graph_uses_32_bit_csr_and_matches_oracle(oracle, sig):
    """n > 32768: the device CSR falls back from 16-bit to 32-bit column |
    sign entries (the packed sweep and the bucket kernel branch per node);
    ideal and timing-spread profiles against the oracle."""
    from paper_2601_14476_b200.model import MaxCutGraph
    rng = np.random.default_rng(3)
    n = 33000
    a, b = rng.integers(0, n, 70000), rng.integers(0, n, 70000)
    pairs = sorted({(int(min(x, y)), int(max(x, y))) for x, y in zip(a, b) if x != y})
    g = MaxCutGraph.from_edges(n, [(i, j, int(rng.choice([-1, 1]))) for i, j in pairs])
    model = maxcut_to_ising(g)
    assert model.n == 33000
    sch = derive_schedule(model, 12, 10)
    T = 40
    seeds = [streams.trial_seed(2, k) for k in range(T)]
    vc = VariabilityConfig(*sig)
    profs = None if vc.is_ideal else [
        sample_variability(vc, g.n, np.random.default_rng(streams.profile_seed(s))) for s in seeds]
    keys = [streams.run_key(s) for s in seeds]
    b = _native.Batch(model, sch, keys, profile_rows=profile_rows(profs, model.n), graph=g)
    plan = _native.Plan(b)
    assert plan.info()["path"] == "packed"
    plan.run()
    got = plan.download()
    plan.close()
    want = oracle.anneal_batch(model, sch, "psa", profs or VariabilityProfile.ideal(model.n), keys,
                               graph=g)
    for k in ("spins", "inputs", "counts", "energy_trace", "cut_trace", "best_cut"):
        assert np.array_equal(got[k], want[k]), k


def test_cached_one_shot_plans_are_keyed_by_model_and_schedule(bench_graphs, monkeypatch):
    """Kept plans never leak between shapes: two structure-matched graphs of
    the same size (G81 analog and a relabelled torus) and two schedules give
    the results of fresh uncached calls."""
    import torch
    g = bench_graphs("G81")
    perm = np.random.default_rng(5).permutation(g.n)
    from paper_2601_14476_b200.model import MaxCutGraph
    g2 = MaxCutGraph.from_edges(g.n, [(int(min(perm[i], perm[j])), int(max(perm[i], perm[j])), int(w))
                                      for i, j, w in zip(g.edge_i, g.edge_j, g.edge_w)])
    keys = streams.run_keys(streams.trial_seeds(0, 600))
    batches = []
    for graph in (g, g2):
        model = maxcut_to_ising(graph)
        for cycles in (30, 31):
            batches.append(_native.Batch(model, derive_schedule(model, cycles, 10), keys, graph=graph))
    _native.plan_cache_clear()
    got = []
    for b in batches + batches:
        out = {k: torch.empty(v.shape, dtype=getattr(torch, str(v.dtype)), pin_memory=True).numpy()
               for k, v in b.alloc_outputs().items()}
        got.append({k: v.copy() for k, v in _native.anneal_batch(b, out=out)[0].items()})
    monkeypatch.setenv("PBSA_PLAN_CACHE", "0")
    for j, b in enumerate(batches + batches):
        want, _ = _native.anneal_batch(b)
        for k in _native.OUT_ORDER:
            assert np.array_equal(got[j][k], want[k]), (j, k)
    _native.plan_cache_clear()


@pytest.mark.parametrize("name,sig,rng", [("G55", (0, 0, 0), "replay"), ("G60", (0.5, 0.5, 0.5), "replay"),
                                          ("G55", (0, 0, 0), "philox"), ("G22", (0, 0, 0.7), "replay")])
@pytest.mark.parametrize("order", ["1", "0"])
def test_degree_order_is_bitwise_neutral(oracle, bench_graphs, monkeypatch, name, sig, rng, order):
    """The degree-sorted processing order of irregular graphs (warps take
    nodes of similar degree; labels, spin layout and draws unchanged) on the
    packed sweep and the bucket kernel, forced on and off: equal to the oracle."""
    monkeypatch.setenv("PBSA_DEGREE_ORDER", order)
    monkeypatch.setenv("PBSA_RESIDENT", "0")
    g = bench_graphs(name)
    model = maxcut_to_ising(g)
    sch = derive_schedule(model, 30, 10)
    T = 70
    seeds = [streams.trial_seed(4, k) for k in range(T)]
    vc = VariabilityConfig(*sig)
    profs = None if vc.is_ideal else [
        sample_variability(vc, g.n, np.random.default_rng(streams.profile_seed(s))) for s in seeds]
    keys = [streams.run_key(s) for s in seeds]
    seed = 0x2468_ACE0
    b = _native.Batch(model, sch, keys, profile_rows=profile_rows(profs, model.n), graph=g, rng=rng,
                      rng_seed=seed)
    plan = _native.Plan(b)
    plan.run()
    got = plan.download()
    plan.close()
    extra = dict(rng="philox", rng_seed=seed) if rng == "philox" else {}
    want = oracle.anneal_batch(model, sch, "psa", profs or VariabilityProfile.ideal(model.n), keys,
                               graph=g, **extra)
    for k in ("spins", "inputs", "counts", "energy_trace", "cut_trace", "best_cut"):
        assert np.array_equal(got[k], want[k]), k


# ------------------------------------------ native (device-drawn) variability profiles

def test_native_profiles_are_the_reference_distributions():
    """pbsa_native_profiles: lam ~ N(1, s_l^2), delta ~ N(0, s_d^2),
    period = max(1, rint(t_res (1 + N(0, s_n^2)))) (pbit.py:57-75) -- moments,
    the period histogram against numpy's draw of the same law, shard
    invariance (trial k's profile depends only on its global index)."""
    sig = (0.5, 0.3, 0.5)
    lam, delta, per = _native.native_profiles(0xABC, 0, 512, 4000, 10, 1000, sig)
    assert abs(lam.mean() - 1.0) < 0.003 and abs(lam.std() - 0.5) < 0.003
    assert abs(delta.mean()) < 0.002 and abs(delta.std() - 0.3) < 0.002
    ref = sample_variability(VariabilityConfig(*sig), 2_048_000, np.random.default_rng(3)).period
    for p in range(1, 25):
        assert abs((per == p).mean() - (ref == p).mean()) < 0.003, p
    lam2, delta2, per2 = _native.native_profiles(0xABC, 256, 256, 4000, 10, 1000, sig)
    assert np.array_equal(lam[256:], lam2) and np.array_equal(per[256:], per2)
    assert np.array_equal(delta[256:], delta2)


@pytest.mark.parametrize("name,sig,trials,cycles", [("G81", (0.5, 0.5, 0.5), 96, 30),
                                                    ("G55", (0.7, 0.2, 0.0), 64, 40),
                                                    ("G1", (0.0, 0.0, 0.8), 40, 30)])
def test_native_profile_runs_match_oracle_on_their_profiles(oracle, bench_graphs, name, sig, trials,
                                                            cycles):
    """A native-profile plan (profiles drawn on the device at plan creation,
    bucket / plain variability kernels) equals the oracle's Philox run on the
    same profiles, fetched with pbsa_native_profiles."""
    g = bench_graphs(name)
    model = maxcut_to_ising(g)
    sch = derive_schedule(model, cycles, 10)
    seed = 0x51DE_5EED
    keys = [streams.run_key(streams.trial_seed(9, k)) for k in range(trials)]
    b = _native.Batch(model, sch, keys, graph=g, rng="philox", rng_seed=seed, native_sigmas=sig)
    got, _ = _native.anneal_batch(b)
    lam, delta, per = _native.native_profiles(seed, 0, trials, g.n, 10, cycles, sig)
    profs = [VariabilityProfile(lam[k], delta[k], per[k], 10) for k in range(trials)]
    want = oracle.anneal_batch(model, sch, "psa", profs, keys, graph=g, rng="philox", rng_seed=seed)
    for k in ("spins", "inputs", "counts", "energy_trace", "cut_trace", "best_cut"):
        assert np.array_equal(got[k], want[k]), k


@pytest.mark.parametrize("name,sig,trials", [("G81", (0.5, 0.5, 0.5), 256), ("G1", (0.0, 0.0, 0.5), 128),
                                             ("G55", (1.0, 0.0, 0.0), 256)])
def test_native_profile_cut_statistics_match_reference(bench_graphs, golden_analogs, name, sig, trials):
    """ExperimentSpec(rng='philox', native_profiles=True): the profiles come
    from the device, not numpy; mean final cut and mean per-trial best cut
    within 0.5 % of the best-known cut of the reference's replayed run."""
    g = bench_graphs(name)
    best_known = golden_analogs[name]["best_known_analog"]
    spec = engine.ExperimentSpec(graph=name, algo=AlgorithmConfig(Algorithm.PSA),
                                 variability=VariabilityConfig(*sig), cycles=1000, trials=trials)
    rep = engine.run_trials(spec, {name: g})
    nat = engine.run_trials(dataclasses.replace(spec, rng="philox", native_profiles=True), {name: g})
    assert abs(nat.mean_cut - rep.mean_cut) <= 0.005 * best_known, (nat.mean_cut, rep.mean_cut)
    b_rep = np.mean([r.best_cut for r in rep.results])
    b_nat = np.mean([r.best_cut for r in nat.results])
    assert abs(b_nat - b_rep) <= 0.005 * best_known, (b_nat, b_rep)


# ------------------------------------------------ launch shapes of the packed sweep

@pytest.mark.parametrize("name,trials", [("G77", 1024), ("G81", 512), ("G55", 4096)])
def test_launch_shapes_are_bitwise_neutral(oracle, bench_graphs, monkeypatch, name, trials):
    """The word-phase width and chunk balance the wave model picks
    (plan.cu choose_phases), and forced alternatives (one phase, other widths,
    balance on/off): every shape equals the oracle bit for bit."""
    g = bench_graphs(name)
    model = maxcut_to_ising(g)
    sch = derive_schedule(model, 6, 10)
    seeds = [streams.trial_seed(6, k) for k in range(trials)]
    keys = [streams.run_key(s) for s in seeds]
    b = _native.Batch(model, sch, keys, graph=g)
    want = oracle.anneal_batch(model, sch, "psa", VariabilityProfile.ideal(model.n), keys, graph=g)
    W = trials // 32
    shapes = [{}, {"PBSA_PACKED_PHASE_WORDS": "0", "PBSA_BALANCE_CHUNKS": "0"},
              {"PBSA_PACKED_PHASE_WORDS": str(max(1, W // 3)), "PBSA_BALANCE_CHUNKS": "1"},
              {"PBSA_PACKED_PHASE_WORDS": str(max(1, W // 2 + 1)), "PBSA_BALANCE_CHUNKS": "0"},
              # the 1-D grid (per-warp division) and the L1 tile prefetch paths
              {"PBSA_GRID2D": "0", "PBSA_CACHE_PREFETCH": "1"},
              # one cut flush per warp instead of per block (warps per word not a multiple of 4)
              {"PBSA_CTA_FLUSH": "0", "PBSA_WARPS_PER_WORD": "37"}]
    knobs = ("PBSA_PACKED_PHASE_WORDS", "PBSA_BALANCE_CHUNKS", "PBSA_GRID2D", "PBSA_CACHE_PREFETCH",
             "PBSA_CTA_FLUSH", "PBSA_WARPS_PER_WORD")
    seen = set()
    for env in shapes:
        for k in knobs:
            monkeypatch.delenv(k, raising=False)
        for k, v in env.items():
            monkeypatch.setenv(k, v)
        plan = _native.Plan(b)
        lay = plan.layout()
        plan.run()
        got = plan.download()
        plan.close()
        seen.add((lay["phase_words"], lay["warps_per_word"]))
        for k in ("spins", "inputs", "counts", "energy_trace", "cut_trace", "best_cut"):
            assert np.array_equal(got[k], want[k]), (env, lay, k)
    assert len(seen) >= 3, seen


@pytest.mark.parametrize("name,trials,sig,kernel", [
    ("G1", 128, (0, 0, 0), "resident"),
    ("G81", 4096, (0, 0, 0), "packed"),
    ("G55", 4096, (0.5, 0.5, 0.5), "packed_bucket"),
    ("G22", 1024, (0.0, 0.0, 0.5), "resident_timing"),
    ("G60", 1000, (0.5, 0.5, 0.0), "packed")])
def test_shortest_runs_match_oracle(oracle, bench_graphs, name, trials, sig, kernel):
    """Two cycles (the shortest schedule the API admits) on every kernel
    family at its production batch shape: the first cycle's sweep, the one
    cut pass per phase and the last-cycle outputs (inputs, counts) meet with
    no steady state in between; equal to the oracle bit for bit."""
    g = bench_graphs(name)
    model = maxcut_to_ising(g)
    sch = derive_schedule(model, 2, 10)
    seeds = [streams.trial_seed(8, k) for k in range(trials)]
    vc = VariabilityConfig(*sig)
    profs = None if vc.is_ideal else [
        sample_variability(vc, g.n, np.random.default_rng(streams.profile_seed(s))) for s in seeds]
    keys = [streams.run_key(s) for s in seeds]
    b = _native.Batch(model, sch, keys, profile_rows=profile_rows(profs, model.n), graph=g)
    plan = _native.Plan(b)
    assert plan.info()["kernel"] == kernel, plan.info()
    plan.run()
    got = plan.download()
    plan.close()
    want = oracle.anneal_batch(model, sch, "psa", profs or VariabilityProfile.ideal(model.n), keys, graph=g)
    for k in ("spins", "inputs", "counts", "energy_trace", "cut_trace", "best_cut"):
        assert np.array_equal(got[k], want[k]), k


@pytest.mark.parametrize("env", [{}, {"PBSA_GRID2D": "1"}, {"PBSA_BUCKET": "0"}])
def test_bucket_kernel_shapes_match_oracle(oracle, bench_graphs, monkeypatch, env):
    """The period-bucket kernel on the 2-D grid (default 1-D) and the
    fallback timing kernel, on a timing-spread batch: equal to the oracle."""
    for k, v in env.items():
        monkeypatch.setenv(k, v)
    g = bench_graphs("G55")
    model = maxcut_to_ising(g)
    sch = derive_schedule(model, 4, 10)
    seeds = [streams.trial_seed(9, k) for k in range(256)]
    vc = VariabilityConfig(0.5, 0.5, 0.5)
    profs = [sample_variability(vc, g.n, np.random.default_rng(streams.profile_seed(s))) for s in seeds]
    keys = [streams.run_key(s) for s in seeds]
    b = _native.Batch(model, sch, keys, profile_rows=profile_rows(profs, model.n), graph=g)
    plan = _native.Plan(b)
    want_kernel = "packed_timing" if env.get("PBSA_BUCKET") == "0" else "packed_bucket"
    assert plan.info()["kernel"] == want_kernel, plan.info()
    plan.run()
    got = plan.download()
    plan.close()
    want = oracle.anneal_batch(model, sch, "psa", profs, keys, graph=g)
    for k in ("spins", "inputs", "counts", "energy_trace", "cut_trace", "best_cut"):
        assert np.array_equal(got[k], want[k]), k
