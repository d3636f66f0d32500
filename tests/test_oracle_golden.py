"""Pin the CPU oracle (oracle/psa_oracle.c) to the reference's own outputs.

The golden fixtures were produced by importing the reference package
(tests/golden/make_golden.py); the oracle must reproduce them bit-for-bit
before it is trusted as the checker for the CUDA path.
"""

from __future__ import annotations

import numpy as np
import pytest

from cases import BENCH_CASES, bench_inputs, small_case


def test_oracle_stream_kats(oracle, golden_streams):
    # pinned values of /root/reference/pkg/tests/test_streams.py:26-45
    assert oracle.mix64(1) == 0x10A81D8AD3D870A3
    assert oracle.stream_u64(42, 3, 7, 123) == 0xB71C3C338A17B8FA
    assert oracle.run_key(0) == 0x9D9A85784BF1C21D
    assert oracle.trial_seed(0, 0) == 0x805BF55D41EBCFB0
    assert oracle.trial_seed(0, 1) == 0xDA28150A69217582
    assert oracle.profile_seed(12345) == 0xB62E0384700FB443
    assert oracle.uniform01(9, 3, 5, 17) == 0.2934698501022247
    for z, want in golden_streams["mix64"].items():
        assert oracle.mix64(int(z)) == int(want)
    for key, tag, a, b, want, u in golden_streams["grid"]:
        assert oracle.stream_u64(int(key), tag, int(a), b) == int(want)
        assert oracle.uniform01(int(key), tag, int(a), b) == float.fromhex(u)


@pytest.mark.parametrize("pname", ["ideal", "varied"])
@pytest.mark.parametrize("kind", ["psa", "tapsa", "spsa"])
def test_oracle_small_case_matches_reference(oracle, golden_small, pname, kind):
    g, model, sch, profiles = small_case()
    assert np.array_equal(np.stack([g.edge_i, g.edge_j, g.edge_w]), golden_small["edges"])
    prof = profiles[pname]
    alpha = 3 if kind == "tapsa" else 1
    for seed in (0, 1):
        from paper_2601_14476_b200 import streams
        out = oracle.anneal_batch(model, sch, kind, prof, [streams.run_key(seed)], graph=g,
                                  alpha=alpha, p_stall=0.4, threads=1)
        p = f"{pname}_{kind}_{seed}_"
        assert np.array_equal(out["spins"][0], golden_small[p + "spins"])
        assert np.array_equal(out["inputs"][0], golden_small[p + "inputs"])
        assert np.array_equal(out["hist"][0], golden_small[p + "hist"])
        assert np.array_equal(out["counts"][0], golden_small[p + "counts"])
        assert np.array_equal(out["i0_trace"][0], golden_small[p + "i0"])
        assert np.array_equal(out["energy_trace"][0], golden_small[p + "energy"])
        assert np.array_equal(out["cut_trace"][0], golden_small[p + "cut"])
        assert out["best_cut"][0] == golden_small[p + "best"]


# one representative trial per benchmark config keeps the CPU suite short
ORACLE_BENCH = [("g1_psa_s0", [0, 3]), ("g1_psa_s5", [1]), ("g1_tapsa_s0", [0]),
                ("g1_spsa_s0", [1]), ("g22_psa_s5", [1024]), ("g55_psa_s5", [0, 4095]),
                ("g81_psa_s0", [2047]), ("g81_psa_s5", [0])]


@pytest.mark.parametrize("tag,trials", ORACLE_BENCH)
def test_oracle_benchmark_runs_match_reference(oracle, golden_bench, bench_graphs, tag, trials):
    name, kind, sig, _ = BENCH_CASES[tag]
    graph = bench_graphs(name)
    model, sch, cfg, seeds, profs, keys = bench_inputs(graph, kind, sig, trials)
    out = oracle.anneal_batch(model, sch, kind.value, profs if profs else _ideal(graph.n), keys,
                              graph=graph, alpha=cfg.kernel_alpha, p_stall=cfg.p_stall)
    for idx, k in enumerate(trials):
        p = f"{tag}_{k}_"
        assert np.array_equal(out["spins"][idx], golden_bench[p + "spins"]), p
        assert np.array_equal(out["cut_trace"][idx], golden_bench[p + "cut"]), p
        assert out["best_cut"][idx] == golden_bench[p + "best"]
        assert out["counts"][idx].sum() == golden_bench[p + "counts_sum"]
        assert np.array_equal(out["inputs"][idx], golden_bench[p + "inputs"]), p


def _ideal(n):
    from paper_2601_14476_b200.pbit import VariabilityProfile
    return VariabilityProfile.ideal(n)


def test_profile_golden_prefix(golden_bench, bench_graphs):
    # host profile sampling reproduces the reference draws (pbit.py:57-75)
    for tag in ("g55_psa_s5", "g22_psa_s5", "g81_psa_s5"):
        name, kind, sig, _ = BENCH_CASES[tag]
        *_, profs, _ = bench_inputs(bench_graphs(name), kind, sig, [0])
        p = f"{tag}_0_"
        assert np.array_equal(profs[0].lam[:3], golden_bench[p + "lam3"])
        assert np.array_equal(profs[0].delta[:3], golden_bench[p + "delta3"])
        assert np.array_equal(profs[0].period[:8], golden_bench[p + "period8"])


@pytest.mark.parametrize("name,kind,sig", [("G1", "psa", (0.0, 0.0, 0.3)),
                                           ("G47", "tapsa", (0.5, 0.0, 0.0)),
                                           ("G48", "spsa", (0.0, 0.5, 0.0))])
def test_oracle_acceptance_criterion_7_specs(oracle, golden_acceptance, bench_graphs, name, kind, sig):
    """Variability runs of all three rules (test_acceptance.py:205-230 specs:
    120 cycles, 6 trials, seed 2, default alpha 4 / p_stall 0.5)."""
    from paper_2601_14476_b200 import streams
    from paper_2601_14476_b200.annealer import derive_schedule
    from paper_2601_14476_b200.model import maxcut_to_ising
    from paper_2601_14476_b200.pbit import VariabilityConfig, sample_variability
    g = bench_graphs(name)
    model = maxcut_to_ising(g)
    sch = derive_schedule(model, 120, 10)
    seeds = [streams.trial_seed(2, k) for k in range(6)]
    profs = [sample_variability(VariabilityConfig(*sig), g.n,
                                np.random.default_rng(streams.profile_seed(s))) for s in seeds]
    out = oracle.anneal_batch(model, sch, kind, profs, [streams.run_key(s) for s in seeds], graph=g,
                              alpha=4, p_stall=0.5)
    assert np.array_equal(out["cut_trace"], golden_acceptance[f"c7_{name}_{kind}_cut_traces"])
    assert np.array_equal(out["energy_trace"], golden_acceptance[f"c7_{name}_{kind}_energy_traces"])


def test_oracle_philox_matches_random123_kats(oracle):
    """The native stream's generator, pinned by the published Random123
    known-answer vectors (the reference has no Philox; see include/pbsa.h)."""
    kats = [
        ([0, 0, 0, 0], [0, 0], [0x6627E8D5, 0xE169C58D, 0xBC57AC4C, 0x9B00DBD8]),
        ([0xFFFFFFFF] * 4, [0xFFFFFFFF] * 2, [0x408F276D, 0x41C83B0E, 0xA20BC7C6, 0x6D5451FD]),
        ([0x243F6A88, 0x85A308D3, 0x13198A2E, 0x03707344], [0xA4093822, 0x299F31D0],
         [0xD16CFE09, 0x94FDCCEB, 0x5001E420, 0x24126EA1]),
    ]
    for ctr, key, want in kats:
        assert oracle.philox4x32_10(ctr, key) == want


def test_oracle_philox_mode_is_a_different_stream_with_the_same_schedule(oracle):
    """rng="philox" changes only the activation draws: same i0 trace, same
    initial spins, same update counts; different trajectories."""
    from paper_2601_14476_b200.annealer import derive_schedule
    from paper_2601_14476_b200.model import maxcut_to_ising
    from paper_2601_14476_b200.pbit import VariabilityProfile
    from cases import random_graph
    g = random_graph(40, 3, p_edge=0.15)
    model = maxcut_to_ising(g)
    sch = derive_schedule(model, 30, 10)
    keys = [oracle.run_key(oracle.trial_seed(0, k)) for k in range(8)]
    prof = VariabilityProfile.ideal(model.n)
    a = oracle.anneal_batch(model, sch, "psa", prof, keys, graph=g)
    b = oracle.anneal_batch(model, sch, "psa", prof, keys, graph=g, rng="philox", rng_seed=99)
    c = oracle.anneal_batch(model, sch, "psa", prof, keys[4:], graph=g, rng="philox",
                            rng_seed=99, first_trial=4)
    assert np.array_equal(a["i0_trace"], b["i0_trace"])
    assert np.array_equal(a["counts"], b["counts"])
    assert not np.array_equal(a["cut_trace"], b["cut_trace"])
    for k in ("spins", "cut_trace", "energy_trace", "inputs"):
        assert np.array_equal(b[k][4:], c[k])
