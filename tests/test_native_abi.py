"""The C-ABI library (CPU-side checks, no GPU compute).

* libpbsa.so loads and exports every function include/pbsa.h declares;
* the host build of the device tanh (libm_tanh.cuh) equals the system libm
  bit-for-bit -- the property that makes varied-profile runs replay the
  reference exactly;
* the packed path's integer activation threshold equals the reference's
  floating-point decision ``r + t >= 0`` (_kernels.py:149-152) exactly;
* compute entry points fail loudly (no CPU fallback) without a GPU.
"""

from __future__ import annotations

import math
import re
from fractions import Fraction
from pathlib import Path

import numpy as np
import pytest

from paper_2601_14476_b200 import _native

HEADER = Path(__file__).resolve().parents[1] / "include" / "pbsa.h"


def declared_functions() -> list[str]:
    text = re.sub(r"/\*.*?\*/", "", HEADER.read_text(), flags=re.S)
    return sorted(set(re.findall(r"\b(pbsa_[a-z0-9_]+)\s*\(", text)))


def test_library_exports_every_declared_symbol():
    lib = _native.load()
    names = declared_functions()
    assert len(names) >= 14
    for name in names:
        assert hasattr(lib, name), name
    assert set(names) == set(_native.EXPORTED)
    assert lib.pbsa_abi_version() == 1


def test_host_tanh_port_equals_libm():
    lib = _native.load()
    rng = np.random.default_rng(11)
    xs = np.concatenate([rng.uniform(-25, 25, 60_000), rng.uniform(-1.5, 1.5, 60_000),
                         np.ldexp(rng.uniform(0.5, 1.0, 30_000), rng.integers(-70, 6, 30_000)),
                         -np.ldexp(rng.uniform(0.5, 1.0, 30_000), rng.integers(-70, 6, 30_000)),
                         np.array([0.0, -0.0, 22.0, -22.0, 21.99999, 1.0, -1.0, 0.5 * math.log(3)])])
    bad = [x for x in xs if lib.pbsa_libm_tanh_host(float(x)).hex() != math.tanh(float(x)).hex()]
    assert not bad, bad[:5]


def _decision_exact(t: float, u53: int) -> bool:
    """The reference decision r + t >= 0 with r = 2 (u / 2^53) - 1."""
    r = 2.0 * (u53 * 2.0 ** -53) - 1.0
    return r + t >= 0.0


def test_threshold_matches_reference_decision():
    lib = _native.load()
    rng = np.random.default_rng(12)
    ts = [math.tanh(x) for x in np.concatenate([rng.normal(0, 2, 3000), rng.normal(0, 1e-6, 500)])]
    ts += [1.0, -1.0, 0.0, -0.0, math.tanh(20.0), math.tanh(-20.0), 2.0 ** -60, -(2.0 ** -60)]
    for t in ts:
        thr = int(lib.pbsa_threshold_host(t))
        if thr == (1 << 64) - 1:  # never +1
            assert not _decision_exact(t, (1 << 53) - 1)
            continue
        assert thr % 2048 == 0
        U = thr >> 11
        # exact rational threshold
        assert U == max(0, math.ceil((1 - Fraction(t)) * 2 ** 52))
        for u in (U - 1, U, U + 1):
            if 0 <= u < (1 << 53):
                assert _decision_exact(t, u) == (u >= U), (t, u)


def test_compute_calls_fail_loudly_without_gpu():
    if _native.device_count() > 0:
        pytest.skip("a GPU is visible")
    with pytest.raises(RuntimeError, match="no CUDA device"):
        _native.require_device(0)
    from paper_2601_14476_b200 import annealer, model, pbit
    g = model.MaxCutGraph.from_edges(3, [(0, 1, 1), (1, 2, 1)])
    m = model.maxcut_to_ising(g)
    sch = annealer.derive_schedule(m, 5)
    with pytest.raises(RuntimeError):
        annealer.run_anneal(m, sch, annealer.AlgorithmConfig(annealer.Algorithm.PSA),
                            pbit.VariabilityProfile.ideal(3), seed=0, graph=g)


# Random123 known-answer vectors for Philox4x32-10 (kat_vectors, philox4x32_10):
# (counter, key, output)
PHILOX_KATS = [
    ([0, 0, 0, 0], [0, 0], [0x6627E8D5, 0xE169C58D, 0xBC57AC4C, 0x9B00DBD8]),
    ([0xFFFFFFFF] * 4, [0xFFFFFFFF] * 2, [0x408F276D, 0x41C83B0E, 0xA20BC7C6, 0x6D5451FD]),
    ([0x243F6A88, 0x85A308D3, 0x13198A2E, 0x03707344], [0xA4093822, 0x299F31D0],
     [0xD16CFE09, 0x94FDCCEB, 0x5001E420, 0x24126EA1]),
]


def test_host_philox_matches_random123_kats():
    for ctr, key, want in PHILOX_KATS:
        assert _native.philox_host(ctr, key) == want


def test_host_philox_equals_oracle_philox(oracle):
    rng = np.random.default_rng(3)
    for _ in range(2000):
        ctr = [int(x) for x in rng.integers(0, 2 ** 32, 4)]
        key = [int(x) for x in rng.integers(0, 2 ** 32, 2)]
        assert _native.philox_host(ctr, key) == oracle.philox4x32_10(ctr, key)


def _native_decision(t: float, x: int) -> bool:
    """The oracle's native decision: r = (2X + 1) 2^-32 - 1, +1 iff r + t >= 0."""
    r = (2.0 * x + 1.0) * 2.0 ** -32 - 1.0
    return r + t >= 0.0


def test_native_threshold_matches_native_decision():
    lib = _native.load()
    rng = np.random.default_rng(12)
    ts = np.concatenate([np.tanh(rng.uniform(-30, 30, 3000)), rng.uniform(-1, 1, 3000),
                         np.ldexp(rng.uniform(-1, 1, 1000), rng.integers(-60, 0, 1000)),
                         np.array([-1.0, 1.0, 0.0, -0.0, 2.0 ** -33, -(2.0 ** -33),
                                   1 - 2.0 ** -53, -1 + 2.0 ** -53])])
    for t in ts:
        T = int(lib.pbsa_threshold_native_host(float(t)))
        assert 0 <= T <= 2 ** 32
        if T < 2 ** 32:
            assert _native_decision(float(t), T)
        if T > 0:
            assert not _native_decision(float(t), T - 1)


def test_launch_shape_model_picks_the_measured_best_phase_widths():
    """The word-phase width plan creation picks (plan.cu choose_phases, host
    export) for B200 parameters -- 148 SMs x blocks per SM x 4 warps, 5/8 of
    the 126.5 MiB L2 -- against the widths measured fastest on one B200
    (profiles/r02_summary.md, "Word-phase width"): G81 13, G77 19, G67 26,
    G60 43, one phase for G55 and G48 at 4096 trials; two phases of 16 words
    for the 1024-trial G81 shard, one phase at 512 trials."""
    import ctypes
    lib = _native.load()
    budget = 132644864 * 5 // 8

    def pick(n, words, blocks):
        bal = ctypes.c_int()
        pw = lib.pbsa_choose_phases_host((n + 31) // 32, words, 148 * blocks * 4, budget, ctypes.byref(bal))
        return pw, bal.value

    assert pick(20000, 128, 7) == (13, 1)
    assert pick(14000, 128, 7)[0] == 19
    assert pick(10000, 128, 7)[0] == 26
    assert pick(7000, 128, 8)[0] == 43
    assert pick(5000, 128, 8)[0] == 128
    assert pick(3000, 128, 7)[0] == 128
    assert pick(20000, 32, 7)[0] == 16
    assert pick(20000, 16, 7)[0] == 16
    # no L2 budget: always one phase; otherwise equal phases only
    for n, words in ((20000, 128), (9000, 100), (800, 7)):
        bal = ctypes.c_int()
        assert lib.pbsa_choose_phases_host((n + 31) // 32, words, 4144, 0, ctypes.byref(bal)) == words
        pw = lib.pbsa_choose_phases_host((n + 31) // 32, words, 4144, budget, ctypes.byref(bal))
        nph = -(-words // pw)
        assert -(-words // nph) == pw
