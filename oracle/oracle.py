"""ctypes front-end for the C restatement in ``psa_oracle.c``.

TEST INFRASTRUCTURE ONLY -- imported by ``tests/``, ``__graft_entry__.smoke()``
and ``bench.py``'s ``cpu_baseline`` / ``--impl reference`` leg as the checker.
The product path (``paper_2601_14476_b200``) never imports this module.

The entry points take duck-typed objects carrying the reference's attribute
names (``IsingModel.indptr/indices/values/h/edge_*``, ``MaxCutGraph.edge_*``,
``VariabilityProfile.lam/delta/period``, ``AnnealSchedule.i0_min/beta/
cycles/t_res``), so the same call works on the reference's own objects and on
the product package's mirrors.  Results use the reference's 8-tuple order of
``_kernels.anneal_loop`` (/root/reference/pkg/src/pbitsa/_kernels.py:175).
"""

from __future__ import annotations

import ctypes
import os
import subprocess
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
LIB_PATH = HERE / "_build" / "liboracle.so"

ALGO_CODES = {"psa": 0, "tapsa": 1, "spsa": 2}
MASK64 = (1 << 64) - 1

_lib = None


def build() -> Path:
    subprocess.run(["make", "-s", "-C", str(HERE)], check=True)
    return LIB_PATH


def lib() -> ctypes.CDLL:
    global _lib
    if _lib is None:
        if not LIB_PATH.exists():
            build()
        L = ctypes.CDLL(str(LIB_PATH))
        u64, i64, dbl, ptr = ctypes.c_uint64, ctypes.c_int64, ctypes.c_double, ctypes.c_void_p
        L.orc_mix64.restype = u64
        L.orc_mix64.argtypes = [u64]
        L.orc_stream_u64.restype = u64
        L.orc_stream_u64.argtypes = [u64, u64, u64, u64]
        L.orc_u01.restype = dbl
        L.orc_u01.argtypes = [u64, u64, u64, u64]
        L.orc_tanh.restype = dbl
        L.orc_tanh.argtypes = [dbl]
        L.orc_philox4x32_10.restype = None
        L.orc_philox4x32_10.argtypes = [ptr, ptr, ptr]
        L.orc_anneal_batch_rng.restype = ctypes.c_int
        L.orc_anneal_batch_rng.argtypes = (
            [i64, ctypes.c_int, i64, ptr, ptr, ptr, ptr, i64, ptr, ptr, ptr, i64, ptr, ptr, ptr,
             ptr, ptr, ptr, i64, dbl, dbl, i64, i64, ctypes.c_int, i64, dbl, ptr,
             ctypes.c_int, u64, i64]
            + [ptr] * 8
        )
        L.orc_anneal_batch.restype = ctypes.c_int
        L.orc_anneal_batch.argtypes = (
            [i64, ctypes.c_int, i64, ptr, ptr, ptr, ptr, i64, ptr, ptr, ptr, i64, ptr, ptr, ptr,
             ptr, ptr, ptr, i64, dbl, dbl, i64, i64, ctypes.c_int, i64, dbl, ptr]
            + [ptr] * 8
        )
        _lib = L
    return _lib


# ---------------------------------------------------------------- streams

def mix64(z: int) -> int:
    return int(lib().orc_mix64(z & MASK64))


def stream_u64(key: int, tag: int, a: int = 0, b: int = 0) -> int:
    return int(lib().orc_stream_u64(key & MASK64, tag & MASK64, a & MASK64, b & MASK64))


def uniform01(key: int, tag: int, a: int = 0, b: int = 0) -> float:
    return float(lib().orc_u01(key & MASK64, tag & MASK64, a & MASK64, b & MASK64))


def philox4x32_10(ctr, key) -> list[int]:
    """Philox4x32-10 of a 4-word counter under a 2-word key (native RNG mode)."""
    c = (ctypes.c_uint32 * 4)(*[int(x) & 0xFFFFFFFF for x in ctr])
    k = (ctypes.c_uint32 * 2)(*[int(x) & 0xFFFFFFFF for x in key])
    o = (ctypes.c_uint32 * 4)()
    lib().orc_philox4x32_10(ctypes.addressof(c), ctypes.addressof(k), ctypes.addressof(o))
    return list(o)


def run_key(seed: int) -> int:
    """streams.py:58-60"""
    return stream_u64(seed, 1, 0, 0)


def trial_seed(base_seed: int, index: int) -> int:
    """streams.py:63-68"""
    return stream_u64(base_seed, 5, index, 0)


def profile_seed(seed: int) -> int:
    """streams.py:71-73"""
    return stream_u64(seed, 6, 0, 0)


# ------------------------------------------------------------------ anneal

def _c(a, dtype):
    return np.ascontiguousarray(a, dtype=dtype)


def _p(a) -> int:
    return a.ctypes.data if a.size else 0


def anneal_batch(model, schedule, algo: str, profiles, keys, graph=None, alpha: int = 1,
                 p_stall: float = 0.5, threads: int | None = None, rng: str = "replay",
                 rng_seed: int = 0, first_trial: int = 0) -> dict:
    """Run len(keys) trials of anneal_loop on the CPU (restated in C).

    ``profiles`` is one profile object shared by all trials or a sequence
    with one per trial.  ``alpha`` follows annealer.py:235 (1 unless TAPSA).
    Returns a dict of stacked per-trial arrays in the anneal_loop order.
    ``rng="philox"`` draws the activation uniforms from the native Philox
    stream of global trials ``first_trial + t`` under ``rng_seed`` (the CUDA
    library's PBSA_RNG_PHILOX mode) instead of the reference's counter hash.
    """
    if rng not in ("replay", "philox"):
        raise ValueError(f"rng must be 'replay' or 'philox', got {rng!r}")
    keys = np.asarray([int(k) & MASK64 for k in keys], dtype=np.uint64)
    T = int(keys.size)
    n = int(model.n)
    if hasattr(profiles, "lam"):
        lam, delta, period, stride = (_c(profiles.lam, np.float64), _c(profiles.delta, np.float64),
                                      _c(profiles.period, np.int64), 0)
    else:
        lam = _c(np.stack([p.lam for p in profiles]), np.float64)
        delta = _c(np.stack([p.delta for p in profiles]), np.float64)
        period = _c(np.stack([p.period for p in profiles]), np.int64)
        stride = n
    indptr, indices = _c(model.indptr, np.int64), _c(model.indices, np.int64)
    values, h = _c(model.values, np.float64), _c(model.h, np.float64)
    me_i, me_j, me_w = (_c(model.edge_i, np.int64), _c(model.edge_j, np.int64),
                        _c(model.edge_w, np.float64))
    if graph is not None:
        ge_i, ge_j, ge_w = (_c(graph.edge_i, np.int64), _c(graph.edge_j, np.int64),
                            _c(graph.edge_w, np.int64))
    else:
        ge_i = ge_j = ge_w = np.empty(0, np.int64)
    C = int(schedule.cycles)
    code = ALGO_CODES[algo] if isinstance(algo, str) else int(algo)
    out = dict(
        spins=np.empty((T, n), np.int8), inputs=np.empty((T, n)),
        hist=np.empty((T, n, alpha)), counts=np.empty((T, n), np.int64),
        i0_trace=np.empty((T, C)), energy_trace=np.empty((T, C)),
        cut_trace=np.empty((T, C), np.int64), best_cut=np.empty(T, np.int64),
    )
    rc = lib().orc_anneal_batch_rng(
        T, int(threads or os.cpu_count() or 1), n, _p(indptr), _p(indices), _p(values), _p(h),
        int(me_i.size), _p(me_i), _p(me_j), _p(me_w), int(ge_i.size), _p(ge_i), _p(ge_j),
        _p(ge_w), _p(lam), _p(delta), _p(period), stride, float(schedule.i0_min),
        float(schedule.beta), C, int(schedule.t_res), code, int(alpha), float(p_stall),
        _p(keys), int(rng == "philox"), int(rng_seed) & MASK64, int(first_trial),
        *(_p(out[k]) for k in ("spins", "inputs", "hist", "counts", "i0_trace",
                                          "energy_trace", "cut_trace", "best_cut")))
    if rc != 0:
        raise RuntimeError(f"oracle anneal failed with status {rc}")
    return out
