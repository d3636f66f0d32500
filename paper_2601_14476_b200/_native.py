"""ctypes binding of the C ABI in include/pbsa.h (libpbsa.so, built in-tree).

This is the only route from the Python API to the compute: there is no CPU
fallback.  If the library is missing or no CUDA device is visible, every
compute entry point raises ``RuntimeError``.  ctypes releases the GIL for the
duration of each call, so trials sharded over threads/devices overlap.
"""

from __future__ import annotations

import ctypes
import os
from pathlib import Path

import numpy as np

LIB_PATH = Path(os.environ.get("PBSA_LIB") or
                Path(__file__).resolve().parent / "_lib" / "libpbsa.so")

PBSA_OK = 0
PATH_PACKED, PATH_GENERAL = 1, 2
RNG_MODES = {"replay": 0, "philox": 1}  # include/pbsa.h PBSA_RNG_*

_lib: ctypes.CDLL | None = None

_P = ctypes.c_void_p
_I64 = ctypes.c_int64
_F64 = ctypes.c_double

# (name, restype, argtypes)
_SIGNATURES = [
    ("pbsa_abi_version", ctypes.c_int, []),
    ("pbsa_last_error", ctypes.c_char_p, []),
    ("pbsa_device_count", ctypes.c_int, [ctypes.POINTER(ctypes.c_int)]),
    ("pbsa_plan_create", ctypes.c_int,
     [ctypes.c_int, _I64, _P, _P, _P, _P, _I64, _P, _P, _P, _I64, _P, _P, _P, _P, _P, _P, _I64,
      _F64, _F64, _I64, _I64, ctypes.c_int, _I64, _F64, _I64, _P, ctypes.POINTER(_P)]),
    ("pbsa_plan_create_ex", ctypes.c_int,
     [ctypes.c_int, _I64, _P, _P, _P, _P, _I64, _P, _P, _P, _I64, _P, _P, _P, _P, _P, _P, _I64,
      _F64, _F64, _I64, _I64, ctypes.c_int, _I64, _F64, _I64, _P, ctypes.c_int, ctypes.c_uint64,
      _I64, ctypes.POINTER(_P)]),
    ("pbsa_plan_run", ctypes.c_int, [_P, ctypes.POINTER(ctypes.c_float)]),
    ("pbsa_plan_download", ctypes.c_int, [_P] + [_P] * 8),
    ("pbsa_plan_summary", ctypes.c_int, [_P, ctypes.POINTER(_I64), ctypes.POINTER(_I64),
                                         ctypes.POINTER(_I64)]),
    ("pbsa_plan_info", ctypes.c_int, [_P, ctypes.POINTER(ctypes.c_int), ctypes.POINTER(_I64),
                                      ctypes.POINTER(_F64), ctypes.POINTER(_I64),
                                      ctypes.POINTER(_I64)]),
    ("pbsa_plan_kernel", ctypes.c_int, [_P, ctypes.POINTER(ctypes.c_int), ctypes.POINTER(ctypes.c_int)]),
    ("pbsa_plan_layout", ctypes.c_int, [_P, ctypes.POINTER(_I64), ctypes.POINTER(ctypes.c_int),
                                        ctypes.POINTER(ctypes.c_int), ctypes.POINTER(ctypes.c_int)]),
    ("pbsa_plan_bytes", ctypes.c_int, [_P, ctypes.POINTER(_I64), ctypes.POINTER(_I64)]),
    ("pbsa_plan_destroy", ctypes.c_int, [_P]),
    ("pbsa_anneal_loop_batch", ctypes.c_int,
     [ctypes.c_int, _I64, _P, _P, _P, _P, _I64, _P, _P, _P, _I64, _P, _P, _P, _P, _P, _P, _I64,
      _F64, _F64, _I64, _I64, ctypes.c_int, _I64, _F64, _I64, _P] + [_P] * 8
     + [ctypes.POINTER(ctypes.c_float)]),
    ("pbsa_anneal_loop_batch_ex", ctypes.c_int,
     [ctypes.c_int, _I64, _P, _P, _P, _P, _I64, _P, _P, _P, _I64, _P, _P, _P, _P, _P, _P, _I64,
      _F64, _F64, _I64, _I64, ctypes.c_int, _I64, _F64, _I64, _P, ctypes.c_int, ctypes.c_uint64,
      _I64] + [_P] * 8 + [ctypes.POINTER(ctypes.c_float)]),
    ("pbsa_plan_cache_clear", ctypes.c_int, []),
    ("pbsa_plan_create_np", ctypes.c_int,
     [ctypes.c_int, _I64, _P, _P, _P, _P, _I64, _P, _P, _P, _I64, _P, _P, _P, _P,
      _F64, _F64, _I64, _I64, ctypes.c_int, _I64, _F64, _I64, _P, ctypes.c_uint64, _I64,
      ctypes.POINTER(_P)]),
    ("pbsa_anneal_loop_batch_np", ctypes.c_int,
     [ctypes.c_int, _I64, _P, _P, _P, _P, _I64, _P, _P, _P, _I64, _P, _P, _P, _P,
      _F64, _F64, _I64, _I64, ctypes.c_int, _I64, _F64, _I64, _P, ctypes.c_uint64, _I64]
     + [_P] * 8 + [ctypes.POINTER(ctypes.c_float)]),
    ("pbsa_native_profiles", ctypes.c_int,
     [ctypes.c_int, ctypes.c_uint64, _I64, _I64, _I64, _I64, _I64, _P, _P, _P, _P]),
    ("pbsa_last_call_bytes", ctypes.c_int, [ctypes.POINTER(_I64), ctypes.POINTER(_I64)]),
    ("pbsa_anneal_loop_batch_devices", ctypes.c_int,
     [_P, ctypes.c_int, _I64, _P, _P, _P, _P, _I64, _P, _P, _P, _I64, _P, _P, _P, _P, _P, _P, _I64,
      _F64, _F64, _I64, _I64, ctypes.c_int, _I64, _F64, _I64, _P, ctypes.c_int, ctypes.c_uint64,
      _I64] + [_P] * 8 + [ctypes.POINTER(ctypes.c_float)]),
    ("pbsa_debug_stream_u64", ctypes.c_int, [ctypes.c_int, _I64, _P, _P, _P, _P, _P]),
    ("pbsa_debug_tanh", ctypes.c_int, [ctypes.c_int, _I64, _P, _P]),
    ("pbsa_debug_philox", ctypes.c_int, [ctypes.c_int, _I64, _P, _P, _P]),
    ("pbsa_debug_var_prefilter", ctypes.c_int, [ctypes.c_int, _I64, _P, _P, _P, _P, _P, _P]),
    ("pbsa_format_trace_csv", ctypes.c_int, [_I64, _I64, _P, _P, _P, _P, _P, _I64,
                                              ctypes.POINTER(_I64)]),
    ("pbsa_libm_tanh_host", _F64, [_F64]),
    ("pbsa_threshold_host", ctypes.c_uint64, [_F64]),
    ("pbsa_threshold_native_host", ctypes.c_uint64, [_F64]),
    ("pbsa_philox_host", None, [_P, _P, _P]),
    ("pbsa_choose_phases_host", _I64, [_I64, _I64, _I64, _I64, ctypes.POINTER(ctypes.c_int)]),
]

EXPORTED = [name for name, _, _ in _SIGNATURES]

# pbsa_plan_kernel codes (include/pbsa.h PBSA_KERNEL_*)
KERNELS = {1: "packed", 2: "packed_timing", 3: "resident", 4: "resident_timing", 5: "active_fast",
           6: "active", 7: "full", 8: "packed_bucket"}


def load() -> ctypes.CDLL:
    """Load libpbsa.so; raises RuntimeError (never falls back) if it is absent."""
    global _lib
    if _lib is None:
        # PBSA_LIB: an alternative in-tree build of the same library (A/B
        # experiments of compile-time variants, tools/); default the product build
        path = Path(os.environ.get("PBSA_LIB") or LIB_PATH)
        if not path.exists():
            raise RuntimeError(
                f"CUDA library {path} is not built; run __graft_entry__.build() "
                "(there is no CPU fallback for the annealing sweep)")
        lib = ctypes.CDLL(str(path))
        for name, res, args in _SIGNATURES:
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        _lib = lib
    return _lib


def _check(rc: int) -> None:
    if rc != PBSA_OK:
        msg = load().pbsa_last_error().decode(errors="replace")
        if rc == -1:
            raise ValueError(msg)
        raise RuntimeError(f"pbsa error {rc}: {msg}")


def device_count() -> int:
    c = ctypes.c_int(0)
    rc = load().pbsa_device_count(ctypes.byref(c))
    return c.value if rc == PBSA_OK else 0


def require_device(device: int) -> None:
    n = device_count()
    if n < 1:
        raise RuntimeError("no CUDA device visible: the p-bit sweep runs only on the GPU "
                           "(libpbsa.so, sm_100a); there is no CPU fallback")
    if not 0 <= device < n:
        raise RuntimeError(f"device {device} out of range (have {n})")


def _ptr(a) -> int:
    return 0 if a is None or a.size == 0 else a.ctypes.data


def _c(a, dtype):
    return np.ascontiguousarray(a, dtype=dtype)


class Batch:
    """Host-side arguments of one batched anneal_loop call (_kernels.py:69-91)."""

    def __init__(self, model, schedule, keys, profile_rows=None, graph=None, algo_code=0,
                 alpha=1, p_stall=0.5, rng="replay", rng_seed=0, first_trial=0, native_sigmas=None):
        if rng not in RNG_MODES:
            raise ValueError(f"rng must be one of {sorted(RNG_MODES)}, got {rng!r}")
        # native_sigmas: (sigma_lambda, sigma_delta, sigma_nu) -- the profiles
        # are drawn on the device (pbsa_plan_create_np; Philox stream only)
        self.native_sigmas = None
        if native_sigmas is not None:
            if profile_rows is not None:
                raise ValueError("native_sigmas replace profile_rows; give one")
            if rng != "philox":
                raise ValueError("native profiles need rng='philox'")
            self.native_sigmas = np.ascontiguousarray([float(x) for x in native_sigmas], dtype=np.float64)
            if self.native_sigmas.size != 3:
                raise ValueError("native_sigmas holds (sigma_lambda, sigma_delta, sigma_nu)")
        self.rng, self.rng_seed, self.first_trial = rng, int(rng_seed), int(first_trial)
        self.n = int(model.n)
        self.indptr = _c(model.indptr, np.int64)
        self.indices = _c(model.indices, np.int64)
        self.values = _c(model.values, np.float64)
        self.h = _c(model.h, np.float64)
        self.me_i = _c(model.edge_i, np.int64)
        self.me_j = _c(model.edge_j, np.int64)
        self.me_w = _c(model.edge_w, np.float64)
        if graph is not None:
            self.ge_i = _c(graph.edge_i, np.int64)
            self.ge_j = _c(graph.edge_j, np.int64)
            self.ge_w = _c(graph.edge_w, np.int64)
        else:
            self.ge_i = self.ge_j = self.ge_w = np.empty(0, np.int64)
        self.keys = np.asarray(keys, dtype=np.uint64)
        self.T = int(self.keys.size)
        # profile_rows: None (ideal), or (lam, delta, period, stride)
        if profile_rows is None:
            self.lam = self.delta = self.period = None
            self.stride = 0
        else:
            lam, delta, period, stride = profile_rows
            self.lam, self.delta = _c(lam, np.float64), _c(delta, np.float64)
            self.period, self.stride = _c(period, np.int64), int(stride)
        self.i0_min, self.beta = float(schedule.i0_min), float(schedule.beta)
        self.cycles, self.t_res = int(schedule.cycles), int(schedule.t_res)
        self.algo, self.alpha, self.p_stall = int(algo_code), int(alpha), float(p_stall)

    def _args(self):
        return (self.n, _ptr(self.indptr), _ptr(self.indices), _ptr(self.values), _ptr(self.h),
                int(self.me_i.size), _ptr(self.me_i), _ptr(self.me_j), _ptr(self.me_w),
                int(self.ge_i.size), _ptr(self.ge_i), _ptr(self.ge_j), _ptr(self.ge_w),
                _ptr(self.lam), _ptr(self.delta), _ptr(self.period), self.stride,
                self.i0_min, self.beta, self.cycles, self.t_res, self.algo, self.alpha,
                self.p_stall, self.T, _ptr(self.keys), RNG_MODES[self.rng],
                self.rng_seed & 0xFFFFFFFFFFFFFFFF, self.first_trial)

    def _args_np(self):
        """pbsa_*_np arguments: the model, the sigmas in place of the profile
        arrays, the schedule and rule, keys, seed and first trial."""
        return (self.n, _ptr(self.indptr), _ptr(self.indices), _ptr(self.values), _ptr(self.h),
                int(self.me_i.size), _ptr(self.me_i), _ptr(self.me_j), _ptr(self.me_w),
                int(self.ge_i.size), _ptr(self.ge_i), _ptr(self.ge_j), _ptr(self.ge_w),
                self.native_sigmas.ctypes.data, self.i0_min, self.beta, self.cycles, self.t_res,
                self.algo, self.alpha, self.p_stall, self.T, _ptr(self.keys),
                self.rng_seed & 0xFFFFFFFFFFFFFFFF, self.first_trial)

    def alloc_outputs(self) -> dict:
        T, n, C = self.T, self.n, self.cycles
        return dict(spins=np.empty((T, n), np.int8), inputs=np.empty((T, n)),
                    hist=np.empty((T, n, self.alpha)), counts=np.empty((T, n), np.int64),
                    i0_trace=np.empty((T, C)), energy_trace=np.empty((T, C)),
                    cut_trace=np.empty((T, C), np.int64), best_cut=np.empty(T, np.int64))


OUT_ORDER = ("spins", "inputs", "hist", "counts", "i0_trace", "energy_trace", "cut_trace",
             "best_cut")


def anneal_batch(batch: Batch, device: int = 0, out: dict | None = None) -> tuple[dict, float]:
    """One-shot pbsa_anneal_loop_batch; returns (outputs, device milliseconds).
    ``out`` may supply preallocated (e.g. page-locked) output arrays shaped
    like ``batch.alloc_outputs()``."""
    lib = load()
    require_device(device)
    if out is None:
        out = batch.alloc_outputs()
    ms = ctypes.c_float(0.0)
    if batch.native_sigmas is not None:
        _check(lib.pbsa_anneal_loop_batch_np(device, *batch._args_np(),
                                             *(_ptr(out[k]) for k in OUT_ORDER), ctypes.byref(ms)))
    else:
        _check(lib.pbsa_anneal_loop_batch_ex(device, *batch._args(),
                                             *(_ptr(out[k]) for k in OUT_ORDER), ctypes.byref(ms)))
    return out, float(ms.value)


def anneal_batch_devices(batch: Batch, devices, out: dict | None = None) -> tuple[dict, float]:
    """pbsa_anneal_loop_batch_devices: the batch's trials sharded over a
    device-ordinal list inside the library (one host thread, plan and stream
    per shard); outputs identical to anneal_batch.  Returns (outputs, the
    largest shard's device milliseconds)."""
    lib = load()
    devs = np.ascontiguousarray([int(d) for d in devices], dtype=np.int32)
    if devs.size == 0:
        raise ValueError("need at least one device")
    for d in set(devs.tolist()):
        require_device(d)
    if out is None:
        out = batch.alloc_outputs()
    ms = ctypes.c_float(0.0)
    _check(lib.pbsa_anneal_loop_batch_devices(devs.ctypes.data, int(devs.size), *batch._args(),
                                              *(_ptr(out[k]) for k in OUT_ORDER), ctypes.byref(ms)))
    return out, float(ms.value)


def native_profiles(rng_seed: int, first_trial: int, trials: int, n: int, t_res: int, cycles: int,
                    sigmas, device: int = 0):
    """The (lam, delta, period) [trials][n] arrays a native-profile plan with
    this seed and first trial draws on the device (pbsa_native_profiles;
    periods clamped to cycles * t_res, which fires identically)."""
    lib = load()
    require_device(device)
    sig = np.ascontiguousarray([float(x) for x in sigmas], dtype=np.float64)
    lam, delta = np.empty((trials, n)), np.empty((trials, n))
    period = np.empty((trials, n), np.int64)
    _check(lib.pbsa_native_profiles(device, int(rng_seed) & 0xFFFFFFFFFFFFFFFF, int(first_trial), int(trials),
                                    int(n), int(t_res), int(cycles), sig.ctypes.data, _ptr(lam), _ptr(delta),
                                    _ptr(period)))
    return lam, delta, period


def plan_cache_clear() -> None:
    """Free the one-shot plans the library keeps for repeated calls
    (pbsa_plan_cache_clear)."""
    _check(load().pbsa_plan_cache_clear())


def last_call_bytes() -> tuple[int, int]:
    """(host->device, device->host) bytes of this thread's last one-shot call."""
    a, b = _I64(), _I64()
    _check(load().pbsa_last_call_bytes(ctypes.byref(a), ctypes.byref(b)))
    return a.value, b.value


def device_list() -> list[int] | None:
    """PBSA_DEVICES=0,1,... (comma-separated ordinals): the device list
    engine.run_trials shards over when the spec names none; None if unset."""
    v = os.environ.get("PBSA_DEVICES", "").strip()
    if not v:
        return None
    return [int(x) for x in v.split(",") if x.strip()]


class Plan:
    """Device-resident batch: create once, run many times (bench `value` path)."""

    def __init__(self, batch: Batch, device: int = 0):
        lib = load()
        require_device(device)
        self.batch, self.device = batch, device
        h = _P()
        if batch.native_sigmas is not None:
            _check(lib.pbsa_plan_create_np(device, *batch._args_np(), ctypes.byref(h)))
        else:
            _check(lib.pbsa_plan_create_ex(device, *batch._args(), ctypes.byref(h)))
        self._h = h

    def run(self) -> float:
        ms = ctypes.c_float(0.0)
        _check(load().pbsa_plan_run(self._h, ctypes.byref(ms)))
        return float(ms.value)

    def download(self) -> dict:
        out = self.batch.alloc_outputs()
        _check(load().pbsa_plan_download(self._h, *(_ptr(out[k]) for k in OUT_ORDER)))
        return out

    def summary(self) -> tuple[int, int, int]:
        a, b, c = _I64(), _I64(), _I64()
        _check(load().pbsa_plan_summary(self._h, ctypes.byref(a), ctypes.byref(b), ctypes.byref(c)))
        return a.value, b.value, c.value

    def info(self) -> dict:
        path, launches, sweeps, words = ctypes.c_int(), _I64(), _I64(), _I64()
        ms = _F64()
        _check(load().pbsa_plan_info(self._h, ctypes.byref(path), ctypes.byref(launches),
                                     ctypes.byref(ms), ctypes.byref(sweeps), ctypes.byref(words)))
        kern, cs = ctypes.c_int(), ctypes.c_int()
        _check(load().pbsa_plan_kernel(self._h, ctypes.byref(kern), ctypes.byref(cs)))
        return dict(path={1: "packed", 2: "general"}.get(path.value, "?"),
                    kernel=KERNELS.get(kern.value, "?"), cluster_size=cs.value,
                    launches=launches.value, sweep_ms_mean=ms.value,
                    sweep_launches=sweeps.value, words=words.value)

    def layout(self) -> dict:
        """Launch shape of a launched packed plan (pbsa_plan_layout)."""
        pw, ch, wpw, cache = _I64(), ctypes.c_int(), ctypes.c_int(), ctypes.c_int()
        _check(load().pbsa_plan_layout(self._h, ctypes.byref(pw), ctypes.byref(ch), ctypes.byref(wpw),
                                       ctypes.byref(cache)))
        return dict(phase_words=pw.value, chains=ch.value, warps_per_word=wpw.value,
                    hash_cache=bool(cache.value))

    def transfer_bytes(self) -> tuple[int, int]:
        """(host->device bytes at creation, device->host bytes of a full download)."""
        a, b = _I64(), _I64()
        _check(load().pbsa_plan_bytes(self._h, ctypes.byref(a), ctypes.byref(b)))
        return a.value, b.value

    def close(self) -> None:
        if getattr(self, "_h", None):
            load().pbsa_plan_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def debug_stream_u64(keys, tags, a, b, device: int = 0) -> np.ndarray:
    lib = load()
    require_device(device)
    arrs = [np.ascontiguousarray(x, dtype=np.uint64) for x in (keys, tags, a, b)]
    out = np.empty(arrs[0].size, np.uint64)
    _check(lib.pbsa_debug_stream_u64(device, out.size, *(x.ctypes.data for x in arrs),
                                     out.ctypes.data))
    return out


def debug_philox(ctr, key, device: int = 0) -> np.ndarray:
    """Device Philox4x32-10: ctr [m, 4], key [m, 2] (uint32) -> [m, 4]."""
    lib = load()
    require_device(device)
    c = np.ascontiguousarray(ctr, dtype=np.uint32).reshape(-1, 4)
    k = np.ascontiguousarray(key, dtype=np.uint32).reshape(-1, 2)
    out = np.empty_like(c)
    _check(lib.pbsa_debug_philox(device, c.shape[0], c.ctypes.data, k.ctypes.data,
                                 out.ctypes.data))
    return out


def debug_var_prefilter(lam, delta, i0, raw, zh, device: int = 0) -> np.ndarray:
    """Device variability prefilter codes (bit 1 undecided, bit 0 decision)."""
    lib = load()
    require_device(device)
    a = [np.ascontiguousarray(x, dtype=np.float64) for x in (lam, delta, i0)]
    r = np.ascontiguousarray(raw, dtype=np.int32)
    z = np.ascontiguousarray(zh, dtype=np.uint32)
    out = np.empty(z.size, np.uint32)
    _check(lib.pbsa_debug_var_prefilter(device, z.size, *(x.ctypes.data for x in a), r.ctypes.data,
                                        z.ctypes.data, out.ctypes.data))
    return out


def philox_host(ctr, key) -> list[int]:
    """Host build of the device Philox4x32-10 (same source, philox.cuh)."""
    c = (ctypes.c_uint32 * 4)(*[int(x) & 0xFFFFFFFF for x in ctr])
    k = (ctypes.c_uint32 * 2)(*[int(x) & 0xFFFFFFFF for x in key])
    o = (ctypes.c_uint32 * 4)()
    load().pbsa_philox_host(ctypes.addressof(c), ctypes.addressof(k), ctypes.addressof(o))
    return list(o)


def debug_tanh(x, device: int = 0) -> np.ndarray:
    lib = load()
    require_device(device)
    x = np.ascontiguousarray(x, dtype=np.float64)
    out = np.empty_like(x)
    _check(lib.pbsa_debug_tanh(device, x.size, x.ctypes.data, out.ctypes.data))
    return out


def default_device() -> int:
    """Device ordinal from PBSA_DEVICE or LOCAL_RANK (one process per GPU), else 0."""
    for var in ("PBSA_DEVICE", "LOCAL_RANK"):
        v = os.environ.get(var)
        if v is not None and v.strip():
            return int(v)
    return 0


def format_trace_rows(i0_strs: list[bytes], energy_int: np.ndarray, cut: np.ndarray | None) -> bytes:
    """Trace CSV rows (no header) by the library's host formatter
    (pbsa_format_trace_csv): energy_int [T][C] integral energies, cut [T][C]
    or None, i0_strs the repr() bytes of the shared i0 trace."""
    lib = load()
    T, C = energy_int.shape
    text = b"".join(i0_strs)
    off = np.zeros(C + 1, np.int64)
    np.cumsum([len(x) for x in i0_strs], out=off[1:])
    e = np.ascontiguousarray(energy_int, dtype=np.int64)
    c = None if cut is None else np.ascontiguousarray(cut, dtype=np.int64)
    cap = T * (C * 96 + int(off[-1])) + 64  # 4 integers <= 21 chars, ".0", 4 separators
    out = np.empty(cap, np.uint8)
    n = _I64(0)
    tb = ctypes.create_string_buffer(text, len(text) + 1)
    _check(lib.pbsa_format_trace_csv(T, C, ctypes.addressof(tb), off.ctypes.data, e.ctypes.data,
                                     0 if c is None else c.ctypes.data, out.ctypes.data, cap,
                                     ctypes.byref(n)))
    return out[:n.value].tobytes()
