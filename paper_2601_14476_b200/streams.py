"""Counter-hash random streams (host side).

Mirrors the reference stream contract (/root/reference/pkg/src/pbitsa/streams.py:1-73):
every draw is ``absorb(absorb(absorb(key, tag), a), b)`` with ``absorb(h, w) =
mix64((h + 0x9E37...) ^ w)`` and ``mix64`` the splitmix64 finaliser.  The host
uses these only to derive per-trial keys (``trial_seed``, ``run_key``,
``profile_seed``) and the per-trial key prefixes the CUDA kernels start from;
the per-update draws themselves are regenerated on the device by the same
hash (``csrc/pbsa_device.cuh``), so nothing is ever dumped or uploaded.
"""

from __future__ import annotations

import numpy as np

MASK64 = (1 << 64) - 1
GOLDEN_GAMMA = 0x9E3779B97F4A7C15
MIX_M1 = 0xBF58476D1CE4E5B9
MIX_M2 = 0x94D4A04C32684F87
_TWO_M53 = 2.0 ** -53

# Stream tags (streams.py:19-26); they fix every result downstream of a seed.
TAG_RUN, TAG_SPIN, TAG_R, TAG_STALL, TAG_TRIAL, TAG_PROFILE = 1, 2, 3, 4, 5, 6


def mix64(z: int) -> int:
    z &= MASK64
    z = ((z ^ (z >> 30)) * MIX_M1) & MASK64
    z = ((z ^ (z >> 27)) * MIX_M2) & MASK64
    return z ^ (z >> 31)


def absorb(h: int, w: int) -> int:
    return mix64(((h + GOLDEN_GAMMA) & MASK64) ^ (w & MASK64))


def stream_u64(key: int, tag: int, a: int = 0, b: int = 0) -> int:
    return absorb(absorb(absorb(key & MASK64, tag), a), b)


def uniform01(key: int, tag: int, a: int = 0, b: int = 0) -> float:
    return (stream_u64(key, tag, a, b) >> 11) * _TWO_M53


def uniform_signed(key: int, tag: int, a: int = 0, b: int = 0) -> float:
    return 2.0 * uniform01(key, tag, a, b) - 1.0


def run_key(seed: int) -> int:
    return stream_u64(seed & MASK64, TAG_RUN)


def trial_seed(base_seed: int, index: int) -> int:
    if index < 0:
        raise ValueError("trial index must be >= 0")
    return stream_u64(base_seed & MASK64, TAG_TRIAL, index)


def profile_seed(seed: int) -> int:
    return stream_u64(seed & MASK64, TAG_PROFILE)


TAG_NATIVE = 7  # not in the reference: key of the native Philox stream (rng="philox")


def native_seed(base_seed: int) -> int:
    """64-bit Philox key of an experiment's native activation stream (one key
    per experiment; trials are told apart by their global index in the counter)."""
    return stream_u64(base_seed & MASK64, TAG_NATIVE)


# ------------------------------------------------------- vectorised helpers

def _mix64_vec(z: np.ndarray) -> np.ndarray:
    with np.errstate(over="ignore"):
        z = (z ^ (z >> np.uint64(30))) * np.uint64(MIX_M1)
        z = (z ^ (z >> np.uint64(27))) * np.uint64(MIX_M2)
        return z ^ (z >> np.uint64(31))


def absorb_vec(h: np.ndarray, w) -> np.ndarray:
    """Element-wise absorb on uint64 arrays (wrap-around arithmetic)."""
    with np.errstate(over="ignore"):
        return _mix64_vec((np.asarray(h, np.uint64) + np.uint64(GOLDEN_GAMMA))
                          ^ np.asarray(w, np.uint64))


def trial_seeds(base_seed: int, count: int, start: int = 0) -> list[int]:
    """trial_seed(base, k) for k in [start, start + count)."""
    base = absorb(base_seed & MASK64, TAG_TRIAL)
    ks = np.arange(start, start + count, dtype=np.uint64)
    out = absorb_vec(absorb_vec(np.full(count, base, np.uint64), ks), np.uint64(0))
    return [int(x) for x in out]


def run_keys(seeds) -> np.ndarray:
    """run_key(seed) for a sequence of seeds, as uint64."""
    s = np.asarray([int(x) & MASK64 for x in seeds], dtype=np.uint64)
    z = np.zeros_like(s)
    return absorb_vec(absorb_vec(absorb_vec(s, np.uint64(TAG_RUN)), z), z)
