"""Per-trial variability profiles, produced in parallel on the host.

The reference draws each trial's profile with numpy's PCG64 from
``default_rng(profile_seed(seed_k))`` (engine.py:107-112, pbit.py:57-75) one
trial at a time.  The draws must stay exactly those (they are the reference's
random stream), so this module keeps the same numpy calls but fans the trials
out over worker processes that write straight into one shared, stacked
``[trials][n]`` buffer (no pickling of arrays).  For G81 x 4096 trials that is
~5 s single-threaded; with W workers it scales ~W-fold.  Small jobs stay serial.

The pool forks (Python warns when the parent runs threads, e.g. CUDA's): the
children run only numpy's generators on their own row ranges and the shared
anonymous mappings -- no CUDA, no imports, no locks the parent's threads could
hold -- and exit.  Threads instead of processes measured 1.4x, not ~W-fold
(the per-trial numpy calls hold the GIL).
"""

from __future__ import annotations

import mmap
import multiprocessing as mp
import os

import numpy as np

from . import streams
from .pbit import VariabilityConfig, sample_variability

PARALLEL_MIN_ELEMENTS = 4_000_000  # trials * n below this: serial


def _fill(cfg, n, seeds, lam, delta, period, lo, hi):
    for k in range(lo, hi):
        p = sample_variability(cfg, n, np.random.default_rng(streams.profile_seed(seeds[k])))
        lam[k], delta[k], period[k] = p.lam, p.delta, p.period


_CHILD = {}  # set in each forked worker by _init; the parent never touches it


def _init(state):
    _CHILD.clear()
    _CHILD.update(state)


def _worker(args):
    lo, hi = args
    s = _CHILD
    _fill(s["cfg"], s["n"], s["seeds"], s["lam"], s["delta"], s["period"], lo, hi)
    return hi - lo


def sample_profiles(cfg: VariabilityConfig, n: int, seeds, workers: int | None = None):
    """Stacked (lam, delta, period) arrays, row k = the profile of seeds[k]."""
    T = len(seeds)
    if workers is None:
        workers = min(len(os.sched_getaffinity(0)) if hasattr(os, "sched_getaffinity")
                      else (os.cpu_count() or 1), 32)
    if T * n < PARALLEL_MIN_ELEMENTS or workers <= 1 or T < 2 or "fork" not in mp.get_all_start_methods():
        lam, delta = np.empty((T, n)), np.empty((T, n))
        period = np.empty((T, n), np.int64)
        _fill(cfg, n, list(seeds), lam, delta, period, 0, T)
        return lam, delta, period
    # anonymous shared mappings survive fork; workers write their row ranges
    bufs = [mmap.mmap(-1, T * n * 8) for _ in range(3)]
    lam = np.frombuffer(bufs[0], dtype=np.float64).reshape(T, n)
    delta = np.frombuffer(bufs[1], dtype=np.float64).reshape(T, n)
    period = np.frombuffer(bufs[2], dtype=np.int64).reshape(T, n)
    # each call hands its own buffers to its own pool through the initializer
    # (forked children inherit the arguments; nothing module-global is shared
    # between concurrent calls, e.g. run_trials_devices' per-device threads)
    state = dict(cfg=cfg, n=n, seeds=list(seeds), lam=lam, delta=delta, period=period)
    step = (T + workers * 4 - 1) // (workers * 4)
    chunks = [(lo, min(T, lo + step)) for lo in range(0, T, step)]
    with mp.get_context("fork").Pool(workers, initializer=_init, initargs=(state,)) as pool:
        done = sum(pool.map(_worker, chunks))
    if done != T:
        raise RuntimeError("profile workers did not cover every trial")
    # the arrays keep their mappings alive (np.frombuffer holds a reference)
    return lam, delta, period
