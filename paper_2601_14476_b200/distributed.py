"""Trial sharding across GPUs (one process per GPU, torch.distributed).

The reference fans trials out over a thread pool (engine.py:118-123) and its
results are independent of how trials are scheduled because trial k's seed is
``trial_seed(base_seed, k)`` (streams.py:63-68).  The multi-GPU form keeps that
contract: rank r of W anneals the contiguous trial range
``[r*T//W, (r+1)*T//W)`` on its own device with the global trial index kept
for seeding, so every per-trial result is identical for any W.  There is no
exchange during the anneal; the only collective is the end-of-run reduction
(NCCL on GPUs, gloo in the CPU tests):

  * all_reduce(SUM)  of [sum of final cuts, sum of final energies*2, trials]
  * all_reduce(MAX)  of the best cut
  * all_gather       of the per-trial final cuts (T int64) when the exact
                     sample std of ``summarize`` is wanted on every rank.
"""

from __future__ import annotations

import time
from dataclasses import dataclass
from typing import Callable, Mapping

import numpy as np

from .engine import ExperimentSpec, run_trial_range
from .model import MaxCutGraph


def shard_range(total: int, rank: int, world: int, align: int = 4) -> tuple[int, int]:
    """Contiguous trial range of ``rank``.  Interior boundaries are multiples of
    ``align`` (4: the native Philox stream draws four trials per call, so its
    results are shard-invariant only for 4-aligned shards; replay results are
    invariant to any split)."""
    if not 0 <= rank < world:
        raise ValueError(f"rank {rank} outside world of {world}")

    def edge(r: int) -> int:
        return total if r >= world else (total * r // world) // align * align

    return edge(rank), edge(rank + 1)


@dataclass
class ShardSummary:
    """Whole-job statistics, identical on every rank after the reduction."""
    trials: int
    mean_cut: float
    std_cut: float
    best_cut: int
    mean_final_energy: float
    normalized_mean_cut: float | None
    anneal_seconds: float          # max over ranks
    final_cuts: np.ndarray | None  # all trials, in trial order (when gathered)


def default_runner(spec: ExperimentSpec, graph: MaxCutGraph, lo: int, hi: int):
    """Per-rank compute: the GPU batch for trials [lo, hi) on this rank's device.
    Returns (final_cuts[int64], best_cuts[int64], final_energies[float64], seconds)."""
    results, secs = run_trial_range(spec, graph, lo, hi)
    return (np.array([r.final_cut for r in results], np.int64),
            np.array([r.best_cut for r in results], np.int64),
            np.array([r.final_energy for r in results], np.float64), secs)


def run_trials_sharded(spec: ExperimentSpec, graphs: Mapping[str, MaxCutGraph],
                       registry: Mapping[str, int] | None = None, *,
                       runner: Callable | None = None, gather: bool = True,
                       device: str | None = None) -> ShardSummary:
    """Trial-sharded ``run_trials`` over the initialised torch.distributed group."""
    import torch
    import torch.distributed as dist

    world = dist.get_world_size() if dist.is_initialized() else 1
    rank = dist.get_rank() if dist.is_initialized() else 0
    try:
        graph = graphs[spec.graph]
    except KeyError:
        raise KeyError(f"unknown graph {spec.graph!r}; have {sorted(graphs)}") from None
    lo, hi = shard_range(spec.trials, rank, world)
    run = runner or default_runner
    t0 = time.perf_counter()
    if hi > lo:
        cuts, bests, energies, _ = run(spec, graph, lo, hi)
    else:  # an empty shard (T < 4 W with 4-aligned edges) still joins the collectives
        cuts, bests, energies = np.empty(0, np.int64), np.empty(0, np.int64), np.empty(0)
    secs = time.perf_counter() - t0
    if device is None:
        # NCCL: this rank's own GPU (the library's device ordinal, LOCAL_RANK
        # under torchrun), not whatever torch's current device happens to be
        if dist.is_initialized() and dist.get_backend() == "nccl":
            from . import _native
            device = f"cuda:{_native.default_device()}"
            torch.cuda.set_device(device)
        else:
            device = "cpu"

    # integer sums are exact; energies are integers for MAX-CUT models, so the
    # doubled energy sum is exact in int64 as well
    sums = torch.tensor([int(cuts.sum()), int(np.rint(2 * energies.sum())), hi - lo],
                        dtype=torch.int64, device=device)
    best = torch.tensor([int(bests.max()) if bests.size else -(1 << 62)], dtype=torch.int64,
                        device=device)
    wall = torch.tensor([secs], dtype=torch.float64, device=device)
    if world > 1:
        dist.all_reduce(sums, op=dist.ReduceOp.SUM)
        dist.all_reduce(best, op=dist.ReduceOp.MAX)
        dist.all_reduce(wall, op=dist.ReduceOp.MAX)
    total, e2, n = (int(x) for x in sums.tolist())
    all_cuts = None
    std = float("nan")
    if gather:
        if world > 1:
            counts = [shard_range(spec.trials, r, world) for r in range(world)]
            width = max(b - a for a, b in counts)
            buf = torch.full((width,), 0, dtype=torch.int64, device=device)
            buf[: hi - lo] = torch.as_tensor(cuts, dtype=torch.int64, device=device)
            parts = [torch.empty_like(buf) for _ in range(world)]
            dist.all_gather(parts, buf)
            all_cuts = np.concatenate([p[: b - a].cpu().numpy() for p, (a, b) in zip(parts, counts)])
        else:
            all_cuts = cuts.copy()
        f = all_cuts.astype(np.float64)
        std = float(f.std(ddof=1)) if f.size > 1 else 0.0
    mean = total / n
    bk = registry.get(spec.graph) if registry is not None else None
    return ShardSummary(trials=n, mean_cut=mean, std_cut=std, best_cut=int(best.item()),
                        mean_final_energy=(e2 / 2) / n,
                        normalized_mean_cut=(mean / bk) if bk else None,
                        anneal_seconds=float(wall.item()), final_cuts=all_cuts)


def run_trials_devices(spec: ExperimentSpec, graphs: Mapping[str, MaxCutGraph],
                       registry: Mapping[str, int] | None = None, devices=None, *,
                       runner: Callable | None = None):
    """``run_trials`` over several GPUs from ONE process: the device-ordinal
    list of the batched entry.  Trial shards
    ``shard_range(T, r, len(devices))`` run concurrently, one host thread per
    device (the C-ABI call releases the GIL; each call owns its plan and
    stream), and the per-trial results are concatenated in trial order, so
    the summary is identical to the single-device ``run_trials``.  The
    anneal seconds are the wall time of the whole fan-out.

    ``runner(spec, graph, lo, hi, device) -> (results, seconds)`` defaults to
    ``engine.run_trial_range`` (tests inject a CPU runner)."""
    from concurrent.futures import ThreadPoolExecutor

    from . import _native
    from .engine import summarize

    try:
        graph = graphs[spec.graph]
    except KeyError:
        raise KeyError(f"unknown graph {spec.graph!r}; have {sorted(graphs)}") from None
    if devices is None:
        devices = list(range(max(1, _native.device_count())))
    devices = list(devices)
    if not devices:
        raise ValueError("need at least one device")
    run = runner or (lambda s, g, lo, hi, d: run_trial_range(s, g, lo, hi, device=d))
    spans = [shard_range(spec.trials, r, len(devices)) for r in range(len(devices))]
    t0 = time.perf_counter()
    with ThreadPoolExecutor(len(devices)) as ex:
        parts = list(ex.map(lambda a: run(spec, graph, a[0][0], a[0][1], a[1]) if a[0][1] > a[0][0]
                            else ([], 0.0), zip(spans, devices)))
    results = [r for part, _ in parts for r in part]
    best_known = registry.get(spec.graph) if registry is not None else None
    return summarize(results, best_known, time.perf_counter() - t0)
