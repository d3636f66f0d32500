"""Batched experiment runner: ``run_trials``, ``sweep``, ``summarize``.

API mirror of /root/reference/pkg/src/pbitsa/engine.py:1-149.  The reference
fans trials out one ``run_anneal`` per ThreadPoolExecutor task
(engine.py:118-123); here all trials of a spec go to the GPU in ONE batched
``pbsa_anneal_loop_batch`` call (trial-sliced spin words, one CUDA graph per
batch), so ``threads`` no longer matters -- results are identical for any
value, as the reference guarantees for its thread budget.  Trial k's seed is
still ``trial_seed(base_seed, k)`` and its profile is still drawn from
``default_rng(profile_seed(seed_k))`` on the host, so every per-trial result
equals the reference's bit-for-bit.
"""

from __future__ import annotations

import time
from dataclasses import dataclass, replace
from typing import Mapping, Sequence

import numpy as np

from . import _native, streams
from .annealer import (AlgorithmConfig, TrialResult, derive_schedule, profile_rows,
                       results_from_batch)
from .model import MaxCutGraph, maxcut_to_ising
from .pbit import VariabilityConfig, sample_variability
from .profiles import sample_profiles

SWEEP_AXES = ("sigma_lambda", "sigma_delta", "sigma_nu")


@dataclass(frozen=True)
class ExperimentSpec:
    graph: str
    algo: AlgorithmConfig
    variability: VariabilityConfig = VariabilityConfig()
    cycles: int = 1000
    trials: int = 100
    base_seed: int = 0
    threads: int = 1
    resample_variability: bool = True
    # not in the reference: "replay" (default) draws from the reference's
    # counter hash, bit-exact; "philox" from the native Philox4x32-10 stream
    # (include/pbsa.h PBSA_RNG_PHILOX; plain rule, ideal profile)
    rng: str = "replay"
    # not in the reference: device ordinals to shard the trials over (one
    # library-owned host thread and plan per device; results identical to one
    # device); None reads PBSA_DEVICES, else one device (PBSA_DEVICE / LOCAL_RANK)
    devices: tuple | None = None
    # not in the reference: with rng="philox", draw every trial's variability
    # profile on the device from the native stream (pbsa_plan_create_np) instead
    # of numpy's generator -- statistically, not bitwise, the reference's
    native_profiles: bool = False

    def __post_init__(self) -> None:
        if self.rng not in ("replay", "philox"):
            raise ValueError(f"rng must be 'replay' or 'philox', got {self.rng!r}")
        if self.native_profiles and self.rng != "philox":
            raise ValueError("native_profiles needs rng='philox'")
        if self.cycles < 2:
            raise ValueError("cycles must be >= 2")
        if self.trials < 1:
            raise ValueError("trials must be >= 1")
        if self.threads < 1:
            raise ValueError("threads must be >= 1")


@dataclass
class ExperimentSummary:
    mean_cut: float
    std_cut: float
    normalized_mean_cut: float | None
    mean_final_energy: float
    anneal_seconds: float
    results: list[TrialResult]


def summarize(results: Sequence[TrialResult], best_known: int | None = None,
              anneal_seconds: float = 0.0) -> ExperimentSummary:
    cuts = np.array([r.final_cut for r in results], dtype=np.float64)
    mean_cut = float(cuts.mean())
    std_cut = float(cuts.std(ddof=1)) if cuts.size > 1 else 0.0
    normalized = None
    if best_known is not None:
        if not (np.isfinite(best_known) and best_known > 0):
            raise ValueError(f"best-known cut {best_known} is not finite and positive")
        normalized = mean_cut / best_known
    return ExperimentSummary(
        mean_cut=mean_cut, std_cut=std_cut, normalized_mean_cut=normalized,
        mean_final_energy=float(np.mean([r.final_energy for r in results])),
        anneal_seconds=anneal_seconds, results=list(results))


def trial_profiles(spec: ExperimentSpec, n: int, seeds: Sequence[int]):
    """Per-trial profiles exactly as engine.py:102-112 draws them; None when
    the variability config is all-zero (every draw is then the ideal profile)."""
    cfg = spec.variability
    if cfg.sigma_lambda == 0.0 and cfg.sigma_delta == 0.0 and cfg.sigma_nu == 0.0:
        return None
    if not spec.resample_variability:
        fixed = sample_variability(cfg, n, np.random.default_rng(streams.profile_seed(seeds[0])))
        return fixed
    # stacked [trials][n] rows, sampled by parallel worker processes (profiles.py)
    lam, delta, period = sample_profiles(cfg, n, seeds)
    return (lam, delta, period, n)


def run_trial_range(spec: ExperimentSpec, graph: MaxCutGraph, start: int, stop: int,
                    device: int | None = None) -> tuple[list[TrialResult], float]:
    """Trials [start, stop) of ``spec`` on one device (seeds keep their global
    index, so any sharding of the range gives identical per-trial results).
    Returns (results, seconds); seconds covers profile sampling + the
    device anneal + transfers, like the reference's anneal_seconds."""
    model = maxcut_to_ising(graph)
    schedule = derive_schedule(model, spec.cycles, spec.variability.t_res)
    all_seeds = streams.trial_seeds(spec.base_seed, stop, 0)
    seeds = all_seeds[start:stop]
    t0 = time.perf_counter()
    cfg = spec.variability
    native = spec.native_profiles and not (cfg.sigma_lambda == 0.0 and cfg.sigma_delta == 0.0 and
                                           cfg.sigma_nu == 0.0)
    if native:  # drawn on the device from the native stream
        profs = None
    elif spec.resample_variability:
        profs = trial_profiles(spec, model.n, seeds)
    else:
        profs = trial_profiles(spec, model.n, all_seeds[:1])
    batch = _native.Batch(model, schedule, streams.run_keys(seeds),
                          profile_rows=profile_rows(profs, model.n), graph=graph,
                          algo_code=spec.algo.kind.code, alpha=spec.algo.kernel_alpha,
                          p_stall=spec.algo.p_stall, rng=spec.rng,
                          rng_seed=streams.native_seed(spec.base_seed), first_trial=start,
                          native_sigmas=(cfg.sigma_lambda, cfg.sigma_delta, cfg.sigma_nu) if native else None)
    devs = None
    if device is None:
        devs = list(spec.devices) if spec.devices is not None else _native.device_list()
    try:
        if devs is not None and len(devs) > 1 and native:
            # (the library's device fan-out takes profile arrays: shard here)
            return _native_shards(spec, graph, start, stop, devs), time.perf_counter() - t0
        if devs is not None and len(devs) > 1:
            out, _ = _native.anneal_batch_devices(batch, devs)
        else:
            dev = device if device is not None else (devs[0] if devs else _native.default_device())
            out, _ = _native.anneal_batch(batch, device=dev)
    except ValueError as exc:
        raise RuntimeError(f"trials {start}..{stop - 1} of {spec.graph!r} failed: {exc}") from exc
    elapsed = time.perf_counter() - t0
    return results_from_batch(out, seeds, schedule, True), elapsed


def _native_shards(spec: ExperimentSpec, graph: MaxCutGraph, start: int, stop: int, devs):
    """Native-profile trials [start, stop) over several devices: 4-aligned
    shards (the Philox groups), one host thread per device, trial order kept."""
    from concurrent.futures import ThreadPoolExecutor

    from .distributed import shard_range
    spans = [shard_range(stop - start, r, len(devs)) for r in range(len(devs))]
    with ThreadPoolExecutor(len(devs)) as ex:
        parts = list(ex.map(lambda a: run_trial_range(spec, graph, start + a[0][0], start + a[0][1],
                                                      device=a[1])[0] if a[0][1] > a[0][0] else [],
                            zip(spans, devs)))
    return [r for part in parts for r in part]


def run_trials(spec: ExperimentSpec, graphs: Mapping[str, MaxCutGraph],
               registry: Mapping[str, int] | None = None) -> ExperimentSummary:
    try:
        graph = graphs[spec.graph]
    except KeyError:
        raise KeyError(f"unknown graph {spec.graph!r}; have {sorted(graphs)}") from None
    results, elapsed = run_trial_range(spec, graph, 0, spec.trials)
    best_known = registry.get(spec.graph) if registry is not None else None
    return summarize(results, best_known, elapsed)


def sweep(spec: ExperimentSpec, axis: str, values: Sequence[float],
          graphs: Mapping[str, MaxCutGraph],
          registry: Mapping[str, int] | None = None) -> list[ExperimentSummary]:
    if axis not in SWEEP_AXES:
        raise ValueError(f"sweep axis must be one of {SWEEP_AXES}, got {axis!r}")
    if len(values) == 0:
        raise ValueError("sweep needs at least one value")
    for v in values:
        if v < 0:
            raise ValueError(f"sweep value must be >= 0, got {v}")
    try:
        graph = graphs[spec.graph]
    except KeyError:
        raise KeyError(f"unknown graph {spec.graph!r}; have {sorted(graphs)}") from None
    specs = [replace(spec, variability=replace(spec.variability, **{axis: float(v)}))
             for v in values]
    best_known = registry.get(spec.graph) if registry is not None else None
    out: list[ExperimentSummary | None] = [None] * len(specs)
    # Points with variability share the device path, so they run as ONE batch
    # of len(points) * trials trials (same seeds per point, so the sweep stays
    # paired exactly as in the reference).  The ideal point, if any, runs alone
    # on the packed path.
    # (replay stream only: the native Philox stream is indexed by global trial,
    # so batching would give point j the counters of trials j*T.., breaking the
    # pairing; Philox points run one by one)
    grouped = [k for k, s in enumerate(specs)
               if not s.variability.is_ideal and s.resample_variability and s.rng == "replay"]
    for k, s in enumerate(specs):
        if k not in grouped:
            out[k] = run_trials(s, graphs, registry)
    if len(grouped) == 1:
        out[grouped[0]] = run_trials(specs[grouped[0]], graphs, registry)
    elif grouped:
        model = maxcut_to_ising(graph)
        schedule = derive_schedule(model, spec.cycles, spec.variability.t_res)
        seeds = streams.trial_seeds(spec.base_seed, spec.trials, 0)
        t0 = time.perf_counter()
        rows = [trial_profiles(specs[k], model.n, seeds) for k in grouped]
        lam = np.concatenate([r[0] for r in rows])
        delta = np.concatenate([r[1] for r in rows])
        period = np.concatenate([r[2] for r in rows])
        keys = np.tile(streams.run_keys(seeds), len(grouped))
        batch = _native.Batch(model, schedule, keys, profile_rows=(lam, delta, period, model.n),
                              graph=graph, algo_code=spec.algo.kind.code,
                              alpha=spec.algo.kernel_alpha, p_stall=spec.algo.p_stall,
                              rng=spec.rng, rng_seed=streams.native_seed(spec.base_seed))
        res, _ = _native.anneal_batch(batch, device=_native.default_device())
        elapsed = (time.perf_counter() - t0) / len(grouped)
        T = spec.trials
        for j, k in enumerate(grouped):
            part = {name: arr[j * T:(j + 1) * T] for name, arr in res.items()}
            out[k] = summarize(results_from_batch(part, seeds, schedule, True), best_known, elapsed)
    return out
