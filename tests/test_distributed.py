"""Trial sharding over two processes (gloo on the CPU; NCCL on GPUs).

The per-rank compute is injected: here the CPU oracle stands in for the GPU
batch (test infrastructure), so what is exercised is the sharding rule, the
seed bookkeeping and the end-of-run reductions -- the whole multi-GPU path
except the device kernels, which test_gpu_parity.py covers (including shard
invariance at full size).
"""

from __future__ import annotations

import os
import socket
import sys
from pathlib import Path

import numpy as np
import pytest
import torch.multiprocessing as mp

ROOT = Path(__file__).resolve().parents[1]


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def oracle_runner(spec, graph, lo, hi):
    # an empty shard must not reach the runner (the C ABI rejects 0 trials);
    # with 7 trials over 2 ranks rank 0's 4-aligned shard is empty
    assert hi > lo, (lo, hi)
    from oracle import oracle as orc
    from paper_2601_14476_b200 import streams
    from paper_2601_14476_b200.annealer import derive_schedule
    from paper_2601_14476_b200.model import maxcut_to_ising
    from paper_2601_14476_b200.pbit import VariabilityProfile
    model = maxcut_to_ising(graph)
    sch = derive_schedule(model, spec.cycles, spec.variability.t_res)
    seeds = streams.trial_seeds(spec.base_seed, hi)[lo:hi]
    out = orc.anneal_batch(model, sch, spec.algo.kind.value, VariabilityProfile.ideal(model.n),
                           [streams.run_key(s) for s in seeds], graph=graph, threads=2)
    return out["cut_trace"][:, -1].copy(), out["best_cut"].copy(), out["energy_trace"][:, -1].copy(), 0.0


def _spec_and_graphs():
    from paper_2601_14476_b200 import benchmarks
    from paper_2601_14476_b200.annealer import Algorithm, AlgorithmConfig
    from paper_2601_14476_b200.engine import ExperimentSpec
    g, _ = benchmarks.load("G1")
    return ExperimentSpec(graph="G1", algo=AlgorithmConfig(Algorithm.TAPSA, alpha=1), cycles=60,
                          trials=7), {"G1": g}


def _worker(rank, world, port, q):
    sys.path.insert(0, str(ROOT))
    sys.path.insert(0, str(ROOT / "tests"))
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    import torch.distributed as dist
    from paper_2601_14476_b200.distributed import run_trials_sharded
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        spec, graphs = _spec_and_graphs()
        s = run_trials_sharded(spec, graphs, {"G1": 11605}, runner=oracle_runner)
        q.put((rank, s.trials, s.mean_cut, s.std_cut, s.best_cut, s.mean_final_energy,
               s.normalized_mean_cut, s.final_cuts.tolist()))
    finally:
        dist.destroy_process_group()


def test_shard_ranges_cover_trials_exactly():
    from paper_2601_14476_b200.distributed import shard_range
    for total in (1, 7, 100, 4096):
        for world in (1, 2, 3, 8):
            spans = [shard_range(total, r, world) for r in range(world)]
            assert spans[0][0] == 0 and spans[-1][1] == total
            assert all(a[1] == b[0] for a, b in zip(spans, spans[1:]))
    with pytest.raises(ValueError):
        shard_range(10, 2, 2)


def test_two_rank_gloo_sharding_matches_single_process(oracle):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    got = [q.get(timeout=300) for _ in procs]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    # the whole job on one process, through the same runner
    spec, graphs = _spec_and_graphs()
    cuts, bests, energies, _ = oracle_runner(spec, graphs["G1"], 0, spec.trials)
    from paper_2601_14476_b200.engine import summarize

    class R:
        def __init__(self, c, e):
            self.final_cut, self.final_energy = int(c), float(e)
    ref = summarize([R(c, e) for c, e in zip(cuts, energies)], 11605)
    for rank, n, mean, std, best, me, norm, all_cuts in got:
        assert n == spec.trials
        assert all_cuts == cuts.tolist()
        assert mean == ref.mean_cut and std == ref.std_cut
        assert me == ref.mean_final_energy and norm == ref.normalized_mean_cut
        assert best == int(bests.max())


def test_device_list_fan_out_is_trial_ordered_and_exact(oracle):
    """run_trials_devices: shards on several devices (here a CPU runner with
    the oracle) concatenate to the single-device trial order and summary."""
    from paper_2601_14476_b200.distributed import run_trials_devices
    from paper_2601_14476_b200.engine import summarize
    spec, graphs = _spec_and_graphs()
    seen = []

    def runner(s, g, lo, hi, device):
        seen.append((lo, hi, device))
        cuts, bests, energies, secs = oracle_runner(s, g, lo, hi)

        class R:
            def __init__(self, k, c, e):
                self.trial, self.final_cut, self.final_energy = k, int(c), float(e)
        return [R(lo + k, c, e) for k, (c, e) in enumerate(zip(cuts, energies))], secs

    out = run_trials_devices(spec, graphs, {"G1": 11605}, devices=[0, 1, 2], runner=runner)
    spans = sorted((lo, hi) for lo, hi, _ in seen)
    assert spans[0][0] == 0 and spans[-1][1] == spec.trials
    assert all(a[1] == b[0] for a, b in zip(spans, spans[1:]))
    assert len({d for _, _, d in seen}) == len(seen)  # one shard per device
    assert [r.trial for r in out.results] == list(range(spec.trials))
    cuts, _, energies, _ = oracle_runner(spec, graphs["G1"], 0, spec.trials)

    class R:
        def __init__(self, c, e):
            self.final_cut, self.final_energy = int(c), float(e)
    ref = summarize([R(c, e) for c, e in zip(cuts, energies)], 11605)
    assert out.mean_cut == ref.mean_cut and out.std_cut == ref.std_cut
    assert out.normalized_mean_cut == ref.normalized_mean_cut
