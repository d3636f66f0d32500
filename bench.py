"""Benchmark of the B200 pSA sweep (BASELINE.json metric: p-bit updates/s).

Default workload = BASELINE config C4: G81 (20,000-node +-1 torus analog),
plain pSA, ideal devices (sigma = 0), 4096 trials x 1000 cycles x t_res 10,
trials sharded over the N ranks (one process per GPU).  One "step" is one
whole anneal of the batch (init + 1000 sweep launches + the final cut pass +
trace finalisation, replayed as one CUDA graph) followed by the end-of-run
NCCL reduce of the final-cut sum and best cut.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl reference]
    torchrun --nproc-per-node N bench.py --gpus N ...

Prints ONE JSON line on rank 0.  `value` is measured with inputs resident in
HBM (CUDA events around each step on the plan stream, L2 flushed between
steps, max over ranks); `e2e` times the public C-ABI call
pbsa_anneal_loop_batch with host buffers (uploads, run, full download of all
eight outputs).  `--impl reference` times the reference algorithm on the
host cores instead (the C restatement in oracle/, all threads).
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

from paper_2601_14476_b200 import _native, benchmarks, streams  # noqa: E402
from paper_2601_14476_b200.annealer import derive_schedule  # noqa: E402
from paper_2601_14476_b200.model import maxcut_to_ising  # noqa: E402

METRIC = "p-bit updates/s on G81 (20k nodes) x trials, 1/2/4/8 GPU; mean cut/best-known"
UNIT = "updates/s"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["b200", "reference"], default="b200")
    ap.add_argument("--graph", default="G81")
    ap.add_argument("--trials", type=int, default=4096)
    ap.add_argument("--cycles", type=int, default=1000)
    ap.add_argument("--e2e-steps", type=int, default=2)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--rng", choices=["replay", "philox"], default="replay",
                    help="activation stream of the headline run: the reference's counter hash "
                         "(bit-exact, default) or the native Philox4x32-10 stream")
    ap.add_argument("--no-philox-leg", action="store_true",
                    help="skip the extra native-Philox measurement reported under 'philox'")
    ap.add_argument("--cpu-sample-trials", type=int, default=0,
                    help="trials in the CPU baseline sample (default 8 per thread)")
    return ap.parse_args()


def dist_env():
    return (int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1)),
            int(os.environ.get("LOCAL_RANK", 0)))


def shard(total, rank, world):
    # contiguous, 4-aligned interior boundaries (the native Philox stream draws
    # four trials per call; distributed.shard_range)
    from paper_2601_14476_b200.distributed import shard_range
    return shard_range(total, rank, world)


def workload(name, cycles):
    graph, real = benchmarks.load(name)
    model = maxcut_to_ising(graph)
    return graph, real, model, derive_schedule(model, cycles, 10)


def best_known(name, real):
    if real:
        from paper_2601_14476_b200.gset import bundled_best_known
        return bundled_best_known().get(name)
    return benchmarks.ANALOG_BEST_KNOWN.get(name)


def config_dict(args, graph, real, world):
    return {
        "workload": f"{args.graph} {'G-set file' if real else 'structure-matched analog'} "
                    f"(n={graph.n}, m={graph.m}), pSA, sigma=(0,0,0), {args.trials} trials x "
                    f"{args.cycles} cycles x t_res 10, trials sharded over {world} GPU(s)",
        "graph": args.graph, "n": graph.n, "m": graph.m, "trials": args.trials,
        "cycles": args.cycles, "t_res": 10, "algo": "psa",
        "rng": ("replay (reference counter hash)" if args.rng == "replay"
                else "philox (native Philox4x32-10 stream)"),
        "parallelism": f"trial-shard x{world}", "l2": "flushed (512 MiB write) between steps",
    }


# ---------------------------------------------------------------- clocks

class ClockSampler:
    """nvidia-smi clocks and throttle reasons sampled during the timed region."""
    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, device):
        self.device, self.rows, self.proc = device, [], None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.device), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except OSError:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) == 6:
                self.rows.append(parts)

    def __exit__(self, *exc):
        if self.proc:
            self.proc.terminate()
            self.proc.wait(timeout=5)

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unavailable"]}
        sm = [float(r[0]) for r in self.rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[k] for r in self.rows for k in range(4) if r[2 + k] == "Active"})
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": reasons,
                "samples": len(self.rows)}


# ------------------------------------------------------------- CPU legs

def cpu_threads():
    try:
        return len(os.sched_getaffinity(0))
    except AttributeError:
        return os.cpu_count() or 1


def oracle_sample(graph, model, sch, trials, threads):
    """Time the CPU restatement of the reference loop (oracle/) on `trials`
    trials of the same workload; returns (updates/s, seconds)."""
    from oracle import oracle as orc  # test infrastructure: the CPU baseline leg only
    from paper_2601_14476_b200.pbit import VariabilityProfile
    orc.build()
    keys = streams.run_keys(streams.trial_seeds(0, trials))
    prof = VariabilityProfile.ideal(model.n)
    t0 = time.perf_counter()
    out = orc.anneal_batch(model, sch, "psa", prof, keys, graph=graph, threads=threads)
    dt = time.perf_counter() - t0
    updates = int(out["counts"].sum())
    return updates / dt, dt


def run_reference(args):
    rank, world, _ = dist_env()
    if rank != 0:
        return
    graph, real, model, sch = workload(args.graph, args.cycles)
    threads = cpu_threads()
    sample = args.cpu_sample_trials or threads
    for _ in range(args.warmup):
        oracle_sample(graph, model, sch, sample, threads)
    rates, secs = [], 0.0
    for _ in range(args.steps):
        r, dt = oracle_sample(graph, model, sch, sample, threads)
        rates.append(r)
        secs += dt
    value = sample * graph.n * args.cycles * args.steps / secs
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT,
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1e3 * secs / args.steps, "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": config_dict(args, graph, real, world),
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": threads, "kind": "port",
                         "sample": f"{sample} of {args.trials} trials per step (first trial "
                                   f"indices, same seeds), {args.cycles} cycles; C restatement "
                                   "of _kernels.anneal_loop (oracle/psa_oracle.c), pthreads"},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ------------------------------------------------------------- GPU leg

def load_profile_traffic():
    """dram bytes per sweep launch from the committed ncu capture, if any."""
    p = ROOT / "profiles" / "sweep_traffic.json"
    if p.exists():
        try:
            return json.loads(p.read_text()).get("dram_bytes_per_launch")
        except (ValueError, OSError):
            return None
    return None


def algorithmic_bytes_per_update(graph):
    """B = d + 1 + (2.125 nnz + 4 (n+1)) / (32 n)."""
    n, nnz = graph.n, 2 * graph.m
    return nnz / n + 1 + (2.125 * nnz + 4 * (n + 1)) / (32 * n)


def alu_ceiling(n, trials, cycles, local, flush):
    """Measured instruction ceiling of the sweep (SURVEY 8(d) "measure it with
    an RNG-only kernel"): the same packed kernel, launch shape and schedule on
    an edgeless graph of the same n and trials, so only the per-update draw,
    threshold lookup and decision remain.  Returns updates/s."""
    import torch
    from paper_2601_14476_b200.annealer import AnnealSchedule
    from paper_2601_14476_b200.model import IsingModel
    model = IsingModel.from_edges(n, [], h=np.zeros(n))
    sch = AnnealSchedule(i0_min=0.05, i0_max=5.0, beta=0.01 ** (1.0 / (cycles - 1)), cycles=cycles,
                         t_res=10)
    b = _native.Batch(model, sch, streams.run_keys(streams.trial_seeds(7, trials)))
    plan = _native.Plan(b, device=local)
    best = 0.0
    for _ in range(3):
        flush.zero_()
        torch.cuda.synchronize()
        plan.run()
        best = max(best, trials * n * cycles / (plan.info()["sweep_ms_mean"] * cycles * 1e-3))
    plan.close()
    return best


def peaks():
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        d = json.loads(p.read_text())
        return float(d["hbm_gbs"]), "measured"
    return 6650.0, "fallback"


def main():
    args = parse()
    if args.impl == "reference":
        run_reference(args)
        return
    rank, world, local = dist_env()
    torch = None
    if world > 1:
        import torch
        import torch.distributed as dist
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    else:
        import torch
        torch.cuda.set_device(local)

    graph, real, model, sch = workload(args.graph, args.cycles)
    lo, hi = shard(args.trials, rank, world)
    seeds = streams.trial_seeds(0, hi)[lo:hi]
    nseed = streams.native_seed(0)
    batch = _native.Batch(model, sch, streams.run_keys(seeds), graph=graph, rng=args.rng,
                          rng_seed=nseed, first_trial=lo)
    plan = _native.Plan(batch, device=local)
    flush = torch.empty(512 << 20, dtype=torch.uint8, device=f"cuda:{local}")

    def barrier():
        torch.cuda.synchronize()
        if world > 1:
            torch.distributed.barrier()

    def reduce_summary():
        return reduce_summary_of(plan)

    def reduce_summary_of(p):
        s, b, u = p.summary()
        t = torch.tensor([s, u], dtype=torch.int64, device=f"cuda:{local}")
        m = torch.tensor([b], dtype=torch.int64, device=f"cuda:{local}")
        if world > 1:
            torch.distributed.all_reduce(t)
            torch.distributed.all_reduce(m, op=torch.distributed.ReduceOp.MAX)
        return int(t[0]), int(m[0]), int(t[1])

    for _ in range(args.warmup):
        flush.zero_()
        plan.run()
        reduce_summary()
    barrier()
    dev_ms = 0.0
    t_wall = time.perf_counter()
    with ClockSampler(local) as clk:
        for _ in range(args.steps):
            flush.zero_()
            torch.cuda.synchronize()
            dev_ms += plan.run()
            cut_sum, best, updates = reduce_summary()
    barrier()
    wall_ms = 1e3 * (time.perf_counter() - t_wall)
    info = plan.info()
    h2d, d2h = plan.transfer_bytes()
    plan.close()

    # the other stream on the same workload (same timing rules), reported
    # beside the headline: the native Philox mode of the same packed sweep
    other = None
    if not args.no_philox_leg:
        alt = "philox" if args.rng == "replay" else "replay"
        ob = _native.Batch(model, sch, streams.run_keys(seeds), graph=graph, rng=alt,
                           rng_seed=nseed, first_trial=lo)
        oplan = _native.Plan(ob, device=local)
        for _ in range(args.warmup):
            flush.zero_()
            oplan.run()
        barrier()
        oms = 0.0
        for _ in range(args.steps):
            flush.zero_()
            torch.cuda.synchronize()
            oms += oplan.run()
            ocut, obest, _ = reduce_summary_of(oplan)
        barrier()
        oinfo = oplan.info()
        oplan.close()
        other = (alt, oms / args.steps, ocut, obest, oinfo)
    del flush

    # end-to-end through the public C ABI call with host buffers: inputs are
    # uploaded and all eight outputs downloaded inside every timed call, into
    # page-locked host arrays the caller allocated once (as a serving loop would)
    pinned = {k: torch.empty(v.shape, dtype=getattr(torch, str(v.dtype)), pin_memory=True).numpy()
              for k, v in batch.alloc_outputs().items()}
    _native.anneal_batch(batch, device=local, out=pinned)  # warm the allocator pools
    barrier()
    e2e_ms = 0.0
    for _ in range(args.e2e_steps):
        t0 = time.perf_counter()
        out, _ = _native.anneal_batch(batch, device=local, out=pinned)
        s_local = int(out["cut_trace"][:, -1].sum())
        e2e_ms += 1e3 * (time.perf_counter() - t0)
    barrier()

    step_ms = dev_ms / args.steps
    e2e_step_ms = e2e_ms / args.e2e_steps
    if world > 1:
        v = torch.tensor([step_ms, e2e_step_ms, other[1] if other else 0.0],
                         dtype=torch.float64, device=f"cuda:{local}")
        torch.distributed.all_reduce(v, op=torch.distributed.ReduceOp.MAX)
        step_ms, e2e_step_ms = float(v[0]), float(v[1])
        if other:
            other = (other[0], float(v[2])) + other[2:]
    total_updates = args.trials * graph.n * args.cycles
    assert updates == total_updates, (updates, total_updates)

    if rank != 0:
        torch.distributed.barrier()
        torch.distributed.destroy_process_group()
        return

    B = algorithmic_bytes_per_update(graph)
    flush = torch.empty(512 << 20, dtype=torch.uint8, device=f"cuda:{local}")
    alu = alu_ceiling(graph.n, hi - lo, min(args.cycles, 200), local, flush)
    del flush
    upd_per_launch = (hi - lo) * graph.n
    achieved = B * upd_per_launch / (info["sweep_ms_mean"] * 1e-3) / 1e9
    peak, peak_kind = peaks()
    traffic = load_profile_traffic()
    cpu = None
    if world == 1 and not args.no_cpu_baseline:
        threads = cpu_threads()
        sample = args.cpu_sample_trials or min(args.trials, 8 * threads)
        rate, secs = oracle_sample(graph, model, sch, sample, threads)
        cpu = {"value": rate, "unit": UNIT, "cores": threads, "kind": "port",
               "sample": f"first {sample} of {args.trials} trials (same seeds), {args.cycles} "
                         f"cycles, {secs:.1f} s; C restatement of _kernels.anneal_loop "
                         "(oracle/psa_oracle.c), one trial per pthread"}
    bk = best_known(args.graph, real)
    line = {
        "metric": METRIC,
        "value": total_updates / (step_ms * 1e-3),
        "unit": UNIT,
        "n_gpus": world,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": step_ms,
        "higher_is_better": True,
        "scaling": "strong",
        "vs_baseline": None,
        "dtype": "u64",
        "data": "synthetic (seeded structure-matched G-set analog; "
                + ("replayed reference RNG)" if args.rng == "replay" else "native Philox RNG)"),
        "config": config_dict(args, graph, real, world),
        "quality": {"mean_final_cut": cut_sum / args.trials, "best_cut": best,
                    "best_known": bk,
                    "mean_cut_over_best_known": (cut_sum / args.trials / bk) if bk else None},
        "e2e": {"value": total_updates / (e2e_step_ms * 1e-3), "unit": UNIT,
                "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
                "api": "pbsa_anneal_loop_batch (host buffers)", "ms_per_step": e2e_step_ms},
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                     "frac": achieved / peak, "traffic": traffic,
                     "peak_source": peak_kind,
                     "kernel": info["path"] + "_sweep",
                     "kernel_ms_mean": info["sweep_ms_mean"],
                     "bytes_per_update": B, "updates_per_launch": upd_per_launch,
                     "alu_ceiling": {"value": alu, "unit": UNIT,
                                     "frac": (upd_per_launch / (info["sweep_ms_mean"] * 1e-3)) / alu,
                                     "how": "same packed kernel and launch shape on an edgeless graph "
                                            "of the same n and trials (draw + threshold + decision only)"}},
        "cpu_baseline": cpu,
        other[0] if other else "philox": None if other is None else {
            "value": total_updates / (other[1] * 1e-3), "unit": UNIT, "ms_per_step": other[1],
            "kernel_ms_mean": other[4]["sweep_ms_mean"],
            "stream": ("native Philox4x32-10 (PBSA_RNG_PHILOX), same packed sweep and timing rules"
                       if other[0] == "philox" else "replayed reference counter hash"),
            "quality": {"mean_final_cut": other[2] / args.trials, "best_cut": other[3],
                        "mean_cut_over_best_known": (other[2] / args.trials / bk) if bk else None}},
        "clocks": clk.summary(),
        "gpu_launches": info["launches"] * args.steps,
        "wall_ms_timed_region": wall_ms,
    }
    print(json.dumps(line), flush=True)
    if world > 1:
        torch.distributed.barrier()
        torch.distributed.destroy_process_group()


if __name__ == "__main__":
    main()
