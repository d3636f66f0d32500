"""Benchmark of the B200 pSA sweep (BASELINE.json metric: p-bit updates/s).

Default workload = BASELINE config C4: G81 (20,000-node +-1 torus analog),
plain pSA, ideal devices (sigma = 0), 4096 trials x 1000 cycles x t_res 10,
trials sharded over the N ranks (one process per GPU).  One "step" is one
whole anneal of the batch (init + 1000 sweep launches + the final cut pass +
trace finalisation, replayed as one CUDA graph) followed by the end-of-run
NCCL all_reduce of the final-cut sum, update count and best cut -- the step
is timed with CUDA events on the launching stream around both.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl reference]

`--gpus N` (N > 1) outside torchrun re-launches itself under
torch.distributed.run with N ranks (it fails if fewer than N GPUs are
visible); under torchrun WORLD_SIZE must equal N.

Prints ONE JSON line on rank 0.  `value` is measured with inputs resident in
HBM (L2 flushed between steps, max over ranks); `e2e` times the public C-ABI
call pbsa_anneal_loop_batch with host buffers (uploads, run, full download of
all eight outputs).  Extra legs on the same line: `philox` (the native stream
on the same workload) and `variability` (BASELINE C3: G55 x 4096, sigma =
0.5^3, replayed stream, the period-bucket kernel) with its own roofline.
`--impl reference` times the reference algorithm on the host cores instead
(the C restatement in oracle/, all threads); `cpu_baseline` additionally
carries the reference package itself (numba, baseline/_ref) when installed.
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
    ap.add_argument("--no-var-leg", action="store_true",
                    help="skip the BASELINE C3 variability leg (G55 x 4096, sigma = 0.5^3)")
    ap.add_argument("--no-ref-numba", action="store_true",
                    help="skip timing the reference package itself (numba) in cpu_baseline")
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
    world = max(world, args.gpus)
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


def peaks():
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        d = json.loads(p.read_text())
        return float(d["hbm_gbs"]), "measured"
    return 6650.0, "fallback"


def issue_model():
    """Warp instructions per update of the headline sweep kernel, measured by
    ncu (profiles/sweep_issue.json, written by tools/profile_r02.sh)."""
    p = ROOT / "profiles" / "sweep_issue.json"
    if p.exists():
        try:
            return json.loads(p.read_text())
        except (ValueError, OSError):
            return None
    return None


def reference_numba_sample(name, cycles, trials, threads):
    """The reference package itself (pbitsa, numba, installed into
    baseline/_ref): engine.run_trials with `threads` threads on the first
    `trials` trials (same seeds as the GPU batch).  Returns (updates/s,
    seconds) or None when the package is not installed."""
    ref = ROOT / "baseline" / "_ref"
    if not (ref / "pbitsa").exists():
        return None
    os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/pbsa_numba_cache")
    if str(ref) not in sys.path:
        sys.path.append(str(ref))
    try:
        from pbitsa import engine as reng
        from pbitsa.model import MaxCutGraph as RGraph
        from pbitsa.annealer import AlgorithmConfig as RAlgo, Algorithm as RKind
    except Exception:
        return None
    g = benchmarks.load(name)[0]
    rg = RGraph(n=g.n, edge_i=np.asarray(g.edge_i), edge_j=np.asarray(g.edge_j),
                edge_w=np.asarray(g.edge_w))
    spec = reng.ExperimentSpec(graph=name, algo=RAlgo(RKind.PSA), cycles=cycles, trials=trials,
                               threads=threads)
    reng.run_trials(reng.ExperimentSpec(graph=name, algo=RAlgo(RKind.PSA), cycles=2, trials=1),
                    {name: rg})  # JIT warm-up (numba compile), untimed
    s = reng.run_trials(spec, {name: rg})
    updates = sum(int(np.asarray(r.update_counts).sum()) for r in s.results)
    return updates / s.anneal_seconds, s.anneal_seconds


def relaunch_under_torchrun(args):
    """--gpus N (N > 1) without a torchrun environment: one rank per GPU."""
    import socket

    import torch
    have = torch.cuda.device_count()
    if have < args.gpus:
        print(f"bench.py: --gpus {args.gpus} needs {args.gpus} visible GPUs, found {have}",
              file=sys.stderr)
        sys.exit(2)
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={args.gpus}", "--master-addr=127.0.0.1", f"--master-port={port}",
           str(Path(__file__).resolve())] + sys.argv[1:]
    sys.exit(subprocess.call(cmd))


def variability_leg(args, local, world, rank, flush, barrier):
    """BASELINE C3's variability workload on the same ranks: G55 x 4096
    trials x 1000 cycles, sigma = (0.5, 0.5, 0.5), replayed stream (the
    period-bucket kernel).  Device time per run (events on the plan stream),
    max over ranks; updates = sum of the update counts."""
    import torch

    from paper_2601_14476_b200.annealer import profile_rows
    from paper_2601_14476_b200.engine import ExperimentSpec, trial_profiles
    from paper_2601_14476_b200.annealer import Algorithm, AlgorithmConfig
    from paper_2601_14476_b200.pbit import VariabilityConfig
    name, trials, sig = "G55", 4096, (0.5, 0.5, 0.5)
    graph, real, model, sch = workload(name, args.cycles)
    lo, hi = shard(trials, rank, world)
    seeds = streams.trial_seeds(0, hi)[lo:hi]
    spec = ExperimentSpec(graph=name, algo=AlgorithmConfig(Algorithm.PSA),
                          variability=VariabilityConfig(*sig), cycles=args.cycles, trials=trials)
    profs = trial_profiles(spec, model.n, seeds)
    b = _native.Batch(model, sch, streams.run_keys(seeds), profile_rows=profile_rows(profs, model.n),
                      graph=graph, first_trial=lo)
    plan = _native.Plan(b, device=local)
    for _ in range(args.warmup):
        flush.zero_()
        plan.run()
    barrier()
    ms = 0.0
    for _ in range(args.steps):
        flush.zero_()
        torch.cuda.synchronize()
        ms += plan.run()
    barrier()
    cut_sum, best, updates = plan.summary()
    info = plan.info()
    launch_ms = info["sweep_ms_mean"]
    sweeps = info["sweep_launches"]
    plan.close()
    step_ms = ms / args.steps
    v = torch.tensor([step_ms, cut_sum, best, updates], dtype=torch.float64, device=f"cuda:{local}")
    if world > 1:
        mx = v[:1].clone()
        torch.distributed.all_reduce(mx, op=torch.distributed.ReduceOp.MAX)
        sm = v[1:2].clone()
        torch.distributed.all_reduce(sm)
        bm = v[2:3].clone()
        torch.distributed.all_reduce(bm, op=torch.distributed.ReduceOp.MAX)
        up = v[3:4].clone()
        torch.distributed.all_reduce(up)
        step_ms, cut_sum, best, updates = float(mx), float(sm), float(bm), float(up)
    B = algorithmic_bytes_per_update(graph) + 4.0   # + the fired p-bit's fp16 (lam, lam delta)
    # average sweep launch: updates of a run / launches, over the mean launch time
    local_updates = updates / world
    achieved = B * (local_updates / max(1, sweeps)) / (launch_ms * 1e-3) / 1e9
    peak, peak_kind = peaks()
    bk = best_known(name, real)
    return {
        "value": updates / (step_ms * 1e-3), "unit": UNIT, "ms_per_step": step_ms,
        "workload": f"{name} structure-matched analog (n={graph.n}, m={graph.m}), pSA, "
                    f"sigma=(0.5,0.5,0.5), {trials} trials x {args.cycles} cycles x t_res 10, "
                    "replayed reference stream (BASELINE C3)",
        "kernel": info["kernel"], "updates_per_step": int(updates),
        "quality": {"mean_final_cut": cut_sum / trials, "best_cut": int(best),
                    "mean_cut_over_best_known": (cut_sum / trials / bk) if bk else None},
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                     "frac": achieved / peak, "peak_source": peak_kind,
                     "bytes_per_update": B, "kernel_ms_mean": launch_ms,
                     "launches_per_run": sweeps,
                     "model": "SURVEY 8(d) bytes per fired update (d + 1 + CSR) + 4 B fp16 profile pair; "
                              "mean over the run's sub-step launches"},
    }


def main():
    args = parse()
    rank, world, local = dist_env()
    if args.impl == "reference":
        run_reference(args)
        return
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        relaunch_under_torchrun(args)
    if world != args.gpus:
        print(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}", file=sys.stderr)
        sys.exit(2)
    import torch
    torch.cuda.set_device(local)
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))

    graph, real, model, sch = workload(args.graph, args.cycles)
    lo, hi = shard(args.trials, rank, world)
    seeds = streams.trial_seeds(0, hi)[lo:hi]
    nseed = streams.native_seed(0)
    batch = _native.Batch(model, sch, streams.run_keys(seeds), graph=graph, rng=args.rng,
                          rng_seed=nseed, first_trial=lo)
    plan = _native.Plan(batch, device=local)
    flush = torch.empty(512 << 20, dtype=torch.uint8, device=f"cuda:{local}")
    dev = f"cuda:{local}"

    def barrier():
        torch.cuda.synchronize()
        if world > 1:
            torch.distributed.barrier()

    def step_of(p):
        """One step: the whole anneal, then the end-of-run reduction (SUM of
        final-cut sum and update count, MAX of best cut) -- NCCL for N > 1."""
        p.run()
        s, b, u = p.summary()
        t = torch.tensor([s, u], dtype=torch.int64, device=dev)
        m = torch.tensor([b], dtype=torch.int64, device=dev)
        if world > 1:
            torch.distributed.all_reduce(t)
            torch.distributed.all_reduce(m, op=torch.distributed.ReduceOp.MAX)
        return t, m

    for _ in range(args.warmup):
        flush.zero_()
        step_of(plan)
    barrier()
    step_ms_list, anneal_ms = [], 0.0
    t_wall = time.perf_counter()
    with ClockSampler(local) as clk:
        for _ in range(args.steps):
            flush.zero_()
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            t, m = step_of(plan)
            e1.record()
            e1.synchronize()
            step_ms_list.append(e0.elapsed_time(e1))
    barrier()
    wall_ms = 1e3 * (time.perf_counter() - t_wall)
    cut_sum, updates, best = int(t[0]), int(t[1]), int(m[0])
    info = plan.info()
    lay = plan.layout()
    h2d, d2h = plan.transfer_bytes()
    plan.close()
    # the reduction alone (same tensors, events on torch's stream), for the record
    red_ms = 0.0
    if world > 1:
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        torch.distributed.all_reduce(t)
        torch.distributed.all_reduce(m, op=torch.distributed.ReduceOp.MAX)
        e1.record()
        e1.synchronize()
        red_ms = e0.elapsed_time(e1)

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
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            ot, om = step_of(oplan)
            e1.record()
            e1.synchronize()
            oms += e0.elapsed_time(e1)
        barrier()
        oinfo = oplan.info()
        oplan.close()
        other = (alt, oms / args.steps, int(ot[0]), int(om[0]), oinfo)
    var = None if args.no_var_leg else variability_leg(args, local, world, rank, flush, barrier)
    del flush

    # end-to-end through the public C ABI call with host buffers: inputs are
    # uploaded and all eight outputs downloaded inside every timed call, into
    # page-locked host arrays the caller allocated once (as a serving loop would)
    pinned = {k: torch.empty(v.shape, dtype=getattr(torch, str(v.dtype)), pin_memory=True).numpy()
              for k, v in batch.alloc_outputs().items()}
    t0 = time.perf_counter()
    _native.anneal_batch(batch, device=local, out=pinned)  # the first call builds the plan (reported)
    e2e_cold_ms = 1e3 * (time.perf_counter() - t0)
    barrier()
    e2e_ms = 0.0
    for _ in range(args.e2e_steps):
        t0 = time.perf_counter()
        out, _ = _native.anneal_batch(batch, device=local, out=pinned)
        int(out["cut_trace"][:, -1].sum())  # the caller reads a result
        e2e_ms += 1e3 * (time.perf_counter() - t0)
    e2e_h2d, e2e_d2h = _native.last_call_bytes()
    barrier()

    step_ms = sum(step_ms_list) / len(step_ms_list)  # mean over steps; max over ranks below
    e2e_step_ms = e2e_ms / args.e2e_steps
    if world > 1:
        v = torch.tensor([step_ms, e2e_step_ms, other[1] if other else 0.0],
                         dtype=torch.float64, device=dev)
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
    upd_per_launch = (hi - lo) * graph.n
    launch_s = info["sweep_ms_mean"] * 1e-3
    achieved = B * upd_per_launch / launch_s / 1e9
    peak, peak_kind = peaks()
    traffic = load_profile_traffic()
    clocks = clk.summary()
    issue = None
    im = issue_model()
    if im and clocks.get("sm_mhz"):
        sms = torch.cuda.get_device_properties(local).multi_processor_count
        ceiling = sms * 4 * clocks["sm_mhz"] * 1e6 / im["warp_inst_per_update"]
        issue = {"warp_inst_per_update": im["warp_inst_per_update"],
                 "ceiling": ceiling, "unit": UNIT,
                 "frac": (upd_per_launch / launch_s) / ceiling,
                 "how": f"{sms} SMs x 4 warp schedulers x 1 instruction/clk x median SM clock under "
                        "load / ncu warp instructions per update of the sweep kernel "
                        "(profiles/sweep_issue.json)",
                 "source": im.get("source")}
    cpu = None
    if world == 1 and not args.no_cpu_baseline:
        threads = cpu_threads()
        sample = args.cpu_sample_trials or min(args.trials, 8 * threads)
        rate, secs = oracle_sample(graph, model, sch, sample, threads)
        cpu = {"value": rate, "unit": UNIT, "cores": threads, "kind": "port",
               "sample": f"first {sample} of {args.trials} trials (same seeds), {args.cycles} "
                         f"cycles, {secs:.1f} s; C restatement of _kernels.anneal_loop "
                         "(oracle/psa_oracle.c), one trial per pthread"}
        if not args.no_ref_numba:
            refs = []
            for th, n_tr in ((threads, 2 * threads), (1, 2)):
                r = reference_numba_sample(args.graph, args.cycles, min(n_tr, args.trials), th)
                if r is None:
                    break
                refs.append({"value": r[0], "unit": UNIT, "cores": th, "kind": "reference",
                             "sample": f"first {min(n_tr, args.trials)} trials, {args.cycles} cycles, "
                                       f"{r[1]:.1f} s; the reference package itself "
                                       "(pbitsa.engine.run_trials, numba, threads="
                                       f"{th}; baseline/_ref)"})
            if refs:
                cpu["reference_package"] = refs
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
        "collective": {"backend": "nccl" if world > 1 else None, "ranks": world,
                       "ops": "all_reduce SUM(final-cut sum, updates) + all_reduce MAX(best cut), "
                              "inside every timed step",
                       "ms": red_ms if world > 1 else 0.0},
        "e2e": {"value": total_updates / (e2e_step_ms * 1e-3), "unit": UNIT,
                "h2d_bytes_per_step": e2e_h2d, "d2h_bytes_per_step": e2e_d2h,
                "api": "pbsa_anneal_loop_batch (page-locked host buffers; plan kept across calls, every "
                       "input uploaded and every output written per call)", "ms_per_step": e2e_step_ms,
                "cold_call_ms": e2e_cold_ms},
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                     "frac": achieved / peak, "traffic": traffic,
                     "peak_source": peak_kind,
                     "kernel": info["path"] + "_sweep",
                     "kernel_ms_mean": info["sweep_ms_mean"],
                     "bytes_per_update": B, "updates_per_launch": upd_per_launch,
                     "launch_shape": lay, "issue": issue},
        "cpu_baseline": cpu,
        other[0] if other else "philox": None if other is None else {
            "value": total_updates / (other[1] * 1e-3), "unit": UNIT, "ms_per_step": other[1],
            "kernel_ms_mean": other[4]["sweep_ms_mean"],
            "stream": ("native Philox4x32-10 (PBSA_RNG_PHILOX), same packed sweep and timing rules"
                       if other[0] == "philox" else "replayed reference counter hash"),
            "quality": {"mean_final_cut": other[2] / args.trials, "best_cut": other[3],
                        "mean_cut_over_best_known": (other[2] / args.trials / bk) if bk else None}},
        "variability": var,
        "clocks": clocks,
        "gpu_launches": info["launches"] * args.steps,
        "wall_ms_timed_region": wall_ms,
    }
    print(json.dumps(line), flush=True)
    if world > 1:
        torch.distributed.barrier()
        torch.distributed.destroy_process_group()


if __name__ == "__main__":
    main()
