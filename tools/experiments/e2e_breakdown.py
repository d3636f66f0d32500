"""Where the end-to-end time of one pbsa_anneal_loop_batch-equivalent call goes."""
import sys, time
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[2]))
import numpy as np
import torch
from paper_2601_14476_b200 import _native, benchmarks, streams
from paper_2601_14476_b200.annealer import derive_schedule
from paper_2601_14476_b200.model import maxcut_to_ising

T = int(sys.argv[1]) if len(sys.argv) > 1 else 4096
g, _ = benchmarks.load("G81")
m = maxcut_to_ising(g)
sch = derive_schedule(m, 1000, 10)
b = _native.Batch(m, sch, streams.run_keys(streams.trial_seeds(0, T)), graph=g)
pinned = {k: torch.empty(v.shape, dtype=getattr(torch, str(v.dtype)), pin_memory=True).numpy()
          for k, v in b.alloc_outputs().items()}
for rep in range(3):
    t0 = time.perf_counter(); plan = _native.Plan(b); t1 = time.perf_counter()
    ms = plan.run(); t2 = time.perf_counter()
    lib = _native.load()
    _native._check(lib.pbsa_plan_download(plan._h, *(_native._ptr(pinned[k]) for k in _native.OUT_ORDER)))
    t3 = time.perf_counter(); plan.close(); t4 = time.perf_counter()
    print(f"T={T} create {1e3*(t1-t0):.1f} ms, run {1e3*(t2-t1):.1f} ms (device {ms:.1f}), "
          f"download {1e3*(t3-t2):.1f} ms, destroy {1e3*(t4-t3):.1f} ms, launches {plan.info() if False else ''}")
for rep in range(3):
    t0 = time.perf_counter()
    out, _ = _native.anneal_batch(b, out=pinned)
    t1 = time.perf_counter()
    print(f"one-shot anneal_batch {1e3*(t1-t0):.1f} ms")
