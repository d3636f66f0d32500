import sys, time, ctypes
sys.path.insert(0, '.')
import numpy as np, torch
from paper_2601_14476_b200 import _native, benchmarks, streams
from paper_2601_14476_b200.annealer import derive_schedule
from paper_2601_14476_b200.model import maxcut_to_ising
g, _ = benchmarks.load("G81"); m = maxcut_to_ising(g); sch = derive_schedule(m, 1000, 10)
b = _native.Batch(m, sch, streams.run_keys(streams.trial_seeds(0, 4096)), graph=g)
pinned = {k: torch.empty(v.shape, dtype=getattr(torch, str(v.dtype)), pin_memory=True).numpy() for k, v in b.alloc_outputs().items()}
lib = _native.load()
for drop in ([], ["inputs"], ["inputs", "spins"], ["inputs", "spins", "hist", "counts", "i0_trace"]):
    ptrs = [None if k in drop else _native._ptr(pinned[k]) for k in _native.OUT_ORDER]
    for rep in range(3):
        ms = ctypes.c_float(0)
        t0 = time.perf_counter()
        _native._check(lib.pbsa_anneal_loop_batch_ex(0, *b._args(), *ptrs, ctypes.byref(ms)))
        print(drop, rep, f"{1e3*(time.perf_counter()-t0):.1f} ms wall, device {ms.value:.1f}")
