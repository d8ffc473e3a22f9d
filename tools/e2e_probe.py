"""Time the e2e step variants (eager upload vs deferred per-leaf upload)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_1607_05210_b200 as H
from paper_1607_05210_b200 import workloads as W
wl = W.make(1)
d, m = wl.d, wl.m
sp = H.InnerProductSpace(d)
host = torch.empty((m, d), dtype=torch.float64, pin_memory=True)
host.copy_(wl.values.t())
hv = host.t()
tree = H.build_star(16)
target = H.eps_star_to_target(wl.eps_star, m)
def step(defer, workers):
    t0 = time.perf_counter()
    blk = H.SnapshotBlock(sp, hv, defer_upload=defer)
    torch.cuda.synchronize(); t1 = time.perf_counter()
    la = H.distribute_columns(tree, blk, block_size=512)
    tol = H.assign_tolerances(tree, la, target, omega=0.75)
    res = H.run_parallel(tree, la, tol, worker_count=workers)[0] if workers > 1 else H.run_hapod(tree, la, tol)
    s = res.modes.sigmas.sum()
    torch.cuda.synchronize(); t2 = time.perf_counter()
    return t1 - t0, t2 - t1
for defer in (False, True):
    for workers in (1, 16):
        step(defer, workers)
        a, b = step(defer, workers)
        print(f"defer={defer} workers={workers}: construct {a:.3f}s, rest {b:.3f}s, total {a+b:.3f}s -> {m/(a+b):.0f} cols/s", flush=True)
