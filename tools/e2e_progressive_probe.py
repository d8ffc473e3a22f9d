"""e2e step (config 1, deferred per-leaf uploads, 16 stream workers) under different settings of
D.ProgressiveGram: pairs in flight beside the wave, tail policy, drain streams; off = the wave
executor of the reference (parent after the whole wave).

    python tools/e2e_progressive_probe.py
"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1607_05210_b200 as H  # noqa: E402
from paper_1607_05210_b200 import _device as D  # noqa: E402
from paper_1607_05210_b200 import workloads as W  # noqa: E402

wl = W.make(1)
d, m = wl.d, wl.m
sp = H.InnerProductSpace(d)
host = torch.empty((m, d), dtype=torch.float64, pin_memory=True)
host.copy_(wl.values.t())
hv = host.t()
tree = H.build_star(16)
target = H.eps_star_to_target(wl.eps_star, m)


def step():
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    blk = H.SnapshotBlock(sp, hv, defer_upload=True)
    la = H.distribute_columns(tree, blk, block_size=512)
    tol = H.assign_tolerances(tree, la, target, omega=0.75)
    res = H.run_parallel(tree, la, tol, worker_count=16)[0]
    res.modes.sigmas.sum()
    torch.cuda.synchronize()
    return time.perf_counter() - t0, res.mode_count


settings = [("off", None), ("6/3/0", (6, 3, 0)), ("4/3/0", (4, 3, 0)), ("6/0/0", (6, 0, 0)), ("8/4/0", (8, 4, 0)),
            ("6/5/1", (6, 5, 1)), ("3/2/0", (3, 2, 0))]
for name, cfg in settings:
    D.PROGRESSIVE_GRAM = cfg is not None
    if cfg:
        D.ProgressiveGram.WAVE_INFLIGHT, D.ProgressiveGram.TAIL_CHILDREN, D.ProgressiveGram.TAIL_INFLIGHT = cfg
    step()
    ts = [step() for _ in range(3)]
    best = min(t for t, _ in ts)
    print(f"{name:8s} (in flight / tail children / tail in flight): {[round(t * 1e3) for t, _ in ts]} ms -> "
          f"{m / best:.0f} cols/s, modes {ts[0][1]}", flush=True)
