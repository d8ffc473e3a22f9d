"""Device-resident config-1 step (16 stream workers) with the root Gramian accumulated pair by pair
beside the leaf wave (D.PROGRESSIVE_GRAM_RESIDENT) under different settings of D.ProgressiveGram.

    python tools/resident_progressive_probe.py
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1607_05210_b200 as H  # noqa: E402
from paper_1607_05210_b200 import _device as D  # noqa: E402
from paper_1607_05210_b200 import workloads as W  # noqa: E402

wl = W.make(1)
d, m = wl.d, wl.m
sp = H.InnerProductSpace(d)
tree = H.build_star(16)
maps = H.derive_maps(tree)
full = H.SnapshotBlock(sp, wl.values)
blocks = {leaf: full.column_block(512 * i, 512 * (i + 1)) for i, leaf in enumerate(maps.leaf_order)}
target = H.eps_star_to_target(wl.eps_star, m)
tol = H.assign_tolerances(tree, {leaf: 512 for leaf in maps.leaf_order}, target, omega=0.75)


def step():
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    res, stats = H.run_parallel(tree, H.LeafAssignment(blocks), tol, worker_count=16)
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1), res.mode_count, stats.wave_times[0] * 1e3, float(res.modes.sigmas.sum())


settings = [("off", None), ("8/4/0", (8, 4, 0)), ("4/4/0", (4, 4, 0)), ("2/2/0", (2, 2, 0)), ("4/0/4", (4, 0, 4)),
            ("6/2/2", (6, 2, 2)), ("off", None)]
for name, cfg in settings:
    D.PROGRESSIVE_GRAM_RESIDENT = cfg is not None
    if cfg:
        D.ProgressiveGram.WAVE_INFLIGHT, D.ProgressiveGram.TAIL_CHILDREN, D.ProgressiveGram.TAIL_INFLIGHT = cfg
    step()
    ts = [step() for _ in range(3)]
    print(f"{name:8s} (in flight / tail children / tail in flight): step {[round(t[0]) for t in ts]} ms, "
          f"wave {[round(t[2]) for t in ts]} ms -> {m / min(t[0] for t in ts) * 1e3:.0f} cols/s, modes {ts[0][1]}, "
          f"sigma sum {ts[0][3]!r}", flush=True)
