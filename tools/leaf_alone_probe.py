"""One config-1 leaf POD alone (phases, flops), the 16 leaves one after another, and the 16-worker
wave: how far the wave is from the sum of its parts.

    python tools/leaf_alone_probe.py
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
tree = H.build_star(16)
maps = H.derive_maps(tree)
full = H.SnapshotBlock(sp, wl.values)
blocks = {leaf: full.column_block(512 * i, 512 * (i + 1)) for i, leaf in enumerate(maps.leaf_order)}
target = H.eps_star_to_target(wl.eps_star, m)
tol = H.assign_tolerances(tree, {leaf: 512 for leaf in maps.leaf_order}, target, omega=0.75)
leaf0 = maps.leaf_order[0]
eps = float(tol.epsilons[leaf0])


def one(leaf):
    return H.pod(blocks[leaf], eps)


for rep in range(3):
    D.Profiler.reset(True)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    out = one(leaf0)
    torch.cuda.synchronize()
    t1 = time.perf_counter()
    summ = D.Profiler.summary()
    D.Profiler.reset(False)
    if rep:
        print(f"leaf alone: {1e3 * (t1 - t0):.1f} ms, modes {out.count} | " +
              " ".join(f"{k}={v[1]:.2f}ms/{v[2] / max(v[1], 1e-9) / 1e9:.1f}TF" for k, v in summ.items()), flush=True)

for rep in range(2):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for leaf in maps.leaf_order:
        one(leaf)
    torch.cuda.synchronize()
    print(f"16 leaves one after another: {1e3 * (time.perf_counter() - t0):.1f} ms", flush=True)

for workers in (16, 8, 4, 2):
    for rep in range(2):
        torch.cuda.synchronize()
        res, stats = H.run_parallel(tree, H.LeafAssignment(blocks), tol, worker_count=workers)
        torch.cuda.synchronize()
    print(f"wave with {workers} workers: {stats.wave_times[0] * 1e3:.1f} ms", flush=True)
