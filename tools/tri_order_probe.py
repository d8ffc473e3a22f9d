"""TRI_MIN_ORDER study: config 0 (one node, m = 1,000) and the config-1 leaf wave (16 x 512) with the
tridiagonal H-phase solver switched on at smaller orders.

    python tools/tri_order_probe.py
"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1607_05210_b200 as H  # noqa: E402
from paper_1607_05210_b200 import _device as D  # noqa: E402
from paper_1607_05210_b200 import workloads as W  # noqa: E402

w0 = W.make(0)
b0 = H.SnapshotBlock(H.InnerProductSpace(w0.d), w0.values)
w1 = W.make(1)
sp1 = H.InnerProductSpace(w1.d)
tree = H.build_star(16)
maps = H.derive_maps(tree)
full = H.SnapshotBlock(sp1, w1.values)
blocks = {leaf: full.column_block(512 * i, 512 * (i + 1)) for i, leaf in enumerate(maps.leaf_order)}
tol = H.assign_tolerances(tree, {leaf: 512 for leaf in maps.leaf_order}, H.eps_star_to_target(w1.eps_star, w1.m),
                          omega=0.75)
ref = {}
for thr in (1024, 896, 512, 1024):
    D.TRI_MIN_ORDER = thr
    for rep in range(3):
        D.Profiler.reset(True)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        out = H.pod(b0, w0.eps_star)
        torch.cuda.synchronize()
        dt = time.perf_counter() - t0
        summ = D.Profiler.summary()
        D.Profiler.reset(False)
    sig = np.asarray(out.sigmas)
    ref.setdefault("c0", sig)
    ds = np.max(np.abs(sig[:min(len(sig), len(ref["c0"]))] - ref["c0"][:len(sig)]) / ref["c0"][:len(sig)])
    print(f"thr {thr}: c0 {dt * 1e3:.1f} ms modes {out.count} dsigma vs first {ds:.2e} tri {dict(D.LAST_TRI_DIAG).get('order')} | " +
          " ".join(f"{k}={v[1]:.1f}" for k, v in summ.items()), flush=True)
    D.LAST_TRI_DIAG.clear()
    for rep in range(3):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        res, stats = H.run_parallel(tree, H.LeafAssignment(blocks), tol, worker_count=16)
        torch.cuda.synchronize()
        dt = time.perf_counter() - t0
    sig = np.asarray(res.modes.sigmas)
    ref.setdefault("c1", sig)
    ds = np.max(np.abs(sig - ref["c1"]) / ref["c1"]) if len(sig) == len(ref["c1"]) else float("nan")
    print(f"thr {thr}: c1 step {dt * 1e3:.1f} ms wave {stats.wave_times[0] * 1e3:.1f} ms modes {res.mode_count} "
          f"dsigma vs first {ds:.2e}", flush=True)
