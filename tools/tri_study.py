"""Tridiagonal vs block-Jacobi H-phase eigensolver on a config-1-root-like POD (m columns, reduced
d): node phases timed on the launching stream, mode counts, sigma and subspace differences between
the two paths and against the exact POD (S = Q1 diag(sigma) Q2^T).

    python tools/tri_study.py [d] [m] [repeats] [debug flags] [tri]
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
from oracle import hapod_oracle as O  # noqa: E402

d = int(sys.argv[1]) if len(sys.argv) > 1 else 30000
m = int(sys.argv[2]) if len(sys.argv) > 2 else 8192
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 2
if len(sys.argv) > 4:
    from paper_1607_05210_b200 import _native as N  # noqa: E402
    N.load().hp_set_debug(int(sys.argv[4]))
wl = W.make(1, d=d, m=m)
blk = H.SnapshotBlock(H.InnerProductSpace(d), wl.values)
eps = 0.75 * wl.eps_star
outs = {}
variants = (("tri", 1024), ("jacobi", 1 << 30))
if len(sys.argv) > 5 and sys.argv[5] == "tri":
    variants = variants[:1]
for name, min_order in variants:
    D.TRI_MIN_ORDER = min_order
    for rep in range(reps):
        D.Profiler.reset(True)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        out = H.pod(blk, eps)
        torch.cuda.synchronize()
        dt = time.perf_counter() - t0
        summ = D.Profiler.summary()
        D.Profiler.reset(False)
        ph = " ".join(f"{k}={v[1]:.1f}" for k, v in summ.items())
        print(f"{name} rep {rep}: {dt * 1e3:.1f} ms modes={out.count} | {ph}", flush=True)
    print(name, "diag", out.diagnostics, D.LAST_TRI_DIAG if name == "tri" else "", flush=True)
    outs[name] = (out.count, np.asarray(out.sigmas), np.asarray(out.modes))
if len(variants) < 2:
    sys.exit(0)
na, sa, ma = outs["tri"]
nb, sb, mb = outs["jacobi"]
n = min(na, nb)
print(f"counts tri {na} jacobi {nb}; max rel dsigma {np.max(np.abs(sa[:n] - sb[:n]) / sb[:n]):.3e}")
if na == nb and n <= 6000:
    s = O.principal_angle_sines(ma, mb)
    print(f"angle tri vs jacobi {s.max():.3e}")
