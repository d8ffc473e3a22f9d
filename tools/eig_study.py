"""Root-node eigensolver study: one config-1-root-like POD (m columns, reduced d) with the
node phases timed on the launching stream.  Per-sweep traces come from the explicit debug API
(``hp_set_debug``, include/hapod_b200.h; the library reads no environment variables): pass a
flag mask as the 4th argument (1 = per-sweep trace, 2 = mid-round timing).

    python tools/eig_study.py [d] [m] [repeats] [debug flags]
"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1607_05210_b200 as H  # noqa: E402
from paper_1607_05210_b200 import _device as D  # noqa: E402
from paper_1607_05210_b200 import workloads as W  # noqa: E402

d = int(sys.argv[1]) if len(sys.argv) > 1 else 30000
m = int(sys.argv[2]) if len(sys.argv) > 2 else 8192
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 2
if len(sys.argv) > 4:
    from paper_1607_05210_b200 import _native as N  # noqa: E402
    N.load().hp_set_debug(int(sys.argv[4]))
wl = W.make(1, d=d, m=m)
blk = H.SnapshotBlock(H.InnerProductSpace(d), wl.values)
eps = 0.75 * wl.eps_star
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
    print(f"rep {rep}: {dt * 1e3:.1f} ms modes={out.count} | {ph}", flush=True)
print("diag", out.diagnostics, flush=True)
