"""Polish-floor study: how far below the Gram cutoff the preconditioned eigensolve must resolve
(POLISH_FACTOR: eigenpairs kept for the subspace step; PSTRF_POLISH_MARGIN: where the pivoted
Cholesky stops, as a fraction of that floor) vs time and accuracy against the EXACT POD of
configs 0 and 1 (S = Q1 diag(sigma) Q2^T: span(Q1[:, :N]) and sigma are known).

    python tools/polish_study.py [d1]
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


def ang(a, b):
    s = O.principal_angle_sines(a, b)
    return s.max() if s.size else 0.0


d1 = int(sys.argv[1]) if len(sys.argv) > 1 else 20000
wl0 = W.make(0)
q10 = W.haar_frame(wl0.d, 1000, 0, 1).cpu().numpy()
wl1 = W.make(1, d=d1)
q11 = W.haar_frame(wl1.d, 8192, 1, 1).cpu().numpy()
blk0 = H.SnapshotBlock(H.InnerProductSpace(wl0.d), wl0.values)
tree = H.build_star(16)
leaves = H.distribute_columns(tree, H.SnapshotBlock(H.InnerProductSpace(wl1.d), wl1.values), block_size=512)
tl = H.assign_tolerances(tree, leaves, H.eps_star_to_target(wl1.eps_star, wl1.m), omega=0.75)
for pf, margin in [(1e-2, 0.25), (3e-2, 0.25), (1e-1, 0.25), (1e-1, 1.0), (3e-1, 0.25), (3e-1, 1.0)]:
    D.POLISH_FACTOR, D.PSTRF_POLISH_MARGIN = pf, margin
    H.pod(blk0, wl0.eps_star)
    torch.cuda.synchronize()
    t0 = time.time()
    out = H.pod(blk0, wl0.eps_star)
    torch.cuda.synchronize()
    t_c0 = time.time() - t0
    a0 = ang(out.modes, q10[:, :out.count])
    s0 = np.max(np.abs(out.sigmas - wl0.sigma_exact[:out.count]) / wl0.sigma_exact[:out.count])
    D.Profiler.reset(True)
    torch.cuda.synchronize()
    t0 = time.time()
    res = H.run_hapod(tree, leaves, tl)
    torch.cuda.synchronize()
    t_c1 = time.time() - t0
    summ = D.Profiler.summary(tag=tree.root)
    D.Profiler.reset(False)
    n = res.mode_count
    a1 = ang(res.modes.modes, q11[:, :n])
    s1 = np.max(np.abs(res.modes.sigmas - wl1.sigma_exact[:n]) / wl1.sigma_exact[:n])
    dg = res.modes.diagnostics
    ph = " ".join(f"{k}={v[1]:.0f}" for k, v in summ.items() if v[1] > 5)
    print(f"pf {pf:.0e} margin {margin:.2f}: c0 {t_c0 * 1e3:6.1f} ms N={out.count} angle {a0:.2e} sig {s0:.1e} | "
          f"c1(d={d1}) {t_c1:5.2f} s N={n} nkeep={dg['nkeep']} sweeps={dg['jacobi_sweeps']} angle {a1:.2e} "
          f"sig {s1:.1e} | root {ph}", flush=True)
