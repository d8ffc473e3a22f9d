"""Pivoted-Cholesky truncation study: accuracy vs the exact POD (configs 0, 1) and time."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_1607_05210_b200 as H
from paper_1607_05210_b200 import _device as D, workloads as W
from oracle import hapod_oracle as O

def ang(a, b):
    s = O.principal_angle_sines(a, b); return s.max() if s.size else 0.0

wl0 = W.make(0); q10 = W.haar_frame(wl0.d, 1000, 0, 1).cpu().numpy()
wl1 = W.make(1, d=20000); q11 = W.haar_frame(wl1.d, 8192, 1, 1).cpu().numpy()
for tol in [2.0 ** -52]:
    D.PSTRF_TOL = tol
    try:
        H.pod(H.SnapshotBlock(H.InnerProductSpace(wl0.d), wl0.values), wl0.eps_star)
        torch.cuda.synchronize(); t0 = time.time()
        out = H.pod(H.SnapshotBlock(H.InnerProductSpace(wl0.d), wl0.values), wl0.eps_star)
        torch.cuda.synchronize(); t_c0 = time.time() - t0
        a0 = ang(out.modes, q10[:, :out.count]); s0 = np.max(np.abs(out.sigmas - wl0.sigma_exact[:out.count]) / wl0.sigma_exact[:out.count])
        tree = H.build_star(16)
        leaves = H.distribute_columns(tree, H.SnapshotBlock(H.InnerProductSpace(wl1.d), wl1.values), block_size=512)
        tl = H.assign_tolerances(tree, leaves, H.eps_star_to_target(wl1.eps_star, wl1.m), omega=0.75)
        D.Profiler.reset(True)
        torch.cuda.synchronize(); t0 = time.time()
        res = H.run_hapod(tree, leaves, tl)
        torch.cuda.synchronize(); t_c1 = time.time() - t0
        summ = D.Profiler.summary(); D.Profiler.reset(False)
        n = res.mode_count
        a1 = ang(res.modes.modes, q11[:, :n]); s1 = np.max(np.abs(res.modes.sigmas - wl1.sigma_exact[:n]) / wl1.sigma_exact[:n])
        ph = ", ".join(f"{k} {v[1]:.0f}" for k, v in sorted(summ.items(), key=lambda kv: -kv[1][1])[:4])
        dg = res.modes.diagnostics
        print(f"pstrf tol {tol:.1e}: c0 {t_c0*1e3:6.1f} ms N={out.count} angle {a0:.2e} sig {s0:.1e} | c1(d=20k) {t_c1:5.2f} s "
              f"N={n} nkeep={dg['nkeep']} sweeps={dg['jacobi_sweeps']} angle {a1:.2e} sig {s1:.1e} | {ph}", flush=True)
    except Exception as e:
        print(f"pstrf tol {tol:.1e}: FAILED {e}", flush=True)
