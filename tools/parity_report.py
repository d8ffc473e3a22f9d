"""Parity report for configs 0 and 1 (mini): GPU vs CPU (reference eigh driver evr),
the algorithmic CPU floor (LAPACK evd vs evr on the same snapshots), the rounding floor
(evr on row-permuted snapshots), and everyone against the EXACT left singular vectors
(S = Q1 diag(sigma) Q2^T, so span(Q1[:, :N]) is the exact POD space)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_1607_05210_b200 as H
from paper_1607_05210_b200 import workloads as W
from oracle import hapod_oracle as O

def ang(a, b):
    s = O.principal_angle_sines(a, b)
    return s.max() if s.size else 0.0

def rel(a, b):
    n = min(len(a), len(b))
    return float(np.max(np.abs(a[:n] - b[:n]) / b[:n])) if n else 0.0

def run(cfg, d=None, m=None):
    wl = W.make(cfg, d=d, m=m)
    vals = np.asfortranarray(wl.values.cpu().numpy())
    # exact POD space: Q1 (left factor) -- regenerate exactly as the workload did
    k = min(wl.d, wl.m)
    q1 = W.haar_frame(wl.d, k, cfg, 1).cpu().numpy()
    sig = wl.sigma_exact
    if cfg == 0:
        eps = wl.eps_star
        t0 = time.time(); g = H.pod(H.SnapshotBlock(H.InnerProductSpace(wl.d), wl.values), eps); tg = time.time() - t0
        t0 = time.time(); c = O.pod(vals, eps); tc = time.time() - t0
        c2 = O.pod(vals, eps, driver="evd")
        perm = np.random.default_rng(99).permutation(wl.d)
        c3 = O.pod(np.asfortranarray(vals[perm]), eps)
        c3m = c3.modes[np.argsort(perm)]
        gm, cm = g.modes, c.modes
        gs, cs, c2s, c3s = g.sigmas, c.sigmas, c2.sigmas, c3.sigmas
    else:
        tree = H.build_star(wl.m // 512)
        blk = H.SnapshotBlock(H.InnerProductSpace(wl.d), wl.values)
        leaves = H.distribute_columns(tree, blk, block_size=512)
        tol = H.assign_tolerances(tree, leaves, H.eps_star_to_target(wl.eps_star, wl.m), omega=wl.omega)
        t0 = time.time(); res = H.run_hapod(tree, leaves, tol); tg = time.time() - t0
        ch = [list(x) for x in tree.children]
        order = H.derive_maps(tree).leaf_order
        blocks = {l: vals[:, 512 * i: 512 * (i + 1)] for i, l in enumerate(order)}
        t0 = time.time(); c = O.run_hapod(ch, 0, blocks, list(tol.epsilons)).modes; tc = time.time() - t0
        c2 = O.run_hapod(ch, 0, blocks, list(tol.epsilons), driver="evd").modes
        perm = np.random.default_rng(99).permutation(wl.d)
        c3 = O.run_hapod(ch, 0, {l: np.asfortranarray(v[perm]) for l, v in blocks.items()}, list(tol.epsilons)).modes
        c3m = c3.modes[np.argsort(perm)]
        gm, cm = res.modes.modes, c.modes
        gs, cs, c2s, c3s = res.modes.sigmas, c.sigmas, c2.sigmas, c3.sigmas
    n = len(cs)
    ex = q1[:, :n]
    print(f"config {cfg} d={wl.d} m={wl.m}: counts gpu={len(gs)} cpu(evr)={n} cpu(evd)={len(c2s)} cpu(perm)={len(c3s)}  "
          f"[gpu {tg:.2f}s, cpu {tc:.1f}s]")
    print(f"  max rel dsigma: gpu-vs-cpu {rel(gs, cs):.2e} | evd-vs-evr {rel(c2s, cs):.2e} | perm-vs-evr {rel(c3s, cs):.2e}"
          f" | vs exact: gpu {rel(gs, sig):.2e} cpu {rel(cs, sig):.2e}")
    print(f"  max angle sine: gpu-vs-cpu {ang(gm, cm):.2e} | evd-vs-evr {ang(c2.modes, cm):.2e} | perm-vs-evr {ang(c3m, cm):.2e}"
          f" | vs exact Q1[:, :N]: gpu {ang(gm, ex):.2e} cpu {ang(cm, ex):.2e} evd {ang(c2.modes, ex):.2e}", flush=True)

run(0)
run(1, d=6000, m=2048)
run(1, d=10000, m=4096)
