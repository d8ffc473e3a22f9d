"""Config-1 root eigenvalue accuracy near the Gram cutoff: device eigensolvers vs LAPACK
(scipy eigh on the same device-computed Gram) vs the exact spectrum sigma_i^2.

The leaves keep all 512 modes, so the root Gram has the eigenvalues of S^T S exactly:
sigma_i^2 = 10^(-20 (i-1)/8191)."""
import ctypes, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, scipy.linalg, torch
import paper_1607_05210_b200 as H
from paper_1607_05210_b200 import _device as D, _native as N, workloads as W

d = int(sys.argv[1]) if len(sys.argv) > 1 else 20000
wl = W.make(1, d=d)
m = wl.m
sp = H.InnerProductSpace(d)
tree = H.build_star(16)
blk = H.SnapshotBlock(sp, wl.values)
leaves = H.distribute_columns(tree, blk, block_size=512)
tol = H.assign_tolerances(tree, leaves, H.eps_star_to_target(wl.eps_star, m), omega=0.75)
maps = H.derive_maps(tree)
kids = [H.pod(leaves.blocks[l], tol.epsilons[l]) for l in maps.leaf_order]
parts = []
for k in kids:
    parts.extend(k.scaled_parts())
G, mm, _ = D.gram_full(parts, d)
torch.cuda.synchronize()
exact = wl.sigma_exact ** 2
cut = 4 * 2.0 ** -52 * exact[0] * m
eps_root = tol.epsilons[0]

def trunc(lam):
    lam = np.sort(lam)[::-1]
    lmax = lam[0]
    keep = lam >= 4 * 2.0 ** -52 * lmax * m
    s = np.sqrt(lam[keep])
    tails = np.zeros(s.size + 1)
    tails[:-1] = np.cumsum((s * s)[::-1])[::-1]
    return int(keep.sum()), int(np.argmax(tails <= eps_root ** 2)), lam

def show(name, lam):
    nk, n, lam = trunc(lam)
    idx = np.arange(4530, 4580)
    err = (lam[idx] - exact[idx]) / exact[idx]
    print(f"{name:22s} nkeep={nk} N={n}  rel err near cutoff: max {np.abs(err).max():.2e} median {np.median(np.abs(err)):.2e}; "
          f"top-10 max rel {np.abs((lam[:10]-exact[:10])/exact[:10]).max():.1e}", flush=True)

show("exact", exact)
D.KEEP_SPECTRUM = True
for meth, pol in [("pcjacobi", False), ("pcjacobi", True)]:
    D.EIG_METHOD = meth
    D.POLISH = pol
    D.Profiler.reset(True)
    t0 = time.time()
    out = D.spectrum_and_modes(G, m, parts, d, eps_root, 4 * 2.0 ** -52, False)
    torch.cuda.synchronize()
    dt = time.time() - t0
    summ = D.Profiler.summary()
    D.Profiler.reset(False)
    ph = ", ".join(f"{k} {v[1]:.0f}ms" for k, v in sorted(summ.items(), key=lambda kv: -kv[1][1]))
    print(f"  [{meth} polish={pol}] {dt:.2f}s sweeps={out.sweeps} N={len(out.sigmas)} nkeep={out.nkeep} "
          f"drift={out.drift:.2e} | {ph}")
    lam = D.LAST_SPECTRUM[0]
    show(f"{meth}{'+polish' if pol else ''}", np.concatenate([lam, np.zeros(m - lam.size)]))
g = G.to_numpy()
t0 = time.time()
lam = scipy.linalg.eigh(g, eigvals_only=True)[::-1]
print(f"  [LAPACK dsyevr on the same G] {time.time()-t0:.1f}s")
show("LAPACK eigh", lam)
perm = np.random.default_rng(1).permutation(d)
