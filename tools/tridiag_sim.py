"""NumPy study for the tridiagonal H-phase eigensolver (round 2).

Question: if the block-Jacobi solve of H = L^T L (the preconditioned Gram) is replaced by
Householder tridiagonalisation + Sturm bisection + ONE twisted-factorisation solve per
eigenvalue (no re-orthogonalisation between eigenvectors), does the existing subspace step +
Ritz polish against G still land on the reference's counts / sigma / subspace?

Host only (NumPy / SciPy LAPACK as the stand-in for the device kernels); the snapshots are a
config-1-like star at reduced size.

    python tools/tridiag_sim.py [d] [m] [leaves]
"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import scipy.linalg as sla  # noqa: E402
from scipy.linalg import lapack  # noqa: E402

from oracle import hapod_oracle as O  # noqa: E402
from oracle import hostgen  # noqa: E402

U = 2.0 ** -52
CUTOFF = 4.0 * np.finfo(np.float64).eps
POLISH_FACTOR = 1e-2
PSTRF_MARGIN = 0.25


def twisted_vectors(a, b, lam):
    """Eigenvector of tridiag(a, b) for every shift in lam by one twisted factorisation
    (LDL^T from the top, UDU^T from the bottom, twist at min |gamma_k|)."""
    n, k = a.size, lam.size
    tiny = np.finfo(np.float64).tiny / U
    dp = np.empty((n, k))
    lp = np.empty((n - 1, k))
    dm = np.empty((n, k))
    um = np.empty((n - 1, k))
    dp[0] = a[0] - lam
    for i in range(n - 1):
        piv = np.where(np.abs(dp[i]) < tiny, tiny, dp[i])
        lp[i] = b[i] / piv
        dp[i + 1] = (a[i + 1] - lam) - lp[i] * b[i]
    dm[n - 1] = a[n - 1] - lam
    for i in range(n - 2, -1, -1):
        piv = np.where(np.abs(dm[i + 1]) < tiny, tiny, dm[i + 1])
        um[i] = b[i] / piv
        dm[i] = (a[i] - lam) - um[i] * b[i]
    gamma = dp + dm - (a[:, None] - lam[None, :])
    tw = np.argmin(np.abs(gamma), axis=0)
    z = np.zeros((n, k))
    cols = np.arange(k)
    z[tw, cols] = 1.0
    # upward from the twist
    cur = np.ones(k)
    for i in range(n - 2, -1, -1):
        act = i < tw
        cur = np.where(act, -lp[i] * np.where(i + 1 == tw, 1.0, cur), cur)
        z[i] = np.where(act, cur, z[i])
    cur = np.ones(k)
    for i in range(n - 1):
        act = i >= tw
        cur = np.where(act, -um[i] * np.where(i == tw, 1.0, cur), cur)
        z[i + 1] = np.where(act, cur, z[i + 1])
    z /= np.linalg.norm(z, axis=0)[None, :]
    return z, tw, gamma[tw, cols]


def ldl_factor(a, b, shift):
    """T - shift I = L D L^T (tridiagonal Cholesky-like factorisation)."""
    n = a.size
    d = np.empty(n)
    l = np.empty(n - 1)
    d[0] = a[0] - shift
    for i in range(n - 1):
        l[i] = b[i] / d[i]
        d[i + 1] = (a[i + 1] - shift) - l[i] * b[i]
    return d, l


def negcount(d, lld, lam, pivmin):
    """#eigenvalues of L D L^T below lam (differential stationary qds), vectorised over lam."""
    n = d.size
    t = -lam.copy()
    neg = np.zeros(lam.size, dtype=np.int64)
    for i in range(n - 1):
        dp = d[i] + t
        dp = np.where(np.abs(dp) < pivmin, -pivmin, dp)
        neg += dp < 0
        t = (t / dp) * lld[i] - lam
    dp = d[n - 1] + t
    neg += dp < 0
    return neg


def bisect_rel(d, l, idx_desc, hi0, pivmin, steps=80):
    """Eigenvalue number idx (descending, 0 = largest) of L D L^T to high RELATIVE accuracy."""
    n = d.size
    lld = l * l * d[:-1]
    want = n - 1 - idx_desc  # ascending index: count(lam) <= want  <=> lam <= eig
    lo = np.full(idx_desc.size, 0.0)
    hi = np.full(idx_desc.size, hi0)
    for it in range(steps):
        # geometric midpoint once lo > 0, arithmetic otherwise
        mid = np.where(lo > 0.0, np.sqrt(lo) * np.sqrt(hi), 0.5 * (lo + hi))
        mid = np.where((hi - lo) <= 8 * U * hi, 0.5 * (lo + hi), mid)
        c = negcount(d, lld, mid, pivmin)
        below = c <= want  # eigenvalue `want` is >= mid
        lo = np.where(below, mid, lo)
        hi = np.where(below, hi, mid)
        if np.all(hi - lo <= 2 * U * hi):
            break
    return 0.5 * (lo + hi), it + 1


def getvec(d, l, lam):
    """dlar1v-style eigenvector of L D L^T for each lam: dstqds down, dpqds up, twist at min|gamma|."""
    n, k = d.size, lam.size
    ld = l * d[:-1]
    lld = l * ld
    lplus = np.empty((n - 1, k))
    sarr = np.empty((n, k))
    sarr[0] = 0.0
    s = -lam.copy()
    for i in range(n - 1):
        dplus = d[i] + s
        lplus[i] = ld[i] / dplus
        sarr[i + 1] = s * lplus[i] * l[i]
        s = sarr[i + 1] - lam
    p = np.empty((n, k))
    umin = np.empty((n - 1, k))
    p[n - 1] = d[n - 1] - lam
    for i in range(n - 2, -1, -1):
        dminus = lld[i] + p[i + 1]
        tmp = d[i] / dminus
        umin[i] = l[i] * tmp
        p[i] = p[i + 1] * tmp - lam
    gamma = sarr + p
    gamma = np.where(np.isfinite(gamma), gamma, np.inf)
    tw = np.argmin(np.abs(gamma), axis=0)
    cols = np.arange(k)
    z = np.zeros((n, k))
    z[tw, cols] = 1.0
    cur = np.ones(k)
    for i in range(n - 2, -1, -1):
        act = i < tw
        cur = np.where(act, -lplus[i] * np.where(i + 1 == tw, 1.0, cur), cur)
        z[i] = np.where(act, cur, z[i])
    cur = np.ones(k)
    for i in range(n - 1):
        act = i >= tw
        cur = np.where(act, -umin[i] * np.where(i == tw, 1.0, cur), cur)
        z[i + 1] = np.where(act, cur, z[i + 1])
    z = np.where(np.isfinite(z), z, 0.0)
    ztz = np.sum(z * z, axis=0)
    g = gamma[tw, cols]
    return z / np.sqrt(ztz)[None, :], tw, g, g / ztz, np.abs(g) / np.sqrt(ztz)


def polish(G, Q0, lam0, m, jacobi=sla.eigh):
    """_device.eig_vectors' polish: X = G Q0 / lam, orthonormalise, G2 = X^T G X, eigensolve."""
    X = (G @ Q0) / lam0[None, :]
    C = X.T @ X
    drift = np.max(np.abs(C - np.eye(C.shape[0])))
    try:
        R = np.linalg.cholesky(C)
        X = sla.solve_triangular(R, X.T, lower=True).T
        C = X.T @ X
        R = np.linalg.cholesky(C)
        X = sla.solve_triangular(R, X.T, lower=True).T
        ok = True
    except np.linalg.LinAlgError:
        X, _ = np.linalg.qr(X)
        ok = False
    G2 = X.T @ (G @ X)
    G2 = 0.5 * (G2 + G2.T)
    off = G2 - np.diag(np.diag(G2))
    dg = np.sqrt(np.abs(np.diag(G2)))
    rel_off = np.max(np.abs(off) / (dg[:, None] * dg[None, :]))
    lam, W = jacobi(G2)
    lam, W = lam[::-1], W[:, ::-1]
    return lam, X @ W, drift, ok, rel_off


def truncate(lam, eps, m):
    lam_max = lam[0]
    keep = lam >= CUTOFF * lam_max * m
    lk = lam[keep]
    n = O.truncation_rank(np.sqrt(lk), eps)
    return int(keep.sum()), int(n), float(lk[n:].sum())


def main():
    d = int(sys.argv[1]) if len(sys.argv) > 1 else 3000
    m = int(sys.argv[2]) if len(sys.argv) > 2 else 2048
    nl = int(sys.argv[3]) if len(sys.argv) > 3 else 16
    s, sig_exact, left = hostgen.decay(d, m, 10.0, 1, want_left=True)
    fro = np.linalg.norm(s)
    eps_star = 1e-6 * fro
    target = eps_star / np.sqrt(m)
    children, root = O.star(nl)
    bs = m // nl
    lo = O.leaf_order(children, root)
    blocks = {leaf: s[:, bs * i: bs * (i + 1)] for i, leaf in enumerate(lo)}
    eps = O.assign_tolerances(children, root, {leaf: bs for leaf in lo}, target, omega=0.75)
    # leaves through the oracle, the root by hand
    parts = []
    for leaf in lo:
        md = O.pod(blocks[leaf], eps[leaf])
        parts.append(md.modes * md.sigmas[None, :])
    A = np.hstack(parts)
    mr = A.shape[1]
    eps_root = eps[root]
    print(f"root input {A.shape}, eps_root {eps_root:.3e}")
    G = A.T @ A
    G = 0.5 * (G + G.T)
    t0 = time.time()
    lam_ref = np.linalg.eigvalsh(G)[::-1]
    lam_ref, V_ref = sla.eigh(G, driver="evr")
    lam_ref, V_ref = lam_ref[::-1], V_ref[:, ::-1]
    print(f"eigh(G) {time.time() - t0:.1f} s")
    nk_ref, n_ref, tail_ref = truncate(lam_ref, eps_root, mr)
    print(f"reference: nkeep {nk_ref} N {n_ref} tail {tail_ref:.8e}")

    # pivoted Cholesky stopped like hp_pstrf
    tol = max(U * np.max(np.diag(G)), PSTRF_MARGIN * POLISH_FACTOR * CUTOFF * mr * lam_ref[0])
    c, piv, rank, info = lapack.dpstrf(G, lower=1, tol=tol)
    L = np.tril(c)[:, :rank]
    P = np.zeros((mr, mr))
    P[piv - 1, np.arange(mr)] = 1.0
    L = P @ L  # rows back in the original order
    print(f"pstrf rank {rank} of {mr}; |G - L L^T| / lam_max = {np.max(np.abs(G - L @ L.T)) / lam_ref[0]:.2e}")
    H = L.T @ L
    H = 0.5 * (H + H.T)
    floor_k = POLISH_FACTOR * CUTOFF * mr

    def finish(name, lamH, W):
        K = int((lamH >= floor_k * lamH[0]).sum())
        Q0 = (L @ W[:, :K]) / np.sqrt(lamH[:K])[None, :]
        orth0 = np.max(np.abs(Q0.T @ Q0 - np.eye(K)))
        lam, V, drift, ok, rel_off = polish(G, Q0, lamH[:K], mr)
        nk, n, tail = truncate(lam, eps_root, mr)
        ncmp = min(n, n_ref)
        ds = np.max(np.abs(np.sqrt(lam[:ncmp]) - np.sqrt(lam_ref[:ncmp])) / np.sqrt(lam_ref[:ncmp]))
        Uo = A @ V[:, :n]
        Uo /= np.linalg.norm(Uo, axis=0)[None, :]
        Uo, _ = np.linalg.qr(Uo)
        r = Uo - left[:, :n] @ (left[:, :n].T @ Uo)
        ang = np.sqrt(max(np.linalg.eigvalsh(r.T @ r)[-1], 0.0))
        print(f"{name:28s} K {K} |Q0^TQ0-I| {orth0:.2e} X drift {drift:.2e} cholqr {'ok' if ok else 'FAIL'} "
              f"G2 rel off {rel_off:.2e} | nkeep {nk} N {n} tail rel {abs(tail - tail_ref) / tail_ref:.1e} "
              f"dsigma {ds:.2e} angle vs exact {ang:.2e}")

    # reference subspace angle
    Ur = A @ V_ref[:, :n_ref]
    Ur, _ = np.linalg.qr(Ur)
    r = Ur - left[:, :n_ref] @ (left[:, :n_ref].T @ Ur)
    print(f"reference angle vs exact {np.sqrt(np.linalg.eigvalsh(r.T @ r)[-1]):.2e}")

    lamH, W = sla.eigh(H)
    finish("H by LAPACK (Jacobi stand-in)", lamH[::-1], W[:, ::-1])

    # tridiagonal route
    t0 = time.time()
    c, dd, e, tau, info = lapack.dsytrd(H, lower=1)
    nH = H.shape[0]

    def apply_q(zm):
        # Q = H(1) ... H(n-1), H(i) = I - tau_i v_i v_i^T, v_i = [0.., 1, c[i+2:, i]]
        out = zm.copy()
        for i in range(nH - 2, -1, -1):
            v = np.concatenate([[1.0], c[i + 2:, i]])
            out[i + 1:] -= tau[i] * np.outer(v, v @ out[i + 1:])
        return out
    t_trd = time.time() - t0
    t0 = time.time()
    ev = sla.eigh_tridiagonal(dd, e, eigvals_only=True, lapack_driver="stebz")[::-1]
    K = int((ev >= 0.5 * floor_k * ev[0]).sum())
    z, tw, gam = twisted_vectors(dd, e, ev[:K])
    t_vec = time.time() - t0
    resid = np.max(np.abs(gam) / np.linalg.norm(z, axis=0)) / ev[0]
    zz = z.T @ z
    orth = np.abs(zz - np.eye(K))
    print(f"tridiag: sytrd {t_trd:.1f} s, bisect+twisted {t_vec:.1f} s, K {K}, max resid/lam_max {resid:.2e}, "
          f"max |z^T z - I| {orth.max():.2e}")
    # where does orthogonality degrade
    for lo_, hi_ in [(0, K // 4), (K // 4, K // 2), (K // 2, 3 * K // 4), (3 * K // 4, K - 50), (K - 50, K)]:
        print(f"   eigs {lo_}-{hi_}: lam/lam_max {ev[lo_] / ev[0]:.1e}..{ev[hi_ - 1] / ev[0]:.1e} "
              f"max off-orth {orth[lo_:hi_, :].max():.2e}")
    Wt = apply_q(z)
    lam_t = ev[:K].copy()
    Wfull = np.zeros((rank, rank))
    Wfull[:, :K] = Wt
    lam_full = np.full(rank, 0.0)
    lam_full[:K] = lam_t
    finish("H by tridiag+bisect+twisted", lam_full, Wfull)
    # with Rayleigh quotients of H for lambda
    rq = np.einsum("ij,ij->j", Wt, H @ Wt)
    lam_full2 = lam_full.copy()
    lam_full2[:K] = rq
    order = np.argsort(-lam_full2[:K])
    Wfull2 = Wfull.copy()
    Wfull2[:, :K] = Wt[:, order]
    lam_full2[:K] = rq[order]
    finish("  ... with Rayleigh lambda", lam_full2, Wfull2)

    # MRRR-lite: one definite root representation T - shift I = L D L^T, relative bisection, dlar1v
    t0 = time.time()
    tnorm = max(np.abs(dd).max(), np.abs(e).max())
    lam_min = ev[-1]
    shift = lam_min - 16 * U * tnorm * 4
    dfac, lfac = ldl_factor(dd, e, shift)
    print(f"mrrr: lam_min(T)/lam_max {lam_min / ev[0]:.2e} shift/lam_max {shift / ev[0]:.2e} min d {dfac.min() / ev[0]:.2e} "
          f"max |l| {np.abs(lfac).max():.2e}")
    pivmin = np.finfo(np.float64).tiny * max(1.0, np.max(e * e))
    Kw = int((ev >= 0.5 * floor_k * ev[0]).sum())
    lam_s, its = bisect_rel(dfac, lfac, np.arange(Kw), 2.0 * (ev[0] - shift), pivmin)
    relgap = np.abs(np.diff(lam_s)) / lam_s[:-1]
    zz_, tw, g, rqc, res = getvec(dfac, lfac, lam_s)
    print(f"mrrr: {its} bisection steps, K {Kw}, min relgap {relgap.min():.2e}, max |rqcorr|/lam {np.max(np.abs(rqc) / lam_s):.2e}, "
          f"max resid/lam {np.max(res / lam_s):.2e}, {time.time() - t0:.1f} s")
    for rq_it in range(2):
        orth = np.abs(zz_.T @ zz_ - np.eye(Kw))
        print(f"   pass {rq_it}: max |z^T z - I| {orth.max():.2e}; last 50: {orth[Kw - 50:].max():.2e}; "
              f"|T z - lam z|/lam_max {np.max(np.abs(dd[:, None] * zz_ + np.vstack([e[:, None] * zz_[1:], np.zeros((1, Kw))]) + np.vstack([np.zeros((1, Kw)), e[:, None] * zz_[:-1]]) - (lam_s + shift)[None, :] * zz_)) / ev[0]:.2e}")
        if rq_it == 0:
            lam_s = lam_s + rqc
            zz_, tw, g, rqc, res = getvec(dfac, lfac, lam_s)
    Wm = apply_q(zz_)
    lam_m = lam_s + shift
    Wfull = np.zeros((rank, rank))
    Wfull[:, :Kw] = Wm
    lam_full = np.zeros(rank)
    lam_full[:Kw] = lam_m
    finish("H by tridiag + MRRR-lite", lam_full, Wfull)


if __name__ == "__main__":
    main()
