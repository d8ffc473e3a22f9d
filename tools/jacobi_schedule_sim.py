"""NumPy simulation of the block-Jacobi schedule on the preconditioned root matrix H = L^T L
(L = pivoted Cholesky of a config-1-like Gramian): full round-robin sweeps vs "band" sweeps
that pair only nearby blocks, measured by max|h_ij| / max h_ii per sweep and by the number of
64x64 rounds (each round costs one full apply on the device).  CPU only.

    python tools/jacobi_schedule_sim.py [m] [decades]
"""
import sys
import time

import numpy as np
import scipy.linalg as sl

BW = 32


def build_h(m, decades, seed=1):
    rng = np.random.default_rng(seed)
    q, r = np.linalg.qr(rng.standard_normal((m, m)))
    q *= np.sign(np.diag(r))[None, :]
    sig2 = 10.0 ** (-2.0 * decades * np.arange(m) / (m - 1))
    g = (q * sig2[None, :]) @ q.T
    g = 0.5 * (g + g.T)
    u = 2.0 ** -52
    c, piv, rank, info = sl.lapack.dpstrf(g, lower=1, tol=4 * u * m * 1e-2 * 0.25)
    L = np.tril(c)[:, :rank]
    h = L.T @ L
    return h, sig2


def circle_rounds(nb):
    m = nb - 1
    rounds = []
    for r in range(m):
        pairs = [(m, r)]
        for k in range(1, nb // 2):
            pairs.append(((r + k) % m, (r - k) % m))
        rounds.append([(min(a, b), max(a, b)) for a, b in pairs])
    return rounds


def band_rounds(nb, band):
    """for offset d = 1..band: pair block i with i + d inside runs of 2d (every block used when
    possible); returns a list of pairings (disjoint pairs)."""
    rounds = []
    for d in range(1, band + 1):
        for phase in range(2):
            pairs = []
            used = set()
            start = phase * d
            i = start
            while i + d < nb:
                for j in range(d):
                    a, b = i + j, i + j + d
                    if b < nb and a not in used and b not in used:
                        pairs.append((a, b))
                        used.update((a, b))
                i += 2 * d
            if pairs:
                rounds.append(pairs)
    return rounds


def run_round(h, pairs):
    n = h.shape[0]
    J = np.eye(n)
    for a, b in pairs:
        idx = np.r_[a * BW:(a + 1) * BW, b * BW:(b + 1) * BW]
        sub = h[np.ix_(idx, idx)]
        w, v = np.linalg.eigh(sub)
        order = np.argsort(-w, kind="stable")
        J[np.ix_(idx, idx)] = v[:, order]
    return J.T @ h @ J


def off_ratio(h):
    d = np.abs(np.diag(h)).max()
    o = np.abs(h - np.diag(np.diag(h))).max()
    return o / d


def simulate(h0, schedule, label):
    h = h0.copy()
    rounds = 0
    t0 = time.time()
    out = []
    for name, rlist in schedule:
        for pairs in rlist:
            h = run_round(h, pairs)
        rounds += len(rlist)
        out.append((name, rounds, off_ratio(h)))
        print(f"  [{label}] {name:10s} rounds {rounds:5d} off/diag {out[-1][2]:.3e}  ({time.time() - t0:.0f}s)",
              flush=True)
        if out[-1][2] < 16 * 2.0 ** -52:
            break
    return out


def main():
    m = int(sys.argv[1]) if len(sys.argv) > 1 else 2048
    decades = float(sys.argv[2]) if len(sys.argv) > 2 else 10.0 * m / 8192
    h, _ = build_h(m, decades)
    n = h.shape[0]
    nb = -(-n // BW)
    nb += nb & 1
    hp = np.zeros((nb * BW, nb * BW))
    hp[:n, :n] = h
    print(f"m={m} decades={decades:.2f} r={n} blocks={nb} initial off/diag {off_ratio(hp):.3e}", flush=True)
    full = circle_rounds(nb)
    simulate(hp, [("full", full)] * 14, "full sweeps")
    for band in (4, 8):
        br = band_rounds(nb, band)
        simulate(hp, [("band", br)] * 6 + [("full", full)] * 10, f"band {band} x6 then full")


if __name__ == "__main__":
    main()
