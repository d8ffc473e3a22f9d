"""NumPy simulation: block Jacobi on H = L^T L (config-1-like spectrum) with a per-sweep
threshold schedule -- a block pair is rotated in sweep s only if its largest coupling
|h_ij| / sqrt(h_ii h_jj) (or absolute |h_ij| / max h_ii) exceeds tau_s.  Counts the rotated
pairs (each costs one row/column apply on the device) until the absolute criterion
16u * max h_ii holds.  CPU only.

    python tools/jacobi_threshold_sim.py [m] [decades] [mode]
"""
import sys
import time

import numpy as np

sys.path.insert(0, __file__.rsplit("/", 2)[0] + "/tools")
from jacobi_schedule_sim import BW, build_h, circle_rounds  # noqa: E402

U = 2.0 ** -52


def sweep(h, rounds, tau_abs, tau_rel, stats):
    n = h.shape[0]
    dmax = np.abs(np.diag(h)).max()
    worked = 0
    for pairs in rounds:
        J = None
        todo = []
        dg = np.abs(np.diag(h))
        for a, b in pairs:
            ia = slice(a * BW, (a + 1) * BW)
            ib = slice(b * BW, (b + 1) * BW)
            blk = h[ia, ib]
            # also the within-block couplings (diagonal tiles are part of the 64x64 problem)
            sub_a = h[ia, ia] - np.diag(np.diag(h[ia, ia]))
            sub_b = h[ib, ib] - np.diag(np.diag(h[ib, ib]))
            ab = max(np.abs(blk).max(), np.abs(sub_a).max(), np.abs(sub_b).max())
            if ab <= 16 * U * dmax:
                continue
            sc = np.sqrt(np.outer(dg[ia], dg[ib])) + 1e-300
            rel = max((np.abs(blk) / sc).max(),
                      (np.abs(sub_a) / (np.sqrt(np.outer(dg[ia], dg[ia])) + 1e-300)).max(),
                      (np.abs(sub_b) / (np.sqrt(np.outer(dg[ib], dg[ib])) + 1e-300)).max())
            if ab / dmax < tau_abs or rel < tau_rel:
                continue
            todo.append((a, b))
        if not todo:
            continue
        worked += len(todo)
        for a, b in todo:
            idx = np.r_[a * BW:(a + 1) * BW, b * BW:(b + 1) * BW]
            sub = h[np.ix_(idx, idx)]
            w, v = np.linalg.eigh(sub)
            order = np.argsort(-w, kind="stable")
            v = v[:, order]
            h[idx, :] = v.T @ h[idx, :]
            h[:, idx] = h[:, idx] @ v
    stats.append(worked)
    off = np.abs(h - np.diag(np.diag(h))).max() / np.abs(np.diag(h)).max()
    return off


def run(h0, nb, schedule, label):
    h = h0.copy()
    rounds = circle_rounds(nb)
    stats = []
    t0 = time.time()
    npairs_sweep = sum(len(p) for p in rounds)
    for s in range(30):
        ta, tr = schedule(s, stats)
        off = sweep(h, rounds, ta, tr, stats)
        print(f"  [{label}] sweep {s}: tau_abs {ta:.1e} tau_rel {tr:.1e} rotated {stats[-1]}/{npairs_sweep} "
              f"off/diag {off:.3e} ({time.time() - t0:.0f}s)", flush=True)
        if stats[-1] == 0 and ta == 0 and tr == 0:
            break
    print(f"  [{label}] total rotated pairs {sum(stats)} = {sum(stats) / npairs_sweep:.2f} full sweeps", flush=True)


def main():
    m = int(sys.argv[1]) if len(sys.argv) > 1 else 2048
    decades = float(sys.argv[2]) if len(sys.argv) > 2 else 10.0 * m / 8192
    mode = sys.argv[3] if len(sys.argv) > 3 else "all"
    h, _ = build_h(m, decades)
    n = h.shape[0]
    nb = -(-n // BW)
    nb += nb & 1
    hp = np.zeros((nb * BW, nb * BW))
    hp[:n, :n] = h
    print(f"m={m} decades={decades} r={n} blocks={nb}", flush=True)
    if mode in ("all", "base"):
        run(hp, nb, lambda s, st: (0.0, 0.0), "baseline")
    if mode in ("all", "rel"):
        # relative threshold: start at 1e-2, divide by 10 per sweep, then none
        run(hp, nb, lambda s, st: (0.0, max(0.0, 10.0 ** (-2 - s)) if s < 6 else 0.0), "rel 1e-2 /10")
    if mode in ("all", "abs"):
        run(hp, nb, lambda s, st: (10.0 ** (-3 - 2 * s) if s < 6 else 0.0, 0.0), "abs 1e-3 /100")


if __name__ == "__main__":
    main()
