"""Parity fixture for BASELINE config 1 at its real tree shape (16 leaves x 512 columns
+ the 8,192-column root), at the reduced row count d' = 10,000.

Config 1 is S = Q1 diag(sigma) Q2^T, so every node's Gram matrix is independent of
Q1 and of d in exact arithmetic: node sizes at d' are the full-size ones (SURVEY.md
0.3: leaves keep 512, the root keeps 4,549 of nkeep 4,562).  Run in the build
container, where the unmodified reference imports:

    python tests/golden/make_c1_fixture.py --variant ref    # hapod.run_hapod (the reference)
    python tests/golden/make_c1_fixture.py --variant evd    # oracle, LAPACK divide & conquer
    python tests/golden/make_c1_fixture.py --variant perm   # oracle, row-permuted snapshots
    python tests/golden/make_c1_fixture.py --merge          # floors + committed fixture

Each variant takes ~40 min (the root's Python MGS loop, pod.py:227-237).  The
reference run is also the committed full-tree CPU timing of config 1 at d'
(BASELINE.md section 3).  Output: tests/golden/c1_d10000.npz / .json -- the
reference's root sigma, lambda head, counts, tails, l2 error, the angles of every
CPU variant to the EXACT span Q1[:, :N], and the CPU-vs-CPU floors.  The GPU test
(tests/test_gpu_c1_fixture.py) regenerates S with oracle.hostgen on the box.
"""

from __future__ import annotations

import argparse
import json
import math
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, REPO)
from oracle import hostgen  # noqa: E402

D_PRIME = 10_000
M = 8_192
SEED = 1
OUT_TMP = os.environ.get("C1FIX_TMP", "/tmp/c1fix")


def exact_angle_sines(q1n: np.ndarray, u: np.ndarray) -> np.ndarray:
    """Principal-angle sines between span(q1n) and span(u) (both orthonormal):
    singular values of the residual R = U - Q (Q^T U), via eig(R^T R)."""
    r = u - q1n @ (q1n.T @ u)
    ev = np.linalg.eigvalsh(r.T @ r)
    return np.sqrt(np.clip(ev[::-1], 0.0, None))


def projection_l2(s: np.ndarray, u: np.ndarray) -> float:
    """||S - U U^T S||_F (the total-reading projection error of BASELINE.json)."""
    c = u.T @ s
    return float(math.sqrt(max(0.0, float(np.sum(s * s)) - float(np.sum(c * c)))))


def projection_l2_direct(s: np.ndarray, u: np.ndarray) -> float:
    r = s - u @ (u.T @ s)
    return float(np.linalg.norm(r))


def run_variant(variant: str):
    os.makedirs(OUT_TMP, exist_ok=True)
    t0 = time.time()
    s, sig_exact, left = hostgen.decay(D_PRIME, M, 10.0, SEED, want_left=True)
    t_gen = time.time() - t0
    fro = float(np.linalg.norm(s))
    eps_star = 1e-6 * fro
    target = eps_star / math.sqrt(M)
    rec: dict = {"variant": variant, "d": D_PRIME, "m": M, "seed": SEED, "fro": fro, "eps_star": eps_star,
                 "target": target, "gen_s": t_gen}
    lam_root = None
    if variant == "ref":
        sys.path.insert(0, os.environ.get("HAPOD_REF_SRC", "/root/reference/pkg/src"))
        import hapod  # the unmodified reference
        podmod = sys.modules["hapod.pod"]
        seen = []
        orig = podmod._from_spectrum

        def spy(lam_desc, *a, **k):  # record every node's eigenvalues (no behaviour change)
            seen.append(np.array(lam_desc))
            return orig(lam_desc, *a, **k)

        podmod._from_spectrum = spy
        tree = hapod.build_star(16)
        block = hapod.SnapshotBlock(hapod.InnerProductSpace(D_PRIME), s)
        leaves = hapod.distribute_columns(tree, block, block_size=512)
        tol = hapod.assign_tolerances(tree, leaves, target, omega=0.75)
        t1 = time.time()
        res = hapod.run_hapod(tree, leaves, tol)
        rec["run_s"] = time.time() - t1
        rec["reports"] = [dict(node=r.node, leaf=r.is_leaf, n_in=r.input_count, n_out=r.output_mode_count,
                               eps=r.local_epsilon, tail=r.discarded_tail_energy, wall_s=r.wall_time)
                          for r in res.reports]
        rec["apriori"] = res.apriori_error_bound
        rec["epsilons"] = [float(e) for e in tol.epsilons]
        sig = np.asarray(res.modes.sigmas)
        modes = np.asarray(res.modes.modes)
        lam_root = seen[-1]
        rec["root_tail"] = float(res.modes.tail_energy)
        rec["numpy"] = np.__version__
        import scipy
        rec["scipy"] = scipy.__version__
        try:
            import threadpoolctl
            rec["blas"] = [f"{i.get('internal_api')} {i.get('version')} {i.get('architecture')} "
                           f"threads={i.get('num_threads')}" for i in threadpoolctl.threadpool_info()]
        except Exception:
            pass
        rec["cpu"] = open("/proc/cpuinfo").read().split("model name")[1].split("\n")[0].strip(": \t")
        rec["nproc"] = os.cpu_count()
    else:
        from oracle import hapod_oracle as O
        perm = None
        vals = s
        if variant == "perm":
            perm = np.random.default_rng(99).permutation(D_PRIME)
            vals = np.asfortranarray(s[perm])
        children = [list(range(1, 17))] + [[] for _ in range(16)]
        blocks = {leaf: vals[:, 512 * (leaf - 1): 512 * leaf] for leaf in range(1, 17)}
        n_leaf = [512] * 16
        eps = O.assign_tolerances(children, 0, {leaf: 512 for leaf in range(1, 17)}, target, 0.75)
        del n_leaf
        t1 = time.time()
        run = O.run_hapod(children, 0, blocks, eps, driver=("evd" if variant == "evd" else None))
        rec["run_s"] = time.time() - t1
        sig = run.modes.sigmas
        modes = run.modes.modes
        if perm is not None:
            inv = np.argsort(perm)
            modes = np.ascontiguousarray(modes[inv])
        lam_root = run.modes.lam_desc
        rec["root_tail"] = float(run.modes.tail_energy)
        rec["reports"] = [dict(node=int(v), n_out=int(c), tail=float(t), n_in=int(n))
                          for v, (c, t, n) in sorted(run.node_outputs.items())]
    n = int(sig.size)
    lam_max = float(lam_root[0])
    nkeep = int(np.count_nonzero(lam_root >= 4.0 * 2.0 ** -52 * lam_max * M))
    rec.update(N=n, nkeep=nkeep, lam_max=lam_max)
    t2 = time.time()
    ang = exact_angle_sines(left[:, :n], modes)
    rec["l2"] = projection_l2_direct(s, modes)
    rec["metrics_s"] = time.time() - t2
    np.save(os.path.join(OUT_TMP, f"{variant}_modes.npy"), modes)
    np.savez(os.path.join(OUT_TMP, f"{variant}.npz"), sigmas=sig, lam=lam_root, exact_angles=ang,
             sigma_exact=sig_exact, checksum=hostgen.checksum(s))
    with open(os.path.join(OUT_TMP, f"{variant}.json"), "w") as f:
        json.dump(rec, f, indent=1)
    print(json.dumps({k: v for k, v in rec.items() if k != "reports"}))


def merge():
    from oracle import hapod_oracle as O
    recs, arrs, modes = {}, {}, {}
    for v in ("ref", "evd", "perm"):
        with open(os.path.join(OUT_TMP, f"{v}.json")) as f:
            recs[v] = json.load(f)
        arrs[v] = dict(np.load(os.path.join(OUT_TMP, f"{v}.npz")))
        modes[v] = np.load(os.path.join(OUT_TMP, f"{v}_modes.npy"), mmap_mode="r")
    ref = arrs["ref"]
    out = {"ref/sigmas": ref["sigmas"], "ref/lam_head": ref["lam"][: recs["ref"]["nkeep"] + 64],
           "ref/exact_angles": ref["exact_angles"], "checksum": ref["checksum"],
           "sigma_exact": ref["sigma_exact"][: recs["ref"]["nkeep"] + 64]}
    meta = {"d": D_PRIME, "m": M, "seed": SEED, "generator": "oracle.hostgen.decay(10000, 8192, 10.0, seed=1)",
            "reference": {k: v for k, v in recs["ref"].items()}}
    n_ref = recs["ref"]["N"]
    for v in ("evd", "perm"):
        a = arrs[v]
        n = min(n_ref, recs[v]["N"])
        rel = np.abs(a["sigmas"][:n] - ref["sigmas"][:n]) / ref["sigmas"][:n]
        ang = O.principal_angle_sines(np.asarray(modes["ref"]), np.asarray(modes[v]))
        out[f"{v}/sigmas"] = a["sigmas"]
        out[f"{v}/exact_angles"] = a["exact_angles"]
        out[f"{v}/rel_dsigma_vs_ref"] = rel
        meta[v] = {k: recs[v][k] for k in ("N", "nkeep", "lam_max", "root_tail", "l2", "run_s", "fro")}
        meta[v]["max_rel_dsigma_vs_ref"] = float(rel.max())
        meta[v]["max_angle_vs_ref"] = float(ang.max())
        meta[v]["max_angle_vs_exact"] = float(a["exact_angles"].max())
        meta[v]["checksum_maxdiff_vs_ref"] = float(np.max(np.abs(a["checksum"] - ref["checksum"])))
    meta["ref_max_angle_vs_exact"] = float(ref["exact_angles"].max())
    meta["floor"] = {"rel_dsigma": max(meta["evd"]["max_rel_dsigma_vs_ref"], meta["perm"]["max_rel_dsigma_vs_ref"]),
                     "angle_vs_ref": max(meta["evd"]["max_angle_vs_ref"], meta["perm"]["max_angle_vs_ref"]),
                     "angle_vs_exact": max(meta["ref_max_angle_vs_exact"], meta["evd"]["max_angle_vs_exact"],
                                           meta["perm"]["max_angle_vs_exact"])}
    np.savez_compressed(os.path.join(HERE, "c1_d10000.npz"), **out)
    with open(os.path.join(HERE, "c1_d10000.json"), "w") as f:
        json.dump(meta, f, indent=1)
    print(json.dumps(meta["floor"]))


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("--variant", choices=["ref", "evd", "perm"])
    ap.add_argument("--merge", action="store_true")
    a = ap.parse_args()
    if a.merge:
        merge()
    else:
        run_variant(a.variant)
