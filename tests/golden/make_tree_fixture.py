"""Parity fixtures for BASELINE configs 3 and 4 at their REAL tree shapes, reduced row count.

  config 3: star of 64 leaves x 512 columns + the ~19,000-column root      (d' = 1,200)
  config 4: 8 chains of 16 slices x 512 columns under one root, zero leaf
            tolerance (hierarchy.py:182-222)                                (d' = 1,000)

The snapshots come from ``oracle/hostgen.py`` (NumPy Philox: the same bytes on any host up to
libm/BLAS roundings, compared through ``hostgen.checksum``).  Run in the build container,
where the unmodified reference imports:

    python tests/golden/make_tree_fixture.py --config 3 --variant ref    # hapod.run_hapod
    python tests/golden/make_tree_fixture.py --config 3 --variant evd    # oracle, LAPACK evd
    python tests/golden/make_tree_fixture.py --config 3 --variant perm   # oracle, permuted rows
    python tests/golden/make_tree_fixture.py --config 3 --merge          # floors + fixture

Output: tests/golden/c{3,4}_tree.npz / .json -- the reference's root sigma and modes, every
node's (input, output) counts, tail, projection l2, and the CPU-vs-CPU floors of sigma, angle
and l2 (evd / perm against the reference).  tests/test_gpu_tree_fixtures.py regenerates the
snapshots on the GPU box and runs the device tree against them.
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

OUT_TMP = os.environ.get("TREEFIX_TMP", "/tmp/treefix")

SPEC = {3: dict(d=1_200, leaves=64, block=512, rel=1e-5, omega=0.75, seed=3),
        4: dict(d=1_000, chains=8, per=16, block=512, rel=1e-4, omega=0.8, seed=4)}


def snapshots(cfg: int) -> np.ndarray:
    """The fixture's snapshot matrix (d' x m, Fortran order), slice by slice as the device
    generator builds its slices (one noise stream per 512-column slice)."""
    sp = SPEC[cfg]
    blk = sp["block"]
    nsl = sp["leaves"] if cfg == 3 else sp["chains"] * sp["per"]
    m = nsl * blk
    out = np.empty((sp["d"], m), order="F")
    for b in range(nsl):
        cols = np.arange(b * blk, (b + 1) * blk)
        out[:, cols] = (hostgen.sine(sp["d"], cols, sp["seed"], b) if cfg == 3
                        else hostgen.mixed(sp["d"], cols, m, sp["seed"], b))
    return out


def tree_children(cfg: int):
    """Children lists (root 0).  Config 3: star(64).  Config 4: 8 build_chain(16) subtrees
    under a root (tree.py:181-198 numbering inside each chain)."""
    sp = SPEC[cfg]
    if cfg == 3:
        n = sp["leaves"]
        return [list(range(1, n + 1))] + [[] for _ in range(n)]
    children = [[]]
    per = sp["per"]
    for _ in range(sp["chains"]):
        sub = [[] for _ in range(2 * per - 1)]
        for j in range(per - 1):
            v = 0 if j == 0 else 2 * j - 1
            sub[v] = [2 * j + 1, 2 * j + 2]
        off = len(children)
        children[0].append(off)
        children.extend([[off + k for k in kids] for kids in sub])
    return children


def dfs_leaves(children, root=0):
    out, stack = [], [root]
    while stack:
        v = stack.pop()
        if not children[v]:
            out.append(v)
        else:
            stack.extend(reversed(children[v]))
    return out


def projection_l2(s, u):
    r = s - u @ (u.T @ s)
    return float(np.linalg.norm(r))


def run_variant(cfg: int, variant: str):
    os.makedirs(OUT_TMP, exist_ok=True)
    sp = SPEC[cfg]
    s = snapshots(cfg)
    d, m = s.shape
    fro = float(np.linalg.norm(s))
    eps_star = sp["rel"] * fro
    target = eps_star / math.sqrt(m)
    children = tree_children(cfg)
    order = dfs_leaves(children)
    blk = sp["block"]
    rec = dict(config=cfg, variant=variant, d=d, m=m, fro=fro, eps_star=eps_star, target=target, omega=sp["omega"],
               nodes=len(children))
    if variant == "ref":
        sys.path.insert(0, os.environ.get("HAPOD_REF_SRC", "/root/reference/pkg/src"))
        import hapod  # the unmodified reference
        tree = hapod.RootedTree(tuple(tuple(c) for c in children), 0)
        assert list(hapod.derive_maps(tree).leaf_order) == order
        block = hapod.SnapshotBlock(hapod.InnerProductSpace(d), s)
        leaves = hapod.distribute_columns(tree, block, block_size=blk)
        tol = hapod.assign_tolerances(tree, leaves, target, omega=sp["omega"], zero_leaf_tolerance=(cfg == 4))
        t1 = time.time()
        res = hapod.run_hapod(tree, leaves, tol)
        rec["run_s"] = time.time() - t1
        rec["reports"] = [dict(node=r.node, leaf=r.is_leaf, n_in=r.input_count, n_out=r.output_mode_count,
                               eps=r.local_epsilon, tail=r.discarded_tail_energy) for r in res.reports]
        rec["epsilons"] = [float(e) for e in tol.epsilons]
        rec["apriori"] = res.apriori_error_bound
        sig = np.asarray(res.modes.sigmas)
        modes = np.asarray(res.modes.modes)
        rec["root_tail"] = float(res.modes.tail_energy)
        import scipy
        rec["numpy"], rec["scipy"] = np.__version__, scipy.__version__
        rec["nproc"] = os.cpu_count()
    else:
        from oracle import hapod_oracle as O
        vals = s
        perm = None
        if variant == "perm":
            perm = np.random.default_rng(99).permutation(d)
            vals = np.asfortranarray(s[perm])
        blocks = {leaf: vals[:, blk * i: blk * (i + 1)] for i, leaf in enumerate(order)}
        eps = O.assign_tolerances(children, 0, {leaf: blk for leaf in order}, target, sp["omega"],
                                  zero_leaf_tolerance=(cfg == 4))
        t1 = time.time()
        run = O.run_hapod(children, 0, blocks, eps, driver=("evd" if variant == "evd" else None))
        rec["run_s"] = time.time() - t1
        sig = run.modes.sigmas
        modes = run.modes.modes
        if perm is not None:
            modes = np.ascontiguousarray(modes[np.argsort(perm)])
        rec["root_tail"] = float(run.modes.tail_energy)
        rec["reports"] = [dict(node=int(v), n_out=int(c), tail=float(t), n_in=int(n))
                          for v, (c, t, n) in sorted(run.node_outputs.items())]
    rec["N"] = int(sig.size)
    rec["l2"] = projection_l2(s, modes)
    np.savez(os.path.join(OUT_TMP, f"c{cfg}_{variant}.npz"), sigmas=sig, modes=modes, checksum=hostgen.checksum(s))
    with open(os.path.join(OUT_TMP, f"c{cfg}_{variant}.json"), "w") as f:
        json.dump(rec, f, indent=1)
    print(json.dumps({k: v for k, v in rec.items() if k not in ("reports", "epsilons")}), flush=True)


def merge(cfg: int):
    from oracle import hapod_oracle as O
    recs, arrs = {}, {}
    for v in ("ref", "evd", "perm"):
        with open(os.path.join(OUT_TMP, f"c{cfg}_{v}.json")) as f:
            recs[v] = json.load(f)
        arrs[v] = dict(np.load(os.path.join(OUT_TMP, f"c{cfg}_{v}.npz")))
    ref = arrs["ref"]
    meta = {"config": cfg, "spec": SPEC[cfg], "generator": "oracle/hostgen.py (sine / mixed, one noise stream per slice)",
            "reference": recs["ref"]}
    n_ref = recs["ref"]["N"]
    floor = {"rel_dsigma": 0.0, "angle": 0.0, "l2_rel": 0.0, "tail_rel": 0.0, "count_diff": 0}
    for v in ("evd", "perm"):
        a = arrs[v]
        n = min(n_ref, recs[v]["N"])
        rel = np.abs(a["sigmas"][:n] - ref["sigmas"][:n]) / ref["sigmas"][:n]
        ang = O.principal_angle_sines(ref["modes"], a["modes"])
        meta[v] = {"N": recs[v]["N"], "l2": recs[v]["l2"], "root_tail": recs[v]["root_tail"], "run_s": recs[v]["run_s"],
                   "max_rel_dsigma_vs_ref": float(rel.max()), "max_angle_vs_ref": float(ang.max()),
                   "node_counts_equal": [r["n_out"] for r in recs[v]["reports"]] ==
                                        [r["n_out"] for r in sorted(recs["ref"]["reports"], key=lambda r: r["node"])]}
        floor["rel_dsigma"] = max(floor["rel_dsigma"], float(rel.max()))
        floor["angle"] = max(floor["angle"], float(ang.max()))
        floor["l2_rel"] = max(floor["l2_rel"], abs(recs[v]["l2"] - recs["ref"]["l2"]) / recs["ref"]["l2"])
        if recs["ref"]["root_tail"] > 0:
            floor["tail_rel"] = max(floor["tail_rel"], abs(recs[v]["root_tail"] - recs["ref"]["root_tail"])
                                    / recs["ref"]["root_tail"])
        floor["count_diff"] = max(floor["count_diff"], abs(recs[v]["N"] - n_ref))
    meta["floor"] = floor
    np.savez_compressed(os.path.join(HERE, f"c{cfg}_tree.npz"), sigmas=ref["sigmas"], modes=ref["modes"],
                        checksum=ref["checksum"])
    with open(os.path.join(HERE, f"c{cfg}_tree.json"), "w") as f:
        json.dump(meta, f, indent=1)
    print(json.dumps(floor))


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, choices=[3, 4], required=True)
    ap.add_argument("--variant", choices=["ref", "evd", "perm"])
    ap.add_argument("--merge", action="store_true")
    a = ap.parse_args()
    if a.merge:
        merge(a.config)
    else:
        run_variant(a.config, a.variant)
