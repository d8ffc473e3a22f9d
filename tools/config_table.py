"""Per-configuration device throughput on ONE B200 (snapshot cols/s, fp64), data generation
excluded: every slice / leaf / matrix is generated before its node's work starts and the
node work is bracketed by CUDA events on the launching stream (a device synchronize on both
sides).  Configs 2 and 4 stream their slices (one resident at a time, as in the reference's
incremental driver); config 3's 306 GB root input needs the row-distributed root on >= 4 GPUs,
so on one GPU only its 64 leaf PODs are timed (reported as such).  Prints one JSON line per
config.

    python tools/config_table.py [--configs 0 2 3 4] [--reps 2]
"""
import argparse
import json
import math
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1607_05210_b200 as H  # noqa: E402
from paper_1607_05210_b200 import workloads as W  # noqa: E402


class Clock:
    """Sum of CUDA-event intervals (each bracketed by device synchronizes)."""

    def __init__(self):
        self.ms = 0.0

    def __enter__(self):
        torch.cuda.synchronize()
        self.e0 = torch.cuda.Event(enable_timing=True)
        self.e0.record()
        return self

    def __exit__(self, *exc):
        e1 = torch.cuda.Event(enable_timing=True)
        e1.record()
        torch.cuda.synchronize()
        self.ms += self.e0.elapsed_time(e1)
        return False


def run_c0():
    wl = W.make(0)
    sp = H.InnerProductSpace(wl.d)
    blk = H.SnapshotBlock(sp, wl.values)
    eps = wl.eps_star  # one node, omega = 1: the root tolerance is eps* itself
    H.pod(blk, eps)
    c = Clock()
    with c:
        out = H.pod(blk, eps)
    return dict(cols=wl.m, ms=c.ms, modes=out.count, note="pod() of the resident 20,000 x 1,000 block")


def run_c2():
    cfg = W.CONFIGS[2]
    d, m, nsl = cfg["d"], cfg["m"], cfg["m"] // cfg["block"]
    target = H.eps_star_to_target(cfg["rel"] * W.frobenius_norm(2), m)
    sp = H.InnerProductSpace(d)
    sess = H.incremental_open(target, cfg["omega"], nsl)
    c = Clock()
    for b in range(nsl):
        blk = H.SnapshotBlock(sp, W.slice_values(2, b))  # generated + finiteness-checked, untimed
        with c:
            sess.push(blk)
        del blk
    with c:
        res = sess.finalize()
    return dict(cols=m, ms=c.ms, modes=res.mode_count,
                note="IncrementalSession over 64 streamed slices of 500,000 x 512")


def run_c3():
    cfg = W.CONFIGS[3]
    d, nl = cfg["d"], cfg["m"] // cfg["block"]
    sp = H.InnerProductSpace(d)
    target = H.eps_star_to_target(cfg["rel"] * W.frobenius_norm(3), cfg["m"])
    tree = H.build_star(nl)
    counts = {leaf: cfg["block"] for leaf in H.derive_maps(tree).leaf_order}
    tol = H.assign_tolerances(tree, counts, target, omega=cfg["omega"])
    eps_leaf = tol.epsilons[H.derive_maps(tree).leaf_order[0]]
    c = Clock()
    modes = []
    for b in range(nl):
        blk = H.SnapshotBlock(sp, W.slice_values(3, b))
        with c:
            out = H.pod(blk, eps_leaf)
        modes.append(out.count)
        del blk, out
    return dict(cols=cfg["m"], ms=c.ms, modes=f"leaves {min(modes)}-{max(modes)}",
                note="64 leaf PODs of 2,000,000 x 512 only: the root (306 GB input) needs the "
                     "row-distributed root on >= 4 GPUs")


C4_WORKERS = 1


def run_c4():
    cfg = W.CONFIGS[4]
    d, m = cfg["d"], cfg["m"]

    def chains_under_root(chains, per):
        children = [[]]
        for _ in range(chains):
            sub = H.build_chain(per)
            off = len(children)
            children[0].append(off + sub.root)
            children.extend([[off + k for k in kids] for kids in sub.children])
        return H.RootedTree(tuple(tuple(k) for k in children), 0)

    tree = chains_under_root(8, 16)
    order = H.derive_maps(tree).leaf_order
    slice_of = {leaf: i for i, leaf in enumerate(order)}
    counts = {leaf: cfg["block"] for leaf in order}
    eps_star = cfg["rel"] * W.frobenius_norm(4)
    tol = H.assign_tolerances(tree, counts, H.eps_star_to_target(eps_star, m), omega=cfg["omega"],
                              zero_leaf_tolerance=True)
    sp = H.InnerProductSpace(d)
    gen = Clock()

    def source(v):
        with gen:
            return H.SnapshotBlock(sp, W.slice_values(4, slice_of[v]))

    total = Clock()
    if C4_WORKERS > 1:
        # concurrent chains: slice generation overlaps other chains' work, so it stays inside
        # the timed region (not subtracted)
        def source_plain(v):
            return H.SnapshotBlock(sp, W.slice_values(4, slice_of[v]))
        with total:
            res = H.run_hapod_streaming(tree, source_plain, counts, tol, worker_count=C4_WORKERS)
        return dict(cols=m, ms=total.ms, modes=res.mode_count,
                    note=f"root over 8 chains of 16 streamed slices of 1,000,000 x 512, chains on {C4_WORKERS} "
                         "stream workers (slice generation INCLUDED in the time)")
    with total:
        res = H.run_hapod_streaming(tree, source, counts, tol)
    return dict(cols=m, ms=total.ms - gen.ms, modes=res.mode_count,
                note="root over 8 chains of 16 streamed slices of 1,000,000 x 512 (generation time "
                     f"{gen.ms / 1e3:.1f} s subtracted)")


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--configs", type=int, nargs="*", default=[0, 2, 3, 4])
    ap.add_argument("--c4-workers", type=int, default=1, help="config 4: chains on this many stream workers")
    a = ap.parse_args()
    global C4_WORKERS
    C4_WORKERS = a.c4_workers
    fns = {0: run_c0, 2: run_c2, 3: run_c3, 4: run_c4}
    for k in a.configs:
        t0 = time.time()
        r = fns[k]()
        r.update(config=k, name=W.CONFIGS[k]["name"], n_gpus=1, cols_per_s=round(r["cols"] / (r["ms"] * 1e-3), 1),
                 ms=round(r["ms"], 2), wall_s=round(time.time() - t0, 1))
        print(json.dumps(r), flush=True)


if __name__ == "__main__":
    main()
