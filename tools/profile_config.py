"""Time one BASELINE config end to end on the GPU with a per-phase breakdown.

    python tools/profile_config.py --config 1 [--d 200000] [--workers 1]
"""
import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np
import torch

import paper_1607_05210_b200 as H
from paper_1607_05210_b200 import _device as D
from paper_1607_05210_b200 import workloads as W


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, default=1)
    ap.add_argument("--d", type=int, default=None)
    ap.add_argument("--m", type=int, default=None)
    ap.add_argument("--workers", type=int, default=1)
    ap.add_argument("--repeat", type=int, default=1)
    a = ap.parse_args()
    t0 = time.time()
    wl = W.make(a.config, d=a.d, m=a.m)
    torch.cuda.synchronize()
    print(f"generated c{a.config} {wl.d}x{wl.m} in {time.time() - t0:.1f}s, eps*={wl.eps_star:.4e}", flush=True)
    sp = H.InnerProductSpace(wl.d)
    blk = H.SnapshotBlock(sp, wl.values)
    if a.config == 0:
        tree = H.RootedTree(((),), 0)
    else:
        tree = H.build_star(max(1, wl.m // wl.block))
    leaves = H.distribute_columns(tree, blk, block_size=wl.block if a.config else None)
    tol = H.assign_tolerances(tree, leaves, wl.target, omega=wl.omega)
    for rep in range(a.repeat):
        D.Profiler.reset(True)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        if a.workers > 1:
            res, stats = H.run_parallel(tree, leaves, tol, worker_count=a.workers)
            print("   wave times (s):", [round(w, 3) for w in stats.wave_times])
        else:
            res = H.run_hapod(tree, leaves, tol)
        torch.cuda.synchronize()
        dt = time.perf_counter() - t0
        summ = D.Profiler.summary()
        print(f"rep {rep}: {dt:.3f}s  -> {wl.m / dt:.1f} cols/s ; modes {res.mode_count}")
        for k, (n, ms, fl) in sorted(summ.items(), key=lambda kv: -kv[1][1]):
            tf = fl / (ms * 1e-3) / 1e12 if ms > 0 and fl else 0.0
            print(f"   {k:12s} n={n:4d} {ms:10.2f} ms  {fl:.3e} flop  {tf:6.2f} TF/s")
        for r in res.reports:
            if not r.is_leaf or r.node < 3:
                print("   node", r.node, "in", r.input_count, "out", r.output_mode_count, f"{r.wall_time:.3f}s",
                      getattr(res.modes, "diagnostics", None) if r.node == res.root_node else "")
    err = H.actual_mean_error(blk, res.modes) * wl.m
    print(f"l2 error {np.sqrt(err):.4e} vs eps* {wl.eps_star:.4e}  apriori {res.apriori_error_bound:.4e}")


if __name__ == "__main__":
    main()
