"""Allocator / phase diagnostics for one config: per-step cudaMalloc counts and phase times."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1607_05210_b200 as H
from paper_1607_05210_b200 import _device as D, workloads as W

wl = W.make(1)
sp = H.InnerProductSpace(wl.d)
blk = H.SnapshotBlock(sp, wl.values)
tree = H.build_star(16)
leaves = H.distribute_columns(tree, blk, block_size=512)
tol = H.assign_tolerances(tree, leaves, wl.target, omega=wl.omega)
for rep in range(4):
    st0 = torch.cuda.memory_stats()
    D.Profiler.reset(True)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    res, stats = H.run_parallel(tree, leaves, tol, worker_count=16)
    torch.cuda.synchronize()
    dt = time.perf_counter() - t0
    st1 = torch.cuda.memory_stats()
    root = D.Profiler.summary(tag=tree.root)
    print(f"rep {rep}: {dt:.3f}s waves {[round(w, 3) for w in stats.wave_times]} "
          f"mallocs {st1.get('num_device_alloc', 0) - st0.get('num_device_alloc', 0)} "
          f"frees {st1.get('num_device_free', 0) - st0.get('num_device_free', 0)} "
          f"retries {st1.get('num_alloc_retries', 0) - st0.get('num_alloc_retries', 0)} "
          f"peak {st1['allocated_bytes.all.peak'] / 1e9:.1f} GB reserved {torch.cuda.memory_reserved() / 1e9:.1f} GB")
    print("   root:", {k: round(v[1], 1) for k, v in sorted(root.items(), key=lambda kv: -kv[1][1])})
