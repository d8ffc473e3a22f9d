"""Timeline of one config-1 HAPOD step (16 leaves on stream workers + root): per node, the
start/end of each phase relative to the step start (CUDA events), to see how the leaf wave
overlaps.

    python tools/leaf_timeline.py [d] [workers] [e2e]

e2e: the leaves are column views of a pinned HOST buffer uploaded on demand through the shared
copy stream (bench.py's e2e leg), so the timeline shows how the 13 GB transfer overlaps the wave.
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1607_05210_b200 as H  # noqa: E402
from paper_1607_05210_b200 import _device as D  # noqa: E402
from paper_1607_05210_b200 import workloads as W  # noqa: E402

d = int(sys.argv[1]) if len(sys.argv) > 1 else 200000
workers = int(sys.argv[2]) if len(sys.argv) > 2 else 16
wl = W.make(1, d=d)
sp = H.InnerProductSpace(d)
tree = H.build_star(16)
e2e = len(sys.argv) > 3 and sys.argv[3] == "e2e"
if e2e:
    host = torch.empty((wl.m, d), dtype=torch.float64, pin_memory=True)
    host.copy_(wl.values.t())
    src = host.t()
else:
    src = wl.values


def make_leaves():
    return H.distribute_columns(tree, H.SnapshotBlock(sp, src, defer_upload=e2e), block_size=512)


leaves = make_leaves()
tol = H.assign_tolerances(tree, leaves, H.eps_star_to_target(wl.eps_star, wl.m), omega=0.75)
for rep in range(2):
    if e2e:
        leaves = make_leaves()
    D.Profiler.reset(True)
    torch.cuda.synchronize()
    t0 = torch.cuda.Event(enable_timing=True)
    t0.record()
    res, _ = H.run_parallel(tree, leaves, tol, worker_count=workers)
    torch.cuda.synchronize()
    recs = list(D.Profiler.records)
    D.Profiler.reset(False)
spans = {}
for name, e0, e1, _fl, tag in recs:
    a, b = t0.elapsed_time(e0), t0.elapsed_time(e1)
    spans.setdefault(tag, []).append((name, a, b))
for tag in sorted(spans, key=lambda t: min(x[1] for x in spans[t])):
    ph = spans[tag]
    lo, hi = min(x[1] for x in ph), max(x[2] for x in ph)
    order = " ".join(f"{n}@{a:.0f}-{b:.0f}" for n, a, b in sorted(ph, key=lambda x: x[1]) if b - a > 1.0)
    print(f"node {tag}: {lo:7.1f} .. {hi:7.1f} ms | {order}", flush=True)
