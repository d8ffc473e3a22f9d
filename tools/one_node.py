"""Run the c1 root-like node once (for ncu): pod of a 8192-column decay block at reduced d."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_1607_05210_b200 as H
from paper_1607_05210_b200 import workloads as W
d = int(sys.argv[1]) if len(sys.argv) > 1 else 50000
m = int(sys.argv[2]) if len(sys.argv) > 2 else 8192
wl = W.make(1, d=d, m=m)
blk = H.SnapshotBlock(H.InnerProductSpace(d), wl.values)
eps = 0.75 * wl.eps_star
out = H.pod(blk, eps)
torch.cuda.synchronize()
print("modes", out.count, out.diagnostics)
