"""Time the DMMA GEMM engine at the config-1 contraction shapes (CUDA events, warm).

    python tools/gemm_bench.py [all|gram|asm] [--d D] [--m M] [--n N] [--reps R]
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_1607_05210_b200 import _device as D, _native as N

ap = argparse.ArgumentParser()
ap.add_argument("only", nargs="?", default="all")
ap.add_argument("--d", type=int, default=200_000)
ap.add_argument("--m", type=int, default=None)
ap.add_argument("--n", type=int, default=None)
ap.add_argument("--reps", type=int, default=5)
a = ap.parse_args()
lib = N.load()
st = D._stream


def timeit(fn, reps):
    fn()
    torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


d = a.d
mmax = max([a.m or 0, 8192])
A = D.DevMat.empty(d, mmax)
A.storage.normal_()
if a.only in ("all", "gram"):
    for m in ([a.m] if a.m else [512, 2048, 8192]):
        G = D.DevMat.empty(m, m)
        ws = D._ws(lib.hp_gram_workspace_bytes(d, m))
        S = A.view_cols(0, m)
        ms = timeit(lambda: N.check(lib.hp_gram(S.vecset(), d, m, None, G.ptr, G.ld, ws.data_ptr(), ws.numel(), st()),
                                    "g"), a.reps)
        fl = d * m * (m + 1)
        print(f"gram     d={d} m={m:5d}: {ms:8.3f} ms  {fl / ms / 1e9:7.2f} TF/s (algorithmic, symmetric counted once)",
              flush=True)
if a.only in ("all", "asm"):
    shapes = [(a.m, a.n)] if a.m else [(512, 512), (8192, 4549)]
    for (m, n) in shapes:
        V = D.DevMat.empty(m, n)
        V.storage.normal_()
        sig = torch.ones(n, dtype=torch.float64, device="cuda")
        U = D.DevMat.empty(d, n)
        ws = D._ws(lib.hp_assemble_workspace_bytes(d, m, n))
        S = A.view_cols(0, m)
        ms = timeit(lambda: N.check(lib.hp_assemble(S.vecset(), d, m, V.ptr, V.ld, sig.data_ptr(), n, U.ptr, U.ld,
                                                    ws.data_ptr(), ws.numel(), st()), "a"), a.reps)
        fl = 2.0 * d * m * n
        print(f"assemble d={d} m={m:5d} N={n:5d}: {ms:8.3f} ms  {fl / ms / 1e9:7.2f} TF/s", flush=True)
