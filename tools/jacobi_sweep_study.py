"""Eigensolver convergence/time study on c0's Gramian and a random symmetric matrix."""
import ctypes, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_1607_05210_b200 import _device as D, _native as N, workloads as W
lib = N.load()

def run(g_dev, n, label):
    lam = torch.empty(n, dtype=torch.float64, device="cuda")
    V = D.DevMat.empty(n, n)
    ws = D._ws(lib.hp_syev_workspace_bytes(n))
    sw = ctypes.c_int(0)
    torch.cuda.synchronize(); t0 = time.perf_counter()
    N.check(lib.hp_syev(g_dev.ptr, g_dev.ld, n, lam.data_ptr(), V.ptr, V.ld, n, D.JACOBI_TOL_REL, D.JACOBI_TOL_ABS, 0.0, 0.0,
                        80, 1, ctypes.byref(sw), None, ws.data_ptr(), ws.numel(), D._stream()), "syev")
    torch.cuda.synchronize(); dt = time.perf_counter() - t0
    print(f"{label:28s} n={n:5d} sweeps={sw.value:3d} time={dt*1e3:9.1f} ms", flush=True)
    return lam.cpu().numpy()

for n, kind in [(1000, "c0gram"), (512, "c1leaf"), (2048, "c1root2048")]:
    if kind == "c0gram":
        wl = W.make(0)
        S = D.upload(wl.values)
    elif kind == "c1leaf":
        wl = W.make(1, d=20000, m=512)
        S = D.upload(wl.values)
    else:
        wl = W.make(1, d=20000, m=2048)
        S = D.upload(wl.values)
    G, m, _ = D.gram_full([D.Part(S)], S.rows)
    ev = run(G, m, kind)
