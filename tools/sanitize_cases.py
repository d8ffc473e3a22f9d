"""Small shapes of every hot-path kernel for compute-sanitizer:

    compute-sanitizer --tool memcheck|racecheck|synccheck|initcheck python tools/sanitize_cases.py

One POD that runs the whole node pipeline (TMA SYRK, pstrf_panel_sm, jac_apply + jac_round over
several block pairs, subspace step + Ritz polish, truncate, reconstruction, drift SYRK, signs), one
that triggers the CholQR re-orthonormalisation (chol_inv_run + upper-triangular TMA GEMM), one
incremental merge (block Gram), a 4-leaf star on stream workers, and plain hp_syev / hp_gemm calls
through the C-ABI.  Results are checked against the oracle so a sanitizer-clean run is also a
correct one.
"""
import ctypes
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1607_05210_b200 as H  # noqa: E402
from paper_1607_05210_b200 import _device as D  # noqa: E402
from paper_1607_05210_b200 import _native as N  # noqa: E402
from oracle import hapod_oracle as O  # noqa: E402

lib = N.load()
small = "--small" in sys.argv   # racecheck is ~100x slower: fewer block pairs


def st():
    return ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)


def check_pod(vals, eps, name):
    sp = H.InnerProductSpace(vals.shape[0])
    out = H.pod(H.SnapshotBlock(sp, vals), eps)
    ref = O.pod(vals, eps)
    assert out.count == ref.count, (name, out.count, ref.count)
    assert np.allclose(out.sigmas, ref.sigmas, rtol=1e-9), name
    print(f"[sanitize] {name}: {out.count} modes, reorthonormalized={out.diagnostics['reorthonormalized']}", flush=True)
    return out


d, m = (700, 160) if small else (1500, 300)
vals = O.synthetic_decay(d, m, 0.05, seed=1)
check_pod(vals, 1e-3 * float(np.linalg.norm(vals)), "pod (decay)")

# clustered / tiny sigmas -> drift > 1e-8 -> CholQR
rng = np.random.default_rng(3)
q1, _ = np.linalg.qr(rng.standard_normal((d, m)))
q2, _ = np.linalg.qr(rng.standard_normal((m, m)))
sig = 10.0 ** (-9.0 * np.arange(m) / (m - 1))
s2 = (q1 * sig) @ q2.T
out = check_pod(s2, 1e-7 * float(np.linalg.norm(s2)), "pod (10 decades, CholQR)")

# incremental merge: block Gram
sp = H.InnerProductSpace(d)
half = m // 2
prior = H.pod(H.SnapshotBlock(sp, vals[:, :half]), 1e-4)
merged = H.block_gramian_pod(prior, H.SnapshotBlock(sp, vals[:, half:]), 1e-3)
pr = O.pod(vals[:, :half], 1e-4)
mr = O.block_gramian_pod(pr, vals[:, half:], 1e-3)
assert merged.count == mr.count
print(f"[sanitize] block_gramian_pod: {merged.count} modes", flush=True)

# star(4) on stream workers (concurrent kernels on 4 streams)
tree = H.build_star(4)
leaves = H.distribute_columns(tree, H.SnapshotBlock(sp, vals))
tol = H.assign_tolerances(tree, leaves, 1e-3, omega=0.75)
res, _ = H.run_parallel(tree, leaves, tol, worker_count=4)
print(f"[sanitize] star(4) run_parallel: {res.mode_count} modes", flush=True)

# C-ABI: hp_syev on an indefinite matrix (plain Jacobi path), hp_gemm with edges
n = 130 if small else 200
q, _ = np.linalg.qr(rng.standard_normal((n, n)))
lam = np.sort(rng.uniform(-1, 4, n))[::-1]
g = (q * lam) @ q.T
g = 0.5 * (g + g.T)
G = D.upload(g)
lam_d = torch.empty(n, dtype=torch.float64, device="cuda")
V = D.DevMat.empty(n, n)
w = torch.empty(max(int(lib.hp_syev_workspace_bytes(n)), 16), dtype=torch.uint8, device="cuda")
sweeps = ctypes.c_int(0)
N.check(lib.hp_syev(G.ptr, G.ld, n, lam_d.data_ptr(), V.ptr, V.ld, n, D.JACOBI_TOL_REL, D.JACOBI_TOL_ABS, 0.0, 0.0, 60,
                    1, ctypes.byref(sweeps), None, w.data_ptr(), w.numel(), st()), "syev")
ev = lam_d.cpu().numpy()
assert np.allclose(ev, np.linalg.eigvalsh(g)[::-1], atol=1e-11)
print(f"[sanitize] hp_syev n={n}: {sweeps.value} sweeps", flush=True)
torch.cuda.synchronize()
print("[sanitize] all cases ok", flush=True)
