"""Time the CholQR building blocks (Cholesky + triangular inverse, full re-orthonormalisation)
at root sizes with CUDA events on the launching stream.

    python tools/chol_bench.py [n ...]
"""
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_1607_05210_b200 import _device as D  # noqa: E402
from paper_1607_05210_b200 import _native as N  # noqa: E402

lib = N.load()
st = D._stream()


def timed(fn, reps=3):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


for n in [int(a) for a in sys.argv[1:]] or [1024, 4549, 5368]:
    m = 8192 if n > 1024 else 20000
    g = torch.Generator(device="cuda").manual_seed(n)
    X = D.DevMat.empty(m, n)
    X.tensor().copy_(torch.randn(m, n, generator=g, device="cuda", dtype=torch.float64))
    C = D.DevMat.empty(n, n)
    drift = torch.zeros(1, dtype=torch.float64, device="cuda")
    ws = D._ws(lib.hp_drift_workspace_bytes(m, n))
    t_syrk = timed(lambda: lib.hp_drift(X.ptr, X.ld, m, n, C.ptr, C.ld, drift.data_ptr(), ws.data_ptr(),
                                         ws.numel(), st))
    C0 = C.clone()
    Cw = D.DevMat.empty(n, n)
    Linv = D.DevMat.empty(n, n)
    info = ctypes.c_int(0)
    cws = D._ws(lib.hp_chol_inverse_workspace_bytes(n))

    def chol():
        Cw.tensor().copy_(C0.tensor())
        N.check(lib.hp_chol_inverse(Cw.ptr, Cw.ld, n, Linv.ptr, Linv.ld, ctypes.byref(info), cws.data_ptr(),
                                    cws.numel(), st), "chol_inverse")

    t_copy = timed(lambda: Cw.tensor().copy_(C0.tensor()))
    t_chol = timed(chol) - t_copy
    rws = D._ws(lib.hp_reortho_workspace_bytes(m, n))
    Xw = D.DevMat.empty(m, n)
    passes = ctypes.c_int(0)

    def reortho():
        Xw.tensor().copy_(X.tensor())
        Cw.tensor().copy_(C0.tensor())
        N.check(lib.hp_reorthonormalize(Xw.ptr, Xw.ld, m, n, Cw.ptr, Cw.ld, 1e-3, ctypes.byref(passes),
                                        rws.data_ptr(), rws.numel(), st), "reortho")

    t_re = timed(reortho) - t_copy - timed(lambda: Xw.tensor().copy_(X.tensor()))
    print(f"n={n} m={m}: SYRK {t_syrk:.2f} ms ({m * n * (n + 1) / t_syrk / 1e9:.1f} TF/s), "
          f"potrf+trtri {t_chol:.2f} ms, reortho (1 pass, info {info.value}) {t_re:.2f} ms "
          f"[TRMM ideal {m * n * n / 33e12 * 1e3:.2f} ms]", flush=True)

# the CholQR TRMM (B upper triangular) against a plain GEMM of the same shape
for n in [int(a) for a in sys.argv[1:]] or [1024, 4549, 5368]:
    m = 8192 if n > 1024 else 20000
    A = D.DevMat.empty(m, n)
    A.tensor().normal_()
    B = D.DevMat.empty(n, n)
    B.tensor().normal_()
    Y = D.DevMat.empty(m, n)
    for b_upper in (0, 1):
        ws = D._ws(lib.hp_gemm_workspace_bytes(m, n, n, 0, b_upper))
        t = timed(lambda: N.check(lib.hp_gemm(0, 0, m, n, n, A.vecset(), B.vecset(), 1.0, 0.0, Y.ptr, Y.ld, None, None,
                                               None, 0, b_upper, ws.data_ptr(), ws.numel(), st), "gemm"))
        fl = (1.0 if b_upper else 2.0) * m * n * n
        print(f"gemm NN m={m} n=k={n} b_upper={b_upper}: {t:.2f} ms, {fl / t / 1e9:.1f} TF/s (algorithmic)", flush=True)
