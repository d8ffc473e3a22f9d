"""Kernel-level parity of libhapod_b200.so against the CPU oracle / numpy, called
through the C-ABI (ctypes).  Needs a B200."""

import ctypes

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("no CUDA device", allow_module_level=True)

from paper_1607_05210_b200 import _device as D  # noqa: E402
from paper_1607_05210_b200 import _native as N  # noqa: E402

lib = N.load()


def st():
    return ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)


def ws(nbytes):
    return torch.empty(max(int(nbytes), 16), dtype=torch.uint8, device="cuda")


@pytest.mark.parametrize("d,m", [(1, 1), (7, 3), (100, 17), (1000, 128), (4099, 129), (20000, 512), (3, 300)])
def test_gram_matches_numpy(d, m):
    rng = np.random.default_rng(d * 7 + m)
    a = rng.standard_normal((d, m))
    A = D.upload(a)
    G = D.DevMat.empty(m, m)
    w = ws(lib.hp_gram_workspace_bytes(d, m))
    N.check(lib.hp_gram(A.vecset(), d, m, None, G.ptr, G.ld, w.data_ptr(), w.numel(), st()), "gram")
    g = G.to_numpy()
    ref = a.T @ a
    assert np.array_equal(g, g.T)  # exactly symmetric
    assert np.max(np.abs(g - ref)) <= 1e-13 * max(1.0, np.max(np.abs(ref))) * np.sqrt(d)


@pytest.mark.parametrize("d,m", [(20000, 256), (30000, 384), (50000, 640), (9000, 1000), (40000, 130),
                                 (200000, 512)])
def test_gram_small_symmetric_outputs_split(d, m):
    """Small symmetric outputs (2..8 tile columns, split-K): the re-dealt diagonal tiles, the
    longest-first block order and the makespan-modelled split count (hp_gemm.cu, diag_aware_splits)
    against float64 NumPy (gramian, pod.py:208-211)."""
    g0 = torch.Generator(device="cuda").manual_seed(d + m)
    A = D.DevMat.empty(d, m)
    A.tensor().copy_(torch.randn(d, m, generator=g0, device="cuda", dtype=torch.float64))
    G = D.DevMat.empty(m, m)
    w = ws(lib.hp_gram_workspace_bytes(d, m))
    N.check(lib.hp_gram(A.vecset(), d, m, None, G.ptr, G.ld, w.data_ptr(), w.numel(), st()), "gram")
    g = G.to_numpy()
    a = A.to_numpy()
    ref = a.T @ a
    assert np.array_equal(g, g.T)
    assert np.max(np.abs(g - ref)) <= 1e-13 * max(1.0, np.max(np.abs(ref))) * np.sqrt(d)


@pytest.mark.parametrize("n", [128, 200, 512, 640])
def test_diagonal_tile_path_is_bitwise_the_regular_path(n):
    """A diagonal block of a Gramian through the symmetric launch (diagonal tiles re-dealt over the
    consumer warps, mma_ktile_diag) against the same block as a plain pair product (regular 2 x 4
    warp grid): both unsplit, so every entry with row <= column must agree bit for bit."""
    d = 3000
    rng = np.random.default_rng(n)
    U = D.upload(np.asfortranarray(rng.standard_normal((d, n))))
    sig = torch.tensor(10.0 ** rng.uniform(-2, 0, n), device="cuda")
    sym = D.DevMat.empty(n, n, zero=True)
    full = D.DevMat.empty(n, n, zero=True)
    N.check(lib.hp_gram_pair(U.vecset(), sig.data_ptr(), n, U.vecset(), sig.data_ptr(), n, d, 1, sym.ptr, sym.ld,
                             st()), "symmetric pair")
    N.check(lib.hp_gram_pair(U.vecset(), sig.data_ptr(), n, U.vecset(), sig.data_ptr(), n, d, 0, full.ptr, full.ld,
                             st()), "plain pair")
    a, b = sym.to_numpy(), full.to_numpy()
    iu = np.triu_indices(n)
    assert np.array_equal(a[iu], b[iu])
    assert np.array_equal(a, a.T)


@pytest.mark.parametrize("odd", [False, True])
def test_gram_colscale_and_table(odd):
    rng = np.random.default_rng(5)
    d = 333 if odd else 334
    parts = [rng.standard_normal((d, c)) for c in (5, 0, 40, 13)]
    scales = [rng.uniform(0.5, 2.0, p.shape[1]) for p in parts]
    devparts = [D.Part(D.upload(p), torch.from_numpy(s).cuda()) for p, s in zip(parts, scales)]
    G, m, keep = D.gram_full(devparts, d)
    joined = np.hstack([p * s for p, s in zip(parts, scales)])
    ref = joined.T @ joined
    assert np.allclose(G.to_numpy(), ref, rtol=1e-13, atol=1e-12)


@pytest.mark.parametrize("M,N_,K", [(1, 1, 1), (300, 70, 33), (20000, 257, 512), (129, 130, 1000)])
def test_gemm_nn_with_divide(M, N_, K):
    rng = np.random.default_rng(M + N_ + K)
    a = rng.standard_normal((M, K))
    b = rng.standard_normal((K, N_))
    dv = rng.uniform(0.5, 2.0, N_)
    A, B = D.upload(a), D.upload(b)
    C = D.DevMat.empty(M, N_)
    dvd = torch.from_numpy(dv).cuda()
    w = ws(lib.hp_gemm_workspace_bytes(M, N_, K, 0, 0))
    N.check(lib.hp_gemm(0, 1, M, N_, K, A.vecset(), B.vecset(), 1.0, 0.0, C.ptr, C.ld, None, None, dvd.data_ptr(),
                        0, 0, w.data_ptr(), w.numel(), st()), "gemm")
    ref = (a @ b) / dv[None, :]
    assert np.allclose(C.to_numpy(), ref, rtol=1e-12, atol=1e-11)


def test_gemm_nt_sym_and_upper():
    rng = np.random.default_rng(3)
    M, K = 200, 64
    p = rng.standard_normal((M, K))
    c0 = rng.standard_normal((M, M))
    c0 = c0 + c0.T
    P, C = D.upload(p), D.upload(c0)
    w = ws(lib.hp_gemm_workspace_bytes(M, M, K, 1, 0))
    N.check(lib.hp_gemm(0, 0, M, M, K, P.vecset(), P.vecset(), -1.0, 1.0, C.ptr, C.ld, None, None, None, 1, 0,
                        w.data_ptr(), w.numel(), st()), "syrk")
    assert np.allclose(C.to_numpy(), c0 - p @ p.T, rtol=1e-12, atol=1e-11)
    # upper-triangular B, N-major
    x = rng.standard_normal((500, 150))
    l = np.tril(rng.standard_normal((150, 150)))
    X, L = D.upload(x), D.upload(l)
    Y = D.DevMat.empty(500, 150)
    N.check(lib.hp_gemm(0, 0, 500, 150, 150, X.vecset(), L.vecset(), 1.0, 0.0, Y.ptr, Y.ld, None, None, None, 0, 1,
                        None, 0, st()), "trmm")
    assert np.allclose(Y.to_numpy(), x @ l.T, rtol=1e-12, atol=1e-11)


@pytest.mark.parametrize("bk", [0, 1])
@pytest.mark.parametrize("M,K", [(200, 64), (515, 128), (1000, 130)])
def test_gemm_symmetric_update_modes(M, K, bk):
    """C -= P P^T with an M-major A (the pivoted Cholesky's and the tridiagonalisation's trailing
    updates): sym = 1 writes both triangles (16-byte words and, with an N-major B, 16-byte mirrored
    words on the tiles above the diagonal); sym = 2 updates the upper triangle only and must leave
    the strictly lower part of C untouched.  Ragged last tiles in both directions."""
    rng = np.random.default_rng(M + K + bk)
    p = rng.standard_normal((M, K))
    c0 = rng.standard_normal((M, M))
    c0 = c0 + c0.T
    P = D.upload(p)
    Bop = P if bk == 0 else D.upload(np.asfortranarray(p.T))  # K-major B: vector n holds p[n, :]
    want = c0 - p @ p.T
    for sym in (1, 2):
        C = D.upload(c0)
        w = ws(lib.hp_gemm_workspace_bytes(M, M, K, sym, 0))
        N.check(lib.hp_gemm(0, bk, M, M, K, P.vecset(), Bop.vecset(), -1.0, 1.0, C.ptr, C.ld, None, None, None, sym,
                            0, w.data_ptr(), w.numel(), st()), "symmetric update")
        got = C.to_numpy()
        iu = np.triu_indices(M)
        assert np.allclose(got[iu], want[iu], rtol=1e-12, atol=1e-11)
        il = np.tril_indices(M, -1)
        if sym == 1:
            assert np.array_equal(got, got.T)
        else:
            assert np.array_equal(got[il], c0[il])


@pytest.mark.parametrize("M,N_,K", [(300, 70, 33), (2000, 257, 512)])
def test_gemm_accumulate_beta(M, N_, K):
    """C = 0.5 C - A B with an M-major A: the read-modify-write epilogue (16-byte words)."""
    rng = np.random.default_rng(M * 3 + N_ + K)
    a = rng.standard_normal((M, K))
    b = rng.standard_normal((K, N_))
    c0 = rng.standard_normal((M, N_))
    A, B, C = D.upload(a), D.upload(b), D.upload(c0)
    w = ws(lib.hp_gemm_workspace_bytes(M, N_, K, 0, 0))
    N.check(lib.hp_gemm(0, 1, M, N_, K, A.vecset(), B.vecset(), -1.0, 0.5, C.ptr, C.ld, None, None, None, 0, 0,
                        w.data_ptr(), w.numel(), st()), "gemm")
    assert np.allclose(C.to_numpy(), 0.5 * c0 - a @ b, rtol=1e-12, atol=1e-11)


@pytest.mark.parametrize("ak,bk", [(1, 1), (0, 1), (0, 0), (1, 0)])
@pytest.mark.parametrize("M,N_,K", [(1, 1, 1), (130, 257, 37), (256, 128, 40_001), (517, 300, 16), (64, 700, 4098)])
def test_gemm_layouts_edges(ak, bk, M, N_, K):
    """Every operand layout of the GEMM engine (the TMA-staged kernel for 16-byte aligned
    operands): partial edge tiles in M and N, a partial last k tile (K % 16 != 0, staged with
    zero fill), split-K with the fixed-order reduction, and a pointer-table operand."""
    rng = np.random.default_rng(M * 31 + N_ * 7 + K + 1000 * ak + 100 * bk)
    a = rng.standard_normal((M, K))
    b = rng.standard_normal((K, N_))
    A = D.upload(np.asfortranarray(a.T) if ak else a)     # K-major: vectors m with contiguous k
    B = D.upload(b if bk else np.asfortranarray(b.T))     # K-major: vectors n with contiguous k
    ref = a @ b
    tol = 1e-13 * np.sqrt(K) * max(1.0, np.abs(ref).max())
    for table in (False, True):
        if table:
            # the same operands addressed through per-vector pointer tables (children's mode blocks)
            va, ta = D._concat_parts([D.Part(A.view_cols(0, A.cols // 2)), D.Part(A.view_cols(A.cols // 2, A.cols))])[::3]
            vb, tb = D._concat_parts([D.Part(B.view_cols(0, B.cols // 3)), D.Part(B.view_cols(B.cols // 3, B.cols))])[::3]
        else:
            va, vb = A.vecset(), B.vecset()
        C = D.DevMat.empty(M, N_)
        w = ws(lib.hp_gemm_workspace_bytes(M, N_, K, 0, 0))
        N.check(lib.hp_gemm(ak, bk, M, N_, K, va, vb, 1.0, 0.0, C.ptr, C.ld, None, None, None, 0, 0,
                            w.data_ptr(), w.numel(), st()), "gemm")
        err = np.abs(C.to_numpy() - ref).max()
        assert err <= tol, (table, err, tol)


@pytest.mark.parametrize("n", [1, 2, 5, 64, 65, 200, 512, 1000])
def test_syev_matches_eigh(n):
    rng = np.random.default_rng(n)
    q, _ = np.linalg.qr(rng.standard_normal((n, n)))
    lam = np.sort(rng.uniform(-1, 4, n))[::-1]
    g = (q * lam) @ q.T
    g = 0.5 * (g + g.T)
    G = D.upload(g)
    lam_d = torch.empty(n, dtype=torch.float64, device="cuda")
    V = D.DevMat.empty(n, n)
    w = ws(lib.hp_syev_workspace_bytes(n))
    sweeps = ctypes.c_int(0)
    N.check(lib.hp_syev(G.ptr, G.ld, n, lam_d.data_ptr(), V.ptr, V.ld, n, D.JACOBI_TOL_REL, D.JACOBI_TOL_ABS, 0.0, 0.0, 60, 1,
                        ctypes.byref(sweeps), None, w.data_ptr(), w.numel(), st()), "syev")
    ev = lam_d.cpu().numpy()
    ref = np.linalg.eigvalsh(g)[::-1]
    print("syev n", n, "sweeps", sweeps.value, "err", np.max(np.abs(ev - ref)))
    assert np.all(np.diff(ev) <= 0)
    assert np.allclose(ev, ref, rtol=0, atol=1e-13 * max(1, np.abs(ref).max()) * np.sqrt(n))
    v = V.to_numpy()
    assert np.max(np.abs(v.T @ v - np.eye(n))) < 1e-12 * np.sqrt(n)
    assert np.max(np.abs(g @ v - v * ev[None, :])) < 1e-12 * np.sqrt(n) * max(1, np.abs(ref).max())


def test_syev_graded_psd_gram():
    # a method-of-snapshots Gramian with a 1e-16 spread, as in SURVEY 0.2
    rng = np.random.default_rng(1)
    d, m = 3000, 300
    q1, _ = np.linalg.qr(rng.standard_normal((d, m)))
    q2, _ = np.linalg.qr(rng.standard_normal((m, m)))
    sig = 10.0 ** (-8 * np.arange(m) / (m - 1))
    s = (q1 * sig) @ q2.T
    g = s.T @ s
    g = 0.5 * (g + g.T)
    G = D.upload(g)
    lam_d = torch.empty(m, dtype=torch.float64, device="cuda")
    V = D.DevMat.empty(m, m)
    w = ws(lib.hp_syev_workspace_bytes(m))
    sweeps = ctypes.c_int(0)
    N.check(lib.hp_syev(G.ptr, G.ld, m, lam_d.data_ptr(), V.ptr, V.ld, m, D.JACOBI_TOL_REL, D.JACOBI_TOL_ABS, 0.0, 0.0, 60, 1,
                        ctypes.byref(sweeps), None, w.data_ptr(), w.numel(), st()), "syev")
    ev = lam_d.cpu().numpy()
    import scipy.linalg
    ref = scipy.linalg.eigh(g, eigvals_only=True)[::-1]
    keep = ref >= 4 * 2.0 ** -52 * ref[0] * m
    err = np.abs(ev[keep] - ref[keep]) / ref[0]
    print("graded: sweeps", sweeps.value, "max abs err / lam_max", err.max())
    assert err.max() < 1e-14
    v = V.to_numpy()
    print("graded: V orthogonality", np.max(np.abs(v.T @ v - np.eye(m))))
    assert np.max(np.abs(v.T @ v - np.eye(m))) < 1e-13


def _ref_truncate(lam, eps, cutoff, m):
    """pod.py:281-289 verbatim arithmetic: keep mask, sqrt, truncation_rank, np.sum tail."""
    from oracle.hapod_oracle import truncation_rank
    keep = lam >= cutoff * lam[0] * m
    lk = lam[keep]
    s = np.sqrt(lk)
    n = truncation_rank(s, eps)
    return int(keep.sum()), n, float(np.sum(lk[n:])), s


@pytest.mark.parametrize("seed", range(4))
def test_truncate_kernel_bitwise(seed):
    """K3 bit-for-bit against the reference's NumPy arithmetic: the count, N, every sigma and
    the tail energy (sequential reversed cumsum of sigma*sigma, pairwise np.sum) -- including
    budgets placed exactly on a tail value and one ulp either side of it."""
    rng = np.random.default_rng(900 + seed)
    cutoff = 4 * 2.0 ** -52
    for trial in range(30):
        n = int(rng.integers(1, 20000 if trial % 5 == 0 else 3000))
        lam = np.sort(rng.exponential(1.0, n) ** 4 * 10.0 ** rng.uniform(-12, 0, n))[::-1].copy()
        s = np.sqrt(lam[lam >= cutoff * lam[0] * n])
        tails = np.cumsum((s * s)[::-1])[::-1]
        k = int(rng.integers(0, s.size))
        base = float(np.sqrt(tails[k]))
        for eps in (float(rng.uniform(0, 1) * np.sqrt(lam.sum())), base, np.nextafter(base, 0.0),
                    np.nextafter(base, np.inf), 0.0):
            ld = torch.from_numpy(lam.copy()).cuda()
            sig = torch.empty(n, dtype=torch.float64, device="cuda")
            info = torch.empty(4, dtype=torch.float64, device="cuda")
            N.check(lib.hp_truncate(ld.data_ptr(), n, eps, cutoff, n, sig.data_ptr(), info.data_ptr(), st()),
                    "trunc")
            lam_max, nkeep, N_, tail = info.cpu().tolist()
            rk, rn, rtail, rs = _ref_truncate(lam, eps, cutoff, n)
            assert int(nkeep) == rk and int(N_) == rn, (trial, eps)
            assert tail == rtail, (trial, eps, tail, rtail)
            assert np.array_equal(sig.cpu().numpy()[:rk], rs)


def test_signs_and_reortho():
    rng = np.random.default_rng(2)
    d, n = 5000, 200
    # badly conditioned but full-rank columns -> drift > 1e-8
    q, _ = np.linalg.qr(rng.standard_normal((d, n)))
    u = q @ (np.eye(n) + 1e-5 * rng.standard_normal((n, n)))
    U = D.upload(u)
    C = D.DevMat.empty(n, n)
    drift = torch.zeros(1, dtype=torch.float64, device="cuda")
    w = ws(lib.hp_drift_workspace_bytes(d, n))
    N.check(lib.hp_drift(U.ptr, U.ld, d, n, C.ptr, C.ld, drift.data_ptr(), w.data_ptr(), w.numel(), st()), "drift")
    ref_drift = np.max(np.abs(u.T @ u - np.eye(n)))
    assert float(drift.item()) == pytest.approx(ref_drift, rel=1e-6)
    w = ws(lib.hp_reortho_workspace_bytes(d, n))
    passes = ctypes.c_int(0)
    N.check(lib.hp_reorthonormalize(U.ptr, U.ld, d, n, C.ptr, C.ld, float(drift.item()), ctypes.byref(passes),
                                    w.data_ptr(), w.numel(), st()), "reortho")
    assert passes.value == 1  # drift ~1e-4: one CholQR pass
    qq = U.to_numpy()
    assert np.max(np.abs(qq.T @ qq - np.eye(n))) < 1e-13
    # same Q as Gram-Schmidt (positive diagonal R)
    qr_q, r = np.linalg.qr(u)
    qr_q = qr_q * np.sign(np.diag(r))[None, :]
    assert np.max(np.abs(qq - qr_q)) < 1e-9
    N.check(lib.hp_signs(U.ptr, U.ld, d, n, None, 0, 0, None, st()), "signs")
    s = U.to_numpy()
    pick = np.argmax(np.abs(s), axis=0)
    assert np.all(s[pick, np.arange(n)] > 0)


@pytest.mark.parametrize("scale,graded", [(1e-1, True), (8e-2, False)])
def test_reortho_two_pass_and_shifted(scale, graded):
    rng = np.random.default_rng(4)
    d, n = 3000, 150
    q, _ = np.linalg.qr(rng.standard_normal((d, n)))
    # graded columns: kappa ~ 1e6 (scale 1e-1) .. forces CholQR2 / shifted CholQR3
    u = q @ (np.eye(n) + scale * rng.standard_normal((n, n))) * np.logspace(0, -6 * graded, n)[None, :]
    U = D.upload(u)
    C = D.DevMat.empty(n, n)
    drift = torch.zeros(1, dtype=torch.float64, device="cuda")
    w = ws(lib.hp_drift_workspace_bytes(d, n))
    N.check(lib.hp_drift(U.ptr, U.ld, d, n, C.ptr, C.ld, drift.data_ptr(), w.data_ptr(), w.numel(), st()), "drift")
    w = ws(lib.hp_reortho_workspace_bytes(d, n))
    passes = ctypes.c_int(0)
    N.check(lib.hp_reorthonormalize(U.ptr, U.ld, d, n, C.ptr, C.ld, float(drift.item()), ctypes.byref(passes),
                                    w.data_ptr(), w.numel(), st()), "reortho")
    qq = U.to_numpy()
    assert passes.value >= 2
    assert np.max(np.abs(qq.T @ qq - np.eye(n))) < 1e-12
    qr_q, r = np.linalg.qr(u)
    qr_q = qr_q * np.sign(np.diag(r))[None, :]
    # same span (Q unique up to rounding ~ u kappa)
    assert np.linalg.norm(qr_q - qq @ (qq.T @ qr_q)) < 1e-6


@pytest.mark.parametrize("n,cuts", [(300, [0, 128, 256, 320]), (200, [0, 64, 256]), (512, [0, 192, 192, 512]),
                                    (97, [0, 64, 128])])
def test_syev_rows_partition_is_bitwise_the_full_solve(n, cuts):
    """hp_syev_rows (one rank's share of a replicated eigensolve): eigenvalues, sweeps and every
    accumulated row of V are bit-identical to the full solve, whatever the row partition --
    including an empty share and shares without the padding rows."""
    rng = np.random.default_rng(n)
    q, _ = np.linalg.qr(rng.standard_normal((n, n)))
    lam = np.sort(10.0 ** rng.uniform(-9, 0, n))[::-1]
    g = (q * lam) @ q.T
    g = 0.5 * (g + g.T)
    G = D.upload(g)
    npad = int(lib.hp_syev_padded_order(n))
    assert cuts[-1] == npad

    def solve(a, b):
        lam_d = torch.empty(n, dtype=torch.float64, device="cuda")
        V = D.DevMat.empty(n, n)
        w = ws(lib.hp_syev_workspace_bytes(n))
        sweeps = ctypes.c_int(0)
        if a is None:
            N.check(lib.hp_syev(G.ptr, G.ld, n, lam_d.data_ptr(), V.ptr, V.ld, n, D.JACOBI_TOL_REL, D.JACOBI_TOL_ABS, 0.0,
                                0.0, 60, 0, ctypes.byref(sweeps), None, w.data_ptr(), w.numel(), st()), "syev")
        else:
            N.check(lib.hp_syev_rows(G.ptr, G.ld, n, lam_d.data_ptr(), V.ptr, V.ld, n, D.JACOBI_TOL_REL,
                                     D.JACOBI_TOL_ABS, 0.0, 0.0, 60, ctypes.byref(sweeps), None, a, b, w.data_ptr(),
                                     w.numel(), st()), "syev_rows")
        return lam_d.cpu().numpy(), V.to_numpy(), sweeps.value

    lam_full, v_full, sw_full = solve(None, None)
    merged = np.full_like(v_full, np.nan)
    for a, b in zip(cuts[:-1], cuts[1:]):
        lam_p, v_p, sw_p = solve(a, b)
        assert np.array_equal(lam_p, lam_full) and sw_p == sw_full
        merged[a:min(b, n)] = v_p[a:min(b, n)]
    assert np.array_equal(merged, v_full)
    assert np.max(np.abs(v_full.T @ v_full - np.eye(n))) < 1e-12 * np.sqrt(n)


def _tri_solve(g, floor_rel, relgap_min=1e-9):
    n = g.shape[0]
    G = D.upload(g)
    lam_d = torch.empty(n, dtype=torch.float64, device="cuda")
    W = D.DevMat.empty(n, n)
    w = ws(lib.hp_syev_tri_workspace_bytes(n))
    k = ctypes.c_int64(0)
    status = ctypes.c_int(1)
    diag = (ctypes.c_double * 8)()
    N.check(lib.hp_syev_tri(G.ptr, G.ld, n, floor_rel, relgap_min, lam_d.data_ptr(), W.ptr, W.ld, ctypes.byref(k),
                            ctypes.byref(status), diag, w.data_ptr(), w.numel(), st()), "syev_tri")
    torch.cuda.synchronize()
    return status.value, int(k.value), lam_d.cpu().numpy(), W.to_numpy(), list(diag)


@pytest.mark.parametrize("n,decades", [(2, 1), (3, 2), (65, 3), (130, 6), (517, 10), (1024, 12), (1500, 13)])
def test_syev_tri_graded_spectrum_vs_eigh(n, decades):
    """hp_syev_tri (tridiagonalisation + relative multisection + twisted factorisation, no
    re-orthogonalisation) on graded positive definite matrices -- the preconditioned Gramians
    H = L^T L of a node POD (eigh at pod.py:329): eigenvalues to u * lambda_max, numerically
    orthogonal eigenvectors, small residuals; odd / even orders, partial last panels."""
    rng = np.random.default_rng(n)
    q, _ = np.linalg.qr(rng.standard_normal((n, n)))
    lam = 10.0 ** (-decades * np.arange(n) / max(n - 1, 1))
    g = (q * lam) @ q.T
    g = 0.5 * (g + g.T)
    floor_rel = 10.0 ** (-decades - 0.5)
    status, k, ev, w, diag = _tri_solve(g, floor_rel)
    ref = np.linalg.eigvalsh(g)[::-1]
    print(f"syev_tri n={n}: status {status} K {k} min relgap {diag[0]:.2e} max resid {diag[1]:.2e}")
    assert status == 0
    assert k == int((ref >= floor_rel * ref[0]).sum()) == n
    assert np.max(np.abs(ev[:k] - ref[:k])) <= 64 * 2.0 ** -52 * ref[0] * max(1.0, np.sqrt(n) / 8)
    assert np.all(ev[k:] == 0.0)
    wk = w[:, :k]
    orth = np.max(np.abs(wk.T @ wk - np.eye(k)))
    res = np.max(np.abs(g @ wk - wk * ev[None, :k])) / ref[0]
    print(f"   |ev - ref| / lam_max {np.max(np.abs(ev[:k] - ref[:k])) / ref[0]:.2e} orth {orth:.2e} resid {res:.2e}")
    assert orth <= 1e-10
    assert res <= 1e-13 * max(1.0, np.sqrt(n) / 4)


def test_syev_tri_floor_selects_leading_pairs():
    rng = np.random.default_rng(7)
    n = 700
    q, _ = np.linalg.qr(rng.standard_normal((n, n)))
    lam = 10.0 ** (-15 * np.arange(n) / (n - 1))
    g = (q * lam) @ q.T
    g = 0.5 * (g + g.T)
    status, k, ev, w, diag = _tri_solve(g, 1e-9)
    ref = np.linalg.eigvalsh(g)[::-1]
    assert status == 0
    kref = int((ref >= 1e-9 * ref[0]).sum())
    assert abs(k - kref) <= 1
    assert np.max(np.abs(ev[:k] - ref[:k])) <= 1e-13 * ref[0]
    wk = w[:, :k]
    assert np.max(np.abs(wk.T @ wk - np.eye(k))) <= 1e-10
    # the computed vectors span the leading invariant subspace
    vref = np.linalg.eigh(g)[1][:, ::-1][:, : k - 5]
    assert np.linalg.norm(vref - wk @ (wk.T @ vref), 2) <= 1e-6


def test_syev_tri_declines_clusters():
    """A spectrum with (numerically) multiple eigenvalues cannot be resolved without
    re-orthogonalisation: the solver must decline (status 1) so that the caller runs hp_syev."""
    n = 300
    rng = np.random.default_rng(3)
    q, _ = np.linalg.qr(rng.standard_normal((n, n)))
    lam = np.concatenate([np.full(n // 2, 2.0), np.full(n - n // 2, 1.0)])
    g = (q * lam) @ q.T
    g = 0.5 * (g + g.T)
    status, k, ev, w, diag = _tri_solve(g, 1e-12)
    print("clustered: status", status, "min relgap", diag[0])
    assert status == 1
    status, *_ = _tri_solve(np.eye(n), 1e-12)
    assert status == 1


def test_syev_tri_order_4200():
    """A root-sized order (trailing matrix larger than the L2 at the start): eigenvalues, residuals
    and orthogonality as for the small orders."""
    test_syev_tri_graded_spectrum_vs_eigh(4200, 11)
