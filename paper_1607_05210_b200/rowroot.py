"""Row-distributed root node: the multi-GPU root of a star-like tree.

A root whose input does not fit one GPU (config 3: 64 children x 2,000,000 x ~299 fp64 =
306 GB) -- or whose Gram / reconstruction should run on every GPU (config 1 at N > 1) -- is
evaluated with its input split by ROWS instead of gathered on rank 0:

  1. layout    every rank learns each child's column count and sigma (all_gather of a few
               KB); the root's columns are the children's modes in child-list order
               (hierarchy.py:284-291) scaled by sigma (pod.py:160-162).
  2. exchange  grouped point-to-point (NCCL send/recv): rank p sends rows [b_q, b_{q+1}) of
               every child block it owns to rank q, which lands them in its row block S_q
               (rows_q x m, column-major) -- an all-to-all of the sigma-scaled mode blocks.
  3. Gram      G = sum_q S_q^T D S_q D: each rank's partial SYRK, all_reduce (sum).
  4. eigen     rank 0 runs the node eigensolve + truncation (pod.py:329-331, 278-289) and
               broadcasts (lambda_max, nkeep, N, tail), sigma and the N kept eigenvectors.
  5. modes     U_q = S_q D V / sigma on every rank (pod.py:333-334).
  6. drift     C = sum_q U_q^T U_q (all_reduce), drift = max|C - I| (pod.py:245-247); above
               1e-8 one CholQR pass U_q <- U_q L^-T with L L^T = C computed identically on
               every rank (a second pass when the drift exceeds 1e-1) -- the span of the MGS
               sweep of pod.py:227-237.
  7. signs     per column the largest |u| over ALL rows, first global index on ties
               (pod.py:214-224): local candidates all_gathered, the winner's sign all_reduced.

The protocol is written against torch.distributed and an "arith" object that provides the
node arithmetic on one row block: ``DeviceRowArith`` (the sm_100a kernels of
libhapod_b200.so, NCCL) here, a NumPy restatement in the CPU tests (gloo).  Results are
deterministic for a given world size; they differ from the single-GPU root only by the
summation order of the Gram over rows (rounding level).
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass

import numpy as np

DRIFT_TOL = 1e-8          # pod.py:247
SINGLE_PASS_DRIFT = 1e-1  # one CholQR pass is orthonormal to the rounding level below this drift


def row_bounds(d: int, world: int, align: int = 16) -> list:
    """Row block boundaries b_0 = 0 < ... < b_world = d, interior boundaries multiples of
    ``align`` (16-byte aligned column slices for the TMA GEMM)."""
    out = [0]
    for q in range(1, world):
        b = (d * q // world) // align * align
        out.append(max(out[-1], min(b, d)))
    out.append(d)
    return out


@dataclass
class RootLayout:
    order: list          # [(child id, part index)] in child-list order
    owner: dict          # (child, part) -> rank
    cols: dict           # (child, part) -> column count
    offset: dict         # (child, part) -> first root column
    scale: np.ndarray    # m: sigma-scale of every root column (1 for passthrough columns)
    m: int


def gather_layout(children: list, local: dict, rank: int, world: int, group=None) -> RootLayout:
    """``local``: child id -> list of (matrix, scale ndarray or None) parts held on this rank."""
    import torch.distributed as dist
    mine = {c: [(arith_cols(mat), None if sc is None else np.asarray(sc, dtype=np.float64)) for mat, sc in parts]
            for c, parts in local.items()}
    everyone = [None] * world
    dist.all_gather_object(everyone, (rank, mine), group=group)
    owner, cols, scales = {}, {}, {}
    for r, info in everyone:
        for c, parts in info.items():
            for k, (n, s) in enumerate(parts):
                owner[(c, k)] = r
                cols[(c, k)] = n
                scales[(c, k)] = s
    order, offset, at, scale = [], {}, 0, []
    for c in children:
        k = 0
        while (c, k) in owner:
            order.append((c, k))
            offset[(c, k)] = at
            n = cols[(c, k)]
            scale.append(np.ones(n) if scales[(c, k)] is None else scales[(c, k)])
            at += n
            k += 1
    return RootLayout(order, owner, cols, offset, np.concatenate(scale) if scale else np.zeros(0), at)


def arith_cols(mat) -> int:
    return int(mat.cols) if hasattr(mat, "cols") else int(mat.shape[1])


def exchange_rows(layout: RootLayout, local: dict, bounds: list, rank: int, world: int, arith, group=None):
    """All-to-all of the children's row slices: returns this rank's row block S_q."""
    import torch.distributed as dist
    r0, r1 = bounds[rank], bounds[rank + 1]
    S = arith.empty_rowblock(r1 - r0, layout.m)
    ops, keep = [], []
    for (c, k) in layout.order:
        p = layout.owner[(c, k)]
        off, n = layout.offset[(c, k)], layout.cols[(c, k)]
        if n == 0:
            continue
        if p == rank:
            mat = local[c][k][0]
            for q in range(world):
                q0, q1 = bounds[q], bounds[q + 1]
                if q1 <= q0:
                    continue
                if q == rank:
                    arith.copy_rows(mat, q0, q1, S, off)
                else:
                    buf = arith.row_slice(mat, q0, q1)
                    keep.append(buf)
                    ops.append(dist.P2POp(dist.isend, arith.flat(buf), q, group=group))
        elif r1 > r0:
            ops.append(dist.P2POp(dist.irecv, arith.cols_view(S, off, n), p, group=group))
    if ops:
        for w in dist.batch_isend_irecv(ops):
            w.wait()
    arith.sync()
    del keep
    return S


@dataclass
class RowRootResult:
    U_rows: object        # this rank's row block of the root modes (rows_q x N)
    sigmas: np.ndarray
    tail: float
    lam_max: float
    nkeep: int
    drift: float
    reorthed: bool
    bounds: list
    m: int


def row_root_pod(S_q, layout: RootLayout, bounds: list, eps: float, cutoff: float, rank: int, world: int, arith,
                 group=None) -> RowRootResult:
    import torch
    import torch.distributed as dist
    m = layout.m
    r0, r1 = bounds[rank], bounds[rank + 1]
    scale = arith.vector(layout.scale)
    # 3. Gram
    G = arith.gram(S_q, scale)
    dist.all_reduce(arith.flat(G), group=group)
    # 4. eigen on rank 0, broadcast
    info = arith.vector(np.zeros(4))
    if rank == 0:
        lam_max, nkeep, n_modes, tail, V, sig = arith.eig(G, m, eps, cutoff)
        info = arith.vector(np.array([lam_max, nkeep, n_modes, tail], dtype=np.float64))
    del G
    dist.broadcast(info, 0, group=group)
    lam_max, nkeep, n_modes, tail = (float(x) for x in arith.to_host(info))
    nkeep, n_modes = int(nkeep), int(n_modes)
    if not (lam_max > 0.0) or n_modes == 0:
        return RowRootResult(arith.empty(r1 - r0, 0), np.zeros(0), tail if lam_max > 0.0 else 0.0, lam_max,
                             nkeep if lam_max > 0.0 else 0, 0.0, False, bounds, m)
    if rank != 0:
        V = arith.empty(m, n_modes)
        sig = arith.vector(np.zeros(n_modes))
    dist.broadcast(arith.flat(V), 0, group=group)
    dist.broadcast(sig, 0, group=group)
    # 5. modes of this row block
    U = arith.assemble(S_q, scale, V, sig)
    del V
    # 6. drift and CholQR on the global Gram of the modes
    C = arith.syrk(U)
    dist.all_reduce(arith.flat(C), group=group)
    drift = arith.drift(C)
    reorthed = False
    if drift > DRIFT_TOL:
        U = arith.cholqr_apply(U, C)
        if drift > SINGLE_PASS_DRIFT:
            C = arith.syrk(U)
            dist.all_reduce(arith.flat(C), group=group)
            U = arith.cholqr_apply(U, C)
        reorthed = True
    # 7. signs: global first-index argmax of |u| per column
    vals, idx = arith.col_absmax(U, r0)
    allv = [torch.zeros_like(vals) for _ in range(world)]
    alli = [torch.zeros_like(idx) for _ in range(world)]
    dist.all_gather(allv, vals, group=group)
    dist.all_gather(alli, idx, group=group)
    hv = np.stack([arith.to_host(v) for v in allv])
    hi = np.stack([arith.to_host(i) for i in alli]).astype(np.int64)
    hv = np.where(hi < 0, -1.0, hv)
    win_rank = np.zeros(n_modes, dtype=np.int64)
    for j in range(n_modes):
        best = (-2.0, 1 << 62, -1)
        for q in range(world):
            v, i = hv[q, j], hi[q, j]
            if v > best[0] or (v == best[0] and i < best[1]):
                best = (v, i, q)
        win_rank[j] = best[2]
    mine = np.where(win_rank == rank)[0]
    local_sign = np.zeros(n_modes)
    if mine.size:
        local_sign[mine] = arith.entry_signs(U, hi[rank, mine] - r0, mine)
    sgn = arith.vector(local_sign)
    dist.all_reduce(sgn, group=group)
    s = arith.to_host(sgn)
    s = np.where(s < 0.0, -1.0, 1.0)
    U = arith.flip(U, arith.vector(s))
    return RowRootResult(U, np.asarray(arith.to_host(sig), dtype=np.float64), tail, lam_max, nkeep, drift,
                         reorthed, bounds, m)


def gather_rows(res: RowRootResult, d: int, rank: int, world: int, arith, group=None):
    """The root modes assembled on rank 0 (d x N); None on the other ranks."""
    import torch.distributed as dist
    n = int(res.sigmas.size)
    if rank != 0:
        if n and res.bounds[rank + 1] > res.bounds[rank]:
            dist.send(arith.flat(arith.compact(res.U_rows)), 0, group=group)
        return None
    full = arith.empty(d, n)
    if n:
        arith.copy_rows_into(res.U_rows, full, res.bounds[0])
        for q in range(1, world):
            q0, q1 = res.bounds[q], res.bounds[q + 1]
            if q1 > q0:
                buf = arith.empty_compact(q1 - q0, n)
                dist.recv(arith.flat(buf), q, group=group)
                arith.copy_rows_into(buf, full, q0)
    return full


# ------------------------------------------------------------------------------------ device
class DeviceRowArith:
    """The row-block arithmetic on the B200: libhapod_b200.so kernels (DMMA TMA GEMMs, the
    pivoted-Cholesky / block-Jacobi eigensolver, CholQR, sign argmax).  Matrices are DevMat;
    collectives see their storage tensors (NCCL)."""

    def __init__(self):
        from . import _device as D
        from . import _native as N
        self.D, self.N = D, N
        self.lib = N.load()
        self.torch = D.torch

    # -- storage helpers
    def empty(self, rows, cols):
        return self.D.DevMat.empty(rows, cols)

    def empty_rowblock(self, rows, cols):
        # row blocks receive children's slices in place: compact columns (ld == rows, rows even)
        if rows % 2:
            raise ValueError("the row-distributed root needs an even row count per rank (even d)")
        st = self.torch.empty(max(rows * cols, 1), dtype=self.torch.float64, device="cuda")
        return self.D.DevMat(st, rows, cols, max(rows, 2))

    def empty_compact(self, rows, cols):
        st = self.torch.empty(max(rows * cols, 1), dtype=self.torch.float64, device="cuda")
        return self.D.DevMat(st, rows, cols, max(rows, 1))

    def compact(self, M):
        if M.ld == M.rows:
            return M
        out = self.empty_compact(M.rows, M.cols)
        self._copy(M, 0, M.rows, out, 0, 0)
        return out

    def flat(self, M):
        if hasattr(M, "storage"):
            return M.storage[M.offset: M.offset + M.ld * M.cols] if M.cols else M.storage[:0]
        return M

    def cols_view(self, M, off, n):
        # receive target: rows_q x n contiguous iff ld == rows (row blocks are allocated compact)
        assert M.ld == M.rows or M.rows == 0, "row block must be compact to receive in place"
        return M.storage[M.offset + off * M.ld: M.offset + (off + n) * M.ld]

    def vector(self, a):
        return self.torch.from_numpy(np.ascontiguousarray(a, dtype=np.float64)).to("cuda")

    def to_host(self, t):
        return t.cpu().numpy()

    def sync(self):
        self.torch.cuda.current_stream().synchronize()

    def _copy(self, src, r0, r1, dst, dr0, dc0):
        rows, cols = r1 - r0, src.cols
        if rows and cols:
            self.N.check(self.lib.hp_scale(src.ptr + 8 * r0, src.ld, rows, cols, None, None, None,
                                           dst.ptr + 8 * (dc0 * dst.ld + dr0), dst.ld, self.D._stream()), "row copy")

    def row_slice(self, mat, q0, q1):
        out = self.empty_compact(q1 - q0, mat.cols)
        self._copy(mat, q0, q1, out, 0, 0)
        return out

    def copy_rows(self, mat, q0, q1, S, off):
        self._copy(mat, q0, q1, S, 0, off)

    def copy_rows_into(self, block, full, r0):
        self._copy(block, 0, block.rows, full, r0, 0)

    # -- arithmetic
    def gram(self, S, scale):
        G, _, _ = self.D.gram_full([self.D.Part(S, scale)], S.rows)
        return G

    def eig(self, G, m, eps, cutoff):
        ev = self.D.eig_vectors(G, m, eps, cutoff)
        if not (ev.lam_max > 0.0) or ev.n_modes == 0:
            return ev.lam_max, ev.nkeep, ev.n_modes, ev.tail, None, None
        V = self.empty(m, ev.n_modes)
        self._copy(ev.Vn, 0, m, V, 0, 0)
        return ev.lam_max, ev.nkeep, ev.n_modes, ev.tail, V, ev.sig_dev.contiguous()

    def assemble(self, S, scale, V, sig):
        m, n = V.rows, V.cols
        Vs = self.empty(m, n)
        st = self.D._stream()
        self.N.check(self.lib.hp_scale(V.ptr, V.ld, m, n, scale.data_ptr(), None, None, Vs.ptr, Vs.ld, st), "scale V")
        U = self.empty(S.rows, n)
        if S.rows:
            ws = self.D._ws(self.lib.hp_assemble_workspace_bytes(S.rows, m, n))
            with self.D._phase("assemble", 2.0 * S.rows * m * n):
                self.N.check(self.lib.hp_assemble(S.vecset(), S.rows, m, Vs.ptr, Vs.ld, sig.data_ptr(), n, U.ptr, U.ld,
                                                  ws.data_ptr(), ws.numel(), st), "assemble")
        return U

    def syrk(self, U):
        n = U.cols
        C = self.empty(n, n)
        if U.rows:
            ws = self.D._ws(self.lib.hp_gram_workspace_bytes(U.rows, n))
            with self.D._phase("drift", float(U.rows) * n * (n + 1)):
                self.N.check(self.lib.hp_gram(U.vecset(), U.rows, n, None, C.ptr, C.ld, ws.data_ptr(), ws.numel(),
                                              self.D._stream()), "U^T U")
        else:
            C.storage.zero_()
        return C

    def drift(self, C):
        out = self.torch.zeros(1, dtype=self.torch.float64, device="cuda")
        self.N.check(self.lib.hp_gram_drift(C.ptr, C.ld, C.rows, out.data_ptr(), self.D._stream()), "drift")
        return float(out.item())

    def cholqr_apply(self, U, C):
        n = U.cols
        Cw = self.D.DevMat(C.storage.clone(), n, n, C.ld)
        Linv = self.empty(n, n)
        ws = self.D._ws(self.lib.hp_chol_inverse_workspace_bytes(n))
        info = ctypes.c_int(0)
        self.N.check(self.lib.hp_chol_inverse(Cw.ptr, Cw.ld, n, Linv.ptr, Linv.ld, ctypes.byref(info), ws.data_ptr(),
                                              ws.numel(), self.D._stream()), "CholQR factor")
        if info.value != 0:
            raise np.linalg.LinAlgError("row-distributed CholQR: the modes' Gram is not positive definite")
        Y = self.empty(U.rows, n)
        if U.rows:
            gws = self.D._ws(self.lib.hp_gemm_workspace_bytes(U.rows, n, n, 0, 1))
            with self.D._phase("reortho", float(U.rows) * n * n):
                self.N.check(self.lib.hp_gemm(0, 0, U.rows, n, n, U.vecset(), Linv.vecset(), 1.0, 0.0, Y.ptr, Y.ld,
                                              None, None, None, 0, 1, gws.data_ptr(), gws.numel(), self.D._stream()),
                             "U L^-T")
        return Y

    def col_absmax(self, U, row_offset):
        n = U.cols
        vals = self.torch.empty(max(n, 1), dtype=self.torch.float64, device="cuda")[:n]
        idx = self.torch.empty(max(n, 1), dtype=self.torch.int64, device="cuda")[:n]
        if U.rows == 0:
            vals.fill_(-1.0)
            idx.fill_(-1)
        elif n:
            self.N.check(self.lib.hp_col_absmax(U.ptr, U.ld, U.rows, n, row_offset, vals.data_ptr(), idx.data_ptr(),
                                                self.D._stream()), "column argmax")
        return vals, idx

    def entry_signs(self, U, rows, cols):
        t = U.tensor()
        r = self.torch.from_numpy(np.asarray(rows, dtype=np.int64)).cuda()
        c = self.torch.from_numpy(np.asarray(cols, dtype=np.int64)).cuda()
        v = t[r, c].cpu().numpy()
        return np.where(v < 0.0, -1.0, 1.0)

    def flip(self, U, s):
        if U.rows and U.cols:
            self.N.check(self.lib.hp_scale(U.ptr, U.ld, U.rows, U.cols, None, None, s.data_ptr(), U.ptr, U.ld,
                                           self.D._stream()), "signs")
        return U
