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
  3. Gram      G = sum_s S_s^T D S_s D over EIGHT FIXED ROW SHARDS s (independent of the
               rank count): one SYRK per shard, the eight partials added in one fixed
               binary tree ((0+1)+(2+3))+((4+5)+(6+7)); a sum whose operands live on two
               ranks moves the right operand to the left one (send/recv), so every
               rounding is the same at 1, 2, 4 or 8 ranks.
  4. eigen     rank 0 runs the node eigensolve + truncation (pod.py:329-331, 278-289) and
               broadcasts (lambda_max, nkeep, N, tail), sigma and the N kept eigenvectors.
  5. modes     U_s = S_s D V / sigma per shard (pod.py:333-334).
  6. drift     C = sum_s U_s^T U_s (the same fixed tree, then broadcast), drift = max|C - I|
               (pod.py:245-247); above
               1e-8 one CholQR pass U_q <- U_q L^-T with L L^T = C computed identically on
               every rank (a second pass when the drift exceeds 1e-1) -- the span of the MGS
               sweep of pod.py:227-237.
  7. signs     per column the largest |u| over ALL rows, first global index on ties
               (pod.py:214-224): local candidates all_gathered, the winner's sign all_reduced.

The protocol is written against torch.distributed and an "arith" object that provides the
node arithmetic on one row block: ``DeviceRowArith`` (the sm_100a kernels of
libhapod_b200.so, NCCL) here, a NumPy restatement in the CPU tests (gloo).  Every GEMM
runs on one fixed shard (its split-K plan depends only on the shard's shape) and every sum
over shards follows the fixed tree, so the root's modes are bitwise identical for any rank
count dividing the shard set; they differ from the single-GPU run_hapod root only by the
summation order of the Gram over rows (rounding level).
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass

import numpy as np

DRIFT_TOL = 1e-8          # pod.py:247
SINGLE_PASS_DRIFT = 1e-1  # one CholQR pass is orthonormal to the rounding level below this drift


NSHARDS = 8  # fixed row shards of a distributed root: the reduction order never depends on N


def row_bounds(d: int, nshards: int = NSHARDS, align: int = 16) -> list:
    """Shard boundaries b_0 = 0 < ... < b_nshards = d, interior boundaries multiples of
    ``align`` (16-byte aligned column slices for the TMA GEMM)."""
    out = [0]
    for q in range(1, nshards):
        b = (d * q // nshards) // align * align
        out.append(max(out[-1], min(b, d)))
    out.append(d)
    return out


def shard_owner(world: int, nshards: int = NSHARDS) -> list:
    """shard -> rank: contiguous chunks (rank q owns shards [q n / w, (q+1) n / w))."""
    if not 1 <= world <= nshards:
        raise ValueError(f"the row-distributed root needs 1..{nshards} ranks, got {world}")
    return [(s * world) // nshards for s in range(nshards)]


def rank_bounds(shards: list, world: int) -> list:
    """Row block of every rank: the union of its shards (contiguous)."""
    own = shard_owner(world, len(shards) - 1)
    out = [0] * (world + 1)
    for q in range(world):
        mine = [s for s in range(len(own)) if own[s] == q]
        out[q] = shards[mine[0]] if mine else shards[-1]
    out[world] = shards[-1]
    for q in range(world - 1, -1, -1):  # ranks without shards: empty block at the next start
        out[q] = min(out[q], out[q + 1])
    return out


def tree_reduce(partial, owner: list, rank: int, arith, group=None, lo: int = 0, hi: int | None = None):
    """Sum of the per-shard partials over shards [lo, hi) in the FIXED binary tree
    (left + right at every level), held by the owner of shard lo; None on other ranks.
    ``partial(s)`` computes shard s's term (called on its owner only).  A level whose
    operands sit on two ranks sends the right operand to the left owner (NCCL / gloo p2p);
    at most log2(NSHARDS) + 1 partials are alive on a rank."""
    import torch.distributed as dist
    hi = len(owner) if hi is None else hi
    if hi - lo == 1:
        return partial(lo) if owner[lo] == rank else None
    mid = (lo + hi) // 2
    left = tree_reduce(partial, owner, rank, arith, group, lo, mid)
    right = tree_reduce(partial, owner, rank, arith, group, mid, hi)
    a, b = owner[lo], owner[mid]
    if a == b:
        return arith.add(left, right) if rank == a else None
    if rank == b:
        dist.send(arith.flat(right), a, group=group)
        return None
    if rank == a:
        buf = arith.like(left)
        dist.recv(arith.flat(buf), b, group=group)
        return arith.add(left, buf)
    return None


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


def row_root_pod(S_q, layout: RootLayout, shards: list, eps: float, cutoff: float, rank: int, world: int, arith,
                 group=None, split_eig: bool = True) -> RowRootResult:
    """Steps 3-7 on this rank's row block S_q (rows bounds[rank]..bounds[rank+1] of the root
    input); ``shards``: the fixed shard boundaries (row_bounds)."""
    import torch
    import torch.distributed as dist
    m = layout.m
    owner = shard_owner(world, len(shards) - 1)
    bounds = rank_bounds(shards, world)
    r0, r1 = bounds[rank], bounds[rank + 1]
    mine = [s for s in range(len(owner)) if owner[s] == rank]

    def local(s):  # shard s as local row range of this rank's block
        return shards[s] - r0, shards[s + 1] - r0

    scale = arith.vector(layout.scale)
    # 3. Gram: per-shard SYRK, fixed-tree sum on rank 0
    G = tree_reduce(lambda s: arith.gram_rows(S_q, *local(s), scale, m), owner, rank, arith, group)
    # 4. eigensolve.  split_eig (default for world > 1): the Gram is broadcast and the eigensolve is
    #    REPLICATED -- every rank runs the same deterministic iteration and accumulates only its own
    #    row slabs of the eigenvector matrix, all-gathered at the end (_device.EigShare; no traffic
    #    inside the iteration); otherwise rank 0 solves alone and broadcasts (lambda_max, nkeep, N,
    #    tail), sigma and the N kept eigenvectors.
    if split_eig and world > 1:
        if rank != 0:
            G = arith.empty(m, m)
        dist.broadcast(arith.flat(G), 0, group=group)
        lam_max, nkeep, n_modes, tail, V, sig = arith.eig(G, m, eps, cutoff, share=(rank, world, group))
        del G
        nkeep, n_modes = int(nkeep), int(n_modes)
        if not (lam_max > 0.0) or n_modes == 0:
            return RowRootResult(arith.empty(r1 - r0, 0), np.zeros(0), tail if lam_max > 0.0 else 0.0, lam_max,
                                 nkeep if lam_max > 0.0 else 0, 0.0, False, bounds, m)
    else:
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
    # 5. modes of this row block, shard by shard
    U = arith.empty_rowblock(r1 - r0, n_modes)
    Vs = arith.scale_rows(V, scale)
    del V
    for s in mine:
        arith.assemble_rows(S_q, *local(s), Vs, sig, U)
    del Vs

    # 6. drift and CholQR on the global Gram of the modes (fixed-tree sum, broadcast)
    def mode_gram(X):
        C = tree_reduce(lambda s: arith.syrk_rows(X, *local(s)), owner, rank, arith, group)
        if rank != 0:
            C = arith.empty(n_modes, n_modes)
        dist.broadcast(arith.flat(C), 0, group=group)
        return C

    C = mode_gram(U)
    drift = arith.drift(C)
    reorthed = False
    if drift > DRIFT_TOL:
        passes = 2 if drift > SINGLE_PASS_DRIFT else 1
        for k in range(passes):
            Linv = arith.chol_inverse(C)
            Y = arith.empty_rowblock(r1 - r0, n_modes)
            for s in mine:
                arith.trmm_rows(U, *local(s), Linv, Y)
            U = Y
            if k + 1 < passes:
                C = mode_gram(U)
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
    mine_cols = np.where(win_rank == rank)[0]
    local_sign = np.zeros(n_modes)
    if mine_cols.size:
        local_sign[mine_cols] = arith.entry_signs(U, hi[rank, mine_cols] - r0, mine_cols)
    sgn = arith.vector(local_sign)
    dist.all_reduce(sgn, group=group)  # exactly one nonzero (+-1) term per column
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

    def like(self, M):
        return self.D.DevMat(self.torch.empty_like(M.storage), M.rows, M.cols, M.ld, M.offset)

    def rows_view(self, M, a, b):
        return self.D.DevMat(M.storage, b - a, M.cols, M.ld, M.offset + a)

    # -- arithmetic
    def add(self, A, B):
        """A <- A + B elementwise (the fixed-tree shard sum)."""
        n = A.ld * A.cols
        if n:
            self.N.check(self.lib.hp_add(A.ptr, B.ptr, n, self.D._stream()), "partial sum")
        return A

    def gram_rows(self, S, a, b, scale, m):
        if b <= a:
            return self.D.DevMat.empty(m, m, zero=True)
        G, _, _ = self.D.gram_full([self.D.Part(self.rows_view(S, a, b), scale)], b - a)
        return G

    def eig(self, G, m, eps, cutoff, share=None):
        """``share`` = (rank, world, group): the eigensolve is replicated on every rank and each
        accumulates its own row slabs of the H-phase eigenvector matrix (_device.EigShare)."""
        sh = self.D.EigShare(*share) if share is not None else None
        ev = self.D.eig_vectors(G, m, eps, cutoff, sh)
        if not (ev.lam_max > 0.0) or ev.n_modes == 0:
            return ev.lam_max, ev.nkeep, ev.n_modes, ev.tail, None, None
        V = self.empty(m, ev.n_modes)
        self._copy(ev.Vn, 0, m, V, 0, 0)
        return ev.lam_max, ev.nkeep, ev.n_modes, ev.tail, V, ev.sig_dev.contiguous()

    def scale_rows(self, V, scale):
        m, n = V.rows, V.cols
        Vs = self.empty(m, n)
        self.N.check(self.lib.hp_scale(V.ptr, V.ld, m, n, scale.data_ptr(), None, None, Vs.ptr, Vs.ld,
                                       self.D._stream()), "scale V")
        return Vs

    def assemble_rows(self, S, a, b, Vs, sig, U):
        """rows [a, b) of U <- rows [a, b) of S times Vs / sigma (pod.py:333-334)."""
        if b <= a:
            return
        m, n = Vs.rows, Vs.cols
        Sv, Uv = self.rows_view(S, a, b), self.rows_view(U, a, b)
        ws = self.D._ws(self.lib.hp_assemble_workspace_bytes(b - a, m, n))
        with self.D._phase("assemble", 2.0 * (b - a) * m * n):
            self.N.check(self.lib.hp_assemble(Sv.vecset(), b - a, m, Vs.ptr, Vs.ld, sig.data_ptr(), n, Uv.ptr, Uv.ld,
                                              ws.data_ptr(), ws.numel(), self.D._stream()), "assemble")

    def syrk_rows(self, U, a, b):
        n = U.cols
        if b <= a:
            return self.D.DevMat.empty(n, n, zero=True)
        C = self.empty(n, n)
        Uv = self.rows_view(U, a, b)
        ws = self.D._ws(self.lib.hp_gram_workspace_bytes(b - a, n))
        with self.D._phase("drift", float(b - a) * n * (n + 1)):
            self.N.check(self.lib.hp_gram(Uv.vecset(), b - a, n, None, C.ptr, C.ld, ws.data_ptr(), ws.numel(),
                                          self.D._stream()), "U^T U")
        return C

    def drift(self, C):
        out = self.torch.zeros(1, dtype=self.torch.float64, device="cuda")
        self.N.check(self.lib.hp_gram_drift(C.ptr, C.ld, C.rows, out.data_ptr(), self.D._stream()), "drift")
        return float(self.D.host_read(out)[0])

    def chol_inverse(self, C):
        """L^{-1} for C = L L^T (identical on every rank: same input, same kernels)."""
        n = C.cols
        Cw = self.D.DevMat(C.storage.clone(), n, n, C.ld, C.offset)
        Linv = self.empty(n, n)
        ws = self.D._ws(self.lib.hp_chol_inverse_workspace_bytes(n))
        info = ctypes.c_int(0)
        self.N.check(self.lib.hp_chol_inverse(Cw.ptr, Cw.ld, n, Linv.ptr, Linv.ld, ctypes.byref(info), ws.data_ptr(),
                                              ws.numel(), self.D._stream()), "CholQR factor")
        if info.value != 0:
            raise np.linalg.LinAlgError("row-distributed CholQR: the modes' Gram is not positive definite")
        return Linv

    def trmm_rows(self, U, a, b, Linv, Y):
        """rows [a, b) of Y <- rows [a, b) of U times L^{-T} (upper triangular operand)."""
        if b <= a:
            return
        n = U.cols
        Uv, Yv = self.rows_view(U, a, b), self.rows_view(Y, a, b)
        gws = self.D._ws(self.lib.hp_gemm_workspace_bytes(b - a, n, n, 0, 1))
        with self.D._phase("reortho", float(b - a) * n * n):
            self.N.check(self.lib.hp_gemm(0, 0, b - a, n, n, Uv.vecset(), Linv.vecset(), 1.0, 0.0, Yv.ptr, Yv.ld,
                                          None, None, None, 0, 1, gws.data_ptr(), gws.numel(), self.D._stream()),
                         "U L^-T")

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
