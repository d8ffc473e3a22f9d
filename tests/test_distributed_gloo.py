"""The multi-rank HAPOD protocol (placement, post-order evaluation, child ->
parent payloads over point-to-point send/recv) on CPU with the gloo backend,
world size 2 and 3, the CPU oracle standing in for the node arithmetic.  The
distributed result must be bit-identical to the single-process oracle run."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import paper_1607_05210_b200 as H
from paper_1607_05210_b200 import distributed as DI
from oracle import hapod_oracle as O
from oracle.dist_evaluator import OracleEvaluator


def _case(kind):
    if kind == "star":
        tree = H.build_star(6)
    elif kind == "chain":
        tree = H.build_chain(5)
    else:
        tree = H.build_balanced(9, 2)
    maps = H.derive_maps(tree)
    data = O.synthetic_decay(40, 18 * len(maps.leaves), 0.08, seed=3)
    blocks = {leaf: data[:, 18 * i: 18 * (i + 1)] for i, leaf in enumerate(maps.leaf_order)}
    counts = {leaf: 18 for leaf in maps.leaf_order}
    eps = O.assign_tolerances([list(c) for c in tree.children], tree.root, counts, 1e-2, 0.75,
                              zero_leaf_tolerance=(kind == "chain"))
    return tree, blocks, eps


def _worker(rank, world, port, kind, out_q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        tree, blocks, eps = _case(kind)
        ev = OracleEvaluator([list(c) for c in tree.children], blocks, eps)
        root, reports, stats = DI.run_distributed(tree, ev, rank, world)
        if root is not None:
            out_q.put(("root", rank, root.sigmas, root.modes, stats.recvs))
        else:
            out_q.put(("leafrank", rank, None, None, stats.sends))
    finally:
        dist.destroy_process_group()


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


@pytest.mark.parametrize("kind,world", [("star", 2), ("chain", 2), ("balanced", 3)])
def test_distributed_matches_single_process(kind, world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, kind, q)) for r in range(world)]
    for p in procs:
        p.start()
    msgs = [q.get(timeout=120) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    roots = [m for m in msgs if m[0] == "root"]
    assert len(roots) == 1 and roots[0][1] == 0
    tree, blocks, eps = _case(kind)
    ref = O.run_hapod([list(c) for c in tree.children], tree.root, blocks, eps)
    assert np.array_equal(roots[0][2], ref.modes.sigmas)
    assert np.array_equal(roots[0][3], ref.modes.modes)
    if kind != "chain":  # a chain stays on one rank: no edges cross
        assert roots[0][4] > 0


# ---------------------------------------------------------------------------------------------
# Row-distributed root (rowroot.py): the same protocol as on B200s (all-to-all of row slices,
# all_reduce of the Gram, eigensolve + broadcast on rank 0, all_reduced drift Gram / CholQR,
# global first-index argmax for the signs), with a NumPy restatement of the node arithmetic.
class NumpyRowArith:
    """Matrices are torch CPU tensors stored transposed, shape (cols, rows): column j is
    contiguous, like the column-major DevMat layout the device path uses."""

    def empty(self, rows, cols):
        return torch.zeros((cols, rows), dtype=torch.float64)

    empty_rowblock = empty
    empty_compact = empty

    def compact(self, M):
        return M.contiguous()

    def flat(self, M):
        return M.reshape(-1)

    def cols_view(self, S, off, n):
        return S[off:off + n].reshape(-1)

    def vector(self, a):
        return torch.from_numpy(np.array(a, dtype=np.float64))

    def to_host(self, t):
        return t.numpy()

    def sync(self):
        pass

    def row_slice(self, mat, q0, q1):
        return torch.from_numpy(np.ascontiguousarray(np.asarray(mat)[q0:q1].T))

    def copy_rows(self, mat, q0, q1, S, off):
        S[off:off + np.asarray(mat).shape[1]] = torch.from_numpy(np.ascontiguousarray(np.asarray(mat)[q0:q1].T))

    def copy_rows_into(self, block, full, r0):
        full[:, r0:r0 + block.shape[1]] = block

    @staticmethod
    def _np(M):
        return M.numpy().T

    def like(self, M):
        return torch.empty_like(M)

    def add(self, A, B):
        A += B
        return A

    def gram_rows(self, S, a, b, scale, m):
        x = self._np(S)[a:b] * scale.numpy()[None, :]
        g = x.T @ x
        return torch.from_numpy(np.ascontiguousarray(0.5 * (g + g.T)))

    def eig(self, G, m, eps, cutoff, share=None):
        # share: the replicated eigensolve of the device path (every rank solves; LAPACK is deterministic here)
        import scipy.linalg
        lam, psi = scipy.linalg.eigh(G.numpy())
        lam, psi = lam[::-1], psi[:, ::-1]
        lam_max = lam[0] if lam.size else 0.0
        if lam_max <= 0.0:
            return lam_max, 0, 0, 0.0, None, None
        keep = lam >= cutoff * lam_max * m
        lk = lam[keep]
        sig = np.sqrt(lk)
        n = O.truncation_rank(sig, eps)
        tail = float(np.sum(lk[n:]))
        V = torch.from_numpy(np.ascontiguousarray(psi[:, keep][:, :n].T))
        return lam_max, int(keep.sum()), n, tail, V, torch.from_numpy(sig[:n].copy())

    def scale_rows(self, V, scale):
        return V * scale[None, :]

    def assemble_rows(self, S, a, b, Vs, sig, U):
        u = self._np(S)[a:b] @ self._np(Vs) / sig.numpy()[None, :]
        U[:, a:b] = torch.from_numpy(np.ascontiguousarray(u.T))

    def syrk_rows(self, U, a, b):
        u = self._np(U)[a:b]
        return torch.from_numpy(np.ascontiguousarray(u.T @ u))

    def drift(self, C):
        c = C.numpy()
        return float(np.abs(c - np.eye(c.shape[0])).max()) if c.size else 0.0

    def chol_inverse(self, C):
        import scipy.linalg
        L = np.linalg.cholesky(C.numpy())
        return torch.from_numpy(scipy.linalg.solve_triangular(L, np.eye(L.shape[0]), lower=True))

    def trmm_rows(self, U, a, b, Linv, Y):
        y = self._np(U)[a:b] @ Linv.numpy().T  # U L^{-T}
        Y[:, a:b] = torch.from_numpy(np.ascontiguousarray(y.T))

    def col_absmax(self, U, row_offset):
        u = np.abs(self._np(U))
        n = u.shape[1]
        if u.shape[0] == 0:
            return torch.full((n,), -1.0, dtype=torch.float64), torch.full((n,), -1, dtype=torch.int64)
        return torch.from_numpy(u.max(axis=0).copy()), torch.from_numpy(u.argmax(axis=0).astype(np.int64) + row_offset)

    def entry_signs(self, U, rows, cols):
        v = self._np(U)[rows, cols]
        return np.where(v < 0.0, -1.0, 1.0)

    def flip(self, U, s):
        return U * s[:, None]


class RowOracleEvaluator(OracleEvaluator):
    def __init__(self, children, blocks, eps, d):
        super().__init__(children, blocks, eps)
        self.d = d

    def root_parts(self, res):
        # sigma-scaled modes (ModeSet.scaled, pod.py:160-162); a passthrough keeps unit scale
        return [(np.asfortranarray(res.modes), res.sigmas if res.orthonormal else None)]

    def evaluate_root_rows(self, root, children, local, rank, world, group):
        from paper_1607_05210_b200 import rowroot as RR
        arith = NumpyRowArith()
        layout = RR.gather_layout(children, local, rank, world, group)
        shards = RR.row_bounds(self.d, align=2)
        bounds = RR.rank_bounds(shards, world)
        S = RR.exchange_rows(layout, local, bounds, rank, world, arith, group)
        res = RR.row_root_pod(S, layout, shards, self.eps[root], O.DEFAULT_GRAM_CUTOFF, rank, world, arith, group)
        full = RR.gather_rows(res, self.d, rank, world, arith, group)
        if rank != 0:
            return None
        return O.Modes(res.sigmas, full.numpy().T.copy(), True, res.tail)


def _row_worker(rank, world, port, kind, out_q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        tree, blocks, eps = _case(kind)
        d = next(iter(blocks.values())).shape[0]
        ev = RowOracleEvaluator([list(c) for c in tree.children], blocks, eps, d)
        root, reports, stats = DI.run_distributed(tree, ev, rank, world, root_rows=True)
        out_q.put((rank, None if root is None else (root.sigmas, root.modes, root.tail_energy)))
    finally:
        dist.destroy_process_group()


def _row_run(kind, world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_row_worker, args=(r, world, port, kind, q)) for r in range(world)]
    for p in procs:
        p.start()
    msgs = dict(q.get(timeout=120) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert all(msgs[r] is None for r in range(1, world))
    return msgs[0]


def test_row_distributed_root_bitwise_across_rank_counts():
    """the root's Gram and mode Gram are summed over 8 FIXED row shards in one
    fixed binary tree, and every product runs on one shard -- so 1, 2, 4 and 8 ranks produce
    bitwise identical sigma, modes and tail (the reference is bit-identical across worker
    counts, tests/test_parallel.py:50-58)."""
    runs = {w: _row_run("star", w) for w in (1, 2, 4, 8)}
    s1, m1, t1 = runs[1]
    for w in (2, 4, 8):
        s, mo, t = runs[w]
        assert np.array_equal(s, s1), w
        assert np.array_equal(mo, m1), w
        assert t == t1, w


def test_row_bounds_and_owners():
    from paper_1607_05210_b200 import rowroot as RR
    sh = RR.row_bounds(200_000)
    assert len(sh) == 9 and sh[0] == 0 and sh[-1] == 200_000
    assert all(b % 16 == 0 for b in sh[1:-1]) and all(x <= y for x, y in zip(sh, sh[1:]))
    for w in (1, 2, 3, 4, 5, 8):
        own = RR.shard_owner(w)
        assert own[0] == 0 and own[-1] == w - 1 and own == sorted(own)
        rb = RR.rank_bounds(sh, w)
        assert rb[0] == 0 and rb[-1] == 200_000 and rb == sorted(rb)
    with pytest.raises(ValueError):
        RR.shard_owner(9)


@pytest.mark.parametrize("kind,world", [("star", 2), ("star", 3), ("balanced", 3)])
def test_row_distributed_root_matches_oracle(kind, world):
    """The root evaluated on row blocks by every rank equals the single-process oracle: same
    mode count, sigma and modes to rounding (the Gram is summed over row blocks in another
    order), tail energy alike."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_row_worker, args=(r, world, port, kind, q)) for r in range(world)]
    for p in procs:
        p.start()
    msgs = dict(q.get(timeout=120) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert all(msgs[r] is None for r in range(1, world))
    sig, modes, tail = msgs[0]
    tree, blocks, eps = _case(kind)
    ref = O.run_hapod([list(c) for c in tree.children], tree.root, blocks, eps).modes
    assert sig.size == ref.count
    assert np.allclose(sig, ref.sigmas, rtol=1e-10, atol=0)
    assert np.max(np.abs(modes - ref.modes)) < 1e-8   # same sign convention, same vectors
    assert tail == pytest.approx(ref.tail_energy, rel=1e-6, abs=1e-14)
