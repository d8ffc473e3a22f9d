"""Multi-GPU HAPOD: one process per GPU, child -> parent edges over NCCL.

The tree partitions naturally: every node is placed on a rank,
each rank evaluates its nodes in post-order, and an edge whose child and
parent live on different ranks moves the child's sigma-scaled mode block
(U: d x N float64 and sigma: N) with point-to-point send/recv -- NCCL has no
gather primitive, a gather is grouped send/recv (the paper's MPI runs sent
modes "sequentially to the main node").  No other data
crosses ranks: leaves never move, an interior node's children on the same
rank are consumed in place.

Placement (``plan_placement``): leaves in depth-first order are split into
contiguous, equally sized chunks, chunk r -> rank r; an interior node goes to
the rank of its first child (so a star's root lands on rank 0 and a chain
stays on the rank of its bottom leaf).  Because every node's arithmetic is
the single-GPU kernel sequence with shape-only split-K plans, results are
bitwise identical for any rank count.  With ``root_rows`` the root is instead
evaluated by every rank on a row block of its input (rowroot.py: row
all-to-all, per-shard Grams summed in a fixed tree over 8 row shards,
eigensolve on rank 0 + broadcast) -- needed when the root's input exceeds one
GPU (config 3) -- and is bitwise identical for 1, 2, 4 or 8 ranks.

Edges carry the child's node id in their header and the receiver checks it:
send/recv pairs are matched by posting order only, so a placement that broke
the order would otherwise silently hand a parent the wrong child.

The driver is written against a small evaluator interface so the protocol is
exercised on CPU (gloo, world size 2) by the tests with the CPU oracle as the
node evaluator, and on B200s with the device evaluator below.
"""

from __future__ import annotations

import math
import time
from dataclasses import dataclass

import numpy as np

from .tree import RootedTree, TreeMaps, derive_maps, post_order

__all__ = ["plan_placement", "run_distributed", "DeviceEvaluator", "EdgeStats"]


def plan_placement(tree: RootedTree, world_size: int, maps: TreeMaps | None = None) -> list:
    """node -> rank.  Leaves (DFS order) in contiguous equal chunks; interior
    nodes on their first child's rank."""
    maps = maps or derive_maps(tree)
    order = maps.leaf_order
    k = len(order)
    place = [0] * tree.node_count
    for i, leaf in enumerate(order):
        place[leaf] = min(world_size - 1, (i * world_size) // k)
    for v in post_order(tree):
        if tree.children[v]:
            place[v] = place[tree.children[v][0]]
    return place


@dataclass
class EdgeStats:
    sent_bytes: int = 0
    recv_bytes: int = 0
    sends: int = 0
    recvs: int = 0
    comm_time: float = 0.0


def run_distributed(tree: RootedTree, evaluator, rank: int, world_size: int, placement=None, group=None,
                    root_rows: bool = False):
    """Evaluate the tree across ranks.  Returns (root result on rank 0 / the root's rank,
    None elsewhere; {node: (seconds, result)}; EdgeStats).

    ``evaluator`` provides the node arithmetic and the edge payloads:
    evaluate_leaf(node), evaluate_interior(node, child_results),
    send(result, dst, group, node) -> (async works, bytes), recv(src, group, node) -> (result,
    bytes) (``node``: the child's id, carried in the payload header and verified on receipt);
    with ``root_rows`` also root_parts(result) and evaluate_root_rows(root, children, local,
    rank, world, group): the root is then evaluated by ALL ranks on row blocks of its input
    (rowroot.py) instead of gathering the children's modes on one rank."""
    import torch.distributed as dist

    maps = derive_maps(tree)
    place = placement or plan_placement(tree, world_size, maps)
    live: dict = {}
    reports: dict = {}
    stats = EdgeStats()
    pending_sends = []
    root_kids = set(tree.children[tree.root]) if root_rows else set()
    for v in post_order(tree):
        if place[v] != rank or (root_rows and v == tree.root):
            continue
        kids = tree.children[v]
        started = time.perf_counter()
        if not kids:
            out = evaluator.evaluate_leaf(v)
        else:
            child_results = []
            for c in kids:
                if place[c] == rank:
                    child_results.append(live.pop(c))
                else:
                    t0 = time.perf_counter()
                    res, nbytes = evaluator.recv(place[c], group, c)
                    stats.comm_time += time.perf_counter() - t0
                    stats.recv_bytes += nbytes
                    stats.recvs += 1
                    child_results.append(res)
            out = evaluator.evaluate_interior(v, child_results)
        reports[v] = (time.perf_counter() - started, out)
        parent = maps.parent[v]
        if parent >= 0 and place[parent] != rank and v not in root_kids:
            t0 = time.perf_counter()
            works, nbytes = evaluator.send(out, place[parent], group, v)
            pending_sends.extend(works)
            stats.comm_time += time.perf_counter() - t0
            stats.sent_bytes += nbytes
            stats.sends += 1
        else:
            live[v] = out
    for w in pending_sends:
        w.wait()
    if root_rows:
        started = time.perf_counter()
        local = {c: evaluator.root_parts(live.pop(c)) for c in tree.children[tree.root] if place[c] == rank}
        root = evaluator.evaluate_root_rows(tree.root, list(tree.children[tree.root]), local, rank, world_size, group)
        reports[tree.root] = (time.perf_counter() - started, root)
        return root, reports, stats
    root = live.get(tree.root) if place[tree.root] == rank else None
    return root, reports, stats


# ---------------------------------------------------------------------------- device evaluator
class DeviceEvaluator:
    """B200 node arithmetic (the same kernels as run_hapod) + NCCL payloads.

    Payload of an edge: header int64 [node, count, d, ld, orthonormal], then sigma
    (count float64) and the mode block storage (count x ld float64, column-major)
    as one grouped NCCL send/recv (batch_isend_irecv)."""

    def __init__(self, space, leaf_blocks: dict, tol, backend=None):
        from .pod import PodBackend
        self.space = space
        self.blocks = leaf_blocks
        self.tol = tol
        self.backend = backend or PodBackend()
        self.tree = None

    def bind(self, tree):
        self.tree = tree
        return self

    def evaluate_leaf(self, node):
        from .pod import pod
        return pod(self.blocks[node], self.tol.epsilons[node], self.backend)

    def evaluate_interior(self, node, child_results):
        from .pod import pod_parts
        parts = []
        for ms in child_results:
            if ms.count:
                parts.extend(ms.scaled_parts())
        return pod_parts(self.space, parts, self.tol.epsilons[node], self.backend)

    def root_parts(self, ms):
        """A child's contribution to the root input: its sigma-scaled column blocks
        (ModeSet.scaled, pod.py:160-162) as (DevMat, host scale or None)."""
        return [(p.mat, None if p.scale is None else p.scale.cpu().numpy()) for p in ms.scaled_parts()]

    def evaluate_root_rows(self, root, children, local, rank, world, group):
        from . import _device as D
        from . import rowroot as RR
        from .pod import ModeSet
        arith = RR.DeviceRowArith()
        D.Profiler.set_tag(root)
        d = self.space.dimension
        layout = RR.gather_layout(children, local, rank, world, group)
        shards = RR.row_bounds(d)
        bounds = RR.rank_bounds(shards, world)
        S_q = RR.exchange_rows(layout, local, bounds, rank, world, arith, group)
        res = RR.row_root_pod(S_q, layout, shards, self.tol.epsilons[root], self.backend.gram_eig_cutoff_factor,
                              rank, world, arith, group)
        del S_q
        full = RR.gather_rows(res, d, rank, world, arith, group)
        if rank != 0:
            return None
        if res.sigmas.size == 0:
            return ModeSet._device(self.space, np.zeros(0), [D.Part(D.DevMat.empty(d, 0))], orthonormal=True,
                                   tail_energy=res.tail)
        return ModeSet._device(self.space, res.sigmas, [D.Part(full)], orthonormal=True, tail_energy=res.tail,
                               diagnostics={"lam_max": res.lam_max, "nkeep": res.nkeep, "drift": res.drift,
                                            "reorthonormalized": res.reorthed, "input_count": res.m,
                                            "row_blocks": res.bounds})

    def send(self, ms, dst, group, node):
        """Header [node, count, d, ld, orthonormal] (one op), then sigma and the column-major
        mode storage as ONE grouped NCCL launch (batch_isend_irecv)."""
        import torch
        import torch.distributed as dist
        U = ms.modes_device()
        hdr = torch.tensor([node, ms.count, U.rows, U.ld, int(ms.orthonormal)], dtype=torch.int64, device="cuda")
        works = [dist.isend(hdr, dst, group=group)]
        nbytes = 40
        if ms.count:
            sig = ms.sigmas_device().contiguous()
            body = U.storage[U.offset: U.offset + U.ld * U.cols]
            works.extend(dist.batch_isend_irecv([dist.P2POp(dist.isend, sig, dst, group=group),
                                                 dist.P2POp(dist.isend, body, dst, group=group)]))
            nbytes += sig.numel() * 8 + body.numel() * 8
        return works, nbytes

    def recv(self, src, group, node):
        import torch
        import torch.distributed as dist
        from . import _device as D
        from .pod import ModeSet
        hdr = torch.empty(5, dtype=torch.int64, device="cuda")
        dist.recv(hdr, src, group=group)
        got, count, d, ld, orth = (int(x) for x in D.host_read(hdr))
        if got != node:
            raise RuntimeError(f"edge from rank {src}: expected the modes of node {node}, received node {got}")
        if count == 0:
            return ModeSet._device(self.space, np.zeros(0), [D.Part(D.DevMat.empty(d, 0))], orthonormal=True), 40
        sig = torch.empty(count, dtype=torch.float64, device="cuda")
        store = torch.empty(ld * count, dtype=torch.float64, device="cuda")
        for w in dist.batch_isend_irecv([dist.P2POp(dist.irecv, sig, src, group=group),
                                         dist.P2POp(dist.irecv, store, src, group=group)]):
            w.wait()
        U = D.DevMat(store, d, count, ld)
        sig_host = D.host_read(sig)
        ms = ModeSet._device(self.space, sig_host, [D.Part(U)], orthonormal=bool(orth), sig_dev=sig)
        return ms, 40 + 8 * count + 8 * ld * count
