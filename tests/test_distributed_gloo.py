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


class OracleEvaluator:
    def __init__(self, children, blocks, eps):
        self.children = children
        self.blocks = blocks
        self.eps = eps

    def evaluate_leaf(self, node):
        return O.pod(self.blocks[node], self.eps[node])

    def evaluate_interior(self, node, child_results):
        parts = [r.scaled() for r in child_results if r.count]
        d = next(iter(self.blocks.values())).shape[0]
        stacked = np.hstack(parts) if parts else np.zeros((d, 0))
        return O.pod(stacked, self.eps[node])

    def send(self, res, dst, group):
        hdr = torch.tensor([res.count, res.modes.shape[0], int(res.orthonormal)], dtype=torch.int64)
        works = [dist.isend(hdr, dst, group=group)]
        if res.count:
            works.append(dist.isend(torch.from_numpy(np.ascontiguousarray(res.sigmas)), dst, group=group))
            works.append(dist.isend(torch.from_numpy(np.ascontiguousarray(res.modes.T)), dst, group=group))
        return works, 24 + 8 * res.count * (1 + res.modes.shape[0])

    def recv(self, src, group):
        hdr = torch.empty(3, dtype=torch.int64)
        dist.recv(hdr, src, group=group)
        n, d, orth = (int(x) for x in hdr.tolist())
        if n == 0:
            return O.Modes(np.zeros(0), np.zeros((d, 0))), 24
        sig = torch.empty(n, dtype=torch.float64)
        dist.recv(sig, src, group=group)
        modes = torch.empty((n, d), dtype=torch.float64)
        dist.recv(modes, src, group=group)
        return O.Modes(sig.numpy().copy(), modes.numpy().T.copy(), bool(orth)), 24 + 8 * n * (1 + d)


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
