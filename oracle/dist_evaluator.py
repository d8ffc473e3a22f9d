"""Node evaluator for the multi-rank HAPOD driver with the CPU oracle as the arithmetic --
TEST INFRASTRUCTURE (see oracle/hapod_oracle.py's header).

``paper_1607_05210_b200.distributed.run_distributed`` is written against a small evaluator
interface; this class fills it with NumPy arithmetic and gloo point-to-point payloads, so the
placement / post-order / edge protocol (and ``bench.py --protocol-check``, the CPU rehearsal of
the ``--gpus N`` launch path) run without a GPU.  The reference's counterpart is the pooled
wave executor parallel.py:77-142."""

from __future__ import annotations

import numpy as np
import torch
import torch.distributed as dist

from . import hapod_oracle as O


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

    def send(self, res, dst, group, node):
        hdr = torch.tensor([node, res.count, res.modes.shape[0], int(res.orthonormal)], dtype=torch.int64)
        works = [dist.isend(hdr, dst, group=group)]
        if res.count:
            works.append(dist.isend(torch.from_numpy(np.ascontiguousarray(res.sigmas)), dst, group=group))
            works.append(dist.isend(torch.from_numpy(np.ascontiguousarray(res.modes.T)), dst, group=group))
        return works, 32 + 8 * res.count * (1 + res.modes.shape[0])

    def recv(self, src, group, node):
        hdr = torch.empty(4, dtype=torch.int64)
        dist.recv(hdr, src, group=group)
        got, n, d, orth = (int(x) for x in hdr.tolist())
        assert got == node, (got, node)
        if n == 0:
            return O.Modes(np.zeros(0), np.zeros((d, 0))), 32
        sig = torch.empty(n, dtype=torch.float64)
        dist.recv(sig, src, group=group)
        modes = torch.empty((n, d), dtype=torch.float64)
        dist.recv(modes, src, group=group)
        return O.Modes(sig.numpy().copy(), modes.numpy().T.copy(), bool(orth)), 32 + 8 * n * (1 + d)
