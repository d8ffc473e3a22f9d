"""Acceptance-scale randomized check on the device, after the reference's own acceptance suite
(pkg/tests/test_acceptance.py:67-103 over helpers.random_case, helpers.py:82-114): seeded random
trees of up to 30 nodes, dimensions up to 200, up to 500 columns split at random over the leaves,
exponential-decay data, optional weights, per-node tolerances from keep-everything to
discard-almost-everything with exact zeros.  For every case the device run must

  * stay within the a-priori error budget            (test_error_bound_on_random_trees),
  * never exceed the flat-POD mode count at any node (test_mode_bound_on_random_trees),
  * reproduce the oracle's mode count at EVERY node and its root singular values.
"""

import math

import numpy as np
import pytest
import scipy.linalg

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("no CUDA device", allow_module_level=True)

import paper_1607_05210_b200 as H  # noqa: E402
from oracle import hapod_oracle as O  # noqa: E402

CASES = 200
SEED = 20260819


def _flat_count(values, eps, weights):
    """Mode count of a flat POD by one dense SVD (smallest N with tail energy <= eps^2)."""
    if values.shape[1] == 0:
        return 0
    if eps == 0.0:
        return values.shape[1]
    if weights is not None:
        values = values * np.sqrt(weights)[:, None]
    sig = scipy.linalg.svdvals(values)
    tails = np.concatenate([np.cumsum((sig * sig)[::-1])[::-1], [0.0]])
    return int(np.argmax(tails <= eps * eps))


def _case(rng):
    n = int(rng.integers(1, 31))
    children = [[] for _ in range(n)]
    for v in range(1, n):
        children[int(rng.integers(0, v))].append(v)
    tree = H.RootedTree(tuple(tuple(c) for c in children), 0)
    maps = H.derive_maps(tree)
    d = int(rng.integers(5, 201))
    cols = int(rng.integers(len(maps.leaves), 501))
    data = O.synthetic_decay(d, cols, float(rng.uniform(0.02, 0.8)), seed=int(rng.integers(2 ** 31)))
    w = rng.uniform(0.5, 2.0, d) if rng.random() < 0.25 else None
    probs = rng.random(len(maps.leaves))
    counts = [int(c) for c in rng.multinomial(cols, probs / probs.sum())]
    total = float(np.sum(data ** 2 * (w[:, None] if w is not None else 1.0)))
    eps = rng.uniform(0.0, 0.6, n) ** 2 * (math.sqrt(total) if total > 0 else 1.0)
    eps[rng.random(n) < 0.15] = 0.0
    return tree, maps, d, cols, data, w, counts, eps, total


@pytest.mark.parametrize("tri_min_order,cases", [(None, CASES), (4, 80)])
def test_random_trees_budget_mode_bound_and_oracle_counts(tri_min_order, cases):
    """tri_min_order = 4 sends EVERY preconditioned eigenproblem of order >= 4 through the tridiagonal
    solver (hp_syev_tri; production uses it from order 1,024 up), including the spectra it has to
    decline -- exact zeros, repeated singular values -- which must fall back to block Jacobi."""
    from paper_1607_05210_b200 import _device as D
    saved = D.TRI_MIN_ORDER
    if tri_min_order is not None:
        D.TRI_MIN_ORDER = tri_min_order
    try:
        _run_cases(cases, D if tri_min_order is not None else None)
    finally:
        D.TRI_MIN_ORDER = saved


def _run_cases(ncases, D):
    rng = np.random.default_rng(SEED)
    nodes_checked, worst = 0, 0.0
    tri_done = tri_declined = 0
    for case in range(ncases):
        tree, maps, d, cols, data, w, counts, eps, total = _case(rng)
        sp = H.InnerProductSpace(d, w)
        la = H.distribute_columns(tree, H.SnapshotBlock(sp, data), counts=counts)
        tol = H.ToleranceAssignment(tuple(float(e) for e in eps))
        if D is not None:
            D.LAST_TRI_DIAG.clear()
        res = H.run_hapod(tree, la, tol)
        if D is not None and D.LAST_TRI_DIAG:
            tri_done += D.LAST_TRI_DIAG["status"] == 0
            tri_declined += D.LAST_TRI_DIAG["status"] != 0
        blocks = {leaf: np.asarray(la.blocks[leaf].values) for leaf in maps.leaf_order}
        ref = O.run_hapod([list(c) for c in tree.children], 0, blocks, list(tol.epsilons), weights=w)
        # every node's output count equals the oracle's
        for rep in res.reports:
            assert rep.output_mode_count == ref.node_outputs[rep.node][0], (case, rep.node)
        # mode bound: a node never keeps more modes than a flat POD of its subtree's snapshots
        for rep in res.reports:
            sub = [blocks[u] for u in maps.leaf_order if u in set(maps.subtree_nodes[rep.node])]
            cap = _flat_count(np.hstack(sub), tol.epsilons[rep.node], w)
            assert rep.output_mode_count <= cap, (case, rep.node, rep.output_mode_count, cap)
            nodes_checked += 1
        # error budget
        if res.modes.orthonormal:
            bound_sq = H.error_bound(tree, tol, maps=maps) ** 2
            resid = H.actual_mean_error(H.SnapshotBlock(sp, data), res.modes) * cols
            assert resid <= bound_sq + 1e-8 * max(total, 1.0), (case, resid, bound_sq)
            worst = max(worst, resid - bound_sq)
        # root singular values against the oracle, at the method-of-snapshots floor
        if ref.modes.count and res.modes.orthonormal:
            s = ref.modes.sigmas
            floor = 2.2e-16 * (s[0] / s) ** 2
            rel = np.abs(np.asarray(res.modes.sigmas) - s) / s
            assert np.all(rel <= np.maximum(1e-9, 1e3 * floor)), (case, rel.max())
    print(f"\n[acceptance] {ncases} random trees, {nodes_checked} node outputs: counts equal to the oracle's, "
          f"within flat-POD counts and within budget (worst overshoot {worst:.3e})"
          + (f"; last tridiagonal solve per tree: {tri_done} completed, {tri_declined} declined" if D is not None else ""))
    if D is not None:
        assert tri_done > ncases // 2  # the forced path really ran
