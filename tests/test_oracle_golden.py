"""Pin the CPU oracle (oracle/hapod_oracle.py) against golden vectors produced by
the unmodified reference (tests/golden/make_golden.py).  CPU only."""

import numpy as np
import pytest

from oracle import hapod_oracle as O


def _close(a, b, rtol=1e-10, atol=1e-13):
    a = np.asarray(a)
    b = np.asarray(b)
    assert a.shape == b.shape
    assert np.allclose(a, b, rtol=rtol, atol=atol), float(np.max(np.abs(a - b)))


def test_truncation_rank(golden):
    meta, _ = golden
    for s, e, n in meta["truncation"]:
        assert O.truncation_rank(np.array(s), e) == n


@pytest.mark.parametrize("i", range(5))
def test_pod_random(golden, i):
    meta, arr = golden
    e = meta["pod_rand/eps"][i]
    out = O.pod(arr["pod_rand/input"], e, want_right=True)
    key = f"pod_rand/{i}"
    assert out.count == meta[key]["count"]
    _close(out.sigmas, arr[f"{key}/sigmas"])
    _close(out.modes, arr[f"{key}/modes"], rtol=1e-8, atol=1e-10)
    _close(out.right, arr[f"{key}/right"], rtol=1e-8, atol=1e-10)
    assert out.tail_energy == pytest.approx(meta[key]["tail"], rel=1e-9, abs=1e-14)


def test_pod_weighted(golden):
    meta, arr = golden
    out = O.pod(arr["pod_weighted/input"], 0.4, weights=arr["pod_weighted/weights"])
    assert out.count == meta["pod_weighted"]["count"]
    _close(out.sigmas, arr["pod_weighted/sigmas"])
    _close(out.modes, arr["pod_weighted/modes"], rtol=1e-8, atol=1e-10)


def test_pod_mgs_branch(golden):
    meta, arr = golden
    out = O.pod(arr["pod_mgs/input"], meta["pod_mgs/eps"])
    assert out.drift > 1e-8  # the MGS branch of pod.py:247 is exercised
    assert out.count == meta["pod_mgs"]["count"]
    _close(out.sigmas, arr["pod_mgs/sigmas"], rtol=1e-9)
    _close(out.modes, arr["pod_mgs/modes"], rtol=1e-6, atol=1e-8)


def test_pod_clustered_and_unit(golden):
    meta, arr = golden
    out = O.pod(arr["pod_clustered/input"], 0.2)
    assert out.count == meta["pod_clustered"]["count"]
    _close(out.sigmas, arr["pod_clustered/sigmas"])
    out = O.pod(arr["pod_unit/input"], 0.1)
    assert out.count == 1 and out.sigmas[0] == pytest.approx(2.0, abs=1e-12)
    z = O.pod(np.zeros((4, 3)), 0.5, want_right=True)
    assert z.count == meta["pod_zero"]["count"] and list(z.right.shape) == meta["pod_zero"]["right_shape"]


def test_block_gramian_pod(golden):
    meta, arr = golden
    prior = O.pod(arr["bgp/a"], 0.3)
    _close(prior.modes, arr["bgp/prior/modes"], rtol=1e-8, atol=1e-10)
    out = O.block_gramian_pod(prior, arr["bgp/b"], 1.1)
    assert out.count == meta["bgp/out"]["count"]
    _close(out.sigmas, arr["bgp/out/sigmas"])
    _close(out.modes, arr["bgp/out/modes"], rtol=1e-8, atol=1e-10)
    pr = O.Modes(np.array([2.0, 1.0]), np.eye(6)[:, :2])
    counts = [O.block_gramian_pod(pr, np.zeros((6, 0)), e).count for e in (0.5, 1.5)]
    assert counts == meta["bgp/retrunc"]


def test_star_hapod(golden):
    meta, arr = golden
    vals = O.synthetic_decay(120, 200, 0.05, seed=7)
    assert np.allclose(O_checksum(vals), meta["star/input_checksum"], rtol=1e-12)
    children = [tuple(c) for c in meta["star/tree"]]
    order = O.leaf_order(children, 0)
    counts = {leaf: 50 for leaf in order}
    eps = O.assign_tolerances(children, 0, counts, 1e-2, 0.75)
    assert np.allclose(eps, meta["star/eps"], rtol=1e-15)
    blocks = {leaf: vals[:, 50 * i: 50 * (i + 1)] for i, leaf in enumerate(order)}
    run = O.run_hapod(children, 0, blocks, eps, track=True)
    assert run.modes.count == meta["star"]["count"]
    _close(run.modes.sigmas, arr["star/sigmas"])
    _close(run.modes.modes, arr["star/modes"], rtol=1e-7, atol=1e-9)
    _close(run.right_factor, arr["star/right_factor"], rtol=1e-7, atol=1e-9)
    assert run.apriori_error_bound == pytest.approx(meta["star/bound"], rel=1e-14)
    for node, level, n_in, sub, n_out, tail in meta["star/reports"]:
        c, t, i = run.node_outputs[node]
        assert (c, i) == (n_out, n_in)
        assert t == pytest.approx(tail, rel=1e-8, abs=1e-15)
    assert O.actual_mean_error(vals, run.modes.modes) == pytest.approx(meta["star/mean_error"], rel=1e-9)


def O_checksum(a):
    return [float(a.sum()), float(np.abs(a).sum()), float(a.reshape(-1)[:: max(1, a.size // 97)].sum())]


def test_readme_balanced_example(golden):
    meta, arr = golden
    vals = O.synthetic_decay(400, 2000, 0.05, seed=7)
    assert np.allclose(O_checksum(vals), meta["readme/input_checksum"], rtol=1e-12)
    children = [tuple(c) for c in meta["readme/tree"]]
    order = O.leaf_order(children, 0)
    blocks = {leaf: vals[:, 100 * i: 100 * (i + 1)] for i, leaf in enumerate(order)}
    eps = meta["readme/eps"]
    run = O.run_hapod(children, 0, blocks, eps)
    assert run.modes.count == meta["readme/hapod_count"] == 40
    assert O.pod(vals, eps[0]).count == meta["readme/flat_count"]  # flat POD at the root tolerance
    _close(run.modes.sigmas, arr["readme/sigmas"])


def test_incremental(golden):
    meta, arr = golden
    vals = arr["inc/input"]
    blocks = [vals[:, 20 * j: 20 * (j + 1)] for j in range(6)]
    cur, bound, steps = O.incremental(blocks, 0.05, 0.8)
    assert cur.count == meta["inc"]["count"]
    _close(cur.sigmas, arr["inc/sigmas"])
    _close(cur.modes, arr["inc/modes"], rtol=1e-7, atol=1e-9)
    assert bound == pytest.approx(meta["inc/bound"], rel=1e-14)
    cur, bound, _ = O.incremental(blocks[:4], 0.05, 0.8, planned=10)
    assert cur.count == meta["inc_early"]["count"]
    _close(cur.sigmas, arr["inc_early/sigmas"])
    assert bound == pytest.approx(meta["inc_early/bound"], rel=1e-14)


def test_tolerance_rule(golden):
    meta, _ = golden
    children, root = O.star(4)
    eps = O.assign_tolerances(children, root, {1: 4, 2: 4, 3: 4, 4: 4}, 0.5, 0.75)
    assert eps == pytest.approx(meta["tol/star"], rel=1e-15)
    assert eps[0] == 0.75 * 4 * 0.5  # frozen (test_hierarchy.py:39-44)
    children, root = O.chain(5)
    assert [list(c) for c in children] == meta["tol/chain_tree"]
    assert O.leaf_order(children, root) == meta["tol/chain_leaf_order"]
    counts = {v: 3 for v in range(len(children)) if not children[v]}
    eps = O.assign_tolerances(children, root, counts, 0.2, 0.6, zero_leaf_tolerance=True)
    assert eps == pytest.approx(meta["tol/chain"], rel=1e-15)
