"""Parity of the device HAPOD path (public API) against the CPU oracle and the
golden vectors of the reference.  Needs a B200.

Tolerances: the device Gram has a different summation order than BLAS dgemm,
so singular values agree to ~u*sigma_1^2/sigma_i^2 relative;
for the well-conditioned golden cases that is far below the 1e-10 gate used
here.  Spans are compared through principal angles, never raw entries of
nearly-degenerate modes."""

import math

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("no CUDA device", allow_module_level=True)

import paper_1607_05210_b200 as H  # noqa: E402
from oracle import hapod_oracle as O  # noqa: E402


def euclid(d):
    return H.InnerProductSpace(d)


def angles(ua, ub):
    return O.principal_angle_sines(np.asarray(ua), np.asarray(ub))


def assert_same_modes(dev, ref, sig_rtol=1e-10, ang=1e-8):
    assert dev.count == ref.count
    assert np.allclose(dev.sigmas, ref.sigmas, rtol=sig_rtol, atol=0)
    if ref.count:
        a = angles(dev.modes, ref.modes)
        assert a.size == 0 or a.max() < ang, a.max()


@pytest.mark.parametrize("i", range(5))
def test_pod_golden_random(golden, i):
    meta, arr = golden
    e = meta["pod_rand/eps"][i]
    vals = arr["pod_rand/input"]
    out = H.pod(H.SnapshotBlock(euclid(20), vals), e, want_right=True)
    key = f"pod_rand/{i}"
    assert out.count == meta[key]["count"]
    assert np.allclose(out.sigmas, arr[f"{key}/sigmas"], rtol=1e-12)
    # well separated spectrum: the modes themselves agree (same sign convention)
    assert np.allclose(out.modes, arr[f"{key}/modes"], rtol=1e-8, atol=1e-10)
    assert np.allclose(out.right, arr[f"{key}/right"], rtol=1e-8, atol=1e-10)
    assert out.tail_energy == pytest.approx(meta[key]["tail"], rel=1e-9, abs=1e-13)
    assert out.orthonormal


def test_pod_golden_weighted(golden):
    meta, arr = golden
    w = arr["pod_weighted/weights"]
    out = H.pod(H.SnapshotBlock(H.InnerProductSpace(8, w), arr["pod_weighted/input"]), 0.4)
    assert out.count == meta["pod_weighted"]["count"]
    assert np.allclose(out.sigmas, arr["pod_weighted/sigmas"], rtol=1e-12)
    assert np.allclose(out.modes, arr["pod_weighted/modes"], rtol=1e-8, atol=1e-10)


def test_pod_golden_mgs_branch(golden):
    meta, arr = golden
    out = H.pod(H.SnapshotBlock(euclid(60), arr["pod_mgs/input"]), meta["pod_mgs/eps"])
    assert out.diagnostics["reorthonormalized"]  # drift > 1e-8, like the reference
    assert out.count == meta["pod_mgs"]["count"]
    ref = arr["pod_mgs/sigmas"]
    # sigma_N / sigma_1 ~ e^-19: the Gram rounding floor is u*sigma_1^2/sigma_i^2
    floor = 2.2e-16 * (ref[0] / ref) ** 2
    assert np.all(np.abs(out.sigmas - ref) / ref <= np.maximum(1e-10, 50 * floor))
    g = out.modes.T @ out.modes
    assert np.max(np.abs(g - np.eye(out.count))) < 1e-12


def test_pod_golden_clustered_unit_zero(golden):
    meta, arr = golden
    out = H.pod(H.SnapshotBlock(euclid(12), arr["pod_clustered/input"]), 0.2)
    assert out.count == meta["pod_clustered"]["count"]
    assert np.allclose(out.sigmas, arr["pod_clustered/sigmas"], rtol=1e-12)
    assert np.max(np.abs(out.modes.T @ out.modes - np.eye(out.count))) <= 1e-8
    unit = H.pod(H.SnapshotBlock(euclid(5), arr["pod_unit/input"]), 0.1)
    assert unit.count == 1 and unit.sigmas[0] == pytest.approx(2.0, abs=1e-12)
    assert unit.modes[1, 0] == pytest.approx(1.0, abs=1e-12)
    z = H.pod(H.SnapshotBlock(euclid(4), np.zeros((4, 3))), 0.5, want_right=True)
    assert z.count == 0 and z.right.shape == (3, 0) and z.tail_energy == 0.0
    e = H.pod(H.SnapshotBlock(euclid(4), np.zeros((4, 0))), 0.5, want_right=True)
    assert e.count == 0 and e.right.shape == (0, 0)


def test_pod_passthrough_and_validation():
    rng = np.random.default_rng(31)
    vals = rng.standard_normal((6, 4))
    out = H.pod(H.SnapshotBlock(euclid(6), vals), 0.0, want_right=True)
    assert not out.orthonormal
    assert np.array_equal(out.modes, vals)
    assert np.array_equal(out.sigmas, np.ones(4))
    assert np.array_equal(out.right, np.eye(4))
    with pytest.raises(ValueError):
        H.pod(H.SnapshotBlock(euclid(6), vals), -1e-9)
    bad = np.ones((3, 2))
    bad[1, 1] = np.nan
    with pytest.raises(ValueError):
        H.SnapshotBlock(euclid(3), bad)
    with pytest.raises(ValueError):
        H.pod(H.SnapshotBlock(euclid(6), vals), 0.5, H.PodBackend("svd"))


@pytest.mark.parametrize("seed", range(6))
def test_pod_random_vs_oracle(seed):
    rng = np.random.default_rng(100 + seed)
    d = int(rng.integers(3, 700))
    m = int(rng.integers(1, 260))
    w = rng.uniform(0.3, 3.0, d) if seed % 3 == 0 else None
    vals = O.synthetic_decay(d, m, float(rng.uniform(0.01, 0.3)), seed=seed)
    total = float(np.sum(vals ** 2 * (w[:, None] if w is not None else 1.0)))
    eps = float(rng.uniform(1e-6, 0.5)) * math.sqrt(total)
    ref = O.pod(vals, eps, weights=w, want_right=True)
    out = H.pod(H.SnapshotBlock(H.InnerProductSpace(d, w), vals), eps, want_right=True)
    assert out.count == ref.count
    s1 = ref.sigmas[0] if ref.count else 1.0
    floor = 2.2e-16 * (s1 / np.maximum(ref.sigmas, 1e-300)) ** 2
    assert np.all(np.abs(out.sigmas - ref.sigmas) / ref.sigmas <= np.maximum(1e-10, 100 * floor))
    assert out.tail_energy == pytest.approx(ref.tail_energy, rel=1e-6, abs=1e-12 * total)
    # projection error equals the discarded tail within the gate
    err = H.actual_mean_error(H.SnapshotBlock(H.InnerProductSpace(d, w), vals), out) * m
    ref_err = O.actual_mean_error(vals, ref.modes, w) * m
    assert err == pytest.approx(ref_err, rel=1e-6, abs=1e-9 * total)


def test_block_gramian_pod_golden(golden):
    meta, arr = golden
    sp = euclid(25)
    prior = H.pod(H.SnapshotBlock(sp, arr["bgp/a"]), 0.3)
    assert np.allclose(prior.modes, arr["bgp/prior/modes"], rtol=1e-8, atol=1e-10)
    out = H.block_gramian_pod(prior, H.SnapshotBlock(sp, arr["bgp/b"]), 1.1)
    assert out.count == meta["bgp/out"]["count"]
    assert np.allclose(out.sigmas, arr["bgp/out/sigmas"], rtol=1e-12)
    assert np.allclose(out.modes, arr["bgp/out/modes"], rtol=1e-8, atol=1e-10)
    u = np.zeros((6, 2))
    u[0, 0] = 1.0
    u[1, 1] = 1.0
    pr = H.ModeSet(euclid(6), np.array([2.0, 1.0]), u)
    none = H.SnapshotBlock(euclid(6), np.zeros((6, 0)))
    assert [H.block_gramian_pod(pr, none, e).count for e in (0.5, 1.5)] == meta["bgp/retrunc"]
    raw = H.pod(H.SnapshotBlock(euclid(3), np.eye(3)), 0.0)
    with pytest.raises(ValueError, match="orthonormal"):
        H.block_gramian_pod(raw, H.SnapshotBlock(euclid(3), np.eye(3)), 0.5)


def test_star_golden_and_right_factor(golden):
    meta, arr = golden
    vals = O.synthetic_decay(120, 200, 0.05, seed=7)
    tree = H.build_star(4)
    leaves = H.distribute_columns(tree, H.SnapshotBlock(euclid(120), vals))
    tol = H.assign_tolerances(tree, leaves, 1e-2, omega=0.75)
    assert np.allclose(tol.epsilons, meta["star/eps"], rtol=1e-15)
    res = H.run_hapod(tree, leaves, tol, track_right_factor=True)
    assert res.mode_count == meta["star"]["count"]
    assert np.allclose(res.modes.sigmas, arr["star/sigmas"], rtol=1e-10)
    assert angles(res.modes.modes, arr["star/modes"]).max() < 1e-8
    assert res.apriori_error_bound == pytest.approx(meta["star/bound"], rel=1e-14)
    for node, level, n_in, sub, n_out, tail in meta["star/reports"]:
        r = res.report_for(node)
        assert (r.level, r.input_count, r.subordinate_count, r.output_mode_count) == (level, n_in, sub, n_out)
        assert r.discarded_tail_energy == pytest.approx(tail, rel=1e-7, abs=1e-15)
    lhat = res.right_factor
    assert lhat.shape == (200, res.mode_count)
    assert np.max(np.abs(lhat.T @ lhat - np.eye(res.mode_count))) <= 1e-8
    approx = (res.modes.modes * res.modes.sigmas[None, :]) @ lhat.T
    assert np.sum((vals - approx) ** 2) <= res.apriori_error_bound ** 2 + 1e-8 * np.sum(vals ** 2)
    merr = H.actual_mean_error(H.SnapshotBlock(euclid(120), vals), res.modes)
    assert merr == pytest.approx(meta["star/mean_error"], rel=1e-6)


def test_readme_balanced_example(golden):
    meta, arr = golden
    vals = O.synthetic_decay(400, 2000, 0.05, seed=7)
    tree = H.build_balanced(20, 2)
    assert [list(c) for c in tree.children] == meta["readme/tree"]
    leaves = H.distribute_columns(tree, H.SnapshotBlock(euclid(400), vals), block_size=100)
    tol = H.assign_tolerances(tree, leaves, 1e-2, omega=0.75)
    res = H.run_hapod(tree, leaves, tol)
    assert res.mode_count == meta["readme/hapod_count"] == 40
    assert np.allclose(res.modes.sigmas, arr["readme/sigmas"], rtol=1e-10)
    counts = {r.node: r.output_mode_count for r in res.reports}
    assert counts == {n: c for n, c in meta["readme/counts"]}
    par, stats = H.run_parallel(tree, leaves, tol, worker_count=4)
    assert np.array_equal(par.modes.sigmas, res.modes.sigmas)  # bit-identical for any worker count
    assert np.array_equal(par.modes.modes, res.modes.modes)
    assert stats.peak_resident_modes > 0


def test_incremental_golden(golden):
    meta, arr = golden
    vals = arr["inc/input"]
    sp = euclid(80)
    sess = H.incremental_open(0.05, 0.8, 6)
    for j in range(6):
        sess.push(H.SnapshotBlock(sp, vals[:, 20 * j: 20 * (j + 1)]))
    res = sess.finalize()
    assert res.mode_count == meta["inc"]["count"]
    assert np.allclose(res.modes.sigmas, arr["inc/sigmas"], rtol=1e-10)
    assert angles(res.modes.modes, arr["inc/modes"]).max() < 1e-8
    assert res.apriori_error_bound == pytest.approx(meta["inc/bound"], rel=1e-14)
    got = [[r.node, r.input_count, r.output_mode_count] for r in res.reports]
    want = [[n, i, c] for n, i, e, c, t in meta["inc/reports"]]
    assert got == want
    sess = H.incremental_open(0.05, 0.8, 10)
    for j in range(4):
        sess.push(H.SnapshotBlock(sp, vals[:, 20 * j: 20 * (j + 1)]))
    res = sess.finalize()
    assert res.mode_count == meta["inc_early"]["count"]
    assert np.allclose(res.modes.sigmas, arr["inc_early/sigmas"], rtol=1e-10)
    with pytest.raises(H.SessionError):
        sess.finalize()


def test_chain_run_matches_session():
    rng = np.random.default_rng(47)
    sp = euclid(10)
    raw = [rng.standard_normal((10, c)) for c in (6, 3, 8, 5)]
    blocks = [H.SnapshotBlock(sp, b) for b in raw]
    sess = H.incremental_open(0.15, 0.75, 4)
    for b in blocks:
        sess.push(b)
    inc = sess.finalize()
    tree = H.build_chain(4)
    maps = H.derive_maps(tree)
    la = H.LeafAssignment(dict(zip(maps.leaf_order, blocks)))
    tol = H.assign_tolerances(tree, la, 0.15, omega=0.75, zero_leaf_tolerance=True)
    ref = H.run_hapod(tree, la, tol)
    assert inc.mode_count == ref.mode_count
    assert np.allclose(inc.modes.sigmas, ref.modes.sigmas, rtol=1e-9)
    assert {r.node: r.local_epsilon for r in inc.reports} == pytest.approx(
        {r.node: r.local_epsilon for r in ref.reports})


def test_random_trees_bounds_and_oracle():
    rng = np.random.default_rng(20260819)
    for trial in range(6):
        n = int(rng.integers(1, 14))
        children = [[] for _ in range(n)]
        for v in range(1, n):
            children[int(rng.integers(0, v))].append(v)
        tree = H.RootedTree(tuple(tuple(c) for c in children), 0)
        maps = H.derive_maps(tree)
        d = int(rng.integers(5, 60))
        cols = int(rng.integers(len(maps.leaves), 120))
        data = O.synthetic_decay(d, cols, float(rng.uniform(0.05, 0.6)), seed=trial)
        w = rng.uniform(0.5, 2.0, d) if trial % 3 == 1 else None
        sp = H.InnerProductSpace(d, w)
        probs = rng.random(len(maps.leaves))
        counts = [int(c) for c in rng.multinomial(cols, probs / probs.sum())]
        la = H.distribute_columns(tree, H.SnapshotBlock(sp, data), counts=counts)
        total = float(np.sum(data ** 2 * (w[:, None] if w is not None else 1)))
        eps = rng.uniform(0.0, 0.6, n) ** 2 * math.sqrt(total)
        eps[rng.random(n) < 0.15] = 0.0
        tol = H.ToleranceAssignment(tuple(float(e) for e in eps))
        res = H.run_hapod(tree, la, tol)
        blocks = {leaf: np.asarray(la.blocks[leaf].values) for leaf in maps.leaf_order}
        ref = O.run_hapod([list(c) for c in tree.children], 0, blocks, list(tol.epsilons), weights=w)
        assert res.mode_count == ref.modes.count
        if ref.modes.count:
            s1 = ref.modes.sigmas[0]
            floor = 2.2e-16 * (s1 / ref.modes.sigmas) ** 2
            rel = np.abs(res.modes.sigmas - ref.modes.sigmas) / ref.modes.sigmas
            assert np.all(rel <= np.maximum(1e-9, 1e3 * floor))
        if res.modes.orthonormal:
            bound = H.error_bound(tree, tol, maps=maps)
            resid = H.actual_mean_error(H.SnapshotBlock(sp, data), res.modes) * cols
            assert resid <= bound ** 2 + 1e-8 * max(total, 1.0)


def test_determinism_bitwise():
    vals = O.synthetic_decay(3000, 700, 0.02, seed=11)
    blk = H.SnapshotBlock(euclid(3000), vals)
    a = H.pod(blk, 1e-6 * np.linalg.norm(vals))
    b = H.pod(blk, 1e-6 * np.linalg.norm(vals))
    assert np.array_equal(a.sigmas, b.sigmas)
    assert np.array_equal(a.modes, b.modes)


def test_gramian_public():
    rng = np.random.default_rng(11)
    w = rng.uniform(0.1, 3.0, 6)
    vals = rng.standard_normal((6, 5))
    g = H.gramian(H.SnapshotBlock(H.InnerProductSpace(6, w), vals))
    ref = vals.T @ (w[:, None] * vals)
    assert np.max(np.abs(g - ref)) < 1e-12
    assert np.array_equal(g, g.T)


def test_deferred_upload_matches_eager_and_checks_finiteness():
    vals = O.synthetic_decay(500, 256, 0.05, seed=3)
    sp = euclid(500)
    host = torch.from_numpy(np.asfortranarray(vals).T.copy()).pin_memory().t()  # column-major pinned
    tree = H.build_star(4)
    eager = H.distribute_columns(tree, H.SnapshotBlock(sp, vals))
    lazy = H.distribute_columns(tree, H.SnapshotBlock(sp, host, defer_upload=True))
    tol = H.assign_tolerances(tree, eager, 1e-3, omega=0.75)
    a = H.run_hapod(tree, eager, tol)
    b, _ = H.run_parallel(tree, lazy, tol, worker_count=4)
    assert np.array_equal(a.modes.sigmas, b.modes.sigmas)
    assert np.array_equal(a.modes.modes, b.modes.modes)
    bad = np.array(vals)
    bad[3, 7] = np.inf
    blk = H.SnapshotBlock(sp, bad, defer_upload=True)  # no check yet
    with pytest.raises(ValueError):
        H.pod(blk, 0.1)


@pytest.mark.parametrize("weighted", [False, True])
@pytest.mark.parametrize("d,p,q", [(1, 1, 1), (37, 5, 9), (5000, 64, 130), (20000, 3, 1)])
def test_space_gram_and_norms(weighted, d, p, q):
    """InnerProductSpace.gram / .norms_sq (pod.py:87-97) on the device vs the reference
    arithmetic (oracle ip_gram / ip_norms_sq): host operands in, NumPy out; device in, device out."""
    rng = np.random.default_rng(d + p + q)
    w = rng.uniform(0.5, 2.0, d) if weighted else None
    sp = H.InnerProductSpace(d, w)
    a = rng.standard_normal((d, p))
    b = rng.standard_normal((d, q))
    g = sp.gram(a, b)
    assert isinstance(g, np.ndarray) and g.shape == (p, q)
    ref = O.ip_gram(a, b, w)
    assert np.allclose(g, ref, rtol=1e-13, atol=1e-13 * math.sqrt(d))
    ns = sp.norms_sq(a)
    assert isinstance(ns, np.ndarray) and ns.shape == (p,)
    assert np.allclose(ns, O.ip_norms_sq(a, w), rtol=1e-13)
    gd = sp.gram(torch.from_numpy(a).cuda(), torch.from_numpy(b).cuda())
    assert gd.is_cuda and np.allclose(gd.cpu().numpy(), ref, rtol=1e-13, atol=1e-13 * math.sqrt(d))
    assert np.allclose(sp.norms_sq(torch.from_numpy(a).cuda()).cpu().numpy(), O.ip_norms_sq(a, w), rtol=1e-13)


def test_space_gram_rejects_mismatched_rows():
    sp = H.InnerProductSpace(10)
    with pytest.raises(ValueError):
        sp.gram(np.ones((10, 2)), np.ones((11, 2)))


def test_tridiagonal_path_at_pod_level_and_its_fallback():
    """pod() with the tridiagonal H-phase solver forced on small nodes (production threshold: order
    1,024): same counts / sigma / span as the oracle (pod.py:296-348); a block with two repeated
    singular values makes the solver decline and the block Jacobi take over."""
    from paper_1607_05210_b200 import _device as D
    rng = np.random.default_rng(11)
    d, m = 3000, 400
    q1, _ = np.linalg.qr(rng.standard_normal((d, m)))
    q2, _ = np.linalg.qr(rng.standard_normal((m, m)))
    vals = (q1 * 10.0 ** (-7.0 * np.arange(m) / (m - 1))) @ q2.T
    saved = D.TRI_MIN_ORDER
    try:
        D.TRI_MIN_ORDER = 8
        D.LAST_TRI_DIAG.clear()
        eps = 1e-5 * float(np.linalg.norm(vals))
        out = H.pod(H.SnapshotBlock(euclid(d), vals), eps)
        assert D.LAST_TRI_DIAG.get("status") == 0 and D.LAST_TRI_DIAG["count"] > 100
        ref = O.pod(vals, eps)
        assert out.count == ref.count
        # method-of-snapshots floor of a singular value: u * (sigma_1 / sigma_i)^2 (cf. the MGS golden test)
        floor = 2.2e-16 * (ref.sigmas[0] / ref.sigmas) ** 2
        assert np.all(np.abs(out.sigmas - ref.sigmas) / ref.sigmas <= np.maximum(1e-10, 10 * floor))
        assert angles(out.modes, ref.modes).max() < 1e-6
        # one repeated singular value: the shift next to it resolves the cluster (MRRR's own device)
        D.LAST_TRI_DIAG.clear()
        out = H.pod(H.SnapshotBlock(euclid(d), q1[:, :200]), 0.5)
        assert out.count == 200 and np.allclose(out.sigmas, 1.0, rtol=1e-12)
        # two repeated singular values: the cluster away from the shift has no relative gaps left,
        # the solver declines (status 1) and the block Jacobi takes over
        D.LAST_TRI_DIAG.clear()
        two = np.hstack([2.0 * q1[:, :100], q1[:, 100:200]])
        out = H.pod(H.SnapshotBlock(euclid(d), two), 0.5)
        assert D.LAST_TRI_DIAG.get("status") == 1
        ref = O.pod(two, 0.5)
        assert out.count == ref.count == 200
        assert np.allclose(out.sigmas, ref.sigmas, rtol=1e-12)
        g = out.modes.T @ out.modes
        assert np.max(np.abs(g - np.eye(200))) < 1e-10
    finally:
        D.TRI_MIN_ORDER = saved
