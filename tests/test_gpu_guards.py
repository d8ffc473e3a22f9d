"""Out-of-bounds-write and uninitialised-read detection for the whole node pipeline without
compute-sanitizer (closed on this pool): every matrix and kernel workspace is allocated between
4 KB canary zones with a poisoned payload (``_device.Guards``), the hot path runs on shapes that
exercise every kernel's edge handling (odd sizes, partial tiles, split-K, narrow n tiles, CholQR,
block Gram, stream workers), results are checked against the oracle (a consumed poison NaN
would show), and every canary word must be intact afterwards."""

import math

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("no CUDA device", allow_module_level=True)

import paper_1607_05210_b200 as H  # noqa: E402
from paper_1607_05210_b200 import _device as D  # noqa: E402
from oracle import hapod_oracle as O  # noqa: E402


@pytest.fixture()
def guards():
    D.Guards.enable()
    try:
        yield D.Guards
    finally:
        D.Guards.disable()


def _decay(d, m, decades, seed):
    rng = np.random.default_rng(seed)
    q1, _ = np.linalg.qr(rng.standard_normal((d, m)))
    q2, _ = np.linalg.qr(rng.standard_normal((m, m)))
    sig = 10.0 ** (-decades * np.arange(m) / max(m - 1, 1))
    return np.asfortranarray((q1 * sig) @ q2.T)


@pytest.mark.parametrize("d,m,decades,rel", [(1501, 301, 4.0, 1e-3), (3000, 520, 9.0, 1e-7), (777, 65, 2.0, 1e-2),
                                             (20011, 130, 6.0, 1e-5)])
def test_pod_pipeline_under_guards(guards, d, m, decades, rel):
    vals = _decay(d, m, decades, seed=m)
    eps = rel * float(np.linalg.norm(vals))
    out = H.pod(H.SnapshotBlock(H.InnerProductSpace(d), vals), eps, want_right=True)
    ref = O.pod(vals, eps)
    assert out.count == ref.count
    assert np.all(np.isfinite(out.sigmas)) and np.all(np.isfinite(np.asarray(out.modes)))
    assert np.allclose(out.sigmas, ref.sigmas, rtol=1e-8)
    modes = np.asarray(out.modes)
    if decades <= 6.0:
        assert O.principal_angle_sines(modes, ref.modes).max() < 1e-6
    else:  # boundary modes of a 9-decade spectrum sit at the method-of-snapshots floor: compare the error
        e_dev = np.linalg.norm(vals - modes @ (modes.T @ vals))
        e_ref = np.linalg.norm(vals - ref.modes @ (ref.modes.T @ vals))
        assert abs(e_dev - e_ref) <= 1e-6 * e_ref
    assert np.max(np.abs(modes.T @ modes - np.eye(out.count))) <= 1e-8
    assert guards.check() > 10


def test_chain_star_and_merge_under_guards(guards):
    d, nl, lc = 2500, 6, 70
    vals = _decay(d, nl * lc, 5.0, seed=9)
    sp = H.InnerProductSpace(d)
    target = 1e-4 * float(np.linalg.norm(vals)) / math.sqrt(nl * lc)
    # star on stream workers
    tree = H.build_star(nl)
    leaves = H.distribute_columns(tree, H.SnapshotBlock(sp, vals), block_size=lc)
    tol = H.assign_tolerances(tree, leaves, target, omega=0.75)
    res, _ = H.run_parallel(tree, leaves, tol, worker_count=3)
    order = H.derive_maps(tree).leaf_order
    blocks = {leaf: vals[:, lc * i: lc * (i + 1)] for i, leaf in enumerate(order)}
    ref = O.run_hapod([list(c) for c in tree.children], 0, blocks, list(tol.epsilons))
    assert res.mode_count == ref.modes.count
    assert np.allclose(res.modes.sigmas, ref.modes.sigmas, rtol=1e-8)
    # incremental session: passthrough, plain pod of the join, block-Gram merges (narrow n tiles)
    sess = H.incremental_open(target, 0.9, nl)
    for j in range(nl):
        sess.push(H.SnapshotBlock(sp, vals[:, lc * j: lc * (j + 1)]))
    out = sess.finalize()
    cur, _, _ = O.incremental([vals[:, lc * j: lc * (j + 1)] for j in range(nl)], target, 0.9)
    assert out.mode_count == cur.count
    assert np.allclose(out.modes.sigmas, cur.sigmas, rtol=1e-8)
    assert np.all(np.isfinite(np.asarray(out.modes.modes)))
    assert guards.check() > 50


def test_guards_detect_an_out_of_bounds_write(guards):
    """The detector itself: a deliberate write one element past a guarded matrix must be caught."""
    M = D.DevMat.empty(10, 3)
    n = M.ld * M.cols
    raw = M.storage
    # one double past the payload (inside the tail canary zone)
    past = torch.as_strided(raw, (1,), (1,), raw.storage_offset() + n)
    past.fill_(1.0)
    with pytest.raises(AssertionError):
        guards.check()
