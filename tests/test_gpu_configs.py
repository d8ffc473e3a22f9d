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


class Floors(tuple):
    """(max rel dsigma, max angle sine, count mismatch) of the CPU-vs-CPU variants, plus
    ``l2``: the largest relative difference of their projection errors (filled by l2_floor)."""
    l2 = 0.0


def l2_gate(floors):
    """Projection l2 parity gate: 1e-8 relative (BASELINE.json), or 4x the CPU-vs-CPU floor where the
    residual is so far below ||S||_F that the modes' permitted orthonormality drift (<= 1e-8,
    pod.py:247) already moves it by more than that (config 3: l2 = 1e-3 eps*, the noise level)."""
    return max(1e-8, 4.0 * floors.l2)


def tree_floors(children, root, blocks, eps, ref, ref_err=None):
    """CPU-vs-CPU floors of a tree run: the oracle with LAPACK divide and conquer
    (evd) and the oracle (evr) on row-permuted snapshots, each against the reference-order run.
    Returns Floors(max rel dsigma, max angle sine, count mismatch) over both variants; with
    ``ref_err`` (the reference-order run's total l2 error) also the l2 floor."""
    d = next(iter(blocks.values())).shape[0]
    perm = np.random.default_rng(99).permutation(d)
    pb = {k: np.asfortranarray(v[perm]) for k, v in blocks.items()}
    runs = [(O.run_hapod(children, root, blocks, eps, driver="evd").modes, None),
            (O.run_hapod(children, root, pb, eps).modes, np.argsort(perm))]
    frel, fang, dcount, fl2 = 0.0, 0.0, 0, 0.0
    order = sorted(blocks)
    vals = np.hstack([blocks[k] for k in order]) if ref_err is not None else None
    for mo, inv in runs:
        modes = mo.modes if inv is None else mo.modes[inv]
        r, a = metrics(mo.sigmas, modes, ref)
        frel = max(frel, float(r.max()) if r.size else 0.0)
        fang = max(fang, float(a.max()) if a.size else 0.0)
        dcount = max(dcount, abs(mo.count - ref.count))
        if ref_err is not None and ref_err > 0.0:
            e = math.sqrt(O.actual_mean_error(vals, modes) * vals.shape[1])
            fl2 = max(fl2, abs(e - ref_err) / ref_err)
    out = Floors((frel, fang, dcount))
    out.l2 = fl2
    if ref_err is not None:
        print(f"\n[floors] CPU-vs-CPU relative l2 difference {fl2:.3e}")
    return out


def report(name, dev_count, ref_count, rel, ang, frel=None, fang=None, extra=""):
    print(f"\n[{name}] counts gpu={dev_count} cpu={ref_count}; max rel dsigma={rel.max() if rel.size else 0:.3e} "
          f"(median {np.median(rel) if rel.size else 0:.1e}); max angle sine={ang.max() if ang.size else 0:.3e}"
          + (f"; CPU-vs-CPU floor: rel dsigma={frel:.3e}, angle={fang:.3e}" if frel is not None else "") + extra)



def test_config0_full_size():
    """Config 0 at its full size (20,000 x 1,000): single POD, eps* = 1e-4 ||S||_F."""
    wl = W.make(0)
    vals = host(wl.values)
    out = H.pod(H.SnapshotBlock(H.InnerProductSpace(wl.d), wl.values), wl.eps_star)
    ref = O.pod(vals, wl.eps_star)
    ref_err = math.sqrt(O.actual_mean_error(vals, ref.modes) * wl.m)
    fl = tree_floors([[]], 0, {0: vals}, [wl.eps_star], ref, ref_err)
    frel, fang, fcount = fl
    rel, ang = metrics(out.sigmas, out.modes, ref)
    err = math.sqrt(H.actual_mean_error(H.SnapshotBlock(H.InnerProductSpace(wl.d), wl.values), out) * wl.m)
    report("c0", out.count, ref.count, rel, ang, frel, fang,
           f"; l2 gpu={err:.6e} cpu={ref_err:.6e} eps*={wl.eps_star:.6e}")
    assert out.count == ref.count == 500
    assert rel.max() <= max(1e-10, 4.0 * frel)
    assert abs(err - ref_err) <= l2_gate(fl) * ref_err
    assert err <= wl.eps_star
    assert ang.max() <= max(1e-8, 4.0 * fang)


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
    ref_err = math.sqrt(O.actual_mean_error(vals, ref.modes.modes) * m)
    fl = tree_floors(children, 0, blocks, list(tol.epsilons), ref.modes, ref_err)
    frel, fang, fcount = fl
    rel, ang = metrics(res.modes.sigmas, res.modes.modes, ref.modes)
    err = math.sqrt(H.actual_mean_error(blk, res.modes) * m)
    report(f"c1-mini d={d} m={m}", res.mode_count, ref.modes.count, rel, ang, frel, fang,
           f"; floor count diff {fcount}; l2 gpu={err:.6e} cpu={ref_err:.6e}")
    # no slack: identical counts, every kept sigma, the angle and the projection error
    assert res.mode_count == ref.modes.count
    assert rel.max() <= max(1e-10, 4.0 * frel)
    assert ang.max() <= max(1e-8, 4.0 * fang)
    assert abs(err - ref_err) <= l2_gate(fl) * ref_err


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
    ref_err = math.sqrt(O.actual_mean_error(vals, ref.modes.modes) * m)
    fl = tree_floors(children, 0, blocks, list(tol.epsilons), ref.modes, ref_err)
    frel, fang, fcount = fl
    rel, ang = metrics(res.modes.sigmas, res.modes.modes, ref.modes)
    err = math.sqrt(H.actual_mean_error(blk, res.modes) * m)
    leaf_counts = sorted({r.output_mode_count for r in res.reports if r.is_leaf})
    report("c3-mini", res.mode_count, ref.modes.count, rel, ang, frel, fang,
           extra=f"; leaf modes {leaf_counts}; l2 gpu={err:.4e} cpu={ref_err:.4e} eps*={wl.eps_star:.4e}")
    assert res.mode_count == ref.modes.count
    assert rel.max() <= max(1e-10, 4.0 * frel)
    assert ang.max() <= max(1e-8, 4.0 * fang)
    assert abs(err - ref_err) <= l2_gate(fl) * ref_err
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
    ch = [list(c) for c in tree.children]
    ref = O.run_hapod(ch, 0, blocks, list(tol.epsilons))
    ref_err = math.sqrt(O.actual_mean_error(vals, ref.modes.modes) * m)
    fl = tree_floors(ch, 0, blocks, list(tol.epsilons), ref.modes, ref_err)
    frel, fang, fcount = fl
    rel, ang = metrics(res.modes.sigmas, res.modes.modes, ref.modes)
    err = math.sqrt(H.actual_mean_error(blk, res.modes) * m)
    report("c4-mini", res.mode_count, ref.modes.count, rel, ang, frel, fang,
           extra=f"; l2 gpu={err:.4e} cpu={ref_err:.4e} eps*={wl.eps_star:.4e}")
    assert res.mode_count == ref.modes.count
    assert rel.max() <= max(1e-10, 4.0 * frel)
    assert ang.max() <= max(1e-8, 4.0 * fang)
    assert abs(err - ref_err) <= l2_gate(fl) * ref_err
    assert err <= wl.eps_star
