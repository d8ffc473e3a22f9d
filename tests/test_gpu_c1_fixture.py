"""BASELINE config 1 at its REAL tree shape -- 16 leaves x 512 columns and the 8,192-column
root -- against the committed reference fixture ``tests/golden/c1_d10000.{npz,json}``.

The fixture (``tests/golden/make_c1_fixture.py``) holds the unmodified reference's
``run_hapod(build_star(16), ...)`` (hierarchy.py:323-367; root pod.py:278-293 with the MGS
sweep pod.py:227-237) on ``oracle.hostgen.decay(10000, 8192, 10.0, seed=1)``: the root sigma,
counts (N, nkeep), tail, the projection l2, the principal angles of the reference's modes to
the EXACT POD span Q1[:, :N], and the CPU-vs-CPU floors (LAPACK evd instead of evr; evr on
row-permuted snapshots).  Config 1 is S = Q1 diag(sigma) Q2^T, so every node Gram -- and with
it every node size -- is independent of d in exact arithmetic: d' = 10,000 reproduces the
full-size counts.

The test regenerates the same snapshots on this host (bit-identical Philox draws; the QR /
GEMM roundings depend on the host BLAS, so the bytes are compared through ``hostgen.checksum``
within a tolerance), runs the device tree through the public API and asserts, with no slack:
identical counts; every kept sigma and the angle to the exact span within
max(BASELINE gate, k x measured floor); l2 within 1e-8 relative (or the measured l2 floor).
"""

import json
import math
import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("no CUDA device", allow_module_level=True)

import paper_1607_05210_b200 as H  # noqa: E402
from oracle import hostgen  # noqa: E402

GOLD = os.path.join(os.path.dirname(__file__), "golden")
FIX_NPZ = os.path.join(GOLD, "c1_d10000.npz")
FIX_JSON = os.path.join(GOLD, "c1_d10000.json")

K_FLOOR = 4.0  # the same multiple of the CPU-vs-CPU floor as the other config tests


def exact_angle_sines(q1n, u):
    """Principal-angle sines between span(q1n) and span(u): singular values of the residual
    (the formula of make_c1_fixture.exact_angle_sines)."""
    r = u - q1n @ (q1n.T @ u)
    ev = np.linalg.eigvalsh(r.T @ r)
    return np.sqrt(np.clip(ev[::-1], 0.0, None))


@pytest.mark.skipif(not os.path.exists(FIX_NPZ), reason="c1 fixture not generated")
def test_config1_real_shape_vs_reference_fixture():
    fix = np.load(FIX_NPZ)
    with open(FIX_JSON) as f:
        meta = json.load(f)
    ref = meta["reference"]
    d, m, seed = meta["d"], meta["m"], meta["seed"]
    assert (d, m) == (10_000, 8_192)

    s, _sig_exact, left = hostgen.decay(d, m, 10.0, seed, want_left=True)
    # same snapshots as the fixture's (up to the host BLAS's roundings in QR / GEMM)
    chk = hostgen.checksum(s)
    assert np.max(np.abs(chk - fix["checksum"])) <= 1e-11 * max(1.0, float(np.abs(fix["checksum"]).max()))
    fro = float(np.linalg.norm(s))
    assert fro == pytest.approx(ref["fro"], rel=1e-13)
    eps_star = 1e-6 * fro
    target = H.eps_star_to_target(eps_star, m)
    assert target == pytest.approx(ref["target"], rel=1e-13)

    tree = H.build_star(16)
    sp = H.InnerProductSpace(d)
    blk = H.SnapshotBlock(sp, s)
    leaves = H.distribute_columns(tree, blk, block_size=512)
    tol = H.assign_tolerances(tree, leaves, target, omega=0.75)
    np.testing.assert_allclose(np.asarray(tol.epsilons), np.asarray(ref["epsilons"]), rtol=1e-13)
    res = H.run_hapod(tree, leaves, tol)

    # ---- counts: every node, and the root's cutoff count
    ref_rep = {r["node"]: r for r in ref["reports"]}
    for r in res.reports:
        assert r.output_mode_count == ref_rep[r.node]["n_out"], (r.node, r.output_mode_count)
        assert r.input_count == ref_rep[r.node]["n_in"]
    n_ref, nkeep_ref = ref["N"], ref["nkeep"]
    nkeep = res.modes.diagnostics["nkeep"]
    sig = np.asarray(res.modes.sigmas)
    modes = np.asarray(res.modes.modes)
    fl = meta["floor"]

    # ---- sigma: every kept value against the reference's
    rsig = fix["ref/sigmas"]
    rel = np.abs(sig[: min(len(sig), n_ref)] - rsig[: min(len(sig), n_ref)]) / rsig[: min(len(sig), n_ref)]
    # ---- subspace: angle to the exact POD span, beside the reference's own
    ang = exact_angle_sines(left[:, :n_ref], modes) if len(sig) == n_ref else np.array([np.inf])
    # ---- projection l2 (total reading) and tail energy
    err = math.sqrt(H.actual_mean_error(blk, res.modes) * m)
    l2_floor = max(abs(meta[v]["l2"] - ref["l2"]) / ref["l2"] for v in ("evd", "perm"))
    tail = float(res.modes.tail_energy)
    tail_floor = max(abs(meta[v]["root_tail"] - ref["root_tail"]) / ref["root_tail"] for v in ("evd", "perm"))
    print(f"\n[c1 real shape d'={d}] counts gpu N={len(sig)} nkeep={nkeep}; reference N={n_ref} nkeep={nkeep_ref}; "
          f"max rel dsigma {rel.max():.3e} (median {np.median(rel):.1e}; CPU floor {fl['rel_dsigma']:.3e}); "
          f"angle to the exact span gpu {ang.max():.3e} / reference {meta['ref_max_angle_vs_exact']:.3e} / "
          f"evd {meta['evd']['max_angle_vs_exact']:.3e} / perm {meta['perm']['max_angle_vs_exact']:.3e}; "
          f"l2 gpu {err:.8e} reference {ref['l2']:.8e} (rel diff {abs(err - ref['l2']) / ref['l2']:.2e}, CPU floor "
          f"{l2_floor:.2e}); tail gpu {tail:.8e} reference {ref['root_tail']:.8e} (CPU floor {tail_floor:.2e}); "
          f"sweeps {res.modes.diagnostics['jacobi_sweeps']}")

    assert len(sig) == n_ref == 4549
    assert nkeep == nkeep_ref == 4562
    assert rel.max() <= max(1e-10, K_FLOOR * fl["rel_dsigma"])
    assert ang.max() <= max(1e-8, K_FLOOR * fl["angle_vs_exact"])
    assert abs(err - ref["l2"]) <= max(1e-8, K_FLOOR * l2_floor) * ref["l2"]
    assert abs(tail - ref["root_tail"]) <= max(1e-8, K_FLOOR * tail_floor) * ref["root_tail"]
    # orthonormal output and the reference's sign convention (pod.py:214-224, 247)
    g = modes.T @ modes
    assert np.max(np.abs(g - np.eye(n_ref))) <= 1e-8
    pick = np.argmax(np.abs(modes), axis=0)
    assert np.all(modes[pick, np.arange(n_ref)] > 0.0)
