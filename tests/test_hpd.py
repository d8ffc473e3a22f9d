"""`.hpd` container ingest/egest (paper_1607_05210_b200.hpd) against fixtures written by the
unmodified reference writer (tests/golden/make_hpd_golden.py, io.py:38-51, 128-133).

CPU: the writer reproduces the reference bytes exactly; header/format errors raise
MatrixFormatError like io.py:54-66.  GPU: device ingest (pinned read + one H2D copy), streamed
column blocks into the incremental driver, leaf streaming into run_hapod_streaming, and device
egest of a ModeSet that reads back bit for bit."""

import os
import struct

import numpy as np
import pytest

from paper_1607_05210_b200 import hpd

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def hpd_inputs():
    a = np.arange(35, dtype=np.float64).reshape(7, 5) / 7.0 - 2.0
    a[0, 0] = -0.0
    a[3, 2] = 1e-310
    a[6, 4] = -1.7976931348623157e308
    w = np.linspace(0.5, 2.0, 7)
    s = np.array([3.0, 1.0 / 3.0, 1e-300, 2.0 ** -1074, 0.1])
    return a, w, s


def test_writer_bytes_identical_to_reference(tmp_path):
    a, w, s = hpd_inputs()
    hpd.write_matrix(tmp_path / "p.hpd", a)
    hpd.write_matrix(tmp_path / "w.hpd", a, w)
    hpd.write_floats(tmp_path / "s.txt", s)
    assert (tmp_path / "p.hpd").read_bytes() == open(os.path.join(GOLD, "hpd_plain.hpd"), "rb").read()
    assert (tmp_path / "w.hpd").read_bytes() == open(os.path.join(GOLD, "hpd_weighted.hpd"), "rb").read()
    assert (tmp_path / "s.txt").read_text() == open(os.path.join(GOLD, "hpd_sigmas.txt")).read()
    back = hpd.read_floats(os.path.join(GOLD, "hpd_sigmas.txt"))
    assert np.array_equal(back.view(np.uint64), s.view(np.uint64))


def test_header_and_errors(tmp_path):
    assert hpd.read_matrix_header(os.path.join(GOLD, "hpd_plain.hpd")) == (7, 5, False)
    assert hpd.read_matrix_header(os.path.join(GOLD, "hpd_weighted.hpd")) == (7, 5, True)
    bad = tmp_path / "bad.hpd"
    bad.write_bytes(b"XXXX" + bytes(19))
    with pytest.raises(hpd.MatrixFormatError, match="bad magic"):
        hpd.read_matrix_header(bad)
    bad.write_bytes(struct.pack("<4sHQQB", b"HPD1", 2, 1, 1, 0))
    with pytest.raises(hpd.MatrixFormatError, match="version"):
        hpd.read_matrix_header(bad)
    bad.write_bytes(b"HPD1")
    with pytest.raises(hpd.MatrixFormatError, match="truncated"):
        hpd.read_matrix_header(bad)
    with pytest.raises(ValueError):
        hpd.write_matrix(tmp_path / "x.hpd", np.zeros(3))


torch = pytest.importorskip("torch")


@pytest.mark.gpu
def test_device_ingest_egest_roundtrip(tmp_path):
    if not torch.cuda.is_available():  # pragma: no cover
        pytest.skip("no CUDA device")
    import paper_1607_05210_b200 as H
    a, w, _ = hpd_inputs()
    a[6, 4] = 1.0  # the reference's SnapshotBlock rejects nothing finite; keep the block well scaled
    hpd.write_matrix(tmp_path / "w.hpd", a, w)
    blk = hpd.load_snapshots(tmp_path / "w.hpd")
    assert blk.space.weights is not None and np.array_equal(blk.space.weights, w)
    assert np.array_equal(blk.values.view(np.uint64), a.view(np.uint64))
    rng = np.random.default_rng(1)
    s = rng.standard_normal((3000, 700))
    hpd.write_matrix(tmp_path / "s.hpd", s)
    out = H.pod(hpd.load_snapshots(tmp_path / "s.hpd"), 1e-3 * np.linalg.norm(s))
    hpd.write_matrix(tmp_path / "modes.hpd", out)
    hpd.write_floats(tmp_path / "sigmas.txt", out.sigmas)
    back = hpd.load_snapshots(tmp_path / "modes.hpd")
    assert np.array_equal(back.values, out.modes)
    assert np.array_equal(hpd.read_floats(tmp_path / "sigmas.txt"), out.sigmas)


@pytest.mark.gpu
def test_streamed_file_drivers(tmp_path):
    """A snapshot file streamed block by block into the incremental session and leaf by leaf
    into run_hapod_streaming gives the same results as the in-memory drivers."""
    if not torch.cuda.is_available():  # pragma: no cover
        pytest.skip("no CUDA device")
    import paper_1607_05210_b200 as H
    from oracle import hapod_oracle as O
    vals = O.synthetic_decay(2000, 6 * 256, 0.02, seed=5)
    hpd.write_matrix(tmp_path / "S.hpd", vals)
    sp = H.InnerProductSpace(2000)
    target = 1e-3
    sess = H.incremental_open(target, 0.9, 6)
    for blk in hpd.iter_column_blocks(tmp_path / "S.hpd", 256):
        sess.push(blk)
    streamed = sess.finalize()
    sess = H.incremental_open(target, 0.9, 6)
    for j in range(6):
        sess.push(H.SnapshotBlock(sp, vals[:, 256 * j: 256 * (j + 1)]))
    direct = sess.finalize()
    assert np.array_equal(streamed.modes.sigmas, direct.modes.sigmas)
    assert np.array_equal(streamed.modes.modes, direct.modes.modes)
    tree = H.build_star(6)
    source, counts = hpd.leaf_source(tmp_path / "S.hpd", tree, 256)
    tol = H.assign_tolerances(tree, counts, target, omega=0.75)
    res_s = H.run_hapod_streaming(tree, source, counts, tol)
    leaves = H.distribute_columns(tree, H.SnapshotBlock(sp, vals), block_size=256)
    res_d = H.run_hapod(tree, leaves, tol)
    assert np.array_equal(res_s.modes.sigmas, res_d.modes.sigmas)
    assert np.array_equal(res_s.modes.modes, res_d.modes.modes)
