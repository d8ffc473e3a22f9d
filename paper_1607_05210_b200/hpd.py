"""`.hpd` snapshot / mode container ingest and egest for the B200 path.

The reference's binary container (io.py:1-146): a little-endian header
``<4sHQQB`` = magic ``HPD1``, version 1, rows u64, cols u64, weight flag u8; then the
``rows`` inner-product weights when flagged; then the payload as COLUMN-MAJOR float64.
Column-major float64 with contiguous columns is exactly the device layout of this package
(_device.DevMat), so ingest is one pinned-host read and one host->device copy per block,
and egest one device->host copy and one write -- no transposes, no per-element work.

  read_matrix_header(path)             -> (rows, cols, weighted)            (io.py:71-74)
  load_snapshots(path)                 -> SnapshotBlock on the device       (io.py:114-125)
  iter_column_blocks(path, block)      -> SnapshotBlocks of <= block columns (io.py:95-111)
  leaf_source(path, tree, block_size)  -> leaf_source for run_hapod_streaming: leaf i of the
                                          DFS order reads columns [i*block, (i+1)*block)
  write_matrix(path, modes, weights)   -> byte-identical to io.write_matrix (io.py:38-51)
  write_floats / read_floats           -> sigmas.txt, repr per line (io.py:128-146)

Files written here are read by the reference and vice versa (tests/test_hpd.py checks the
bytes against fixtures written by the unmodified reference).
"""

from __future__ import annotations

import struct

import numpy as np

from .pod import InnerProductSpace, ModeSet, SnapshotBlock

__all__ = ["MatrixFormatError", "read_matrix_header", "load_snapshots", "iter_column_blocks", "leaf_source",
           "write_matrix", "write_floats", "read_floats"]

MAGIC = b"HPD1"
VERSION = 1
_HEADER = struct.Struct("<4sHQQB")


class MatrixFormatError(ValueError):
    """File does not parse as the binary matrix container (io.py:34-35)."""


def _parse(raw: bytes, path):
    if len(raw) < _HEADER.size:
        raise MatrixFormatError(f"{path}: truncated header")
    magic, version, rows, cols, flag = _HEADER.unpack(raw[:_HEADER.size])
    if magic != MAGIC:
        raise MatrixFormatError(f"{path}: bad magic {magic!r}, not a matrix container")
    if version != VERSION:
        raise MatrixFormatError(f"{path}: unsupported container version {version}")
    if flag not in (0, 1):
        raise MatrixFormatError(f"{path}: bad weight flag {flag}")
    return int(rows), int(cols), bool(flag)


def read_matrix_header(path):
    with open(path, "rb") as fh:
        return _parse(fh.read(_HEADER.size), path)


def _open_payload(path):
    fh = open(path, "rb")
    rows, cols, weighted = _parse(fh.read(_HEADER.size), path)
    weights = None
    if weighted:
        wbuf = fh.read(8 * rows)
        if len(wbuf) != 8 * rows:
            fh.close()
            raise MatrixFormatError(f"{path}: truncated weight vector")
        weights = np.frombuffer(wbuf, dtype="<f8").copy()
    return fh, rows, cols, weights, fh.tell()


def _pinned(rows: int, cols: int):
    import torch
    return torch.empty((max(cols, 0), rows), dtype=torch.float64, pin_memory=torch.cuda.is_available())


def _read_cols(fh, path, buf, rows: int, ncols: int, first_col: int):
    view = buf[:ncols].numpy().reshape(-1).view(np.uint8)
    got = fh.readinto(memoryview(view))
    if got != 8 * rows * ncols:
        raise MatrixFormatError(f"{path}: payload ends early at column {first_col + got // (8 * max(rows, 1))}")


def load_snapshots(path) -> SnapshotBlock:
    """The whole container as a device SnapshotBlock (weights -> a weighted space).  The
    column-major payload is read into pinned host memory and copied to the device in one
    transfer (the device finiteness check of SnapshotBlock runs as usual)."""
    fh, rows, cols, weights, _ = _open_payload(path)
    with fh:
        buf = _pinned(rows, cols)
        _read_cols(fh, path, buf, rows, cols, 0)
        if fh.read(1):
            raise MatrixFormatError(f"{path}: payload longer than {rows}x{cols}")
    return SnapshotBlock(InnerProductSpace(rows, weights), buf.t())


def iter_column_blocks(path, block: int, space: InnerProductSpace | None = None):
    """Stream the payload in blocks of ``block`` columns (the last may be shorter), each
    read into a pinned buffer and uploaded as a device SnapshotBlock -- the incremental
    driver's input (``IncrementalSession.push``) straight from disk."""
    if block < 1:
        raise ValueError("block must be positive")
    fh, rows, cols, weights, _ = _open_payload(path)
    space = space or InnerProductSpace(rows, weights)
    with fh:
        buf = _pinned(rows, block)
        done = 0
        while done < cols:
            take = min(block, cols - done)
            _read_cols(fh, path, buf, rows, take, done)
            yield SnapshotBlock(space, buf[:take].t())
            done += take


def leaf_source(path, tree, block_size: int, space: InnerProductSpace | None = None):
    """(leaf_source, leaf_counts) for ``run_hapod_streaming``: leaf i in depth-first order
    holds columns [i*block_size, ...) of the file (distribute_columns, hierarchy.py:141-179),
    read on demand with one seek + one pinned read."""
    from .tree import derive_maps
    fh, rows, cols, weights, data0 = _open_payload(path)
    fh.close()
    space = space or InnerProductSpace(rows, weights)
    order = derive_maps(tree).leaf_order
    if block_size * (len(order) - 1) >= cols or block_size * len(order) < cols:
        raise ValueError(f"{cols} columns do not split into {len(order)} leaves of {block_size}")
    first = {leaf: i * block_size for i, leaf in enumerate(order)}
    counts = {leaf: min(block_size, cols - first[leaf]) for leaf in order}

    def source(v):
        n = counts[v]
        buf = _pinned(rows, n)
        with open(path, "rb") as f:
            f.seek(data0 + 8 * rows * first[v])
            _read_cols(f, path, buf, rows, n, first[v])
        return SnapshotBlock(space, buf.t())

    return source, counts


def write_matrix(path, values, weights=None) -> None:
    """io.write_matrix (io.py:38-51) for NumPy arrays, SnapshotBlocks and device ModeSets:
    a ModeSet's modes come back with one device->host copy of its column-major storage."""
    if isinstance(values, ModeSet):
        mat = values.modes_device()
        rows, cols = mat.rows, mat.cols
        payload = None
        if cols and rows:
            st = mat.storage[mat.offset: mat.offset + mat.ld * cols].view(cols, mat.ld)[:, :rows]
            payload = st.cpu().numpy()          # (cols, rows) C-order == column-major bytes
    else:
        if isinstance(values, SnapshotBlock):
            values = values.values
        values = np.asarray(values, dtype=np.float64)
        if values.ndim != 2:
            raise ValueError(f"matrix must be 2-d, got shape {values.shape}")
        rows, cols = values.shape
        payload = np.ascontiguousarray(values.T, dtype="<f8")
    with open(path, "wb") as fh:
        fh.write(_HEADER.pack(MAGIC, VERSION, rows, cols, 0 if weights is None else 1))
        if weights is not None:
            w = np.asarray(weights, dtype="<f8")
            if w.shape != (rows,):
                raise ValueError(f"weights shape {w.shape} does not match {rows} rows")
            fh.write(w.tobytes())
        if payload is not None:
            fh.write(np.ascontiguousarray(payload, dtype="<f8").tobytes())


def write_floats(path, values) -> None:
    """One float per line, shortest round-trip repr (io.py:128-133)."""
    with open(path, "w") as fh:
        for v in np.asarray(values, dtype=np.float64).reshape(-1):
            fh.write(repr(float(v)))
            fh.write("\n")


def read_floats(path) -> np.ndarray:
    out = []
    with open(path) as fh:
        for ln, line in enumerate(fh, start=1):
            line = line.strip()
            if not line:
                continue
            try:
                out.append(float(line))
            except ValueError:
                raise ValueError(f"{path}:{ln}: not a float: {line!r}") from None
    return np.asarray(out, dtype=np.float64)
