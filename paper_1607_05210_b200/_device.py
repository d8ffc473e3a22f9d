"""Device-side data layout and the per-node POD pipeline on the B200.

Layout in HBM: every snapshot or mode block is a column-major float64 matrix
whose column stride ``ld`` is ``rows`` rounded up to an even count (16-byte
aligned columns, so the GEMM engine can use 16-byte async copies).  Storage
is a torch tensor of shape (cols, ld) -- torch is used for allocation and
streams only; every arithmetic step is a kernel of libhapod_b200.so.

A node's input is a list of *parts* (DevMat, optional per-column scale).  The
concatenation is never materialised: the Gram and reconstruction kernels read
the columns through a device pointer table, and the sigma scaling of
ModeSet.scaled() (pod.py:160-162) is applied as an epilogue scale (Gram) or
folded into the eigenvector rows (reconstruction).
"""

from __future__ import annotations

import ctypes
import math
import threading
from dataclasses import dataclass

import numpy as np

from . import _native as N

try:
    import torch
except ImportError:  # pragma: no cover - torch is part of the image
    torch = None

DRIFT_TOL = 1e-8          # pod.py:247
JACOBI_TOL_REL = 2.0 ** -52
JACOBI_TOL_ABS = 16 * 2.0 ** -52  # absolute off-diagonal trigger, x max|g_ii| (Gram rounding floor)
JACOBI_MAX_SWEEPS = 60
# Eigensolver numerics.  Fixed constants of the product path: the library and this module read
# no environment variables (a stray variable must never change a result).  Studies override
# them explicitly in-process (tools/*.py), never through the environment.
PSTRF_TOL = 2.0 ** -52  # stop pivoting at u * max|G_ii|
# Rayleigh-Ritz polish of the preconditioned eigenpairs against G itself (restores LAPACK-class
# accuracy of the eigenvalues at the Gram cutoff): eigenpairs with lambda above
# POLISH_FACTOR * cutoff * lambda_max * m are re-solved in their own span.
KEEP_SPECTRUM = False   # diagnostics: keep the last node's eigenvalues in LAST_SPECTRUM
LAST_SPECTRUM: list = []
POLISH_FACTOR = 1e-2
PSTRF_POLISH_MARGIN = 0.25
POLISH_TOL_REL = 2.0 ** -52
POLISH_TOL_ABS = 1e-30
# rotations whose angle |g_ij| / |g_jj - g_ii| is below this change no output digit
POLISH_TOL_ANGLE = 1e-14
# absolute trigger of the preconditioned (H = L^T L) phase; the polish carries the final accuracy
PC_TOL_ABS = 16 * 2.0 ** -52
# run_parallel accumulates a star root's Gramian pair by pair beside an upload-bound wave of leaves
PROGRESSIVE_GRAM = True
# ... and also beside a wave of device-resident leaves (their latency-bound phases leave SMs idle)
PROGRESSIVE_GRAM_RESIDENT = False
# Preconditioned eigenproblems of at least this order go through the tridiagonal solver
# (hp_syev_tri: ~4/3 r^3 flops instead of the block Jacobi's ~90 r^3); it declines clustered
# spectra (a relative gap below TRI_RELGAP_MIN), which then take the Jacobi path.  Measured
# (tools/tri_order_probe.py): at order 1,000 (config 0) the H phase takes 14 ms against the block
# Jacobi's 26 ms; at order 512 a LONE solve would also win, but sytrd_panel is a cooperative launch
# over every SM, so 16 concurrent leaf solves serialise (config-1 leaf wave 158 -> 231 ms).
TRI_MIN_ORDER = 896
TRI_RELGAP_MIN = 1e-9
LAST_TRI_DIAG: dict = {}


class Profiler:
    """Optional CUDA-event timing of the node phases on the launching stream
    (used by bench.py for the live roofline; off by default)."""

    enabled = False
    records: list = []
    extra: dict = {}           # kernel-level figures reported by the library itself: name -> (calls, ms, bytes)
    _tag = threading.local()   # the node a thread is evaluating (set by evaluate_node)

    @classmethod
    def reset(cls, enabled=True):
        cls.enabled = enabled
        cls.records = []
        cls.extra = {}

    @classmethod
    def set_tag(cls, tag):
        cls._tag.value = tag

    @classmethod
    def tag(cls):
        return getattr(cls._tag, "value", None)

    @classmethod
    def summary(cls, tag=None):
        """{phase: (launches, total_ms, total_flops)} over all records (or those of one
        tag, e.g. one node) -- synchronises the device."""
        out: dict = {}
        if cls.records:
            torch.cuda.synchronize()
        for name, e0, e1, flops, t in cls.records:
            if tag is not None and t != tag:
                continue
            n, ms, f = out.get(name, (0, 0.0, 0.0))
            out[name] = (n + 1, ms + e0.elapsed_time(e1), f + flops)
        return out


class _phase:
    __slots__ = ("name", "flops", "e0")

    def __init__(self, name, flops=0.0):
        self.name = name
        self.flops = float(flops)
        self.e0 = None

    def __enter__(self):
        if Profiler.enabled:
            self.e0 = torch.cuda.Event(enable_timing=True)
            self.e0.record()
        return self

    def __exit__(self, *exc):
        if self.e0 is not None:
            e1 = torch.cuda.Event(enable_timing=True)
            e1.record()
            Profiler.records.append((self.name, self.e0, e1, self.flops, Profiler.tag()))
        return False


def require_cuda():
    if torch is None or not torch.cuda.is_available():
        raise RuntimeError("the HAPOD B200 path needs a CUDA device (there is no CPU fallback)")
    N.load()


def _stream():
    return ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)


def _ptr(t) -> int:
    return t.data_ptr() if t is not None else 0


def _even(n: int) -> int:
    return n + (n & 1)


class Guards:
    """Debug allocation mode (the pool's substitute for compute-sanitizer memcheck, which is closed
    here): every matrix (DevMat.empty) and kernel workspace (_ws) is allocated with a 4 KB canary
    zone on both sides and a poisoned (signalling-pattern NaN) payload.  ``check()`` verifies that
    no kernel wrote outside its buffer; a kernel that consumes memory it was supposed to have
    written first propagates the poison NaN into results the tests compare with the oracle.
    Off by default; used by tests/test_gpu_guards.py."""

    active = False
    CANARY = 0x7FF8DEADBEEFCAFE   # quiet NaN with a recognisable payload
    POISON = 0x7FF8BAADF00DBAAD
    ZONE = 4096                   # bytes on each side
    _live: list = []
    _lock = threading.Lock()

    @classmethod
    def enable(cls):
        cls._live = []
        cls.active = True

    @classmethod
    def disable(cls):
        cls.active = False
        cls._live = []

    @classmethod
    def alloc(cls, n: int, dtype, zero: bool):
        esz = torch.empty(0, dtype=dtype).element_size()
        nbytes = n * esz
        pad = (-nbytes) % 8
        raw = torch.empty((2 * cls.ZONE + nbytes + pad) // 8, dtype=torch.int64, device="cuda")
        raw.fill_(cls.POISON)
        raw[: cls.ZONE // 8] = cls.CANARY
        raw[(cls.ZONE + nbytes + pad) // 8:] = cls.CANARY
        payload = raw.view(torch.uint8)[cls.ZONE: cls.ZONE + nbytes].view(dtype)
        if zero:
            payload.zero_()
        with cls._lock:
            cls._live.append((raw, nbytes + pad))
        return payload

    @classmethod
    def check(cls) -> int:
        """Number of guarded allocations verified; raises if any canary word changed."""
        torch.cuda.synchronize()
        want = cls.CANARY
        with cls._lock:
            live = list(cls._live)
        for k, (raw, nbytes) in enumerate(live):
            head = raw[: cls.ZONE // 8]
            tail = raw[(cls.ZONE + nbytes) // 8:]
            if not bool((head == want).all()) or not bool((tail == want).all()):
                bad_h = int((head != want).sum())
                bad_t = int((tail != want).sum())
                raise AssertionError(f"guarded allocation {k} ({nbytes} bytes): {bad_h} canary words overwritten "
                                     f"before and {bad_t} after the buffer")
        return len(live)


class DevMat:
    """Column-major float64 matrix on the current CUDA device."""

    __slots__ = ("storage", "rows", "cols", "ld", "offset")

    def __init__(self, storage, rows: int, cols: int, ld: int, offset: int = 0):
        self.storage = storage  # 1-d float64 CUDA tensor
        self.rows = int(rows)
        self.cols = int(cols)
        self.ld = int(ld)
        self.offset = int(offset)  # element offset of column 0

    @staticmethod
    def empty(rows: int, cols: int, zero: bool = False):
        ld = max(_even(rows), 2)
        n = max(ld * cols, 1)
        if Guards.active:
            st = Guards.alloc(n, torch.float64, zero)
        else:
            st = torch.zeros(n, dtype=torch.float64, device="cuda") if zero else \
                torch.empty(n, dtype=torch.float64, device="cuda")
        return DevMat(st, rows, cols, ld)

    @property
    def ptr(self) -> int:
        return self.storage.data_ptr() + 8 * self.offset

    def col_ptr(self, j: int) -> int:
        return self.ptr + 8 * self.ld * j

    def view_cols(self, j0: int, j1: int) -> "DevMat":
        return DevMat(self.storage, self.rows, j1 - j0, self.ld, self.offset + j0 * self.ld)

    def aligned16(self) -> bool:
        return self.ld % 2 == 0 and self.ptr % 16 == 0

    def vecset(self) -> N.VecSet:
        return N.VecSet(self.ptr, self.ld, None, int(self.aligned16()))

    def tensor(self):
        """(rows, cols) torch view (column-major strides)."""
        if self.cols == 0:
            return torch.zeros((self.rows, 0), dtype=torch.float64, device=self.storage.device)
        return self.storage.as_strided((self.rows, self.cols), (1, self.ld), self.storage.storage_offset() + self.offset)

    def to_numpy(self) -> np.ndarray:
        if self.cols == 0 or self.rows == 0:
            return np.zeros((self.rows, self.cols))
        t = self.storage.as_strided((self.cols, self.rows), (self.ld, 1), self.storage.storage_offset() + self.offset)
        host = t.cpu().numpy()  # (cols, rows) C-order == (rows, cols) F-order
        return np.asfortranarray(host.T)

    def clone(self) -> "DevMat":
        out = DevMat.empty(self.rows, self.cols)
        if self.cols and self.rows:
            N.check(N.load().hp_scale(self.ptr, self.ld, self.rows, self.cols, None, None, None,
                                      out.ptr, out.ld, _stream()), "copy")
        return out


_COPY_STREAM = None
_COPY_LOCK = threading.Lock()
_COPY_INFLIGHT: list = []   # completion events of the uploads queued on the copy stream
# at most this many uploads queued at once: any device-to-host read (a memcpy, or a kernel writing
# pinned memory) waits behind the copy engine's pending host-to-device work, so an unbounded queue
# (all 16 leaves of config 1 request their 0.8 GB upload at once) stalls every leaf's first host
# read-back for most of the 13 GB transfer; two in flight keep the DMA engine busy
COPY_MAX_INFLIGHT = 2


def copy_stream():
    """One shared host-to-device copy stream: deferred uploads issued by pooled workers
    serialise on it in request order, so the first leaf computes while the next arrive."""
    global _COPY_STREAM
    if _COPY_STREAM is None:
        _COPY_STREAM = torch.cuda.Stream()
    return _COPY_STREAM


def upload(values, check_finite: bool = True, via=None) -> DevMat:
    """Host (numpy / torch CPU) or device (torch CUDA) d x m array -> DevMat.

    F-contiguous inputs are copied straight into the column-major layout;
    C-contiguous ones are staged and transposed on the device.  ``via``: a copy
    stream for the host-to-device transfer of column-major host inputs (the
    current stream waits on it)."""
    require_cuda()
    lib = N.load()
    if torch.is_tensor(values):
        t = values.detach()
        if t.dtype != torch.float64:
            t = t.to(torch.float64)
    else:
        a = np.asarray(values, dtype=np.float64)
        t = torch.from_numpy(a) if (a.flags.c_contiguous or a.flags.f_contiguous) else \
            torch.from_numpy(np.ascontiguousarray(a))
    if t.dim() != 2:
        raise ValueError(f"snapshot block must be 2-d, got shape {tuple(t.shape)}")
    d, m = int(t.shape[0]), int(t.shape[1])
    out = DevMat.empty(d, m)
    if d and m:
        if t.stride(0) == 1 and t.stride(1) >= d:            # column-major source (possibly a column view)
            src = t.as_strided((m, d), (t.stride(1), 1))
            dst = out.storage[: out.ld * m].view(m, out.ld)[:, :d]
            if via is not None and not t.is_cuda:
                cur = torch.cuda.current_stream()
                # the copy and the event that marks ITS completion are enqueued atomically: with
                # `cur.wait_stream(via)` a worker could also wait for copies other workers enqueued
                # in between (all 16 leaves of config 1 request their upload at once), i.e. for
                # the whole 13 GB transfer before its first kernel
                with _COPY_LOCK:
                    while len(_COPY_INFLIGHT) >= max(1, COPY_MAX_INFLIGHT):
                        _COPY_INFLIGHT.pop(0).synchronize()
                    via.wait_stream(cur)  # the destination was allocated on the current stream
                    with torch.cuda.stream(via):
                        dst.copy_(src, non_blocking=True)
                    done = torch.cuda.Event()
                    done.record(via)
                    _COPY_INFLIGHT.append(done)
                cur.wait_event(done)
            else:
                dst.copy_(src, non_blocking=True)
        else:                                                  # row-major (or strided) source
            tc = t.contiguous() if not (t.is_cuda and t.is_contiguous()) else t
            dev = tc.to("cuda", non_blocking=True) if not tc.is_cuda else tc
            N.check(lib.hp_transpose_rm_to_cm(dev.data_ptr(), d, m, out.ptr, out.ld, _stream()),
                    "upload transpose")
            if not tc.is_cuda:
                torch.cuda.current_stream().synchronize()  # keep the staging buffer alive
        if check_finite:
            bad = torch.zeros(1, dtype=torch.int32, device="cuda")
            N.check(lib.hp_finite_check(out.ptr, out.ld, d, m, bad.data_ptr(), _stream()), "finite")
            if int(host_read(bad)[0]):
                raise ValueError("snapshot block contains non-finite entries")
    return out


_PINNED = threading.local()


def host_read(t) -> np.ndarray:
    """Read a small device tensor on the host: a kernel (hp_read_small) writes it into a
    per-thread PINNED buffer, then an event of the current stream is awaited.  `.item()` /
    `.cpu()` -- any device-to-host memcpy, pinned or not -- was measured to queue behind the copy
    engine's pending host-to-device transfers: under the e2e leg every leaf's finiteness check
    and truncation read-back waited for most of the 13 GB upload queue."""
    flat = t.reshape(-1).contiguous()
    n = flat.numel()
    bufs = getattr(_PINNED, "bufs", None)
    if bufs is None:
        bufs = _PINNED.bufs = {}
    buf = bufs.get(flat.dtype)
    if buf is None or buf.numel() < n:
        buf = bufs[flat.dtype] = torch.empty(max(n, 64), dtype=flat.dtype, pin_memory=True)
    b = buf[:n]
    N.check(N.load().hp_read_small(flat.data_ptr(), b.data_ptr(), n * flat.element_size(), _stream()),
            "read back")
    ev = torch.cuda.Event()
    ev.record()
    ev.synchronize()
    return b.numpy().copy()


def ones(n: int):
    return torch.ones(max(n, 1), dtype=torch.float64, device="cuda")[:n]


@dataclass
class Part:
    """One column block of a node input: columns mat[:, j] * scale[j]."""

    mat: DevMat
    scale: object = None  # 1-d float64 CUDA tensor or None (= all ones)


def _concat_parts(parts: list[Part]):
    """VecSet over the concatenated columns + the concatenated scale (or None)."""
    parts = [p for p in parts if p.mat.cols]
    m = sum(p.mat.cols for p in parts)
    if len(parts) == 1:
        return parts[0].mat.vecset(), parts[0].scale, m, parts
    table = np.empty(m, dtype=np.int64)
    at = 0
    aligned = True
    for p in parts:
        c = p.mat.cols
        table[at:at + c] = p.mat.ptr + 8 * p.mat.ld * np.arange(c, dtype=np.int64)
        aligned &= p.mat.aligned16()
        at += c
    tdev = torch.from_numpy(table).to("cuda", non_blocking=True)
    any_scale = any(p.scale is not None for p in parts)
    scale = None
    if any_scale:
        scale = torch.cat([p.scale if p.scale is not None else ones(p.mat.cols) for p in parts])
    vs = N.VecSet(0, 0, tdev.data_ptr(), int(aligned))
    return vs, scale, m, (parts, tdev)


PACK_MIN_PARTS = 4   # inputs with this many column blocks are packed into one matrix


def pack_parts(parts: list[Part]) -> list[Part]:
    """A node input of many column blocks (an interior node's children) as ONE column-major
    matrix + the concatenated per-column scale, so the Gram and reconstruction GEMMs read it
    with tensor TMA instead of through a pointer table.  The copy moves 2 d m 8 bytes (a few ms
    at the config-1 root against ~1 s of contractions).  Inputs with fewer blocks are returned
    unchanged."""
    live = [p for p in parts if p.mat.cols]
    if len(live) < PACK_MIN_PARTS:
        return parts
    lib = N.load()
    d = live[0].mat.rows
    m = sum(p.mat.cols for p in live)
    out = DevMat.empty(d, m)
    at = 0
    st = _stream()
    for p in live:
        c = p.mat.cols
        # the repo's own copy kernel (hp_scale without scales), not an eager torch copy
        N.check(lib.hp_scale(p.mat.ptr, p.mat.ld, d, c, None, None, None, out.col_ptr(at), out.ld, st), "pack")
        at += c
    scale = None
    if any(p.scale is not None for p in live):
        scale = torch.cat([p.scale if p.scale is not None else ones(p.mat.cols) for p in live])
    return [Part(out, scale)]


def _operand(x) -> tuple:
    """(DevMat, was_host) for a d x k host array / torch tensor / DevMat operand."""
    if isinstance(x, DevMat):
        return x, False
    host = not (torch.is_tensor(x) and x.is_cuda)
    return upload(x, check_finite=False), host


def space_gram(a, b, w_dev=None):
    """InnerProductSpace.gram (pod.py:87-91) on the device: a^T (w * b) by the DMMA GEMM engine
    (w scales b's rows first, as the reference forms w[:, None] * b).  Host inputs give a NumPy
    result, device inputs a CUDA tensor."""
    lib = N.load()
    st = _stream()
    A, ha = _operand(a)
    B, hb = _operand(b)
    if A.rows != B.rows:
        raise ValueError(f"operands have {A.rows} and {B.rows} rows")
    if w_dev is not None and B.cols:
        Bw = DevMat.empty(B.rows, B.cols)
        N.check(lib.hp_scale(B.ptr, B.ld, B.rows, B.cols, w_dev.data_ptr(), None, None, Bw.ptr, Bw.ld, st), "w * b")
        B = Bw
    C = DevMat.empty(A.cols, B.cols, zero=True)
    if A.cols and B.cols and A.rows:
        ws = _ws(lib.hp_gemm_workspace_bytes(A.cols, B.cols, A.rows, 0, 0))
        N.check(lib.hp_gemm(1, 1, A.cols, B.cols, A.rows, A.vecset(), B.vecset(), 1.0, 0.0, C.ptr, C.ld, None, None,
                            None, 0, 0, ws.data_ptr(), ws.numel(), st), "gram")
    return C.to_numpy() if (ha and hb) else C.tensor()


def space_norms_sq(a, w_dev=None):
    """InnerProductSpace.norms_sq (pod.py:93-97) on the device: per column sum_i w_i a_i^2."""
    lib = N.load()
    A, host = _operand(a)
    out = torch.zeros(max(A.cols, 1), dtype=torch.float64, device="cuda")
    if A.cols:
        N.check(lib.hp_col_norms_sq(A.ptr, A.ld, A.rows, A.cols, _ptr(w_dev), out.data_ptr(), _stream()),
                "norms_sq")
    out = out[: A.cols]
    return out.cpu().numpy() if host else out


def weigh_parts(parts: list[Part], sqrt_w) -> list[Part]:
    """Euclidean coordinates of weighted snapshots (InnerProductSpace.weigh, pod.py:76-80)."""
    lib = N.load()
    out = []
    for p in parts:
        x = DevMat.empty(p.mat.rows, p.mat.cols)
        if p.mat.cols:
            N.check(lib.hp_scale(p.mat.ptr, p.mat.ld, p.mat.rows, p.mat.cols, sqrt_w.data_ptr(), None,
                                 None, x.ptr, x.ld, _stream()), "weigh")
        out.append(Part(x, p.scale))
    return out


def _ws(nbytes: int):
    if Guards.active:
        return Guards.alloc(max(int(nbytes), 16), torch.uint8, False)
    return torch.empty(max(int(nbytes), 16), dtype=torch.uint8, device="cuda")


@dataclass
class NodeOutput:
    U: DevMat | None
    sigmas: np.ndarray
    sigmas_dev: object
    tail: float
    right: DevMat | None
    lam_max: float
    nkeep: int
    drift: float
    reorthed: bool
    sweeps: int
    input_count: int


def gram_full(parts: list[Part], d: int):
    """G = D S^T S D for the concatenated (scaled) parts (pod.py:208-211)."""
    lib = N.load()
    vs, scale, m, keep = _concat_parts(parts)
    G = DevMat.empty(m, m)
    if m:
        ws = _ws(lib.hp_gram_workspace_bytes(d, m))
        with _phase("gram", float(d) * m * (m + 1)):
            N.check(lib.hp_gram(vs, d, m, _ptr(scale), G.ptr, G.ld, ws.data_ptr(), ws.numel(), _stream()), "gram")
    return G, m, keep


def gram_block(prior_U: DevMat, prior_sig_dev, fresh: list[Part], d: int):
    """Block Gramian of [Phi*sigma | F] with the diag(sigma^2) top-left block
    written down (pod.py:376-384)."""
    lib = N.load()
    n_old = prior_U.cols
    vs_f, scale_f, m, keep = _concat_parts(fresh)
    total = n_old + m
    G = DevMat.empty(total, total)
    ws = _ws(lib.hp_block_gram_workspace_bytes(d, n_old, m))
    with _phase("gram", 2.0 * d * n_old * m + float(d) * m * (m + 1)):
        N.check(lib.hp_block_gram(prior_U.vecset(), prior_sig_dev.data_ptr(), n_old, vs_f, _ptr(scale_f), m, d,
                                  G.ptr, G.ld, ws.data_ptr(), ws.numel(), _stream()), "block gram")
    return G, total, keep


BJORCK_MAX_DRIFT = 0.05  # Newton-Schulz: quadratic from here
POLISH_ORTH_TOL = 1e-10  # orthonormality the Ritz basis needs (eigenvalues move by at most this, relatively)


def _orthonormalise_basis(X: DevMat, ws, st, ph) -> float:
    """Make X orthonormal (any basis of its span).  Bjorck steps X <- X - X E / 2,
    E = X^T X - I, while max|E| <= BJORCK_MAX_DRIFT (quadratic: drift -> ~drift^2); CholQR
    (hp_reorthonormalize) otherwise.  Returns the initial drift."""
    lib = N.load()
    m, K = X.rows, X.cols
    C = DevMat.empty(K, K)
    drift_dev = torch.zeros(1, dtype=torch.float64, device="cuda")
    N.check(lib.hp_drift(X.ptr, X.ld, m, K, C.ptr, C.ld, drift_dev.data_ptr(), ws.data_ptr(), ws.numel(), st),
            "X^T X")
    drift0 = drift = float(host_read(drift_dev)[0])
    ph.flops += float(m) * K * (K + 1)
    if drift > BJORCK_MAX_DRIFT:
        rws = _ws(lib.hp_reortho_workspace_bytes(m, K))
        passes = ctypes.c_int(0)
        # The max-norm drift of X = G Q0 / lambda is O(1) (its trailing columns are amplified along the
        # larger eigenvectors), but kappa(X) stays ~10: ONE Cholesky-QR pass leaves u kappa^2 ~ 1e-13.
        # hp_reorthonormalize takes a single pass for a declared drift <= 0.1; the result is measured
        # and only a basis still above POLISH_ORTH_TOL gets the second pass.
        N.check(lib.hp_reorthonormalize(X.ptr, X.ld, m, K, C.ptr, C.ld, min(drift, 0.1), ctypes.byref(passes),
                                        rws.data_ptr(), rws.numel(), st), "orthonormalise X")
        ph.flops += passes.value * 2.0 * m * K * K
        if passes.value == 1:
            N.check(lib.hp_drift(X.ptr, X.ld, m, K, C.ptr, C.ld, drift_dev.data_ptr(), ws.data_ptr(), ws.numel(), st),
                    "X^T X")
            ph.flops += float(m) * K * (K + 1)
            drift1 = float(host_read(drift_dev)[0])
            if not (drift1 <= POLISH_ORTH_TOL):
                N.check(lib.hp_reorthonormalize(X.ptr, X.ld, m, K, C.ptr, C.ld, drift1, ctypes.byref(passes),
                                                rws.data_ptr(), rws.numel(), st), "orthonormalise X (second pass)")
                ph.flops += passes.value * 2.0 * m * K * K
        return drift0
    Y = DevMat.empty(m, K)
    orig = X
    for _ in range(6):
        if drift <= 4 * 2.0 ** -52:
            break
        # C := X^T X - I (C holds X^T X); Y = X - X C / 2 ; X <- Y
        N.check(lib.hp_add_diag(C.ptr, C.ld, K, -1.0, st), "C - I")
        N.check(lib.hp_scale(X.ptr, X.ld, m, K, None, None, None, Y.ptr, Y.ld, st), "copy")
        N.check(lib.hp_gemm(0, 1, m, K, K, X.vecset(), C.vecset(), -0.5, 1.0, Y.ptr, Y.ld, None, None, None, 0, 0,
                            ws.data_ptr(), ws.numel(), st), "Bjorck step")
        X, Y = Y, X
        N.check(lib.hp_drift(X.ptr, X.ld, m, K, C.ptr, C.ld, drift_dev.data_ptr(), ws.data_ptr(), ws.numel(), st),
                "X^T X")
        drift = float(host_read(drift_dev)[0])
        ph.flops += 2.0 * m * K * K + float(m) * K * (K + 1)
    if X is not orig:
        N.check(lib.hp_scale(X.ptr, X.ld, m, K, None, None, None, orig.ptr, orig.ld, st), "copy back")
    return drift0


class EigShare:
    """One rank's share of a REPLICATED eigensolve (multi-GPU root): every rank runs
    the same deterministic iteration on the same Gramian, accumulates only its own 64-row slabs of
    the eigenvector matrix (half of a round's DMMA products are V slabs) and the ranks all-gather
    their rows once at the end.  No communication inside the iteration."""

    def __init__(self, rank: int, world: int, group=None):
        self.rank, self.world, self.group = int(rank), int(world), group

    def slab_rows(self, n_padded: int, rank: int | None = None):
        """Rows [a, b) of the padded matrix owned by ``rank`` (whole 64-row slabs, contiguous)."""
        q = self.rank if rank is None else rank
        slabs = n_padded // 64
        return 64 * (q * slabs // self.world), 64 * ((q + 1) * slabs // self.world)

    def allgather_rows(self, V: DevMat, n: int, n_padded: int):
        """Make every row of the n x n matrix V valid on every rank (rank q holds rows slab_rows(q))."""
        if self.world == 1:
            return
        import torch.distributed as dist
        Vt = V.tensor()
        spans = [self.slab_rows(n_padded, q) for q in range(self.world)]
        spans = [(min(a, n), min(b, n)) for a, b in spans]
        width = max(b - a for a, b in spans)
        a, b = spans[self.rank]
        send = torch.zeros((max(width, 1), n), dtype=torch.float64, device="cuda")
        if b > a:
            send[: b - a].copy_(Vt[a:b])
        parts = [torch.empty_like(send) for _ in range(self.world)]
        dist.all_gather(parts, send, group=self.group)
        for q, (qa, qb) in enumerate(spans):
            if q != self.rank and qb > qa:
                Vt[qa:qb].copy_(parts[q][: qb - qa])


def _syev(G: DevMat, n: int, st, name="eigensolve", tol_rel=None, tol_abs=None, keep_floor=0.0, tol_angle=0.0,
          refine=True, share: EigShare | None = None):
    lib = N.load()
    lam = torch.empty(max(n, 1), dtype=torch.float64, device="cuda")
    V = DevMat.empty(n, n)
    ws = _ws(lib.hp_syev_workspace_bytes(n))
    sweeps = ctypes.c_int(0)
    eflops = ctypes.c_double(0.0)
    ph = _phase(name)
    tr = JACOBI_TOL_REL if tol_rel is None else tol_rel
    ta = JACOBI_TOL_ABS if tol_abs is None else tol_abs
    with ph:
        if share is not None and share.world > 1:
            if refine:
                raise ValueError("a shared eigensolve cannot refine its eigenvalues (needs all rows of V)")
            npad = int(lib.hp_syev_padded_order(n))
            a, b = share.slab_rows(npad)
            N.check(lib.hp_syev_rows(G.ptr, G.ld, n, lam.data_ptr(), V.ptr, V.ld, n, tr, ta, float(tol_angle),
                                     float(keep_floor), JACOBI_MAX_SWEEPS, ctypes.byref(sweeps),
                                     ctypes.byref(eflops), a, b, ws.data_ptr(), ws.numel(), st), "eigensolve")
            share.allgather_rows(V, n, npad)
        else:
            N.check(lib.hp_syev(G.ptr, G.ld, n, lam.data_ptr(), V.ptr, V.ld, n, tr, ta, float(tol_angle),
                                float(keep_floor), JACOBI_MAX_SWEEPS, int(refine), ctypes.byref(sweeps),
                                ctypes.byref(eflops), ws.data_ptr(), ws.numel(), st), "eigensolve")
        ph.flops = eflops.value
    return lam, V, sweeps.value


def _syev_tri(H: DevMat, r: int, floor_rel: float, st):
    """Leading eigenpairs (lambda >= floor_rel * lambda_max) of the preconditioned Gramian H by
    hp_syev_tri.  Returns (lam, W) with lam descending and zero past the computed ones, or None
    when the solver declines (clustered spectrum) and the block Jacobi has to run."""
    lib = N.load()
    if r < 2 or r > int(lib.hp_syev_tri_max_order()):
        return None
    try:
        lam = torch.empty(r, dtype=torch.float64, device="cuda")
        W = DevMat.empty(r, r)
        ws = _ws(lib.hp_syev_tri_workspace_bytes(r))  # ~6 r^2 doubles: reflectors, qds factors per eigenvalue
    except torch.cuda.OutOfMemoryError:
        return None  # the block Jacobi needs ~3 r^2 doubles
    k = ctypes.c_int64(0)
    status = ctypes.c_int(1)
    diag = (ctypes.c_double * 8)()
    ph = _phase("eigensolve_tri", 4.0 / 3.0 * float(r) ** 3)
    with ph:
        N.check(lib.hp_syev_tri(H.ptr, H.ld, r, float(floor_rel), TRI_RELGAP_MIN, lam.data_ptr(), W.ptr, W.ld,
                                ctypes.byref(k), ctypes.byref(status), diag, ws.data_ptr(), ws.numel(), st),
                "tridiagonal eigensolve")
        ph.flops += 4.0 * float(r) * r * k.value
    LAST_TRI_DIAG.update(order=r, count=int(k.value), status=int(status.value), min_relgap=diag[0],
                         max_resid=diag[1], sigma=diag[2], sytrd_ms=diag[4], tridiag_ms=diag[5], rqi_max=int(diag[6]))
    if Profiler.enabled:
        # the tridiagonalisation's own time and its algorithmic matrix reads (every column step reads
        # the trailing matrix once: sum_j 8 (r - j)^2 = 8 r^3 / 3 bytes) for the HBM roofline
        n_, ms_, b_ = Profiler.extra.get("sytrd_panel", (0, 0.0, 0.0))
        Profiler.extra["sytrd_panel"] = (n_ + 1, ms_ + diag[4], b_ + 8.0 * float(r) ** 3 / 3.0)
    if status.value != 0:
        return None
    return lam, W


@dataclass
class EigVectors:
    """The spectral half of a node POD: truncation data and the kept eigenvectors of G."""

    lam_max: float
    nkeep: int
    n_modes: int
    tail: float
    sig_dev: object          # sigma_1..sigma_N (device)
    Vn: DevMat | None        # m x N eigenvectors of G, descending
    sweeps: int


def eig_vectors(G: DevMat, m: int, eps: float, cutoff: float, share: EigShare | None = None) -> EigVectors:
    """pod.py:329-331 + 278-289 on the device: eigensolve of the node Gramian, cutoff keep,
    truncation rank and tail, and the N kept eigenvectors.

    Eigensolve (default "pcjacobi"): G = L L^T by pivoted Cholesky (rows of L in
    the original order), H = L^T L, H = W Lambda W^T by block Jacobi, and the
    eigenvectors of G are V = L W Lambda^{-1/2}.  Same eigenpairs as
    eigh(G) (pod.py:329), a handful of Jacobi sweeps instead of dozens."""
    lib = N.load()
    st = _stream()
    if m == 0:
        return EigVectors(0.0, 0, 0, 0.0, ones(0), None, 0)
    Lf = DevMat.empty(m, m)
    piv = torch.empty(max(m, 1), dtype=torch.int32, device="cuda")
    rank = ctypes.c_int64(0)
    ws = _ws(lib.hp_pstrf_workspace_bytes(m))
    with _phase("pstrf", float(m) ** 3 / 3.0):
        # with the polish, pivots below a quarter of its floor (lambda <= POLISH_FACTOR * cutoff
        # * lambda_max * m) only feed directions the subspace step damps anyway
        tol_lam = PSTRF_POLISH_MARGIN * POLISH_FACTOR * float(cutoff) * m
        N.check(lib.hp_pstrf(G.ptr, G.ld, m, Lf.ptr, Lf.ld, piv.data_ptr(), PSTRF_TOL, tol_lam,
                             ctypes.byref(rank), ws.data_ptr(), ws.numel(), st), "pivoted Cholesky")
    del ws
    r = int(rank.value)
    Lr = Lf.view_cols(0, r)
    H = DevMat.empty(r, r)
    if r:
        ws = _ws(lib.hp_gram_workspace_bytes(m, r))
        with _phase("gram", float(m) * r * (r + 1)):
            N.check(lib.hp_gram(Lr.vecset(), m, r, None, H.ptr, H.ld, ws.data_ptr(), ws.numel(), st),
                    "H = L^T L")
        del ws
    # with the polish, H's eigenvalues only select K and scale Q0: no Rayleigh refinement
    # (a multi-GPU root passes `share`: this rank accumulates only its rows of W, all-gathered after)
    # (large H: the tridiagonal solver, replicated on every rank of a multi-GPU root -- deterministic,
    # so the replicas are bitwise equal and nothing is exchanged)
    tri = None
    if r >= TRI_MIN_ORDER:
        tri = _syev_tri(H, r, 0.5 * POLISH_FACTOR * float(cutoff) * m, st)
    if tri is not None:
        lam, W = tri
        sweeps = 0
    else:
        lam, W, sweeps = _syev(H, r, st, tol_abs=PC_TOL_ABS, refine=False, share=share)
    nev = r
    basis, divide = Lf, True
    if r:
        # K = #{lambda_H >= POLISH_FACTOR * cutoff * lambda_max * m}; sig = sqrt(lambda_H[:K])
        sig_h = torch.empty(r, dtype=torch.float64, device="cuda")
        info_h = torch.empty(4, dtype=torch.float64, device="cuda")
        N.check(lib.hp_truncate(lam.data_ptr(), r, 0.0, float(cutoff) * POLISH_FACTOR, m, sig_h.data_ptr(),
                                info_h.data_ptr(), st), "polish count")
        info_hh = host_read(info_h[:2])
        lam_max_h, K = float(info_hh[0]), int(info_hh[1])
        if K:
            # Q0 = L W_K Lambda_K^{-1/2}: approximate eigenvectors of G from the preconditioned solve.
            # One subspace-iteration step X = G Q0 Lambda_K^{-1} damps the components along
            # eigenvectors outside span(Q0) (left there by the Cholesky backward error) by
            # lambda_j / lambda_i; CholQR keeps the descending order; Rayleigh-Ritz on
            # G2 = X^T G X then resolves the mixing inside the span.
            ws = _ws(max(lib.hp_gemm_workspace_bytes(m, K, r, 0, 0), lib.hp_gemm_workspace_bytes(m, K, m, 0, 0),
                         lib.hp_gemm_workspace_bytes(K, K, m, 1, 0)))
            Q0 = DevMat.empty(m, K)
            with _phase("polish_q0", 2.0 * m * r * K):
                N.check(lib.hp_gemm(0, 1, m, K, r, Lr.vecset(), W.vecset(), 1.0, 0.0, Q0.ptr, Q0.ld, None, None,
                                    sig_h.data_ptr(), 0, 0, ws.data_ptr(), ws.numel(), st), "Q0 = L W / sigma")
            X = DevMat.empty(m, K)
            with _phase("polish_x", 2.0 * m * m * K):
                N.check(lib.hp_gemm(0, 1, m, K, m, G.vecset(), Q0.vecset(), 1.0, 0.0, X.ptr, X.ld, None, None,
                                    lam.data_ptr(), 0, 0, ws.data_ptr(), ws.numel(), st), "X = G Q0 / lambda")
            del Q0
            ph = _phase("polish_orth", 0.0)
            with ph:
                # any orthonormal basis of span(X) serves Rayleigh-Ritz: Bjorck / Newton-Schulz steps
                # X <- X (3 I - X^T X) / 2 (two DMMA GEMMs each, no sequential factorisation) while
                # the drift is small, CholQR otherwise
                drift_x = None
                # the trailing columns of X (eigenpairs near the polish floor, where Q0 is least
                # accurate) can be numerically dependent; CholQR keeps nested spans, so on a
                # breakdown the basis is shortened from the tail -- never below the eigenpairs
                # above the Gram cutoff plus half the margin -- and orthonormalised again
                k_cut = int(host_read((lam[:K] >= float(cutoff) * lam_max_h * m).sum())[0])
                k_min = min(K, k_cut + max(1, (K - k_cut) // 2))
                while drift_x is None:
                    try:
                        drift_x = _orthonormalise_basis(X, ws, st, ph)
                    except np.linalg.LinAlgError:
                        if K <= k_min:
                            raise
                        K = max(k_min, K - max(1, (K - k_cut) // 4))
                        X = X.view_cols(0, K)
            T = DevMat.empty(m, K)
            G2 = DevMat.empty(K, K)
            with _phase("polish_rr", 2.0 * m * m * K + float(m) * K * (K + 1)):
                N.check(lib.hp_gemm(0, 1, m, K, m, G.vecset(), X.vecset(), 1.0, 0.0, T.ptr, T.ld, None, None,
                                    None, 0, 0, ws.data_ptr(), ws.numel(), st), "T = G X")
                N.check(lib.hp_gemm(1, 1, K, K, m, X.vecset(), T.vecset(), 1.0, 0.0, G2.ptr, G2.ld, None, None,
                                    None, 1, 0, ws.data_ptr(), ws.numel(), st), "G2 = X^T G X")
            del T, ws
            # G2 is nearly diagonal and graded: relative criterion, but never rotate two
            # eigenvalues that are both below a tenth of the Gram cutoff (pod.py:284)
            floor = 0.1 * float(cutoff) * lam_max_h * m
            lam, W, sweeps2 = _syev(G2, K, st, "eigensolve_polish", tol_rel=POLISH_TOL_REL,
                                    tol_abs=POLISH_TOL_ABS, keep_floor=floor, tol_angle=POLISH_TOL_ANGLE)
            sweeps += sweeps2
            nev = K
            basis, divide = X, False
            del G2, Lf
            Lf = None
    sig = torch.empty(max(m, 1), dtype=torch.float64, device="cuda")
    info = torch.empty(4, dtype=torch.float64, device="cuda")
    with _phase("truncate"):
        N.check(lib.hp_truncate(lam.data_ptr(), nev, float(eps), float(cutoff), m, sig.data_ptr(),
                                info.data_ptr(), st), "truncate")
    if KEEP_SPECTRUM:
        LAST_SPECTRUM[:] = [lam[:nev].cpu().numpy()]
    lam_max, nkeep, n_modes, tail = host_read(info).tolist()
    nkeep, n_modes = int(nkeep), int(n_modes)
    if not (lam_max > 0.0):
        return EigVectors(lam_max, 0, 0, 0.0, ones(0), None, sweeps)
    sig_dev = sig[:n_modes].clone()
    if n_modes == 0:
        return EigVectors(lam_max, nkeep, 0, tail, sig_dev, None, sweeps)
    if basis is not None:
        # eigenvectors of G: V_N = L W_N / sigma_N  (G V = L (L^T L) W / sigma = L W Lambda / sigma), or,
        # after the polish, V_N = Q W_N with Q the orthonormal Ritz basis
        Vn = DevMat.empty(m, n_modes)
        ws = _ws(lib.hp_gemm_workspace_bytes(m, n_modes, nev, 0, 0))
        with _phase("eigvec", 2.0 * m * nev * n_modes):
            N.check(lib.hp_gemm(0, 1, m, n_modes, nev, basis.view_cols(0, nev).vecset(), W.vecset(), 1.0, 0.0,
                                Vn.ptr, Vn.ld, None, None, sig_dev.data_ptr() if divide else None, 0, 0,
                                ws.data_ptr(), ws.numel(), st), "eigenvectors of G")
        del ws, basis
    else:
        Vn = W.view_cols(0, n_modes)
    return EigVectors(lam_max, nkeep, n_modes, tail, sig_dev, Vn, sweeps)


def spectrum_and_modes(G: DevMat, m: int, parts: list[Part], d: int, eps: float, cutoff: float,
                       want_right: bool, sqrt_w=None) -> NodeOutput:
    """pod.py:278-293 on the device: eigensolve + truncation (eig_vectors), reconstruction,
    drift check + re-orthonormalisation, sign convention."""
    lib = N.load()
    st = _stream()
    ev = eig_vectors(G, m, eps, cutoff)
    lam_max, nkeep, n_modes, tail, sig_dev, sweeps = ev.lam_max, ev.nkeep, ev.n_modes, ev.tail, ev.sig_dev, ev.sweeps
    if not (lam_max > 0.0):
        return NodeOutput(None, np.zeros(0), ones(0), 0.0,
                          DevMat.empty(m, 0) if want_right else None, lam_max, 0, 0.0, False,
                          sweeps, m)
    if n_modes == 0:
        return NodeOutput(DevMat.empty(d, 0), np.zeros(0), sig_dev, tail,
                          DevMat.empty(m, 0) if want_right else None, lam_max, nkeep, 0.0, False,
                          sweeps, m)
    Vn = ev.Vn
    vs, scale, m2, keep = _concat_parts(parts)
    assert m2 == m
    if scale is not None:
        Vs = DevMat.empty(m, n_modes)
        N.check(lib.hp_scale(Vn.ptr, Vn.ld, m, n_modes, scale.data_ptr(), None, None, Vs.ptr, Vs.ld, st),
                "scale V")
    else:
        Vs = Vn
    U = DevMat.empty(d, n_modes)
    live = [p for p in parts if p.mat.cols]
    if len(live) <= 1:
        ws = _ws(lib.hp_assemble_workspace_bytes(d, m, n_modes))
        with _phase("assemble", 2.0 * d * m * n_modes):
            N.check(lib.hp_assemble(vs, d, m, Vs.ptr, Vs.ld, sig_dev.data_ptr(), n_modes, U.ptr, U.ld,
                                    ws.data_ptr(), ws.numel(), st), "assemble")
    else:
        # a few column blocks (an incremental merge [Phi sigma | F]): U = sum_p S_p (V_p / sigma),
        # one plain-operand (TMA) GEMM per block accumulating into U -- no pointer table
        rsig = 1.0 / sig_dev
        ws = _ws(max(lib.hp_gemm_workspace_bytes(d, n_modes, p.mat.cols, 0, 0) for p in live))
        with _phase("assemble", 2.0 * d * m * n_modes):
            r0 = 0
            for i, p in enumerate(live):
                c = p.mat.cols
                Vp = DevMat.empty(c, n_modes)  # rows r0..r0+c of V / sigma, 16-byte aligned columns
                N.check(lib.hp_scale(Vs.ptr + 8 * r0, Vs.ld, c, n_modes, None, None, rsig.data_ptr(), Vp.ptr, Vp.ld,
                                     st), "V / sigma")
                N.check(lib.hp_gemm(0, 1, d, n_modes, c, p.mat.vecset(), Vp.vecset(), 1.0, 0.0 if i == 0 else 1.0,
                                    U.ptr, U.ld, None, None, None, 0, 0, ws.data_ptr(), ws.numel(), st),
                        "assemble part")
                r0 += c
        del rsig
    del ws, Vs
    # drift = max |U^T W U - I| (U is in Euclidean coordinates when weighted)
    C = DevMat.empty(n_modes, n_modes)
    drift_dev = torch.zeros(1, dtype=torch.float64, device="cuda")
    ws = _ws(lib.hp_drift_workspace_bytes(d, n_modes))
    with _phase("drift", float(d) * n_modes * (n_modes + 1)):
        N.check(lib.hp_drift(U.ptr, U.ld, d, n_modes, C.ptr, C.ld, drift_dev.data_ptr(), ws.data_ptr(), ws.numel(),
                             st), "drift")
    del ws
    drift = float(host_read(drift_dev)[0])
    reorthed = False
    if drift > DRIFT_TOL:
        ws = _ws(lib.hp_reortho_workspace_bytes(d, n_modes))
        passes = ctypes.c_int(0)
        # CholQR: pass 1 reuses the drift Gram (U L^-T: d N^2 flops); a second pass (SYRK + U L^-T)
        # only when the drift says kappa(U) is not ~1
        ph = _phase("reortho", float(d) * n_modes * n_modes)
        with ph:
            N.check(lib.hp_reorthonormalize(U.ptr, U.ld, d, n_modes, C.ptr, C.ld, drift, ctypes.byref(passes),
                                            ws.data_ptr(), ws.numel(), st), "re-orthonormalisation")
            if passes.value > 1:
                ph.flops += (passes.value - 1) * (float(d) * n_modes * n_modes + float(d) * n_modes * (n_modes + 1))
        del ws
        reorthed = True
    del C
    if sqrt_w is not None:  # back to the space's own coordinates (InnerProductSpace.unweigh)
        N.check(lib.hp_scale(U.ptr, U.ld, d, n_modes, None, sqrt_w.data_ptr(), None, U.ptr, U.ld, st), "unweigh")
    R = None
    if want_right:
        R = Vn.clone()
    with _phase("signs"):
        N.check(lib.hp_signs(U.ptr, U.ld, d, n_modes, R.ptr if R is not None else None,
                             R.ld if R is not None else 0, m if R is not None else 0, None, st), "signs")
    sig_host = host_read(sig_dev)
    return NodeOutput(U, sig_host, sig_dev, float(tail), R, lam_max, nkeep, drift, reorthed, sweeps, m)


def node_pod(parts: list[Part], d: int, eps: float, cutoff: float, want_right: bool, sqrt_w=None,
             gram: "DevMat | None" = None) -> NodeOutput:
    """Full device pod() of the concatenated parts (pod.py:328-337).  ``gram``: the Gramian of the
    (scaled) concatenation when the caller already has it (ProgressiveGram), bit-identical to gram_full's."""
    if sqrt_w is not None:
        parts = weigh_parts(parts, sqrt_w)
        gram = None
    with _phase("pack"):
        parts = pack_parts(parts)
    m = sum(p.mat.cols for p in parts)
    if gram is not None and gram.rows == m and gram.cols == m and m > 0:
        G = gram
    else:
        G, m, _keep = gram_full(parts, d)
    return spectrum_and_modes(G, m, parts, d, eps, cutoff, want_right, sqrt_w)


class ProgressiveGram:
    """The Gramian of a star root's input, hstack(children's sigma-scaled modes) (hierarchy.py:284-291 +
    pod.py:208-211), accumulated child pair by child pair on background streams while later children
    are still being evaluated -- the reference's wave executor (parallel.py:77-142) starts the parent
    only after the whole wave.  Every pair block is an hp_gram_pair (unsplit contraction), so the
    assembled matrix equals hp_gram on the packed concatenation bit for bit as long as that launch is
    unsplit too (hp_gram_single_split); otherwise finish() returns None and the parent computes its
    Gramian as usual.  Used by run_parallel when a wave of leaves is bound by its host-to-device
    copies (deferred uploads), where the GPU would otherwise idle.

    At most WAVE_INFLIGHT pair GEMMs (16 CTAs each, one 128 x 128 tile over the whole contraction per
    CTA) run beside the wave, none once only TAIL_CHILDREN children are outstanding; finish() releases
    the rest on DRAIN_STREAMS streams."""

    WAVE_INFLIGHT = 8    # measured (tools/e2e_progressive_probe.py): 3..8 in flight all land within 2 % of each other
    TAIL_CHILDREN = 4
    TAIL_INFLIGHT = 0
    DRAIN_STREAMS = 10
    _streams: list = []
    _lock = threading.Lock()

    def __init__(self, d: int, children: list[int], slot_cols: list[int]):
        self.d = int(d)
        self.children = list(children)
        self.pos = {c: i for i, c in enumerate(self.children)}
        self.slot, self.width, off = {}, {}, 0
        for c, n in zip(self.children, slot_cols):
            self.slot[c] = off
            self.width[c] = int(n)
            off += _even(int(n))
        self.m_up = off
        self.G = DevMat.empty(off, off, zero=True)
        self.parts: dict = {}      # child -> Part (U, sigma) or None for an empty child
        self.queue: list = []      # pending (row child, column child): upper blocks, rows = the earlier child
        self.events: list = []     # events of launched pairs
        self.ok = True
        main = torch.cuda.current_stream()
        with ProgressiveGram._lock:
            if not ProgressiveGram._streams:  # default (lowest) priority: the stream workers run above it
                ProgressiveGram._streams = [torch.cuda.Stream() for _ in range(self.DRAIN_STREAMS)]
        self.streams = ProgressiveGram._streams
        for s in self.streams:
            s.wait_stream(main)    # the zero fill of G
        self.turn = 0

    def add(self, child: int, modes) -> None:
        """Child ``child`` finished with ModeSet ``modes`` (its stream is idle: evaluate_node ends with a
        device synchronize).  Queues its pairs with every finished sibling and launches what fits."""
        if not self.ok:
            return
        try:
            parts = modes.scaled_parts() if modes.count else []
            if modes.count and (len(parts) != 1 or parts[0].scale is None or not modes.orthonormal
                                or not parts[0].mat.aligned16()
                                or parts[0].mat.cols > self.width[child]):
                self.ok = False
                return
            self.parts[child] = parts[0] if modes.count else None
            if modes.count:
                for other, q in self.parts.items():
                    if q is None or other == child:
                        continue
                    # hp_gram forms the entries with row <= column: rows = the earlier child
                    pair = (child, other) if self.pos[child] < self.pos[other] else (other, child)
                    self.queue.append(pair)
                self.queue.append((child, child))
            # the background work pays while the wave waits for uploads; once only TAIL_CHILDREN children
            # are outstanding the wave is compute-bound and gets the GPU to itself until finish()
            outstanding = len(self.children) - len(self.parts)
            self._pump(self.WAVE_INFLIGHT if outstanding > self.TAIL_CHILDREN else self.TAIL_INFLIGHT)
        except Exception:
            self.ok = False

    def _pump(self, limit: int) -> None:
        self.events = [e for e in self.events if not e.query()]
        lib = N.load()
        while self.queue and len(self.events) < limit:
            a, b = self.queue.pop(0)
            pa, pb = self.parts[a], self.parts[b]
            s = self.streams[self.turn % len(self.streams)]
            self.turn += 1
            dst = self.G.ptr + 8 * (self.slot[a] + self.slot[b] * self.G.ld)
            N.check(lib.hp_gram_pair(pa.mat.vecset(), pa.scale.data_ptr(), pa.mat.cols, pb.mat.vecset(),
                                     pb.scale.data_ptr(), pb.mat.cols, self.d, int(a == b), dst, self.G.ld,
                                     s.cuda_stream), "Gram pair")
            ev = torch.cuda.Event()
            ev.record(s)
            self.events.append(ev)

    def finish(self):
        """Launch what is still queued, make the caller's stream wait for all of it and return the
        Gramian of the compact concatenation (children in list order), or None when the result
        would not be bit-identical to gram_full's."""
        lib = N.load()
        try:
            if not self.ok or set(self.parts) != set(self.children):
                return None
            live = [c for c in self.children if self.parts[c] is not None]
            m = sum(self.parts[c].mat.cols for c in live)
            if len(live) < PACK_MIN_PARTS or not lib.hp_gram_single_split(m, self.d):
                return None
            self._pump(1 << 30)
            main = torch.cuda.current_stream()
            for s in self.streams:
                main.wait_stream(s)
            st = _stream()
            G = self.G
            off, at = {}, 0
            for c in live:
                off[c] = at
                at += self.parts[c].mat.cols
            if any(off[c] != self.slot[c] for c in live):  # children kept fewer modes than their slots: compact
                G = DevMat.empty(m, m)
                for a in live:
                    for b in live:
                        if self.pos[a] > self.pos[b]:
                            continue
                        na, nb = self.parts[a].mat.cols, self.parts[b].mat.cols
                        src = self.G.ptr + 8 * (self.slot[a] + self.slot[b] * self.G.ld)
                        dst = G.ptr + 8 * (off[a] + off[b] * G.ld)
                        N.check(lib.hp_scale(src, self.G.ld, na, nb, None, None, None, dst, G.ld, st), "compact Gram")
            elif m != self.m_up:
                G = self.G.view_cols(0, m)
                G = DevMat(G.storage, m, m, G.ld, G.offset)
            N.check(lib.hp_mirror_upper(G.ptr, G.ld, m, st), "mirror Gram")
            return G
        except Exception:
            return None
        finally:
            self.wait()

    def wait(self) -> None:
        """Nothing of this object may still run once the children's matrices are released."""
        self.queue.clear()
        for s in self.streams:
            torch.cuda.current_stream().wait_stream(s)


def node_block_pod(prior_U: DevMat, prior_sig_dev, fresh: list[Part], d: int, eps: float, cutoff: float,
                   want_right: bool, sqrt_w=None) -> NodeOutput:
    """Device block_gramian_pod (pod.py:376-395)."""
    prior_parts = [Part(prior_U, prior_sig_dev)]
    if sqrt_w is not None:
        prior_parts = weigh_parts(prior_parts, sqrt_w)
        fresh = weigh_parts(fresh, sqrt_w)
    G, total, _keep = gram_block(prior_parts[0].mat, prior_sig_dev, fresh, d)
    return spectrum_and_modes(G, total, prior_parts + list(fresh), d, eps, cutoff, want_right, sqrt_w)


def synchronize():
    if D_AVAILABLE():
        torch.cuda.current_stream().synchronize()


def D_AVAILABLE():
    return torch is not None and torch.cuda.is_available()


def residual_energy(S: DevMat, Phi: DevMat | None, sqrt_w=None) -> float:
    """sum_j ||s_j - Phi Phi^T W s_j||_W^2 with explicit residuals (hierarchy.py:246-253)."""
    lib = N.load()
    st = _stream()
    X = DevMat.empty(S.rows, S.cols)
    N.check(lib.hp_scale(S.ptr, S.ld, S.rows, S.cols, _ptr(sqrt_w), None, None, X.ptr, X.ld, st), "residual copy")
    if Phi is not None and Phi.cols:
        Y = Phi
        if sqrt_w is not None:
            Y = DevMat.empty(Phi.rows, Phi.cols)
            N.check(lib.hp_scale(Phi.ptr, Phi.ld, Phi.rows, Phi.cols, sqrt_w.data_ptr(), None, None, Y.ptr, Y.ld,
                                 st), "weigh modes")
        n, m, d = Y.cols, S.cols, S.rows
        coeff = DevMat.empty(n, m)
        ws = _ws(max(lib.hp_gemm_workspace_bytes(n, m, d, 0, 0), lib.hp_gemm_workspace_bytes(d, m, n, 0, 0)))
        N.check(lib.hp_gemm(1, 1, n, m, d, Y.vecset(), X.vecset(), 1.0, 0.0, coeff.ptr, coeff.ld, None, None, None,
                            0, 0, ws.data_ptr(), ws.numel(), st), "projection coefficients")
        N.check(lib.hp_gemm(0, 1, d, m, n, Y.vecset(), coeff.vecset(), -1.0, 1.0, X.ptr, X.ld, None, None, None,
                            0, 0, ws.data_ptr(), ws.numel(), st), "residual")
    out = torch.zeros(1, dtype=torch.float64, device="cuda")
    ws = _ws(lib.hp_sumsq_workspace_bytes())
    N.check(lib.hp_sumsq(X.ptr, X.ld, X.rows, X.cols, out.data_ptr(), ws.data_ptr(), ws.numel(), st), "sumsq")
    return float(host_read(out)[0])


def block_diag_times(blocks: list, right: DevMat) -> DevMat:
    """stacked_diag(blocks) @ right (hierarchy.py:256-265, 292-295): row block c of
    the result is blocks[c] @ right[off_c : off_c + cols_c, :]."""
    lib = N.load()
    st = _stream()
    rows = sum(b.rows for b in blocks)
    ncol = right.cols
    out = DevMat.empty(rows, ncol, zero=True)
    r = c = 0
    for b in blocks:
        if b.rows and ncol and b.cols:
            rv = N.VecSet(right.ptr + 8 * c, right.ld, None, int(right.ld % 2 == 0 and (right.ptr + 8 * c) % 16 == 0))
            tmp = DevMat.empty(b.rows, ncol)
            ws = _ws(lib.hp_gemm_workspace_bytes(b.rows, ncol, b.cols, 0, 0))
            N.check(lib.hp_gemm(0, 1, b.rows, ncol, b.cols, b.vecset(), rv, 1.0, 0.0, tmp.ptr, tmp.ld, None, None,
                                None, 0, 0, ws.data_ptr(), ws.numel(), st), "right factor")
            N.check(lib.hp_scale(tmp.ptr, tmp.ld, b.rows, ncol, None, None, None, out.ptr + 8 * r, out.ld, st),
                    "right factor place")
        r += b.rows
        c += b.cols
    return out
