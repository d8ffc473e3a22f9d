"""Proper orthogonal decomposition of snapshot blocks -- B200 backend.

Mirrors the public surface of the reference module ``hapod.pod``
(/root/reference/pkg/src/hapod/pod.py:21-31): the same classes, functions,
argument meanings, defaults and exceptions.  What changes is where the data
lives and who computes: snapshot blocks and mode sets are held in HBM
(column-major float64) and every arithmetic step of the method of snapshots
runs in the hand-written sm_100a kernels of ``libhapod_b200.so``:

  Gram SYRK (DMMA)  ->  block-Jacobi eigensolve  ->  truncation scan
  ->  reconstruction GEMM (DMMA)  ->  drift check / CholQR re-orthonormalisation
  ->  sign convention.

NumPy arrays are accepted everywhere the reference accepts them and are
returned by the same attribute names (``ModeSet.modes``, ``.sigmas``,
``.right``, ``SnapshotBlock.values``), copied back lazily.  The ``"svd"``
backend kind of the reference (direct dgesdd, pod.py:338-348) is not part of
the method-of-snapshots hot path and raises instead of silently running on the
CPU.
"""

from __future__ import annotations

import math

import numpy as np

from . import _device as D

__all__ = [
    "DEFAULT_GRAM_CUTOFF",
    "InnerProductSpace",
    "SnapshotBlock",
    "ModeSet",
    "PodBackend",
    "truncation_rank",
    "gramian",
    "pod",
    "block_gramian_pod",
]

#: Gramian eigenvalues below ``factor * lam_max * m`` count as numerical zeros (pod.py:33-34).
DEFAULT_GRAM_CUTOFF = 4.0 * float(np.finfo(np.float64).eps)


def _read_only(a):
    a = np.ascontiguousarray(a, dtype=np.float64)
    a.setflags(write=False)
    return a


def _is_tensor(x):
    return D.torch is not None and D.torch.is_tensor(x)


class InnerProductSpace:
    """R^d with an optional strictly positive diagonal weight vector (pod.py:43-97)."""

    __slots__ = ("dimension", "weights", "_sqrt_w", "_sqrt_w_dev", "_w_dev")

    def __init__(self, dimension, weights=None):
        if int(dimension) != dimension or dimension < 1:
            raise ValueError(f"space dimension must be a positive integer, got {dimension}")
        object.__setattr__(self, "dimension", int(dimension))
        object.__setattr__(self, "_sqrt_w_dev", None)
        object.__setattr__(self, "_w_dev", None)
        if weights is not None:
            w = np.asarray(weights, dtype=np.float64)
            if w.shape != (self.dimension,):
                raise ValueError(f"weights shape {w.shape} does not match dimension {self.dimension}")
            if not np.all(np.isfinite(w)) or np.any(w <= 0.0):
                raise ValueError("weights must be finite and strictly positive")
            object.__setattr__(self, "weights", _read_only(w))
            object.__setattr__(self, "_sqrt_w", _read_only(np.sqrt(w)))
        else:
            object.__setattr__(self, "weights", None)
            object.__setattr__(self, "_sqrt_w", None)

    def __setattr__(self, name, value):
        raise AttributeError("InnerProductSpace is immutable")

    def __repr__(self):
        return f"InnerProductSpace(dimension={self.dimension}, weighted={self.weights is not None})"

    def same_as(self, other: "InnerProductSpace") -> bool:
        if self.dimension != other.dimension:
            return False
        if (self.weights is None) != (other.weights is None):
            return False
        return self.weights is None or bool(np.array_equal(self.weights, other.weights))

    def sqrt_weights_device(self):
        """sqrt(w) as a CUDA tensor (None for the Euclidean space)."""
        if self.weights is None:
            return None
        if self._sqrt_w_dev is None:
            D.require_cuda()
            object.__setattr__(self, "_sqrt_w_dev", D.torch.from_numpy(np.array(self._sqrt_w)).to("cuda"))
        return self._sqrt_w_dev

    def weights_device(self):
        """w as a CUDA tensor (None for the Euclidean space)."""
        if self.weights is None:
            return None
        if self._w_dev is None:
            D.require_cuda()
            object.__setattr__(self, "_w_dev", D.torch.from_numpy(np.array(self.weights)).to("cuda"))
        return self._w_dev

    def gram(self, a, b):
        """All pairwise inner products between the columns of ``a`` and ``b`` (pod.py:87-91):
        ``a.T @ (w * b)``, computed by the DMMA GEMM engine.  NumPy operands give a NumPy
        array, CUDA tensors a CUDA tensor."""
        return D.space_gram(a, b, self.weights_device())

    def norms_sq(self, a):
        """Squared norm of every column (pod.py:93-97), computed on the device."""
        return D.space_norms_sq(a, self.weights_device())

    # host-side coordinate maps with the reference semantics (pod.py:76-84)
    def weigh(self, a):
        if self.weights is None:
            return a
        return a * self._sqrt_w[:, None]

    def unweigh(self, a):
        if self.weights is None:
            return a
        return a / self._sqrt_w[:, None]


class SnapshotBlock:
    """A d x m column block of snapshots living in one space (pod.py:100-121).

    ``values`` may be a NumPy array (any order), a CPU or a CUDA torch tensor.
    By default the block is uploaded to HBM (column-major) and checked for
    non-finite entries on the device at construction, as the reference does on
    the host (pod.py:115-116).

    ``defer_upload=True`` (host inputs only) keeps the host buffer and uploads
    on first device use, on the caller's current CUDA stream; column views
    (``column_block``, ``distribute_columns``) upload only their own columns.
    Under ``run_parallel`` every leaf's host-to-device copy then overlaps the
    other leaves' PODs.  The finiteness check (ValueError) happens at that
    first use instead of at construction."""

    __slots__ = ("space", "_dev", "_host", "_count")

    def __init__(self, space: InnerProductSpace, values, defer_upload: bool = False):
        if _is_tensor(values):
            shape = tuple(values.shape)
        else:
            values = np.asarray(values, dtype=np.float64)
            shape = values.shape
        if len(shape) != 2:
            raise ValueError(f"snapshot block must be 2-d, got shape {shape}")
        if shape[0] != space.dimension:
            raise ValueError(f"snapshot rows {shape[0]} do not match space dimension {space.dimension}")
        object.__setattr__(self, "space", space)
        object.__setattr__(self, "_count", int(shape[1]))
        is_device = _is_tensor(values) and values.is_cuda
        if defer_upload and not is_device:
            object.__setattr__(self, "_host", values)
            object.__setattr__(self, "_dev", None)
            return
        object.__setattr__(self, "_host", None if _is_tensor(values) else values)
        object.__setattr__(self, "_dev", D.upload(values))

    def __setattr__(self, name, value):
        raise AttributeError("SnapshotBlock is immutable")

    @classmethod
    def _from_device(cls, space, dev: "D.DevMat", host=None):
        obj = cls.__new__(cls)
        object.__setattr__(obj, "space", space)
        object.__setattr__(obj, "_count", dev.cols)
        object.__setattr__(obj, "_host", host)
        object.__setattr__(obj, "_dev", dev)
        return obj

    @property
    def count(self) -> int:
        return self._count

    @property
    def device(self) -> "D.DevMat":
        if self._dev is None:  # deferred upload: now, through the shared copy stream
            object.__setattr__(self, "_dev", D.upload(self._host, via=D.copy_stream()))
        return self._dev

    @property
    def values(self) -> np.ndarray:
        if self._host is None:
            object.__setattr__(self, "_host", self._dev.to_numpy())
        v = self._host
        if _is_tensor(v):
            v = v.numpy()
        if isinstance(v, np.ndarray) and v.flags.writeable:
            v = v.view()
            v.setflags(write=False)
        return v

    def column_block(self, j0: int, j1: int) -> "SnapshotBlock":
        """Columns j0:j1 as a new block sharing storage (device view, or a deferred host view)."""
        if self._dev is None:
            obj = SnapshotBlock.__new__(SnapshotBlock)
            object.__setattr__(obj, "space", self.space)
            object.__setattr__(obj, "_count", j1 - j0)
            object.__setattr__(obj, "_host", self._host[:, j0:j1])
            object.__setattr__(obj, "_dev", None)
            return obj
        host = None
        if isinstance(self._host, np.ndarray):
            host = self._host[:, j0:j1]
        return SnapshotBlock._from_device(self.space, self._dev.view_cols(j0, j1), host)


class ModeSet:
    """POD output: left singular vectors with their singular values (pod.py:124-165).

    ``orthonormal=False`` marks the epsilon = 0 passthrough convention.  On the
    device a mode set is a list of column parts (DevMat, scale) whose
    concatenation is ``modes``; an orthonormal result is a single part, a
    passthrough of a merge keeps its parts without an hstack copy."""

    __slots__ = ("space", "sigmas", "orthonormal", "tail_energy", "_parts", "_modes_host", "_right",
                 "_right_host", "_sig_dev", "diagnostics")

    def __init__(self, space, sigmas, modes, orthonormal=True, tail_energy=0.0, right=None):
        s = np.asarray(sigmas, dtype=np.float64).reshape(-1)
        if _is_tensor(modes):
            shape = tuple(modes.shape)
        else:
            modes = np.asarray(modes, dtype=np.float64)
            shape = modes.shape
        if len(shape) != 2 or shape[0] != space.dimension or shape[1] != s.size:
            raise ValueError(f"mode shape {shape} inconsistent with {s.size} sigmas in R^{space.dimension}")
        self._validate_sigmas(s, orthonormal)
        dev = D.upload(modes)
        self._init(space, s, [D.Part(dev, None)], orthonormal, tail_energy, right)
        if not _is_tensor(modes):
            object.__setattr__(self, "_modes_host", _read_only(modes))

    @staticmethod
    def _validate_sigmas(s, orthonormal):
        if s.size and (not np.all(np.isfinite(s)) or np.any(s < 0.0) or np.any(np.diff(s) > 0.0)):
            raise ValueError("sigmas must be finite, nonnegative and non-increasing")
        if not orthonormal and s.size and not np.all(s == 1.0):
            raise ValueError("passthrough mode sets must carry unit sigmas")

    def _init(self, space, s, parts, orthonormal, tail_energy, right):
        object.__setattr__(self, "space", space)
        object.__setattr__(self, "sigmas", _read_only(s))
        object.__setattr__(self, "orthonormal", bool(orthonormal))
        object.__setattr__(self, "tail_energy", float(tail_energy))
        object.__setattr__(self, "_parts", list(parts))
        object.__setattr__(self, "_modes_host", None)
        object.__setattr__(self, "_sig_dev", None)
        object.__setattr__(self, "diagnostics", None)
        if right is None or isinstance(right, D.DevMat):
            object.__setattr__(self, "_right", right)
            object.__setattr__(self, "_right_host", None)
        else:
            object.__setattr__(self, "_right", None)
            object.__setattr__(self, "_right_host", _read_only(np.asarray(right, dtype=np.float64)))

    @classmethod
    def _device(cls, space, sigmas, parts, orthonormal=True, tail_energy=0.0, right=None, sig_dev=None,
                diagnostics=None):
        obj = cls.__new__(cls)
        s = np.asarray(sigmas, dtype=np.float64).reshape(-1)
        cls._validate_sigmas(s, orthonormal)
        obj._init(space, s, parts, orthonormal, tail_energy, right)
        object.__setattr__(obj, "_sig_dev", sig_dev)
        object.__setattr__(obj, "diagnostics", diagnostics)
        return obj

    def __setattr__(self, name, value):
        raise AttributeError("ModeSet is immutable")

    @property
    def count(self) -> int:
        return self.sigmas.size

    @property
    def parts(self):
        return self._parts

    def sigmas_device(self):
        if self._sig_dev is None:
            D.require_cuda()
            object.__setattr__(self, "_sig_dev", D.torch.from_numpy(np.array(self.sigmas)).to("cuda"))
        return self._sig_dev

    def modes_device(self) -> "D.DevMat":
        """The modes as one column-major device matrix (materialises a passthrough concatenation)."""
        if len(self._parts) == 1 and self._parts[0].scale is None:
            return self._parts[0].mat
        out = D.DevMat.empty(self.space.dimension, self.count)
        at = 0
        lib = D.N.load()
        for p in self._parts:
            c = p.mat.cols
            if c:
                D.N.check(lib.hp_scale(p.mat.ptr, p.mat.ld, p.mat.rows, c, None, None, D._ptr(p.scale),
                                       out.col_ptr(at), out.ld, D._stream()), "concatenate")
            at += c
        object.__setattr__(self, "_parts", [D.Part(out, None)])
        return out

    @property
    def modes(self) -> np.ndarray:
        if self._modes_host is None:
            object.__setattr__(self, "_modes_host", _read_only(self.modes_device().to_numpy()))
        return self._modes_host

    @property
    def right(self):
        if self._right_host is None and self._right is not None:
            object.__setattr__(self, "_right_host", _read_only(self._right.to_numpy()))
        return self._right_host

    def right_device(self):
        return self._right

    def scaled(self) -> np.ndarray:
        """Columns sigma_n * phi_n, the snapshots fed to the parent node (pod.py:160-162)."""
        return self.modes * self.sigmas[None, :]

    def scaled_parts(self) -> list:
        """Device view of scaled(): the same parts with sigma folded into their column scales."""
        if self.count == 0:
            return []
        if not self.orthonormal:
            return list(self._parts)  # sigmas are exactly one
        sig = self.sigmas_device()
        out, at = [], 0
        for p in self._parts:
            c = p.mat.cols
            s = sig[at:at + c]
            if p.scale is not None:
                s = p.scale * s
            out.append(D.Part(p.mat, s))
            at += c
        return out

    def as_block(self) -> SnapshotBlock:
        return SnapshotBlock(self.space, self.scaled())


class PodBackend:
    """How the small dense decompositions are carried out (pod.py:168-187).

    kind "gram" is the method of snapshots -- the B200 path.  "svd" is
    accepted by the constructor (reference signature) but pod() raises for it:
    the direct SVD is not on this backend's hot path and there is no CPU
    fallback."""

    __slots__ = ("kind", "gram_eig_cutoff_factor")

    def __init__(self, kind: str = "gram", gram_eig_cutoff_factor: float = DEFAULT_GRAM_CUTOFF):
        if kind not in ("gram", "svd"):
            raise ValueError(f"unknown backend kind {kind!r}, expected 'gram' or 'svd'")
        f = gram_eig_cutoff_factor
        if not (0.0 < f < 1.0):
            raise ValueError(f"gram_eig_cutoff_factor must lie in (0, 1), got {f}")
        object.__setattr__(self, "kind", kind)
        object.__setattr__(self, "gram_eig_cutoff_factor", float(f))

    def __setattr__(self, name, value):
        raise AttributeError("PodBackend is immutable")

    def __eq__(self, other):
        return isinstance(other, PodBackend) and (self.kind, self.gram_eig_cutoff_factor) == (
            other.kind, other.gram_eig_cutoff_factor)

    def __hash__(self):
        return hash((self.kind, self.gram_eig_cutoff_factor))

    def __repr__(self):
        return f"PodBackend(kind={self.kind!r}, gram_eig_cutoff_factor={self.gram_eig_cutoff_factor!r})"


def truncation_rank(sigmas, epsilon: float) -> int:
    """Smallest N whose discarded tail satisfies sum_{n>N} sigma_n^2 <= epsilon^2
    (pod.py:190-205).  Host utility on a short vector; the device path runs the
    same rule inside the truncation kernel."""
    s = np.asarray(sigmas, dtype=np.float64).reshape(-1)
    if s.size and (np.any(s < 0.0) or np.any(np.diff(s) > 0.0)):
        raise ValueError("sigmas must be nonnegative and non-increasing")
    if epsilon < 0.0:
        raise ValueError("epsilon must be nonnegative")
    tails = np.zeros(s.size + 1)
    tails[:-1] = np.cumsum((s * s)[::-1])[::-1]
    return int(np.argmax(tails <= epsilon * epsilon))


def gramian(block: SnapshotBlock) -> np.ndarray:
    """The m x m matrix of pairwise snapshot inner products, exactly symmetric
    (pod.py:208-211), computed by the DMMA SYRK kernel."""
    parts = [D.Part(block.device, None)]
    sw = block.space.sqrt_weights_device()
    if sw is not None:
        parts = D.weigh_parts(parts, sw)
    G, m, _ = D.gram_full(parts, block.space.dimension)
    return G.to_numpy()


def _check_backend(backend):
    backend = backend or PodBackend()
    if backend.kind != "gram":
        raise ValueError("the B200 backend implements the method of snapshots (kind='gram') only; "
                         "kind='svd' has no device path and no CPU fallback")
    return backend


def _empty(space, want_right, input_count=0, tail_energy=0.0):
    # right keeps one row per input column so stacked factors stay aligned (pod.py:254-263)
    return ModeSet._device(space, np.zeros(0), [D.Part(D.DevMat.empty(space.dimension, 0), None)],
                           orthonormal=True, tail_energy=tail_energy,
                           right=D.DevMat.empty(input_count, 0) if want_right else None)


def _passthrough(space, parts, want_right) -> ModeSet:
    """epsilon = 0: the raw columns with unit sigmas (pod.py:266-275)."""
    m = sum(p.mat.cols for p in parts)
    right = None
    if want_right:
        right = np.eye(m)
    return ModeSet._device(space, np.ones(m), parts, orthonormal=False, tail_energy=0.0, right=right)


def _from_node_output(space, out: "D.NodeOutput", want_right) -> ModeSet:
    if out.U is None:  # lam_max <= 0: empty set, right keeps m rows (pod.py:281-283)
        return _empty(space, want_right, input_count=out.input_count)
    diag = {"lam_max": out.lam_max, "nkeep": out.nkeep, "drift": out.drift, "reorthonormalized": out.reorthed,
            "jacobi_sweeps": out.sweeps, "input_count": out.input_count}
    return ModeSet._device(space, out.sigmas, [D.Part(out.U, None)], orthonormal=True, tail_energy=out.tail,
                           right=out.right if want_right else None, sig_dev=out.sigmas_dev, diagnostics=diag)


def pod_parts(space, parts, epsilon: float, backend=None, want_right: bool = False, gram=None) -> ModeSet:
    """pod() of the concatenation of device parts (used by the tree drivers:
    interior nodes pass their children's scaled parts, no hstack copy).  ``gram``: the
    concatenation's Gramian when the driver already accumulated it (D.ProgressiveGram)."""
    if epsilon < 0.0:
        raise ValueError("epsilon must be nonnegative")
    backend = _check_backend(backend)
    parts = [p for p in parts if p.mat.cols]
    if epsilon == 0.0:
        return _passthrough(space, parts, want_right)
    m = sum(p.mat.cols for p in parts)
    if m == 0:
        return _empty(space, want_right)
    out = D.node_pod(parts, space.dimension, epsilon, backend.gram_eig_cutoff_factor, want_right,
                     space.sqrt_weights_device(), gram=gram)
    return _from_node_output(space, out, want_right)


def pod(block: SnapshotBlock, epsilon: float, backend: PodBackend | None = None,
        want_right: bool = False) -> ModeSet:
    """POD of a snapshot block, truncated at squared-error budget epsilon^2
    (pod.py:296-348, method-of-snapshots branch :328-337), on the B200."""
    if epsilon < 0.0:
        raise ValueError("epsilon must be nonnegative")
    _check_backend(backend)
    return pod_parts(block.space, [D.Part(block.device, None)], epsilon, backend, want_right)


def block_gramian_pod(prior: ModeSet, fresh: SnapshotBlock, epsilon: float,
                      cutoff_factor: float = DEFAULT_GRAM_CUTOFF,
                      want_right: bool = False) -> ModeSet:
    """POD of [sigma_1 phi_1, ..., sigma_N phi_N | fresh] without touching old
    inner products (pod.py:351-395): the diag(sigma^2) block is written down,
    only the mixed and fresh blocks are contracted."""
    if not prior.orthonormal:
        raise ValueError("prior modes must be orthonormal (passthrough sets cannot be extended this way)")
    if not prior.space.same_as(fresh.space):
        raise ValueError("prior modes and fresh block live in different spaces")
    if epsilon < 0.0:
        raise ValueError("epsilon must be nonnegative")
    return block_gramian_pod_parts(prior, [D.Part(fresh.device, None)], epsilon, cutoff_factor, want_right)


def block_gramian_pod_parts(prior: ModeSet, fresh_parts, epsilon, cutoff_factor=DEFAULT_GRAM_CUTOFF,
                            want_right=False) -> ModeSet:
    space = prior.space
    n_old = prior.count
    fresh_parts = [p for p in fresh_parts if p.mat.cols]
    backend = PodBackend("gram", cutoff_factor)
    if n_old == 0:
        return pod_parts(space, fresh_parts, epsilon, backend, want_right)
    if epsilon == 0.0:
        return _passthrough(space, prior.scaled_parts() + fresh_parts, want_right)
    out = D.node_block_pod(prior.modes_device(), prior.sigmas_device(), fresh_parts, space.dimension, epsilon,
                           cutoff_factor, want_right, space.sqrt_weights_device())
    return _from_node_output(space, out, want_right)
