"""ctypes binding of libhapod_b200.so (include/hapod_b200.h).

The CUDA library is the ONLY compute path: there is no CPU fallback.  If the
shared object is missing or a CUDA device is absent, every entry point raises.
"""

from __future__ import annotations

import ctypes
import os
import threading

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libhapod_b200.so")
ABI_VERSION = 1

HP_OK, HP_EINVAL, HP_ECUDA, HP_ELINALG, HP_ENOMEM = 0, 1, 2, 3, 4

c_i64 = ctypes.c_int64
c_dbl = ctypes.c_double
c_vp = ctypes.c_void_p
c_int = ctypes.c_int
c_size = ctypes.c_size_t


class VecSet(ctypes.Structure):
    _fields_ = [("base", c_vp), ("ld", c_i64), ("table", c_vp), ("aligned16", c_int)]


_SIGNATURES = {
    "hp_abi_version": (c_int, []),
    "hp_launch_count": (ctypes.c_longlong, []),
    "hp_set_debug": (ctypes.c_int, [ctypes.c_int]),
    "hp_last_error": (ctypes.c_char_p, []),
    "hp_device_sm_count": (c_int, [c_int]),
    "hp_gemm_workspace_bytes": (c_size, [c_i64, c_i64, c_i64, c_int, c_int]),
    "hp_gemm": (c_int, [c_int, c_int, c_i64, c_i64, c_i64, VecSet, VecSet, c_dbl, c_dbl, c_vp, c_i64,
                        c_vp, c_vp, c_vp, c_int, c_int, c_vp, c_size, c_vp]),
    "hp_gram_workspace_bytes": (c_size, [c_i64, c_i64]),
    "hp_gram": (c_int, [VecSet, c_i64, c_i64, c_vp, c_vp, c_i64, c_vp, c_size, c_vp]),
    "hp_gram_single_split": (c_int, [c_i64, c_i64]),
    "hp_gram_pair": (c_int, [VecSet, c_vp, c_i64, VecSet, c_vp, c_i64, c_i64, c_int, c_vp, c_i64, c_vp]),
    "hp_mirror_upper": (c_int, [c_vp, c_i64, c_i64, c_vp]),
    "hp_block_gram_workspace_bytes": (c_size, [c_i64, c_i64, c_i64]),
    "hp_block_gram": (c_int, [VecSet, c_vp, c_i64, VecSet, c_vp, c_i64, c_i64, c_vp, c_i64, c_vp, c_size, c_vp]),
    "hp_pstrf_workspace_bytes": (c_size, [c_i64]),
    "hp_pstrf": (c_int, [c_vp, c_i64, c_i64, c_vp, c_i64, c_vp, c_dbl, c_dbl, ctypes.POINTER(c_i64), c_vp, c_size,
                         c_vp]),
    "hp_syev_workspace_bytes": (c_size, [c_i64]),
    "hp_syev": (c_int, [c_vp, c_i64, c_i64, c_vp, c_vp, c_i64, c_i64, c_dbl, c_dbl, c_dbl, c_dbl, c_int, c_int,
                        ctypes.POINTER(c_int), ctypes.POINTER(c_dbl), c_vp, c_size, c_vp]),
    "hp_syev_padded_order": (c_i64, [c_i64]),
    "hp_syev_rows": (c_int, [c_vp, c_i64, c_i64, c_vp, c_vp, c_i64, c_i64, c_dbl, c_dbl, c_dbl, c_dbl, c_int,
                             ctypes.POINTER(c_int), ctypes.POINTER(c_dbl), c_i64, c_i64, c_vp, c_size, c_vp]),
    "hp_syev_tri_max_order": (c_i64, []),
    "hp_syev_tri_workspace_bytes": (c_size, [c_i64]),
    "hp_syev_tri": (c_int, [c_vp, c_i64, c_i64, c_dbl, c_dbl, c_vp, c_vp, c_i64, ctypes.POINTER(c_i64),
                            ctypes.POINTER(c_int), ctypes.POINTER(c_dbl), c_vp, c_size, c_vp]),
    "hp_truncate": (c_int, [c_vp, c_i64, c_dbl, c_dbl, c_i64, c_vp, c_vp, c_vp]),
    "hp_assemble_workspace_bytes": (c_size, [c_i64, c_i64, c_i64]),
    "hp_assemble": (c_int, [VecSet, c_i64, c_i64, c_vp, c_i64, c_vp, c_i64, c_vp, c_i64, c_vp, c_size, c_vp]),
    "hp_drift_workspace_bytes": (c_size, [c_i64, c_i64]),
    "hp_drift": (c_int, [c_vp, c_i64, c_i64, c_i64, c_vp, c_i64, c_vp, c_vp, c_size, c_vp]),
    "hp_reortho_workspace_bytes": (c_size, [c_i64, c_i64]),
    "hp_reorthonormalize": (c_int, [c_vp, c_i64, c_i64, c_i64, c_vp, c_i64, c_dbl, ctypes.POINTER(c_int),
                                    c_vp, c_size, c_vp]),
    "hp_signs": (c_int, [c_vp, c_i64, c_i64, c_i64, c_vp, c_i64, c_i64, c_vp, c_vp]),
    "hp_transpose_rm_to_cm": (c_int, [c_vp, c_i64, c_i64, c_vp, c_i64, c_vp]),
    "hp_scale": (c_int, [c_vp, c_i64, c_i64, c_i64, c_vp, c_vp, c_vp, c_vp, c_i64, c_vp]),
    "hp_finite_check": (c_int, [c_vp, c_i64, c_i64, c_i64, c_vp, c_vp]),
    "hp_read_small": (c_int, [c_vp, c_vp, c_i64, c_vp]),
    "hp_add_diag": (c_int, [c_vp, c_i64, c_i64, c_dbl, c_vp]),
    "hp_gram_drift": (c_int, [c_vp, c_i64, c_i64, c_vp, c_vp]),
    "hp_add": (c_int, [c_vp, c_vp, c_i64, c_vp]),
    "hp_col_norms_sq": (c_int, [c_vp, c_i64, c_i64, c_i64, c_vp, c_vp, c_vp]),
    "hp_col_absmax": (c_int, [c_vp, c_i64, c_i64, c_i64, c_i64, c_vp, c_vp, c_vp]),
    "hp_chol_inverse_workspace_bytes": (c_size, [c_i64]),
    "hp_chol_inverse": (c_int, [c_vp, c_i64, c_i64, c_vp, c_i64, c_vp, c_vp, c_size, c_vp]),
    "hp_sumsq_workspace_bytes": (c_size, []),
    "hp_sumsq": (c_int, [c_vp, c_i64, c_i64, c_i64, c_vp, c_vp, c_size, c_vp]),
}

EXPORTED = tuple(_SIGNATURES)

_lib = None
_lock = threading.Lock()


class NativeMissing(RuntimeError):
    pass


# set in the target process by Nsight Compute / Nsight Systems / CUPTI-injection tools
_PROFILER_ENV = ("CUDA_INJECTION64_PATH", "NV_COMPUTE_PROFILER_PERFWORKS_DIR", "NV_NSIGHT_INJECTION_PORT_BASE",
                 "NSYS_PROFILING_SESSION_ID")


def load(path: str | None = None):
    """Load (once) and return the ctypes handle; raises if the .so is absent."""
    global _lib
    if _lib is not None:
        return _lib
    with _lock:
        if _lib is not None:
            return _lib
        p = path or LIB_PATH
        if not os.path.exists(p):
            raise NativeMissing(
                f"{p} not found: build it with ./build_native.sh (or __graft_entry__.build()); "
                "there is no CPU fallback")
        lib = ctypes.CDLL(p)
        for name, (res, args) in _SIGNATURES.items():
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        if lib.hp_abi_version() != ABI_VERSION:
            raise NativeMissing(f"ABI mismatch: library {lib.hp_abi_version()} != {ABI_VERSION}")
        if any(v in os.environ for v in _PROFILER_ENV):
            # under an injected per-kernel profiler (ncu crashed on replayed graph launches): launch the
            # Jacobi sweeps directly -- a launch mechanism only, no result depends on it
            lib.hp_set_debug(lib.hp_set_debug(0) | 16)
        _lib = lib
        return lib


def check(rc: int, what: str):
    """Map an hp_status to the reference's exception types."""
    if rc == HP_OK:
        return
    msg = (load().hp_last_error() or b"").decode(errors="replace")
    text = f"{what}: {msg}"
    if rc == HP_EINVAL:
        raise ValueError(text)
    if rc == HP_ELINALG:
        raise np.linalg.LinAlgError(text)
    raise RuntimeError(text)
