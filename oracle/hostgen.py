"""Host-only (NumPy/SciPy) generators of BASELINE inputs -- TEST INFRASTRUCTURE.

Used by the c1 parity fixture (``tests/golden/make_c1_fixture.py``), the GPU
parity test that regenerates the same snapshots on the GPU box, and the
``bench.py --impl reference`` arm, which must not load the product's shared
library.  Nothing here imports ``paper_1607_05210_b200`` or torch.

``decay`` follows the reference's ``synthetic_decay`` convention
(``datagen.py:122-143``): ``SeedSequence(seed).spawn(2)`` -> Philox standard
normal frames, economic ``scipy.linalg.qr`` with diag(R) > 0, S = Q1 diag(sigma)
Q2^T -- with BASELINE.json's spectrum sigma_i = 10^(-decades (i-1)/(k-1))
instead of exp(-rate n).  The Gaussian draws are bit-reproducible on any host;
the QR/GEMM roundings depend on the host's BLAS kernels, so consumers that need
the fixture's exact bytes compare ``checksum`` within a stated tolerance.
"""

from __future__ import annotations

import numpy as np
import scipy.linalg


def haar_frame(rows: int, k: int, seq) -> np.ndarray:
    """datagen.py:133-138 -- Q of a Philox Gaussian rows x k matrix, diag(R) > 0."""
    g = np.random.Generator(np.random.Philox(seq)).standard_normal((rows, k))
    q, r = scipy.linalg.qr(g, mode="economic", overwrite_a=True, check_finite=False)
    signs = np.sign(np.diag(r))
    signs[signs == 0.0] = 1.0
    q *= signs[None, :]
    return q


def decay_spectrum(k: int, decades: float) -> np.ndarray:
    return 10.0 ** (-decades * np.arange(k, dtype=np.float64) / max(k - 1, 1))


def decay(d: int, m: int, decades: float, seed: int, want_left: bool = False):
    """BASELINE configs 0/1: S = Q1 diag(sigma) Q2^T (d x m, Fortran order).

    Returns (S, sigma) or (S, sigma, Q1) -- Q1's leading columns span the exact
    POD space, the reference point of the parity fixture's angle floors."""
    k = min(d, m)
    seq_left, seq_right = np.random.SeedSequence(seed).spawn(2)
    left = haar_frame(d, k, seq_left)
    right = haar_frame(m, k, seq_right)
    sig = decay_spectrum(k, decades)
    s = np.asfortranarray((left * sig[None, :]) @ right.T)
    del right
    return (s, sig, left) if want_left else (s, sig)


CONFIG_DECAY = {0: dict(d=20_000, m=1_000, decades=8.0, rel=1e-4, omega=1.0, block=1_000),
                1: dict(d=200_000, m=8_192, decades=10.0, rel=1e-6, omega=0.75, block=512)}


def checksum(a: np.ndarray) -> np.ndarray:
    """Order-free fingerprint of a snapshot matrix: Frobenius norm, column sums of a fixed
    column sample, and a strided entry sample (compared within a tolerance)."""
    a = np.asarray(a)
    cols = np.arange(0, a.shape[1], max(1, a.shape[1] // 61))
    rows = np.arange(0, a.shape[0], max(1, a.shape[0] // 53))
    return np.concatenate([[np.linalg.norm(a)], a[:, cols].sum(axis=0), a[np.ix_(rows, cols)].reshape(-1)])
