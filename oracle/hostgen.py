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


# ---------------------------------------------------------------------------- configs 2-4 (timing samples)
def pulse(d: int, cols: np.ndarray, seed: int) -> np.ndarray:
    """BASELINE config 2 columns: u_j(x) = exp(-(x - 0.1 - 0.8 t_j)^2 / (2 w_j^2)) on x = linspace(0, 1, d),
    t_j ~ U[0,1], w_j ~ U[0.01, 0.05] per column id (the same Philox streams as the device generator)."""
    rng = np.random.Generator(np.random.Philox(np.random.SeedSequence([int(seed), 2])))
    nmax = int(cols.max()) + 1 if cols.size else 0
    t = rng.uniform(0.0, 1.0, nmax)[cols]
    w = rng.uniform(0.01, 0.05, nmax)[cols]
    x = np.linspace(0.0, 1.0, d)
    z = (x[:, None] - 0.1 - 0.8 * t[None, :]) / w[None, :]
    return np.asfortranarray(np.exp(-0.5 * z * z))


_SINE_COEF: dict = {}


def _sine_coefficients(seed: int, nmax: int, modes: int) -> np.ndarray:
    """Rows 0..nmax-1 of the seeded N(0,1) coefficient stream (drawn row-major, so a prefix does
    not depend on how many rows are drawn); cached, grown in powers of two."""
    have = _SINE_COEF.get((seed, modes))
    if have is None or have.shape[0] < nmax:
        rows = 1 << max(nmax - 1, 1).bit_length()
        rng = np.random.Generator(np.random.Philox(np.random.SeedSequence([int(seed), 3])))
        have = rng.standard_normal((rows, modes))
        _SINE_COEF[(seed, modes)] = have
    return have[:nmax]


def sine(d: int, cols: np.ndarray, seed: int, noise_key: int = 0, modes: int = 300, noise: float = 1e-8) -> np.ndarray:
    """BASELINE config 3 columns: sum_{k<=300} k^-2 a_jk sin(k pi x) + 1e-8 N(0,1).  The coefficient
    stream is the device generator's; the noise stream is NumPy's (the device draws it with the
    CUDA generator), so these are statistically -- not bytewise -- the device's columns: they
    serve the CPU timing samples of bench.py only."""
    nmax = int(cols.max()) + 1 if cols.size else 0
    a = _sine_coefficients(seed, nmax, modes)[cols] / (np.arange(1, modes + 1) ** 2)[None, :]
    x = np.linspace(0.0, 1.0, d)
    basis = np.sin(np.pi * np.arange(1, modes + 1)[None, :] * x[:, None])  # (d, modes)
    out = basis @ a.T
    nrng = np.random.Generator(np.random.Philox(np.random.SeedSequence([int(seed), 5, int(noise_key)])))
    out += noise * nrng.standard_normal(out.shape)
    return np.asfortranarray(out)


def mixed(d: int, cols: np.ndarray, m_total: int, seed: int, noise_key: int = 0) -> np.ndarray:
    """BASELINE config 4 columns: half sine field, half pulses, interleaved by a seeded permutation."""
    perm = np.random.Generator(np.random.Philox(np.random.SeedSequence([int(seed), 4]))).permutation(m_total)
    is_sine = perm[cols] < m_total // 2
    out = np.empty((d, cols.size), order="F")
    if is_sine.any():
        out[:, is_sine] = sine(d, cols[is_sine], seed, noise_key)
    if (~is_sine).any():
        out[:, ~is_sine] = pulse(d, cols[~is_sine], seed)
    return out
