"""Seeded synthetic snapshot sets of the BASELINE.json configurations.

BASELINE.json (``configs``) names five fp64 workloads; there is no public
dataset involved.  The generators below build them on the
device from a seed (data generation is never inside a timed region):

  c0  S = Q1 diag(sigma) Q2^T, 20,000 x 1,000, sigma_i = 10^(-8 (i-1)/999)
  c1  same construction, 200,000 x 8,192, sigma_i = 10^(-10 (i-1)/8191)
  c2  travelling Gaussian pulses, 500,000 x 32,768 (64 slices of 512)
  c3  rank-300 sine field + 1e-8 noise, 2,000,000 x 32,768 (64 leaves of 512)
  c4  half sine field / half pulses, seeded column permutation, 1,000,000 x 65,536

Q1, Q2 are Q factors of seeded standard-Gaussian matrices with diag(R) > 0,
the synthetic_decay convention of the reference (datagen.py:133-138).  Seeds
are c0..c4 = 0..4.  Every generator accepts a reduced row
count ``d`` so the CPU oracle can run the same column structure (the c0/c1
node sizes are d-invariant).
"""

from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np

from . import _device as D

CONFIGS = {
    0: dict(name="c0-single-pod", d=20_000, m=1_000, rel=1e-4, omega=1.0, leaves=1, block=1_000, kind="decay",
            decades=8.0),
    1: dict(name="c1-star16", d=200_000, m=8_192, rel=1e-6, omega=0.75, leaves=16, block=512, kind="decay",
            decades=10.0),
    2: dict(name="c2-chain64", d=500_000, m=32_768, rel=1e-3, omega=0.9, leaves=64, block=512, kind="pulse"),
    3: dict(name="c3-star64", d=2_000_000, m=32_768, rel=1e-5, omega=0.75, leaves=64, block=512, kind="sine"),
    4: dict(name="c4-8chains16", d=1_000_000, m=65_536, rel=1e-4, omega=0.8, leaves=128, block=512, kind="mixed"),
}


def _gen(seed: int, stream_id: int):
    g = D.torch.Generator(device="cuda")
    g.manual_seed(int(seed) * 1_000_003 + int(stream_id))
    return g


def haar_frame(rows: int, k: int, seed: int, stream_id: int):
    """Q factor (diag(R) > 0) of a seeded rows x k standard-Gaussian matrix, on the device."""
    torch = D.torch
    g = torch.randn((rows, k), dtype=torch.float64, device="cuda", generator=_gen(seed, stream_id))
    q, r = torch.linalg.qr(g, mode="reduced")
    sgn = torch.sign(torch.diagonal(r))
    sgn[sgn == 0] = 1.0
    return q * sgn[None, :]


def decay_matrix(d: int, m: int, decades: float, seed: int):
    """S = Q1 diag(sigma) Q2^T with sigma_i = 10^(-decades (i-1)/(m-1)); returns (d x m col-major
    torch tensor, sigma numpy)."""
    torch = D.torch
    k = min(d, m)
    sig = 10.0 ** (-decades * np.arange(k) / max(k - 1, 1))
    q1 = haar_frame(d, k, seed, 1)
    q2 = haar_frame(m, k, seed, 2)
    sdev = torch.from_numpy(sig).to("cuda")
    # column-major d x m: build S^T (m x d, row-major) = Q2 diag(sigma) Q1^T
    st = (q2 * sdev[None, :]) @ q1.t()
    del q1, q2
    return st.t(), sig  # (d, m) view with strides (1, d) == column-major


def pulse_columns(d: int, cols: np.ndarray, seed: int):
    """u_j(x) = exp(-(x - 0.1 - 0.8 t_j)^2 / (2 w_j^2)), x = linspace(0,1,d), t_j ~ U[0,1],
    w_j ~ U[0.01, 0.05] drawn per column id from a counter-based stream (column j of the
    full set is the same whatever slice it is generated in)."""
    torch = D.torch
    t, w = pulse_params(cols, seed)
    x = torch.linspace(0.0, 1.0, d, dtype=torch.float64, device="cuda")
    tt = torch.from_numpy(t).to("cuda")
    ww = torch.from_numpy(w).to("cuda")
    z = (x[None, :] - 0.1 - 0.8 * tt[:, None]) / ww[:, None]
    out = torch.exp(-0.5 * z * z)  # (cols, d) row-major == (d, cols) column-major
    return out.t()


def pulse_params(cols: np.ndarray, seed: int):
    ss = np.random.SeedSequence([int(seed), 2])
    rng = np.random.Generator(np.random.Philox(ss))
    nmax = int(cols.max()) + 1 if cols.size else 0
    t = rng.uniform(0.0, 1.0, nmax)
    w = rng.uniform(0.01, 0.05, nmax)
    return t[cols], w[cols]


_SINE_COEF: dict = {}


def _sine_coefficients(seed: int, nmax: int, modes: int) -> np.ndarray:
    """Rows 0..nmax-1 of the seeded N(0,1) coefficient stream (row j = column j's a_j.);
    the stream is drawn row-major, so a prefix does not depend on how many rows are drawn."""
    have = _SINE_COEF.get((seed, modes))
    if have is None or have.shape[0] < nmax:
        ss = np.random.SeedSequence([int(seed), 3])
        rng = np.random.Generator(np.random.Philox(ss))
        have = rng.standard_normal((max(nmax, 1), modes))
        _SINE_COEF[(seed, modes)] = have
    return have[:nmax]


def sine_columns(d: int, cols: np.ndarray, seed: int, noise_key: int = 0, modes: int = 300, noise: float = 1e-8):
    """S[:, j] = sum_{k<=300} k^-2 a_jk sin(k pi x) + noise * N(0,1), x uniform on [0,1].
    The noise of one generation unit (a 512-column slice, ``noise_key``) comes from its own
    seeded stream, so a slice generated alone equals the same columns of the whole matrix."""
    torch = D.torch
    x = torch.linspace(0.0, 1.0, d, dtype=torch.float64, device="cuda")
    k = torch.arange(1, modes + 1, dtype=torch.float64, device="cuda")
    basis = torch.sin(math.pi * k[:, None] * x[None, :])  # (modes, d)
    nmax = int(cols.max()) + 1 if cols.size else 0
    a = _sine_coefficients(seed, nmax, modes)[cols] / (np.arange(1, modes + 1) ** 2)[None, :]
    coef = torch.from_numpy(a).to("cuda")
    out = coef @ basis  # (cols, d)
    g = torch.Generator(device="cuda")
    g.manual_seed(int(seed) * 7919 + 104729 * int(noise_key) + 1)
    out += noise * torch.randn(out.shape, dtype=torch.float64, device="cuda", generator=g)
    return out.t()


def _mixed_perm(seed: int, m: int) -> np.ndarray:
    return np.random.Generator(np.random.Philox(np.random.SeedSequence([seed, 4]))).permutation(m)


def slice_values(index: int, b: int, d: int | None = None, m: int | None = None, seed: int | None = None):
    """Columns [block*b, block*(b+1)) of config ``index`` as a (d, block) column-major CUDA
    tensor -- the streaming generator of the large configs (c2-c4: one slice resident at a
    time).  ``make`` assembles the same slices, so streamed and whole-matrix runs see
    byte-identical snapshots."""
    cfg = CONFIGS[index]
    d = int(d or cfg["d"])
    m = int(m or cfg["m"])
    seed = index if seed is None else seed
    blk = cfg["block"]
    cols = np.arange(b * blk, min(m, (b + 1) * blk))
    if cfg["kind"] == "pulse":
        return pulse_columns(d, cols, seed)
    if cfg["kind"] == "sine":
        return sine_columns(d, cols, seed, noise_key=b)
    if cfg["kind"] != "mixed":
        raise ValueError(f"config {index} is not generated by slices")
    torch = D.torch
    perm = _mixed_perm(seed, m)
    is_sine = perm[cols] < m // 2
    out = torch.empty((cols.size, d), dtype=torch.float64, device="cuda")
    if is_sine.any():
        out[torch.from_numpy(np.where(is_sine)[0]).cuda()] = sine_columns(d, cols[is_sine], seed, noise_key=b).t()
    if (~is_sine).any():
        out[torch.from_numpy(np.where(~is_sine)[0]).cuda()] = pulse_columns(d, cols[~is_sine], seed).t()
    return out.t()


def frobenius_norm(index: int, d: int | None = None, m: int | None = None, seed: int | None = None) -> float:
    """||S||_F of a sliced config, one slice resident at a time (for eps* at full size)."""
    cfg = CONFIGS[index]
    m = int(m or cfg["m"])
    tot = 0.0
    for b in range((m + cfg["block"] - 1) // cfg["block"]):
        tot += float(D.torch.linalg.vector_norm(slice_values(index, b, d, m, seed)).item()) ** 2
    return math.sqrt(tot)


@dataclass
class Workload:
    """A config instance: device snapshot matrix (column-major) and its parameters."""

    index: int
    d: int
    m: int
    values: object          # torch (d, m) column-major CUDA tensor
    eps_star: float
    omega: float
    leaves: int
    block: int
    sigma_exact: np.ndarray | None = None

    @property
    def target(self) -> float:
        return self.eps_star / math.sqrt(self.m)


def make(index: int, d: int | None = None, m: int | None = None, seed: int | None = None) -> Workload:
    """Build config ``index`` (optionally at a reduced row count d / column count m)."""
    D.require_cuda()
    cfg = CONFIGS[index]
    d = int(d or cfg["d"])
    m = int(m or cfg["m"])
    seed = index if seed is None else seed
    sig = None
    if cfg["kind"] == "decay":
        vals, sig = decay_matrix(d, m, cfg["decades"], seed)
    elif cfg["kind"] == "pulse":
        vals = pulse_columns(d, np.arange(m), seed)
    else:
        # sine / mixed: assembled from the streaming slices (same bytes as a streamed run)
        blk = cfg["block"]
        vals = D.torch.empty((m, d), dtype=D.torch.float64, device="cuda")
        for b in range((m + blk - 1) // blk):
            vals[b * blk: min(m, (b + 1) * blk)] = slice_values(index, b, d, m, seed).t()
        vals = vals.t()
    fro = float(D.torch.linalg.vector_norm(vals).item())
    return Workload(index, d, m, vals, cfg["rel"] * fro, cfg["omega"], cfg["leaves"], cfg["block"], sig)
