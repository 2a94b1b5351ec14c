"""Seeded synthetic inputs shaped like the paper's workloads.

This module is the ONLY code shared by the oracle (oracle/) and the CUDA path
(paper_2211_03339_b200/): it draws random matrices with prescribed spectra and
holds none of the Jacobi method's arithmetic.

Workloads (P:n = /root/reference/PAPER.md line n):
  * Example 1: ``gallery('randsvd', n, -kappa, mode)`` -- a random
    symmetric positive definite matrix A = H diag(lam) H^T with H Haar
    orthogonal and lam prescribed by ``mode``:
      1: lam = [1, 1/k, ..., 1/k]            (one large)
      2: lam = [1, ..., 1, 1/k]              (one small)
      3: lam_i = k^(-(i-1)/(n-1))            (geometric)
      4: lam_i = 1 - (1 - 1/k)(i-1)/(n-1)    (arithmetic)
      5: lam_i = k^(-u_i), u_i ~ U(0,1)      (random, uniform logarithm)
  * Example 2: A = P* diag(lam (x) 1_4) P*^T, n = 4s, with the
    five MATLAB one-liners for lam printed at P:950-954 (modes 3 and 5 are
    indefinite; the formulas win over the caption, reading R18).
  * Example 3: ``gallery('randsvd', [m,n], kappa, mode)`` -- an
    m x n matrix U0 diag(sigma) V0^T with U0 m x n orthonormal, V0 n x n Haar,
    sigma from the same five modes.

Haar matrices are QR factors of Gaussian matrices with the sign of diag(R)
absorbed (the MATLAB ``randn``+``orth`` recipe of P:948).  All host draws use
numpy's PCG64 with an explicit seed; the device variant (``*_torch``) uses a
seeded torch generator on the GPU for the n >= 4096 bench workloads, which the
oracle never runs in full.
"""
from __future__ import annotations

import math

import numpy as np

__all__ = [
    "seed_for", "haar", "stiefel", "spectrum_ex1", "spectrum_ex2", "example1",
    "example2", "example3", "example1_torch", "example3_torch", "rounded_haar",
]


def seed_for(config: int, mode: int, kappa: float, rep: int = 0) -> int:
    """Seed recipe: 2211033390 + 1000 cfg + 100 mode
    + 10 log10(kappa) + rep."""
    return 2211033390 + 1000 * config + 100 * mode + 10 * int(round(math.log10(kappa))) + rep


def _rng(seed: int) -> np.random.Generator:
    return np.random.Generator(np.random.PCG64(seed))


def haar(n: int, rng: np.random.Generator) -> np.ndarray:
    """Haar-distributed orthogonal n x n (QR of a Gaussian, sign-fixed)."""
    g = rng.standard_normal((n, n))
    q, r = np.linalg.qr(g)
    d = np.sign(np.diag(r))
    d[d == 0] = 1.0
    return np.asfortranarray(q * d)


def stiefel(m: int, n: int, rng: np.random.Generator) -> np.ndarray:
    """m x n matrix with Haar-distributed orthonormal columns."""
    g = rng.standard_normal((m, n))
    q, r = np.linalg.qr(g)
    d = np.sign(np.diag(r))
    d[d == 0] = 1.0
    return np.asfortranarray(q * d)


def spectrum_ex1(n: int, kappa: float, mode: int, rng: np.random.Generator | None = None) -> np.ndarray:
    """Example 1 / Example 3 spectra, length n,
    returned in generation order (mode 5 is random)."""
    i = np.arange(n, dtype=np.float64)
    if mode == 1:
        lam = np.full(n, 1.0 / kappa)
        lam[0] = 1.0
    elif mode == 2:
        lam = np.ones(n)
        lam[-1] = 1.0 / kappa
    elif mode == 3:
        lam = kappa ** (-i / max(n - 1, 1))
    elif mode == 4:
        lam = 1.0 - (1.0 - 1.0 / kappa) * i / max(n - 1, 1)
    elif mode == 5:
        if rng is None:
            raise ValueError("mode 5 needs an rng")
        lam = kappa ** (-rng.random(n))
    else:
        raise ValueError(f"mode must be 1..5, got {mode}")
    return lam.astype(np.float64)


def spectrum_ex2(n: int, kappa: float, mode: int, rng: np.random.Generator | None = None) -> np.ndarray:
    """Example 2: lam of length s = n/4, each repeated 4 times
    (``lam (x) 1_4``)."""
    if n % 4:
        raise ValueError("Example 2 needs n = 4 s")
    s = n // 4
    if mode == 1:
        lam = np.concatenate([[1.0], np.ones(s - 1) / kappa])
    elif mode == 2:
        lam = np.concatenate([np.ones(s - 1), [1.0 / kappa]])
    elif mode == 3:
        lam = kappa * np.linspace(-1.0, 0.0, s)
    elif mode == 4:
        lam = 1.0 - (1.0 - 1.0 / kappa) * np.linspace(0.0, 1.0, s)
    elif mode == 5:
        if rng is None:
            raise ValueError("mode 5 needs an rng")
        lam = kappa * (-rng.random(s))
    else:
        raise ValueError(f"mode must be 1..5, got {mode}")
    return np.kron(lam, np.ones(4))


def _sym_from(h: np.ndarray, lam: np.ndarray) -> np.ndarray:
    a = (h * lam) @ h.T
    return np.asfortranarray(0.5 * (a + a.T))


def example1(n: int, kappa: float, mode: int, seed: int):
    """(A, lam_desc): Example 1 matrix and its exact generator spectrum sorted
    descending."""
    rng = _rng(seed)
    lam = spectrum_ex1(n, kappa, mode, rng)
    h = haar(n, rng)
    return _sym_from(h, lam), np.sort(lam)[::-1].copy()


def example2(n: int, kappa: float, mode: int, seed: int):
    """(A, lam_desc): Example 2 (multiplicity 4) matrix and spectrum."""
    rng = _rng(seed)
    lam = spectrum_ex2(n, kappa, mode, rng)
    h = haar(n, rng)
    return _sym_from(h, lam), np.sort(lam)[::-1].copy()


def example3(m: int, n: int, kappa: float, mode: int, seed: int):
    """(A, sigma_desc): Example 3 m x n matrix and its singular values."""
    if m < n:
        raise ValueError("Example 3 needs m >= n")
    rng = _rng(seed)
    sig = spectrum_ex1(n, kappa, mode, rng)
    u0 = stiefel(m, n, rng)
    v0 = haar(n, rng)
    return np.asfortranarray((u0 * sig) @ v0.T), np.sort(sig)[::-1].copy()


def rounded_haar(n: int, seed: int) -> np.ndarray:
    """A Haar matrix rounded to binary32 and back (the input of the MGS
    contract pin, SPEC acceptance criterion 6)."""
    return np.asfortranarray(haar(n, _rng(seed)).astype(np.float32).astype(np.float64))


# --------------------------------------------------------------------------
# Device-side generators for the large bench workloads (n >= 4096), where a
# host LAPACK QR of an n x n Gaussian would dominate setup.  Same recipe, torch
# Philox generator on the GPU; the oracle never runs these sizes in full.
# --------------------------------------------------------------------------
def _torch_haar(n: int, gen, device, m: int | None = None):
    import torch
    rows = n if m is None else m
    g = torch.randn(rows, n, generator=gen, device=device, dtype=torch.float64)
    q, r = torch.linalg.qr(g)
    d = torch.sign(torch.diagonal(r))
    d[d == 0] = 1.0
    return q * d


def _torch_spectrum(n: int, kappa: float, mode: int, gen, device):
    import torch
    if mode == 5:
        u = torch.rand(n, generator=gen, device=device, dtype=torch.float64)
        return kappa ** (-u)
    return torch.from_numpy(spectrum_ex1(n, kappa, mode)).to(device)


def example1_torch(n: int, kappa: float, mode: int, seed: int, device="cuda"):
    """Device Example 1: returns (A column-major as a transposed-contiguous
    torch tensor, lam_desc torch tensor).  A is symmetric, so its row-major and
    column-major images coincide."""
    import torch
    gen = torch.Generator(device=device)
    gen.manual_seed(seed)
    lam = _torch_spectrum(n, kappa, mode, gen, device)
    h = _torch_haar(n, gen, device)
    a = (h * lam) @ h.T
    a = 0.5 * (a + a.T)
    return a.contiguous(), torch.sort(lam, descending=True).values


def example3_torch(m: int, n: int, kappa: float, mode: int, seed: int, device="cuda"):
    """Device Example 3: returns (A as a column-major m x n matrix stored in a
    torch tensor of shape (n, m) row-major -- i.e. A^T contiguous --, sigma)."""
    import torch
    gen = torch.Generator(device=device)
    gen.manual_seed(seed)
    sig = _torch_spectrum(n, kappa, mode, gen, device)
    u0 = _torch_haar(n, gen, device, m=m)
    v0 = _torch_haar(n, gen, device)
    a = (u0 * sig) @ v0.T            # m x n row-major
    return a.T.contiguous(), torch.sort(sig, descending=True).values
