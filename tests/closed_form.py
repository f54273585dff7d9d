"""Closed forms that pin the oracle and the generator from outside both.

Independent mathematics, not a retyping of the oracle: the spectrum and eigenvectors of the
Q1-hex Helmholtz box operator are tensor products of the 1-D P1 eigenpairs, and the box
system is solved directly with the orthonormal DST-I (scipy.fft.dstn type 1), which
diagonalises every Kronecker factor.
"""
import math

import numpy as np
import scipy.fft


def axis_eigs(a: int, h: float):
    """1-D P1 Dirichlet eigenvalues on `a` free nodes: K1 → κ_m, M1 → μ_m, m = 1..a."""
    m = np.arange(1, a + 1)
    th = m * math.pi / (a + 1)
    kap = (2.0 - 2.0 * np.cos(th)) / h
    mu = (h / 3.0) * (2.0 + np.cos(th))
    return kap, mu


def box_eigs(spec, eta: float, k: float | None = None) -> np.ndarray:
    """λ_{pqr} (array indexed [r, q, p] = z, y, x) of A = K − (1+iη)k²M on the free block."""
    a, b, c = spec.free_dims
    kk = spec.k if k is None else k
    kx, mx = axis_eigs(a, spec.h)
    ky, my = axis_eigs(b, spec.h)
    kz, mz = axis_eigs(c, spec.h)
    K = (kz[:, None, None] * my[None, :, None] * mx[None, None, :]
         + mz[:, None, None] * ky[None, :, None] * mx[None, None, :]
         + mz[:, None, None] * my[None, :, None] * kx[None, None, :])
    M = mz[:, None, None] * my[None, :, None] * mx[None, None, :]
    return K - (1.0 + 1j * eta) * kk * kk * M


def free_index(spec) -> np.ndarray:
    """Global row ids of the free block in (z, y, x) C-order."""
    s = 1 if spec.shell else 0
    a, b, c = spec.free_dims
    iz, iy, ix = np.meshgrid(np.arange(c) + s, np.arange(b) + s, np.arange(a) + s, indexing="ij")
    return (ix + spec.nx * (iy + spec.ny * iz)).ravel()


def sine_mode(spec, p: int, q: int, r: int) -> np.ndarray:
    """Tensor sine eigenvector v(ix,iy,iz) = sin(p jx π/(a+1)) sin(q jy π/(b+1)) sin(r jz π/(c+1))
    on the free block (zero on identity rows), as a full-length complex vector."""
    a, b, c = spec.free_dims

    def s(m, d):  # sin(m·j·π/(d+1)) with the integer m·j reduced mod 2(d+1) first (argument ≤ 2π)
        k = (m * np.arange(1, d + 1, dtype=np.int64)) % (2 * (d + 1))
        return np.sin(k * math.pi / (d + 1))

    jx, jy, jz = s(p, a), s(q, b), s(r, c)
    v = np.zeros(spec.n, np.complex128)
    v[free_index(spec)] = (jz[:, None, None] * jy[None, :, None] * jx[None, None, :]).ravel()
    return v


def ident_value(spec) -> float:
    return 8.0 * spec.h / 3.0


def box_solve(spec, b: np.ndarray, eta: float, k: float | None = None) -> np.ndarray:
    """Exact solution of the (untwisted) box system by DST-I diagonalisation."""
    a, bb, c = spec.free_dims
    lam = box_eigs(spec, eta, k)
    idx = free_index(spec)
    x = b / ident_value(spec)                       # identity rows: d·x = b
    bf = b[idx].reshape(c, bb, a)
    xf = scipy.fft.idstn(scipy.fft.dstn(bf, type=1, norm="ortho") / lam, type=1, norm="ortho")
    x[idx] = xf.ravel()
    return x


def box_kappa(spec, eta: float, k: float | None = None) -> float:
    """2-norm condition number (A is normal): max|λ| / min|λ| incl. the identity value d."""
    lam = np.abs(box_eigs(spec, eta, k)).ravel()
    vals = [lam.max(), lam.min()]
    if spec.n > lam.size:
        vals += [ident_value(spec)]
    return max(vals) / min(vals)
