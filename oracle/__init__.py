"""CPU oracle — TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference legs may
import this package.  It shares no code with the CUDA library (paper_2112_11880_b200/) and
the product path never imports it.

Thin ctypes wrapper over ``zk_oracle.c`` (plain C, fp64, -ffp-contract=off).  Each function
cites the passage it follows; see the C file header for the pins and for what is
"parity unpinned".
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_DIR = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_DIR, "zk_oracle.c")
_SO = os.path.join(_DIR, "liboracle.so")
_SO_OMP = os.path.join(_DIR, "liboracle_omp.so")  # timing-only all-core build (ROWWISE loops, see zk_oracle.c)

ORD_SEQ, ORD_REV, ORD_BLOCK256, ORD_NEUMAIER = 0, 1, 2, 3

STATUS = {0: "CONVERGED", 1: "MAXIT", 2: "BREAKDOWN_RHO", 3: "BREAKDOWN_SIGMA",
          4: "BREAKDOWN_OMEGA", 5: "NOT_HPD", 6: "NONFINITE", 7: "ZERO_RHS"}


def build(force: bool = False, omp: bool = False) -> str:
    so = _SO_OMP if omp else _SO
    if force or not os.path.exists(so) or os.path.getmtime(so) < os.path.getmtime(_SRC):
        subprocess.check_call(["gcc", "-O2", "-std=c11", "-ffp-contract=off", "-fno-fast-math", "-fPIC", "-shared"]
                              + (["-fopenmp"] if omp else []) + ["-o", so, _SRC, "-lm"])
    return so


_h = None
_h_omp = None


def use_all_cores(on: bool = True):
    """Route every call through the OpenMP build (bench.py timing only).  Same bits: only the
    independent per-row / per-element loops (ROWWISE in zk_oracle.c) are split over threads."""
    global _h, _h_omp
    if on:
        if _h_omp is None:
            _h_omp = _load(build(omp=True))
        _h = _h_omp
    else:
        _h = _load(build())


def _lib():
    global _h
    if _h is None:
        _h = _load(build())
    return _h


def _load(path):
    lib = ctypes.CDLL(path)
    P, I64, D, I = ctypes.c_void_p, ctypes.c_int64, ctypes.c_double, ctypes.c_int
    lib.oracle_zdotc.argtypes = [I64, P, P, I, P]
    lib.oracle_zdotc.restype = None
    lib.oracle_sumsq.argtypes = [I64, P, I]
    lib.oracle_sumsq.restype = D
    lib.oracle_dznrm2.argtypes = [I64, P, I]
    lib.oracle_dznrm2.restype = D
    lib.oracle_zaxpy.argtypes = [I64, D, D, P, P]
    lib.oracle_zaxpy.restype = None
    lib.oracle_zscal.argtypes = [I64, D, D, P]
    lib.oracle_zscal.restype = None
    lib.oracle_zcsrmv.argtypes = [I64, P, P, P, D, D, P, D, D, P, I]
    lib.oracle_zcsrmv.restype = None
    lib.oracle_zassign.argtypes = [I64, D, D, P]
    lib.oracle_zassign.restype = None
    lib.oracle_zaxmy.argtypes = [I64, P, P]
    lib.oracle_zaxmy.restype = None
    for f in (lib.oracle_bicgstab, lib.oracle_cg, lib.oracle_bicgstab_jacobi, lib.oracle_cocg, lib.oracle_tfqmr):
        f.argtypes = [I64, P, P, P, P, P, D, ctypes.c_int32, I, P, P, P, P]
        f.restype = I
    lib.oracle_bicgstab_l.argtypes = [I64, P, P, P, P, P, D, ctypes.c_int32, I, I, P, P, P, P]
    lib.oracle_bicgstab_l.restype = I
    return lib


def _c128(a) -> np.ndarray:
    a = np.ascontiguousarray(a, dtype=np.complex128)
    return a


def _ptr(a):
    return None if a is None else a.ctypes.data


def zcsrmv(A: dict, x, alpha=1.0, beta=0.0, y=None, order=ORD_SEQ) -> np.ndarray:
    """O1: y ← αAx + βy (T8).  Returns a new array."""
    rp = np.ascontiguousarray(A["row_ptr"], dtype=np.int64)
    col = np.ascontiguousarray(A["col_idx"], dtype=np.int32)
    val = _c128(A["values"])
    x = _c128(x)
    n = len(rp) - 1
    out = np.zeros(n, np.complex128) if y is None else _c128(y).copy()
    alpha, beta = complex(alpha), complex(beta)
    _lib().oracle_zcsrmv(n, _ptr(rp), _ptr(col), _ptr(val), alpha.real, alpha.imag, _ptr(x),
                         beta.real, beta.imag, _ptr(out), order)
    return out


def zdotc(x, y, order=ORD_NEUMAIER) -> complex:
    """O2: Σ conj(x_i) y_i (L1).  Default: compensated (parity reference, L2)."""
    x, y = _c128(x), _c128(y)
    assert x.shape == y.shape
    out = np.zeros(2)
    _lib().oracle_zdotc(len(x), _ptr(x), _ptr(y), order, _ptr(out))
    return complex(out[0], out[1])


def dznrm2(x, order=ORD_NEUMAIER) -> float:
    """O3: sqrt(Σ re² + im²) (L3)."""
    x = _c128(x)
    return float(_lib().oracle_dznrm2(len(x), _ptr(x), order))


def sumsq(x, order=ORD_NEUMAIER) -> float:
    x = _c128(x)
    return float(_lib().oracle_sumsq(len(x), _ptr(x), order))


def zaxpy(alpha, x, y) -> np.ndarray:
    """O4: returns α·x + y."""
    x, out = _c128(x), _c128(y).copy()
    a = complex(alpha)
    _lib().oracle_zaxpy(len(x), a.real, a.imag, _ptr(x), _ptr(out))
    return out


def zscal(alpha, x) -> np.ndarray:
    """O5: returns α·x."""
    out = _c128(x).copy()
    a = complex(alpha)
    _lib().oracle_zscal(len(out), a.real, a.imag, _ptr(out))
    return out


def _solve(fn, A, b, x0, tol, maxit, order, *extra):
    rp = np.ascontiguousarray(A["row_ptr"], dtype=np.int64)
    col = np.ascontiguousarray(A["col_idx"], dtype=np.int32)
    val = _c128(A["values"])
    b = _c128(b)
    n = len(rp) - 1
    x0 = None if x0 is None else _c128(x0)
    x = np.zeros(n, np.complex128)
    iters = ctypes.c_int32(0)
    hist = np.full(maxit + 1, np.nan)
    tr = ctypes.c_double(0.0)
    st = fn(n, _ptr(rp), _ptr(col), _ptr(val), _ptr(b), _ptr(x0), float(tol), int(maxit), order, *extra,
            _ptr(x), ctypes.addressof(iters), _ptr(hist), ctypes.addressof(tr))
    it = iters.value
    return dict(x=x, iters=it, hist=hist[: it + 1].copy(), status=STATUS[st],
                true_relres=tr.value)


def bicgstab(A, b, x0=None, tol=1e-8, maxit=1000, order=ORD_SEQ) -> dict:
    """O6 BiCGStab (§4)."""
    return _solve(_lib().oracle_bicgstab, A, b, x0, tol, maxit, order)


def cg(A, b, x0=None, tol=1e-8, maxit=1000, order=ORD_SEQ) -> dict:
    """O7 CG (north-star addition)."""
    return _solve(_lib().oracle_cg, A, b, x0, tol, maxit, order)


def bicgstab_jacobi(A, b, x0=None, tol=1e-8, maxit=1000, order=ORD_SEQ) -> dict:
    """NEXT-1: Jacobi-preconditioned BiCGStab, the paper's P-Bi-CGSTAB."""
    return _solve(_lib().oracle_bicgstab_jacobi, A, b, x0, tol, maxit, order)


def zassign(n: int, alpha) -> np.ndarray:
    """NEXT-4 ZASSIGN: x_i ← α (PAPER.md T2 P:89-107, read as a fill, L16)."""
    out = np.empty(n, np.complex128)
    a = complex(alpha)
    _lib().oracle_zassign(n, a.real, a.imag, _ptr(out))
    return out


def zaxmy(x, y) -> np.ndarray:
    """NEXT-4 ZAXMY: returns x ⊙ y ("EWProduct", T5)."""
    x, out = _c128(x), _c128(y).copy()
    _lib().oracle_zaxmy(len(x), _ptr(x), _ptr(out))
    return out


def cocg(A, b, x0=None, tol=1e-8, maxit=1000, order=ORD_SEQ) -> dict:
    """NEXT-4 COCG: CG with the unconjugated form, complex symmetric A (van der Vorst & Melissen)."""
    return _solve(_lib().oracle_cocg, A, b, x0, tol, maxit, order)


def tfqmr(A, b, x0=None, tol=1e-8, maxit=1000, order=ORD_SEQ) -> dict:
    """NEXT-2 TFQMR (Freund; Kelley's two-half-step form), the paper's P-TFQMR without M."""
    return _solve(_lib().oracle_tfqmr, A, b, x0, tol, maxit, order)


def bicgstab_l(A, b, x0=None, tol=1e-8, maxit=1000, ell=8, order=ORD_SEQ) -> dict:
    """NEXT-3 BiCGStab(ℓ) (Sleijpen & Fokkema 1993), the paper's P-BiCGSTAB(8) without M (
    S:367-371); iters and hist count outer cycles of 2ℓ SpMVs."""
    assert 1 <= ell <= 8
    return _solve(_lib().oracle_bicgstab_l, A, b, x0, tol, maxit, order, int(ell))
