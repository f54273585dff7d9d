"""Seeded synthetic inputs shared by the CUDA path's tests/bench and the oracle's tests.

This module holds none of the method's arithmetic (no SpMV, dot, norm or Krylov
step): it writes CSR arrays of the discretised Helmholtz operator (C code in
``helmholtz_gen.c``, recipe in SURVEY.md Appendix A / DESIGN.md "Inputs") and
draws seeded random vectors.

Configs:
  C1 Audi3D-1 shape, C2 Audi3D-2, C3 Audi3D-4 (C3T Twingo3D-2), C4 cube 200³, C5 cube 400³,
  plus the other PAPER.md Table 1 levels (A3 = Audi3D-3, T0, T1).
"""
from __future__ import annotations

import ctypes
import math
import os
import subprocess
from dataclasses import dataclass

import numpy as np

_DIR = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_DIR, "helmholtz_gen.c")
_SO = os.path.join(_DIR, "libzkgen.so")


def build(force: bool = False) -> str:
    if force or not os.path.exists(_SO) or os.path.getmtime(_SO) < os.path.getmtime(_SRC):
        subprocess.check_call(
            ["gcc", "-O2", "-fopenmp", "-ffp-contract=off", "-fPIC", "-shared", "-o", _SO, _SRC, "-lm"]
        )
    return _SO


class _Box(ctypes.Structure):
    _fields_ = [
        ("nx", ctypes.c_int64), ("ny", ctypes.c_int64), ("nz", ctypes.c_int64),
        ("shell", ctypes.c_int64), ("pad", ctypes.c_int64),
        ("h", ctypes.c_double), ("k", ctypes.c_double), ("eta", ctypes.c_double),
    ]


_lib_handle = None


def _lib():
    global _lib_handle
    if _lib_handle is None:
        lib = ctypes.CDLL(build())
        P = ctypes.c_void_p
        lib.gen_n_rows.restype = ctypes.c_int64
        lib.gen_n_rows.argtypes = [ctypes.POINTER(_Box)]
        lib.gen_row_nnz.restype = ctypes.c_int64
        lib.gen_row_nnz.argtypes = [ctypes.POINTER(_Box), ctypes.c_int64]
        lib.gen_row_ptr.restype = ctypes.c_int64
        lib.gen_row_ptr.argtypes = [ctypes.POINTER(_Box), ctypes.c_int64, ctypes.c_int64, P]
        lib.gen_fill.restype = None
        lib.gen_fill.argtypes = [ctypes.POINTER(_Box), ctypes.c_int64, ctypes.c_int64, P, P, P, P]
        lib.gen_free_mask.restype = None
        lib.gen_free_mask.argtypes = [ctypes.POINTER(_Box), ctypes.c_int64, ctypes.c_int64, P]
        _lib_handle = lib
    return _lib_handle


@dataclass(frozen=True)
class BoxSpec:
    """Node box Nx×Ny×Nz, spacing h, wavelength lam (k = 2π/λ, L14), Dirichlet shell, pad rows."""

    nx: int
    ny: int
    nz: int
    h: float
    lam: float
    shell: bool = True
    pad: int = 0

    @property
    def k(self) -> float:
        return 2.0 * math.pi / self.lam

    @property
    def free_dims(self):
        s = 2 if self.shell else 0
        return (self.nx - s, self.ny - s, self.nz - s)

    @property
    def n(self) -> int:
        return self.nx * self.ny * self.nz + self.pad

    @property
    def nnz(self) -> int:
        """Closed form: (3a−2)(3b−2)(3c−2) + #identity rows."""
        a, b, c = self.free_dims
        return (3 * a - 2) * (3 * b - 2) * (3 * c - 2) + (self.n - a * b * c)


def cube(N: int, lam: float = 3.5) -> BoxSpec:
    """Unit-cube interior N³, h = 1/(N+1), no identity rows (SURVEY.md App. A 'Scaled cubes')."""
    return BoxSpec(N, N, N, 1.0 / (N + 1), lam, shell=False, pad=0)


# PAPER.md Table 1 shapes fitted in SURVEY.md App. A.
CONFIGS = {
    "C1": BoxSpec(35, 8, 6, 0.133425, 3.5, True, 47),        # Audi3D-1
    "C2": BoxSpec(75, 14, 11, 0.066604, 3.5, True, 87),      # Audi3D-2
    "A3": BoxSpec(144, 31, 19, 0.033289, 3.5, True, 185),    # Audi3D-3
    "C3": BoxSpec(304, 52, 41, 0.016643, 3.5, True, 721),    # Audi3D-4
    "T0": BoxSpec(37, 19, 12, 0.077866, 9.5, True, 3),       # Twingo3D-0
    "T1": BoxSpec(58, 43, 25, 0.038791, 9.5, True, 7),       # Twingo3D-1
    "C3T": BoxSpec(113, 77, 55, 0.019379, 9.5, True, 614),   # Twingo3D-2
    "C4": cube(200),
    "C5": cube(400),
}

ETA = 0.05          # absorbing term of the north star (L14)
SEED_RHS = 42
SEED_TWIST = 43


def _box(spec: BoxSpec, eta: float, k: float | None = None) -> _Box:
    return _Box(spec.nx, spec.ny, spec.nz, 1 if spec.shell else 0, spec.pad, spec.h,
                spec.k if k is None else k, eta)


def twist_phases(n: int, seed: int = SEED_TWIST) -> np.ndarray:
    return np.random.default_rng(seed).uniform(0.0, 2.0 * math.pi, n)


def make_matrix(spec, eta: float = ETA, twist_seed: int | None = None, row_range=None,
                k: float | None = None):
    """CSR arrays of rows [r0, r1) (global column ids).

    Returns dict(row_ptr int64 (local, starts at 0), col_idx int32, values complex128,
    n (global rows), row_begin, nnz (local), free_mask uint8).
    """
    if isinstance(spec, str):
        spec = CONFIGS[spec]
    lib = _lib()
    box = _box(spec, eta, k)
    n = int(lib.gen_n_rows(ctypes.byref(box)))
    r0, r1 = (0, n) if row_range is None else (int(row_range[0]), int(row_range[1]))
    m = r1 - r0
    row_ptr = np.empty(m + 1, dtype=np.int64)
    nnz = int(lib.gen_row_ptr(ctypes.byref(box), r0, r1, row_ptr.ctypes.data))
    col = np.empty(max(nnz, 1), dtype=np.int32)[:nnz]
    val = np.empty(max(nnz, 1), dtype=np.complex128)[:nnz]
    phase = None
    if twist_seed is not None:
        phase = twist_phases(n, twist_seed)
    lib.gen_fill(ctypes.byref(box), r0, r1, row_ptr.ctypes.data, col.ctypes.data, val.ctypes.data,
                 None if phase is None else phase.ctypes.data)
    mask = np.empty(m, dtype=np.uint8)
    lib.gen_free_mask(ctypes.byref(box), r0, r1, mask.ctypes.data)
    return dict(row_ptr=row_ptr, col_idx=col, values=val, n=n, row_begin=r0, nnz=nnz,
                free_mask=mask, spec=spec, eta=eta, phase=phase)


def rand_vector(n: int, seed: int) -> np.ndarray:
    """x_i ~ U[−1,1] + i·U[−1,1] (SPEC S:544 / SURVEY.md §8(d))."""
    rng = np.random.default_rng(seed)
    v = rng.uniform(-1.0, 1.0, size=(n, 2))
    return np.ascontiguousarray(v).view(np.complex128).reshape(n)


def make_rhs(mat: dict, seed: int = SEED_RHS) -> np.ndarray:
    """b ~ U[−1,1]² on free rows, 0 on identity (Dirichlet/pad) rows; rows of this slab only.

    The draw is over all n global rows so every row range sees the same b."""
    n = mat["n"]
    b = rand_vector(n, seed)[mat["row_begin"]: mat["row_begin"] + len(mat["free_mask"])].copy()
    b[mat["free_mask"] == 0] = 0.0
    return b


def row_stats(row_ptr: np.ndarray) -> dict:
    """Row-length statistics of PAPER.md Table 1 columns (n, nnz, mean, sd, max; L13)."""
    lens = np.diff(row_ptr)
    return dict(n=len(lens), nnz=int(row_ptr[-1]), mean=float(lens.mean()), sd=float(lens.std()),
                max=int(lens.max()))


def random_csr(n: int, seed: int, max_len: int = 40, n_cols: int | None = None,
               empty_frac: float = 0.1, one_frac: float = 0.1, integer: bool = False):
    """Random canonical CSR (sorted unique columns per row) with empty rows, 1-nnz rows and rows
    longer than 32 (SURVEY.md §8(c) pins).  integer=True gives Gaussian-integer
    values in [−8,8]² for the exactness pins."""
    rng = np.random.default_rng(seed)
    n_cols = n if n_cols is None else n_cols
    lens = rng.integers(2, max_len + 1, size=n)
    u = rng.random(n)
    lens[u < empty_frac] = 0
    lens[(u >= empty_frac) & (u < empty_frac + one_frac)] = 1
    lens = np.minimum(lens, n_cols)
    row_ptr = np.zeros(n + 1, dtype=np.int64)
    row_ptr[1:] = np.cumsum(lens)
    nnz = int(row_ptr[-1])
    col = np.empty(nnz, dtype=np.int32)
    for i in range(n):
        if lens[i]:
            col[row_ptr[i]:row_ptr[i + 1]] = np.sort(rng.choice(n_cols, size=lens[i], replace=False))
    if integer:
        val = (rng.integers(-8, 9, size=nnz) + 1j * rng.integers(-8, 9, size=nnz)).astype(np.complex128)
    else:
        val = rng.uniform(-1, 1, nnz) + 1j * rng.uniform(-1, 1, nnz)
    return dict(row_ptr=row_ptr, col_idx=col, values=val.astype(np.complex128), n=n, n_cols=n_cols,
                nnz=nnz, row_begin=0)


def int_vector(n: int, seed: int, lo: int = -8, hi: int = 8) -> np.ndarray:
    """Gaussian-integer vector with parts in [lo, hi] (exactness pins)."""
    rng = np.random.default_rng(seed)
    return (rng.integers(lo, hi + 1, size=n) + 1j * rng.integers(lo, hi + 1, size=n)).astype(np.complex128)


def add_long_rows(mat: dict, frac: float = 0.02, target_len: int = 39, scale: float = 1e-3,
                  seed: int = 44) -> dict:
    """NEXT-4 irregular-row stress input (Twingo's max row lengths 33/39, PAPER.md
    T1, which conforming hexes cannot produce): a copy of `mat` in which a random `frac` of the
    free rows gets extra entries at random columns (sorted, unique) until it holds `target_len`,
    with values U[−1,1]² · scale · |diagonal| (weak couplings keep the system well posed).
    Free-row mask, phase and row_begin are carried over; rhs generation is unchanged."""
    rng = np.random.default_rng(seed)
    rp, col, val = mat["row_ptr"], mat["col_idx"], mat["values"]
    n = len(rp) - 1
    n_cols = mat.get("n_cols", mat["n"])
    free = np.flatnonzero(mat["free_mask"]) if "free_mask" in mat else np.arange(n)
    pick = np.zeros(n, dtype=bool)
    pick[rng.choice(free, size=max(1, int(frac * len(free))), replace=False)] = True
    rows_c, rows_v = [], []
    for i in range(n):
        c = col[rp[i]:rp[i + 1]]
        v = val[rp[i]:rp[i + 1]]
        if pick[i] and len(c) < target_len:
            d = np.abs(v[c == i + mat.get("row_begin", 0)]).max() if np.any(c == i + mat.get("row_begin", 0)) else 1.0
            extra = rng.choice(np.setdiff1d(np.arange(n_cols, dtype=np.int64), c), size=target_len - len(c),
                               replace=False).astype(np.int32)
            ev = (rng.uniform(-1, 1, len(extra)) + 1j * rng.uniform(-1, 1, len(extra))) * scale * d
            c = np.concatenate([c, extra])
            v = np.concatenate([v, ev])
            o = np.argsort(c, kind="stable")
            c, v = c[o], v[o]
        rows_c.append(c)
        rows_v.append(v)
    lens = np.array([len(c) for c in rows_c], dtype=np.int64)
    out = dict(mat)
    out["row_ptr"] = np.concatenate([[0], np.cumsum(lens)]).astype(np.int64)
    out["col_idx"] = np.concatenate(rows_c).astype(np.int32)
    out["values"] = np.concatenate(rows_v).astype(np.complex128)
    out["nnz"] = int(out["row_ptr"][-1])
    return out
