"""Pins for the oracle's SpMV and BLAS-1 (SURVEY.md §8(c) 'Pins' rows zcsrmv, zdotc/dznrm2,
zaxpy/zscal).  Each check is fixed by something other than the oracle: dense brute force,
exact integer arithmetic, closed-form eigenvectors and sums, algebraic identities."""
import cmath
import math

import numpy as np
import pytest
import scipy.sparse as sp

import gen
import oracle
from tests import closed_form as cf

ORDERS = [oracle.ORD_SEQ, oracle.ORD_REV, oracle.ORD_BLOCK256, oracle.ORD_NEUMAIER]


def dense(m):
    n = len(m["row_ptr"]) - 1
    return sp.csr_matrix((m["values"], m["col_idx"], m["row_ptr"]),
                         shape=(n, m.get("n_cols", m["n"]))).toarray()


def row_scale(m, x):
    """Σ_j |a_ij||x_j| per row."""
    n = len(m["row_ptr"]) - 1
    A = sp.csr_matrix((np.abs(m["values"]), m["col_idx"], m["row_ptr"]), shape=(n, m.get("n_cols", m["n"])))
    return A @ np.abs(x)


# ---------------------------------------------------------------- zcsrmv (O1)
@pytest.mark.parametrize("seed", [1, 2])
def test_spmv_dense_bruteforce(seed):
    m = gen.random_csr(400, seed=seed, max_len=45)
    x = gen.rand_vector(400, 10 + seed)
    y0 = gen.rand_vector(400, 20 + seed)
    D = dense(m)
    for alpha, beta in [(1, 0), (0.5 - 2j, 0), (1j, -0.25 + 1j)]:
        got = oracle.zcsrmv(m, x, alpha, beta, y0)
        want = alpha * (D @ x) + beta * y0
        tol = 1e-14 * (abs(alpha) * row_scale(m, x) + abs(beta) * np.abs(y0)) + 1e-300
        assert np.all(np.abs(got - want) <= tol)
    # empty rows give β·y (β = 0 ⇒ exactly 0 and y not read: NaN in y is ignored)
    ynan = np.full(400, np.nan + 0j)
    got = oracle.zcsrmv(m, x, 1.0, 0.0, ynan)
    assert np.all(got[np.diff(m["row_ptr"]) == 0] == 0)
    assert np.all(np.isfinite(got))


def test_spmv_integer_exact():
    """Gaussian-integer A and x: every partial sum is an exact integer → bitwise equal to
    exact Python-int arithmetic in any order (pin (5))."""
    m = gen.random_csr(300, seed=7, max_len=40, integer=True)
    x = gen.int_vector(300, 8)
    rp, col, val = m["row_ptr"], m["col_idx"], m["values"]
    want = np.zeros(300, np.complex128)
    for i in range(300):
        sr = si = 0
        for p in range(rp[i], rp[i + 1]):
            a, b = int(val[p].real), int(val[p].imag)
            c, d = int(x[col[p]].real), int(x[col[p]].imag)
            sr += a * c - b * d
            si += a * d + b * c
        want[i] = complex(sr, si)
    for order in (oracle.ORD_SEQ, oracle.ORD_REV):
        assert np.array_equal(oracle.zcsrmv(m, x, order=order), want)


@pytest.mark.parametrize("cfg,modes", [("C1", [(1, 1, 1), (5, 2, 3), (33, 6, 4)]),
                                       ("C2", [(1, 1, 1), (40, 7, 9)])])
def test_spmv_closed_form_eigenvectors(cfg, modes):
    """A·v = λ·v for the tensor-sine modes (App. A), to rounding (pin (2))."""
    spec = gen.CONFIGS[cfg]
    m = gen.make_matrix(spec)
    lam = cf.box_eigs(spec, gen.ETA)
    for (p, q, r) in modes:
        v = cf.sine_mode(spec, p, q, r)
        Av = oracle.zcsrmv(m, v)
        want = lam[r - 1, q - 1, p - 1] * v
        assert np.all(np.abs(Av - want) <= 1e-13 * row_scale(m, v) + 1e-300)


def test_spmv_closed_form_cube64():
    spec = gen.cube(64)
    m = gen.make_matrix(spec)
    lam = cf.box_eigs(spec, gen.ETA)
    v = cf.sine_mode(spec, 3, 17, 60)
    Av = oracle.zcsrmv(m, v)
    assert np.all(np.abs(Av - lam[59, 16, 2] * v) <= 1e-13 * row_scale(m, v) + 1e-300)


def test_spmv_identity_rows_bitwise():
    spec = gen.CONFIGS["C1"]
    m = gen.make_matrix(spec)
    x = gen.rand_vector(spec.n, 5)
    y = oracle.zcsrmv(m, x)
    ident = m["free_mask"] == 0
    d = cf.ident_value(spec)
    assert np.array_equal(y[ident], d * x[ident])


def test_spmv_linearity():
    m = gen.random_csr(500, seed=4)
    x, z = gen.rand_vector(500, 1), gen.rand_vector(500, 2)
    a, b = 0.3 - 1.2j, -2 + 0.5j
    lhs = oracle.zcsrmv(m, a * x + b * z)
    rhs = a * oracle.zcsrmv(m, x) + b * oracle.zcsrmv(m, z)
    assert np.all(np.abs(lhs - rhs) <= 1e-13 * (row_scale(m, np.abs(a * x) + np.abs(b * z))) + 1e-300)


# ---------------------------------------------------------------- zdotc / dznrm2 (O2, O3)
@pytest.mark.parametrize("order", ORDERS)
def test_dot_norm_examples(order):
    assert oracle.zdotc([1j], [1j], order) == 1 + 0j           # conj(i)·i = 1
    assert oracle.zdotc([1], [1j], order) == 1j
    assert oracle.zdotc([1j], [1], order) == -1j
    assert oracle.dznrm2([3 + 4j], order) == 5.0
    assert oracle.dznrm2(np.zeros(17, complex), order) == 0.0
    assert oracle.zdotc(np.zeros(0, complex), np.zeros(0, complex), order) == 0


@pytest.mark.parametrize("order", ORDERS)
def test_dot_integer_exact(order):
    """Gaussian-integer vectors: the sums are exact integers < 2^53 → bitwise (pin (2))."""
    n = 200_000
    x, y = gen.int_vector(n, 1, -90, 90), gen.int_vector(n, 2, -90, 90)
    xr, xi = x.real.astype(np.int64), x.imag.astype(np.int64)
    yr, yi = y.real.astype(np.int64), y.imag.astype(np.int64)
    want = complex(int(np.sum(xr * yr + xi * yi)), int(np.sum(xr * yi - xi * yr)))
    assert oracle.zdotc(x, y, order) == want
    ss = int(np.sum(xr * xr + xi * xi))
    assert oracle.sumsq(x, order) == float(ss)
    assert oracle.dznrm2(x, order) == math.sqrt(ss)            # correctly rounded √ of exact int


def test_dot_closed_forms():
    n = 100_003
    th, ph = 0.37, 1.21
    j = np.arange(n)
    x, y = np.exp(1j * th * j), np.exp(1j * ph * j)
    d = ph - th
    want = (1 - cmath.exp(1j * d * n)) / (1 - cmath.exp(1j * d))   # geometric series
    for order in ORDERS:
        assert abs(oracle.zdotc(x, y, order) - want) <= 1e-12 * n
    # sine orthogonality Σ_{j=1}^{N} sin(jaπ/(N+1)) sin(jbπ/(N+1)) = (N+1)/2 δ_ab
    N = 5000
    jj = np.arange(1, N + 1)
    for a, b in [(3, 3), (3, 4), (17, 1000), (999, 999)]:
        sa = np.sin(jj * a * math.pi / (N + 1)).astype(complex)
        sb = np.sin(jj * b * math.pi / (N + 1)).astype(complex)
        want = (N + 1) / 2 if a == b else 0.0
        assert abs(oracle.zdotc(sa, sb) - want) <= 1e-12 * N
    ones = np.full(n, 1 + 1j)
    assert oracle.sumsq(ones, oracle.ORD_SEQ) == 2.0 * n


def test_dot_symmetries():
    x, y = gen.rand_vector(10_000, 3), gen.rand_vector(10_000, 4)
    for order in ORDERS:
        assert oracle.zdotc(x, y, order) == oracle.zdotc(y, x, order).conjugate()
        dxx = oracle.zdotc(x, x, order)
        assert dxx.imag == 0.0 and dxx.real == oracle.sumsq(x, order)
    # orders agree within the L5 bound |Δ| ≤ 1e-12‖x‖‖y‖
    ref = oracle.zdotc(x, y, oracle.ORD_NEUMAIER)
    scale = oracle.dznrm2(x) * oracle.dznrm2(y)
    for order in ORDERS:
        assert abs(oracle.zdotc(x, y, order) - ref) <= 1e-12 * scale


def test_neumaier_is_accurate():
    """Compensated mode vs exact rational sum (Python fractions via math.fsum)."""
    x, y = gen.rand_vector(300_000, 11), gen.rand_vector(300_000, 12)
    re_terms = x.real * y.real + x.imag * y.imag    # products rounded as in the oracle
    got = oracle.zdotc(x, y, oracle.ORD_NEUMAIER)
    assert abs(got.real - math.fsum(re_terms)) <= 2e-16 * abs(math.fsum(np.abs(re_terms)))


# ---------------------------------------------------------------- zaxpy / zscal (O4, O5)
def test_axpy_scal_exact_alphas():
    x, y = gen.rand_vector(1000, 5), gen.rand_vector(1000, 6)
    assert np.array_equal(oracle.zaxpy(0, x, y), y)
    assert np.array_equal(oracle.zaxpy(1, x, y), x + y)
    assert np.array_equal(oracle.zaxpy(-1, x, y), y - x)
    assert np.array_equal(oracle.zaxpy(1j, x, y), (y.real - x.imag) + 1j * (y.imag + x.real))
    assert np.array_equal(oracle.zaxpy(0.25, x, y), y + 0.25 * x)
    assert np.array_equal(oracle.zscal(1, x), x)
    assert np.array_equal(oracle.zscal(-1, x), -x)
    assert np.array_equal(oracle.zscal(1j, x), -x.imag + 1j * x.real)
    assert np.array_equal(oracle.zscal(8, x), 8 * x)
    assert np.array_equal(oracle.zscal(0, x), np.zeros_like(x))


def test_axpy_scal_spec_examples():
    assert oracle.zaxpy(1, [1 + 1j], [2 - 1j])[0] == 3 + 0j
    assert oracle.zscal(1j, [1 + 0j])[0] == 1j
    xi, yi = gen.int_vector(5000, 1), gen.int_vector(5000, 2)
    a = 3 - 2j
    want = np.array([complex(int(a.real * u.real - a.imag * u.imag + v.real),
                             int(a.real * u.imag + a.imag * u.real + v.imag)) for u, v in zip(xi, yi)])
    assert np.array_equal(oracle.zaxpy(a, xi, yi), want)


# ---------------------------------------------------------------- ZASSIGN / ZAXMY (NEXT-4)
def test_zassign_zaxmy():
    assert np.array_equal(oracle.zassign(5, 1.5 - 2j), np.full(5, 1.5 - 2j))
    assert oracle.zaxmy([1j], [1j])[0] == -1 + 0j                  # i·i = −1
    x, y = gen.int_vector(10_000, 1), gen.int_vector(10_000, 2)
    want = np.array([complex(int(a.real * b.real - a.imag * b.imag), int(a.real * b.imag + a.imag * b.real))
                     for a, b in zip(x, y)])
    assert np.array_equal(oracle.zaxmy(x, y), want)
    ones = np.ones(100, np.complex128)
    y = gen.rand_vector(100, 3)
    assert np.array_equal(oracle.zaxmy(ones, y), y)                 # identity
