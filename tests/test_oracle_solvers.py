"""Pins for the oracle's BiCGStab (O6) and CG (O7) — SURVEY.md §8(c) 'Pins' rows BiCGStab/CG.

Fixed from outside the oracle by: one-step exactness (A = cI), dense LU (numpy.linalg.solve),
DST-I closed-form solves of the box Helmholtz system with κ in closed form, gauge and global
phase invariance (a missing conjugate breaks both), the CG κ bound, true vs recurrence
residual, and constructed breakdowns.  PAPER.md T9/T10 iteration counts: parity unpinned
(other matrices, unnamed preconditioner)."""
import math

import numpy as np
import pytest
import scipy.sparse as sp

import gen
import oracle
from tests import closed_form as cf


def csr_from_dense(D):
    S = sp.csr_matrix(D)
    S.sort_indices()
    return dict(row_ptr=S.indptr.astype(np.int64), col_idx=S.indices.astype(np.int32),
                values=S.data.astype(np.complex128), n=D.shape[0])


def diag_csr(d):
    n = len(d)
    return dict(row_ptr=np.arange(n + 1, dtype=np.int64), col_idx=np.arange(n, dtype=np.int32),
                values=np.asarray(d, np.complex128), n=n)


def twisted(spec, eta):
    """(A_g, D) with A_g = D·A·Dᴴ (L9)."""
    m = gen.make_matrix(spec, eta=eta, twist_seed=gen.SEED_TWIST)
    D = np.exp(1j * m["phase"])
    return m, D


# ------------------------------------------------------------------ BiCGStab
@pytest.mark.parametrize("c", [2.0, -1.0, 1j, 0.3 - 2j])
def test_bicgstab_scalar_identity(c):
    """A = cI converges at the half step of iteration 1 (L6)."""
    b = gen.rand_vector(50, 1)
    r = oracle.bicgstab(diag_csr(np.full(50, c)), b, tol=1e-12)
    assert r["status"] == "CONVERGED" and r["iters"] == 1
    assert np.max(np.abs(r["x"] - b / c)) <= 4e-16 * np.max(np.abs(b / c))
    assert r["hist"][0] == 1.0


@pytest.mark.parametrize("cfg", ["C1", "T0"])
def test_bicgstab_dense_lu(cfg):
    """‖x − x_LU‖/‖x_LU‖ ≤ 1e-7 at tol 1e-10."""
    m = gen.make_matrix(cfg)
    b = gen.make_rhs(m)
    D = sp.csr_matrix((m["values"], m["col_idx"], m["row_ptr"]), shape=(m["n"], m["n"])).toarray()
    x_lu = np.linalg.solve(D, b)
    r = oracle.bicgstab(m, b, tol=1e-10)
    assert r["status"] == "CONVERGED"
    assert np.linalg.norm(r["x"] - x_lu) / np.linalg.norm(x_lu) <= 1e-7


@pytest.mark.parametrize("cfg", ["C1", "C2", "A3"])
def test_bicgstab_dst_exact(cfg):
    """Forward error vs the DST-I exact solution ≤ 2κ·tol, κ in closed form (L12)."""
    spec = gen.CONFIGS[cfg]
    m = gen.make_matrix(spec)
    b = gen.make_rhs(m)
    tol = 1e-8
    r = oracle.bicgstab(m, b, tol=tol)
    xe = cf.box_solve(spec, b, gen.ETA)
    kappa = cf.box_kappa(spec, gen.ETA)
    assert r["status"] == "CONVERGED"
    assert np.linalg.norm(r["x"] - xe) / np.linalg.norm(xe) <= 2 * kappa * tol
    # true vs recurrence residual (S:388 allows 10·tol; we require tol)
    assert abs(r["true_relres"] - r["hist"][-1]) <= tol
    assert r["true_relres"] <= 2 * tol
    # solution-agreement reading L12 is binding literally on C1/C2
    if cfg in ("C1", "C2"):
        assert np.linalg.norm(r["x"] - xe) / np.linalg.norm(xe) <= 1e-6


def test_bicgstab_gauge_invariance():
    """(D·A·Dᴴ, D·b) gives the same count, hist equal to 1e-11 and x_g = D·x (App. B4)."""
    spec = gen.CONFIGS["C2"]
    m = gen.make_matrix(spec)
    mg, D = twisted(spec, gen.ETA)
    b = gen.make_rhs(m)
    r = oracle.bicgstab(m, b, tol=1e-8)
    rg = oracle.bicgstab(mg, D * b, tol=1e-8)
    assert r["iters"] == rg["iters"]
    n = min(12, r["iters"])
    assert np.max(np.abs(r["hist"][:n] - rg["hist"][:n]) / r["hist"][:n]) <= 1e-11
    assert np.linalg.norm(rg["x"] - D * r["x"]) / np.linalg.norm(r["x"]) <= 1e-6


def test_bicgstab_global_phase():
    spec = gen.CONFIGS["C1"]
    m = gen.make_matrix(spec)
    b = gen.make_rhs(m)
    th = 0.7
    mp = dict(m, values=m["values"] * np.exp(1j * th))
    r, rp = oracle.bicgstab(m, b), oracle.bicgstab(mp, b)
    assert r["iters"] == rp["iters"]
    assert np.max(np.abs(r["hist"] - rp["hist"]) / r["hist"]) <= 1e-10
    assert np.linalg.norm(rp["x"] - r["x"] * np.exp(-1j * th)) / np.linalg.norm(r["x"]) <= 1e-7


def test_bicgstab_x0_restart():
    """Restart from the returned x converges immediately (x0 path of O6)."""
    m = gen.make_matrix("C1")
    b = gen.make_rhs(m)
    r = oracle.bicgstab(m, b, tol=1e-8)
    r2 = oracle.bicgstab(m, b, x0=r["x"], tol=1e-7)
    assert r2["status"] == "CONVERGED" and r2["iters"] == 0


def test_bicgstab_statuses():
    # ZERO_RHS
    assert oracle.bicgstab(diag_csr([1, 2]), np.zeros(2))["status"] == "ZERO_RHS"
    # σ = ⟨r̂, A r̂⟩ = 0 for a real skew matrix → BREAKDOWN_SIGMA
    A = csr_from_dense(np.array([[0, 1], [-1, 0]], complex))
    assert oracle.bicgstab(A, np.array([1, 0], complex))["status"] == "BREAKDOWN_SIGMA"
    # MAXIT
    m = gen.make_matrix("C2")
    r = oracle.bicgstab(m, gen.make_rhs(m), tol=1e-14, maxit=3)
    assert r["status"] == "MAXIT" and r["iters"] == 3 and len(r["hist"]) == 4
    # NONFINITE
    bad = dict(m, values=m["values"].copy())
    bad["values"][5] = np.inf
    assert oracle.bicgstab(bad, gen.make_rhs(m))["status"] == "NONFINITE"


def test_bicgstab_order_envelope_small():
    """Summation order perturbs the count only mildly on C2 (L11 context)."""
    m = gen.make_matrix("C2")
    b = gen.make_rhs(m)
    its = [oracle.bicgstab(m, b, order=o)["iters"] for o in (0, 1, 2, 3)]
    assert max(its) - min(its) <= 0.15 * min(its)


# ------------------------------------------------------------------ CG
def test_cg_scalar_identity():
    b = gen.rand_vector(40, 2)
    r = oracle.cg(diag_csr(np.full(40, 3.0)), b)
    assert r["status"] == "CONVERGED" and r["iters"] == 1
    assert np.max(np.abs(r["x"] - b / 3)) <= 4e-16


def test_cg_two_eigenvalues():
    """A = I + uuᴴ has two distinct eigenvalues → CG exact in ≤ 2 iterations."""
    u = gen.rand_vector(60, 3)
    A = np.eye(60) + np.outer(u, u.conj())
    b = gen.rand_vector(60, 4)
    r = oracle.cg(csr_from_dense(A), b, tol=1e-12)
    assert r["status"] == "CONVERGED" and r["iters"] <= 2


@pytest.mark.parametrize("cfg", ["C1", "C2", "A3"])
def test_cg_twisted_closed_form(cfg):
    """CG on the gauge-twisted HPD box (η = 0): x_g = D·x_exact within 2κ·tol and the
    iteration count within the κ bound ⌈ln(2√κ/tol)/ln((√κ+1)/(√κ−1))⌉."""
    spec = gen.CONFIGS[cfg]
    mg, D = twisted(spec, 0.0)
    b = gen.make_rhs(mg)
    tol = 1e-8
    r = oracle.cg(mg, D * b, tol=tol)
    xe = D * cf.box_solve(spec, b, 0.0)
    kappa = cf.box_kappa(spec, 0.0)
    assert r["status"] == "CONVERGED"
    assert np.linalg.norm(r["x"] - xe) / np.linalg.norm(xe) <= 2 * kappa * tol
    sk = math.sqrt(kappa)
    bound = math.ceil(math.log(2 * sk / tol) / math.log((sk + 1) / (sk - 1)))
    assert r["iters"] <= bound
    assert abs(r["true_relres"] - r["hist"][-1]) <= tol


def test_cg_gauge_invariance():
    spec = gen.CONFIGS["C2"]
    m0 = gen.make_matrix(spec, eta=0.0)
    mg, D = twisted(spec, 0.0)
    b = gen.make_rhs(m0)
    r, rg = oracle.cg(m0, b), oracle.cg(mg, D * b)
    assert r["iters"] == rg["iters"]
    assert np.max(np.abs(r["hist"] - rg["hist"]) / r["hist"]) <= 1e-12


def test_cg_not_hpd():
    r = oracle.cg(diag_csr(np.full(10, -1.0)), gen.rand_vector(10, 1))
    assert r["status"] == "NOT_HPD" and r["iters"] == 0
    assert oracle.cg(diag_csr([1.0]), np.zeros(1))["status"] == "ZERO_RHS"


# ------------------------------------------------------------------ Jacobi P-BiCGStab (NEXT-1)
def row_scaled(m, seed=5):
    """(D_s·A, D_s) with a wild complex row scaling D_s (|d| in [e^-3, e^3], random phase)."""
    rng = np.random.default_rng(seed)
    ds = np.exp(rng.uniform(-3, 3, m["n"])) * np.exp(1j * rng.uniform(0, 2 * np.pi, m["n"]))
    rows = np.repeat(np.arange(m["n"]), np.diff(m["row_ptr"]))
    return dict(m, values=m["values"] * ds[rows]), ds


def test_jacobi_diagonal_one_iteration():
    """for diagonal matrices one Jacobi-preconditioned BiCGStab iteration reaches the solution."""
    d = gen.rand_vector(300, 9) + 2.0
    b = gen.rand_vector(300, 10)
    r = oracle.bicgstab_jacobi(diag_csr(d), b, tol=1e-12)
    assert r["status"] == "CONVERGED" and r["iters"] == 1
    assert np.max(np.abs(r["x"] - b / d)) <= 1e-15 * np.max(np.abs(b / d))
    assert oracle.bicgstab(diag_csr(d), b, tol=1e-12)["iters"] > 1


def test_jacobi_undoes_row_scaling():
    """Right-preconditioning with M = diag(D_s·A): the D_s·A system converges like A itself (the box
    diagonal is constant on free rows) and to the DST-I exact solution, while unpreconditioned
    BiCGStab on D_s·A stalls."""
    spec = gen.CONFIGS["C2"]
    m = gen.make_matrix(spec)
    b = gen.make_rhs(m)
    ms, ds = row_scaled(m)
    r = oracle.bicgstab_jacobi(ms, ds * b, tol=1e-8)
    ref = oracle.bicgstab(m, b, tol=1e-8)
    assert r["status"] == "CONVERGED"
    assert abs(r["iters"] - ref["iters"]) <= 0.15 * ref["iters"]
    xe = cf.box_solve(spec, b, gen.ETA)
    assert np.linalg.norm(r["x"] - xe) / np.linalg.norm(xe) <= 2 * cf.box_kappa(spec, gen.ETA) * 1e-8
    assert oracle.bicgstab(ms, ds * b, tol=1e-8, maxit=300)["status"] == "MAXIT"


def test_jacobi_dense_lu_and_missing_diagonal():
    m = gen.make_matrix("C1")
    ms, ds = row_scaled(m, 7)
    b = ds * gen.make_rhs(m)
    D = sp.csr_matrix((ms["values"], ms["col_idx"], ms["row_ptr"]), shape=(m["n"], m["n"])).toarray()
    x_lu = np.linalg.solve(D, b)
    r = oracle.bicgstab_jacobi(ms, b, tol=1e-10)
    assert np.linalg.norm(r["x"] - x_lu) / np.linalg.norm(x_lu) <= 1e-7
    skew = csr_from_dense(np.array([[0, 1], [-1, 0]], complex))   # no stored diagonal
    assert oracle.bicgstab_jacobi(skew, np.array([1, 0], complex))["status"] == "BREAKDOWN_RHO"


# ------------------------------------------------------------------ COCG (NEXT-4)
@pytest.mark.parametrize("c", [2.0, 1j, 0.3 - 2j])
def test_cocg_scalar_identity(c):
    b = gen.rand_vector(80, 1)
    r = oracle.cocg(diag_csr(np.full(80, c)), b, tol=1e-12)
    assert r["status"] == "CONVERGED" and r["iters"] == 1
    assert np.max(np.abs(r["x"] - b / c)) <= 1e-15 * np.max(np.abs(b / c))


def test_cocg_equals_cg_on_real_spd():
    """For real symmetric positive definite A and real b the bilinear and sesquilinear forms agree:
    COCG and CG produce the same iterates (same count, same history)."""
    m = gen.make_matrix("C2", eta=0.0)
    b = gen.make_rhs(m).real.astype(np.complex128)
    r, rc = oracle.cocg(m, b), oracle.cg(m, b)
    assert r["iters"] == rc["iters"]
    assert np.max(np.abs(r["hist"] - rc["hist"]) / rc["hist"]) <= 1e-13
    assert np.max(np.abs(r["x"] - rc["x"])) <= 1e-13 * np.max(np.abs(rc["x"]))


@pytest.mark.parametrize("cfg", ["C1", "C2", "A3"])
def test_cocg_complex_symmetric_closed_form(cfg):
    """COCG on the absorbing (η = 0.05, complex symmetric) box: DST-I exact solution within 2κ·tol."""
    spec = gen.CONFIGS[cfg]
    m = gen.make_matrix(spec)
    b = gen.make_rhs(m)
    r = oracle.cocg(m, b, tol=1e-8)
    assert r["status"] == "CONVERGED"
    xe = cf.box_solve(spec, b, gen.ETA)
    assert np.linalg.norm(r["x"] - xe) / np.linalg.norm(xe) <= 2 * cf.box_kappa(spec, gen.ETA) * 1e-8
    assert abs(r["true_relres"] - r["hist"][-1]) <= 1e-8


def test_cocg_dense_lu_and_breakdown():
    m = gen.make_matrix("C1")
    b = gen.make_rhs(m)
    D = sp.csr_matrix((m["values"], m["col_idx"], m["row_ptr"]), shape=(m["n"], m["n"])).toarray()
    x_lu = np.linalg.solve(D, b)
    r = oracle.cocg(m, b, tol=1e-10)
    assert np.linalg.norm(r["x"] - x_lu) / np.linalg.norm(x_lu) <= 1e-7
    # b = (1, i): bᵀb = 0 → the bilinear form degenerates (quasi-null start): ρ = 0, μ = 0
    A = diag_csr([1.0, 1.0])
    assert oracle.cocg(A, np.array([1, 1j]))["status"] == "BREAKDOWN_SIGMA"


# ------------------------------------------------------------------ TFQMR (NEXT-2)
@pytest.mark.parametrize("c", [2.0, -1.0, 1j, 0.3 - 2j])
def test_tfqmr_scalar_identity(c):
    """identity (scaled) → converges in 1 iteration."""
    b = gen.rand_vector(60, 1)
    r = oracle.tfqmr(diag_csr(np.full(60, c)), b, tol=1e-12)
    assert r["status"] == "CONVERGED" and r["iters"] == 1
    assert np.max(np.abs(r["x"] - b / c)) <= 1e-15 * np.max(np.abs(b / c))


@pytest.mark.parametrize("cfg", ["C1", "C2", "A3"])
def test_tfqmr_closed_form(cfg):
    spec = gen.CONFIGS[cfg]
    m = gen.make_matrix(spec)
    b = gen.make_rhs(m)
    r = oracle.tfqmr(m, b, tol=1e-8)
    assert r["status"] == "CONVERGED"
    xe = cf.box_solve(spec, b, gen.ETA)
    assert np.linalg.norm(r["x"] - xe) / np.linalg.norm(xe) <= 2 * cf.box_kappa(spec, gen.ETA) * 1e-8
    # the quasi-residual bound τ√(m+1) bounds the true residual (Freund 1993)
    assert r["true_relres"] <= r["hist"][-1] * (1 + 1e-6)


def test_tfqmr_bound_and_monotone_tau():
    """Stopped after k iterations (MAXIT) the true residual never exceeds hist[k] = τ√(2k+1)/‖b‖,
    and τ = hist[k]/√(2k+1)·‖b‖ is non-increasing ("monotone quasi-residual")."""
    m = gen.make_matrix("C2")
    b = gen.make_rhs(m)
    full = oracle.tfqmr(m, b, tol=1e-10)
    k = np.arange(1, len(full["hist"]))
    tau = full["hist"][1:] / np.sqrt(2 * k + 1)
    assert np.all(np.diff(tau) <= 1e-15 * tau[:-1])
    for kk in (1, 3, 7, 15):
        r = oracle.tfqmr(m, b, tol=1e-14, maxit=kk)
        assert r["status"] == "MAXIT"
        assert r["true_relres"] <= r["hist"][kk] * (1 + 1e-9)


def test_tfqmr_dense_lu_and_gauge():
    m = gen.make_matrix("C1")
    b = gen.make_rhs(m)
    D = sp.csr_matrix((m["values"], m["col_idx"], m["row_ptr"]), shape=(m["n"], m["n"])).toarray()
    x_lu = np.linalg.solve(D, b)
    r = oracle.tfqmr(m, b, tol=1e-10)
    assert np.linalg.norm(r["x"] - x_lu) / np.linalg.norm(x_lu) <= 1e-7
    mg, Dg = twisted(gen.CONFIGS["C1"], gen.ETA)
    rg = oracle.tfqmr(mg, Dg * b, tol=1e-10)
    assert rg["iters"] == r["iters"]
    assert np.max(np.abs(rg["hist"] - r["hist"]) / r["hist"]) <= 1e-10


# ------------------------------------------------------------------ BiCGStab(ℓ) (NEXT-3)
@pytest.mark.parametrize("cfg", ["C1", "C2", "T0"])
def test_bicgstab_l1_is_bicgstab(cfg):
    """ℓ = 1 reduces to BiCGStab: the independently pinned O6 gives the same count, the
    same residual history (to rounding, first 12 iterations) and the same solution."""
    m = gen.make_matrix(cfg)
    b = gen.make_rhs(m)
    r1 = oracle.bicgstab_l(m, b, tol=1e-8, ell=1)
    r0 = oracle.bicgstab(m, b, tol=1e-8)
    assert r1["status"] == r0["status"] == "CONVERGED" and r1["iters"] == r0["iters"]
    k = min(12, r0["iters"]) + 1
    assert np.max(np.abs(r1["hist"][:k] - r0["hist"][:k]) / r0["hist"][:k]) <= 1e-9
    assert np.linalg.norm(r1["x"] - r0["x"]) / np.linalg.norm(r0["x"]) <= 1e-6


@pytest.mark.parametrize("ell", [1, 2, 8])
@pytest.mark.parametrize("c", [2.0, -1.0, 1j, 0.3 - 2j])
def test_bicgstab_l_scalar_identity(c, ell):
    """One-step exactness: A = cI converges in the first cycle, x = b/c."""
    b = gen.rand_vector(60, 1)
    r = oracle.bicgstab_l(diag_csr(np.full(60, c)), b, tol=1e-12, ell=ell)
    assert r["status"] == "CONVERGED" and r["iters"] == 1
    assert np.max(np.abs(r["x"] - b / c)) <= 1e-15 * np.max(np.abs(b / c))


@pytest.mark.parametrize("ell,neig", [(2, 2), (4, 3), (8, 5)])
def test_bicgstab_l_finite_termination(ell, neig):
    """BiCG with r̃ = r0 terminates after as many steps as A has distinct eigenvalues: with
    ℓ ≥ that number the first cycle's BiCG part already reaches the solution."""
    n = 120
    eig = np.array([1.5, -2.0 + 0.5j, 3.0j, 0.7, 4.0 - 1j])[:neig]
    d = eig[np.arange(n) % neig]
    b = gen.rand_vector(n, 2)
    r = oracle.bicgstab_l(diag_csr(d), b, tol=1e-10, ell=ell)
    assert r["status"] == "CONVERGED" and r["iters"] == 1
    assert np.max(np.abs(r["x"] - b / d)) <= 1e-12 * np.max(np.abs(b / d))


@pytest.mark.parametrize("ell", [2, 4, 8])
def test_bicgstab_l_dense_lu_and_gauge(ell):
    """ℓ = 8 matches the dense LU solution within 1e-7; gauge invariance D·A·Dᴴ,
    D·b (a missing conjugate in the Gram matrix or the BiCG products breaks it)."""
    m = gen.make_matrix("C1")
    b = gen.make_rhs(m)
    D = sp.csr_matrix((m["values"], m["col_idx"], m["row_ptr"]), shape=(m["n"], m["n"])).toarray()
    x_lu = np.linalg.solve(D, b)
    r = oracle.bicgstab_l(m, b, tol=1e-10, ell=ell)
    assert r["status"] == "CONVERGED"
    assert np.linalg.norm(r["x"] - x_lu) / np.linalg.norm(x_lu) <= 1e-7
    mg, Dg = twisted(gen.CONFIGS["C1"], gen.ETA)
    rg = oracle.bicgstab_l(mg, Dg * b, tol=1e-10, ell=ell)
    assert rg["iters"] == r["iters"]
    # ℓ = 8: the Gram matrix of A^j r̂ (j ≤ 8) is ill-conditioned, rounding differences of the
    # twisted run are amplified in the last cycle's tiny residual
    htol = 1e-8 if ell < 8 else 1e-3
    assert np.max(np.abs(rg["hist"] - r["hist"]) / r["hist"]) <= htol
    assert np.linalg.norm(rg["x"] - Dg * r["x"]) / np.linalg.norm(r["x"]) <= 1e-8


@pytest.mark.parametrize("ell", [2, 8])
@pytest.mark.parametrize("cfg", ["C1", "C2", "A3"])
def test_bicgstab_l_closed_form_and_residual_consistency(cfg, ell):
    """DST-I exact solution within 2κ·tol; the recurrence residual (hist) and the true residual
    agree — a wrong x update in the MR part (e.g. γ_j r̂_j instead of γ_j r̂_{j−1}) breaks
    the second, a wrong Gram system slows or stops convergence."""
    spec = gen.CONFIGS[cfg]
    m = gen.make_matrix(spec)
    b = gen.make_rhs(m)
    r = oracle.bicgstab_l(m, b, tol=1e-8, ell=ell)
    assert r["status"] == "CONVERGED"
    xe = cf.box_solve(spec, b, gen.ETA)
    assert np.linalg.norm(r["x"] - xe) / np.linalg.norm(xe) <= 2 * cf.box_kappa(spec, gen.ETA) * 1e-8
    assert abs(r["true_relres"] - r["hist"][-1]) <= 1e-3 * 1e-8 * max(1, ell)


def test_bicgstab_l_cycle_count_scales():
    """A cycle holds ℓ BiCG steps (2ℓ SpMVs): on C2 the cycle count is at most 1.5× BiCGStab's
    iteration count / ℓ (+1) — a wrong MR polynomial (sign, conjugate, index) loses this."""
    m = gen.make_matrix("C2")
    b = gen.make_rhs(m)
    n_bicg = oracle.bicgstab(m, b, tol=1e-8)["iters"]
    for ell in (2, 4, 8):
        r = oracle.bicgstab_l(m, b, tol=1e-8, ell=ell)
        assert r["status"] == "CONVERGED" and r["iters"] <= 1.5 * n_bicg / ell + 1


def test_bicgstab_l_outcomes():
    # BREAKDOWN_SIGMA: γ = ⟨r̃, A r0⟩ = 0 on a real skew matrix
    m = dict(row_ptr=np.array([0, 1, 2]), col_idx=np.array([1, 0], np.int32),
             values=np.array([1, -1], np.complex128), n=2)
    assert oracle.bicgstab_l(m, np.array([1, 0], np.complex128), ell=2)["status"] == "BREAKDOWN_SIGMA"
    mc = gen.make_matrix("C2")
    bc = gen.make_rhs(mc)
    r = oracle.bicgstab_l(mc, bc, tol=1e-14, maxit=3, ell=4)
    assert r["status"] == "MAXIT" and r["iters"] == 3 and np.all(np.isfinite(r["hist"]))
    assert r["true_relres"] == pytest.approx(r["hist"][-1], rel=1e-6)
    assert oracle.bicgstab_l(mc, np.zeros(mc["n"]), ell=2)["status"] == "ZERO_RHS"
    bn = bc.copy()
    bn[0] = np.nan
    assert oracle.bicgstab_l(mc, bn, ell=2)["status"] == "NONFINITE"


@pytest.mark.parametrize("ell", [1, 2, 3, 4, 8])
def test_bicgstab_l_order_spread_within_gpu_bar(ell):
    """The GPU history bars of tests/test_gpu_bicgstab_l.py (HTOL) are derived from the oracle's
    own summation-order spread over the first 6 cycles: recompute the spread
    on C1/C2/T0 and require it to be at least 5× inside the bar, and the bar to be no looser than
    100× the spread (or 1e-10, the BiCGStab bar), so a bar cannot silently drift loose."""
    from tests.test_gpu_bicgstab_l import HTOL
    orders = (oracle.ORD_SEQ, oracle.ORD_REV, oracle.ORD_BLOCK256)
    worst = 0.0
    for cfg in ("C1", "C2", "T0"):
        m = gen.make_matrix(cfg)
        b = gen.make_rhs(m)
        refs = [oracle.bicgstab_l(m, b, tol=1e-8, ell=ell, order=o) for o in orders]
        k = min(6, min(r["iters"] for r in refs)) + 1
        h0 = refs[0]["hist"][:k]
        worst = max(worst, max(np.max(np.abs(r["hist"][:k] - h0) / h0) for r in refs[1:]))
    assert worst * 5 <= HTOL[ell], (ell, worst)
    assert HTOL[ell] <= max(100 * worst, 1e-10), (ell, worst)


def test_oracle_openmp_build_is_bitwise_identical():
    """bench.py's all-core cpu_baseline row uses liboracle_omp.so (ROWWISE loops split over
    threads): it must compute exactly the bits of the plain build (SpMV and a full BiCGStab)."""
    m = gen.make_matrix("C2")
    b = gen.make_rhs(m)
    x = gen.rand_vector(m["n"], 3)
    y1, r1 = oracle.zcsrmv(m, x), oracle.bicgstab(m, b)
    oracle.use_all_cores(True)
    try:
        y2, r2 = oracle.zcsrmv(m, x), oracle.bicgstab(m, b)
    finally:
        oracle.use_all_cores(False)
    assert np.array_equal(y1, y2)
    assert r1["iters"] == r2["iters"] and np.array_equal(r1["x"], r2["x"]) and np.array_equal(r1["hist"], r2["hist"])
