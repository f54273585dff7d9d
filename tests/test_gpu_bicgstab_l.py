"""GPU parity of the device-resident BiCGStab(ℓ) (NEXT-3; zk_solve method ZK_BICGSTAB_L(ℓ)) against
oracle.bicgstab_l.

Bars (iterations are outer cycles of 2ℓ SpMVs):
  * cycle count within [0.95·min, 1.05·max] of the oracle's counts under its summation orders
    (seq, rev, block-256), as for BiCGStab;
  * residual histories over the first 6 cycles to HTOL[ℓ] (1e-10 for ℓ ≤ 2, 1e-9 / 1e-8 / 1e-3
    for ℓ = 3 / 4 / 8): ≈ 10× the oracle's own summation-order spread at that ℓ — the
    minimal-residual step solves a Gram system of A^j r̂ (j ≤ ℓ) whose conditioning amplifies
    rounding (the orders already differ by 9e-5 at ℓ = 8);
  * solutions to 1e-6 relative (C1/C2/T0); true residual ≤ 10·tol;
  * C4 (bench shape, ℓ = 8): DST-I closed form within 2κ·tol, first cycle's residual vs the oracle;
  * outcomes match the oracle's; loop modes bitwise identical; the row-partitioned path on a 1-rank
    communicator is bitwise the local split schedule (multi-rank parity: test_gpu_dist_local.py)."""
import numpy as np
import pytest
import torch

import gen
import oracle
from paper_2112_11880_b200 import zk
from tests import closed_form as cf

pytestmark = pytest.mark.gpu
DEV = "cuda:0"
ORDERS = (oracle.ORD_SEQ, oracle.ORD_REV, oracle.ORD_BLOCK256)


def cuda(a):
    return torch.from_numpy(np.ascontiguousarray(a)).to(DEV)


def gpu_solve(m, b, ell, **kw):
    A = zk.csr_create(m["row_ptr"], m["col_idx"], m["values"], m["n"])
    x0 = kw.pop("x0", None)
    r = zk.solve(A, cuda(b), None if x0 is None else cuda(x0), method="bicgstab_l", ell=ell, **kw)
    r["x"] = r["x"].cpu().numpy()
    return r


def relerr(a, b):
    return np.linalg.norm(a - b) / np.linalg.norm(b)


def diag(d):
    n = len(d)
    return dict(row_ptr=np.arange(n + 1, dtype=np.int64), col_idx=np.arange(n, dtype=np.int32),
                values=np.asarray(d, np.complex128), n=n)


# History bar per ℓ, derived from the ORACLE'S OWN summation-order spread over the first 6 cycles
# on C1/C2/T0 (max over rev / block-256 vs seq; tests/test_oracle_solvers.py::
# test_bicgstab_l_order_spread_within_gpu_bar recomputes it and requires spread ≤ bar/5):
#   ℓ = 1: 1.6e-14, ℓ = 2: 1.5e-12, ℓ = 3: 1.0e-11, ℓ = 4: 6.9e-10, ℓ = 8: 9.2e-5
# — the ℓ×ℓ normal equations of the Gram matrix square its conditioning (DESIGN R18), so the
# rounding of any summation order grows with ℓ.  The bar is ≈ 10× the spread, rounded up.
HTOL = {1: 1e-10, 2: 1e-10, 3: 1e-9, 4: 1e-8, 8: 1e-3}


def htol(ell):
    return HTOL[ell]


@pytest.mark.parametrize("ell", [1, 2, 4, 8])
@pytest.mark.parametrize("cfg", ["C1", "C2", "T0"])
def test_bicgstab_l_parity(cfg, ell, monkeypatch):
    monkeypatch.setenv("ZK_LOOP_MODE", "1")  # the WHILE-graph kernels (mode 5: test_bicgstab_l_cluster_parity)
    m = gen.make_matrix(cfg)
    b = gen.make_rhs(m)
    r = gpu_solve(m, b, ell, tol=1e-8, maxit=1000)
    refs = [oracle.bicgstab_l(m, b, tol=1e-8, ell=ell, order=o) for o in ORDERS]
    its = [q["iters"] for q in refs]
    assert r["status"] == "CONVERGED" and all(q["status"] == "CONVERGED" for q in refs)
    assert 0.95 * min(its) <= r["iters"] <= 1.05 * max(its), (r["iters"], its)
    k = min(6, r["iters"], refs[0]["iters"]) + 1
    assert np.max(np.abs(r["hist"][:k] - refs[0]["hist"][:k]) / refs[0]["hist"][:k]) <= htol(ell)
    assert relerr(r["x"], refs[0]["x"]) <= 1e-6
    assert r["true_relres"] <= 10 * 1e-8
    assert r["loop_mode"] == 1


@pytest.mark.parametrize("ell", [1, 2, 8])
@pytest.mark.parametrize("c", [2.0, -1.0, 1j, 0.3 - 2j])
def test_bicgstab_l_scalar_identity(c, ell):
    """One-step exactness: the first BiCG step reaches x = b/c, exit in cycle 1."""
    n = 1000
    b = gen.rand_vector(n, 1)
    r = gpu_solve(diag(np.full(n, c)), b, ell, tol=1e-12)
    assert r["status"] == "CONVERGED" and r["iters"] == 1
    assert np.max(np.abs(r["x"] - b / c)) <= 1e-15 * np.max(np.abs(b / c))


def test_bicgstab_l_finite_termination():
    """3 distinct eigenvalues, ℓ = 4: the BiCG part of cycle 1 reaches the solution (as the oracle)."""
    n = 3000
    d = np.array([1.5, -2.0 + 0.5j, 3.0j])[np.arange(n) % 3]
    b = gen.rand_vector(n, 2)
    r = gpu_solve(diag(d), b, 4, tol=1e-10)
    assert r["status"] == "CONVERGED" and r["iters"] == 1
    assert np.max(np.abs(r["x"] - b / d)) <= 1e-12 * np.max(np.abs(b / d))


def test_bicgstab_l_outcomes_match_oracle():
    m = dict(row_ptr=np.array([0, 1, 2]), col_idx=np.array([1, 0], np.int32),
             values=np.array([1, -1], np.complex128), n=2)
    b = np.array([1, 0], np.complex128)
    assert gpu_solve(m, b, 2)["status"] == oracle.bicgstab_l(m, b, ell=2)["status"] == "BREAKDOWN_SIGMA"
    mc = gen.make_matrix("C2")
    bc = gen.make_rhs(mc)
    x0 = gen.rand_vector(mc["n"], 5)
    r = gpu_solve(mc, bc, 4, x0=x0, tol=1e-14, maxit=3)
    ref = oracle.bicgstab_l(mc, bc, x0=x0, tol=1e-14, maxit=3, ell=4)
    assert r["status"] == ref["status"] == "MAXIT" and r["iters"] == ref["iters"] == 3
    assert np.max(np.abs(r["hist"] - ref["hist"]) / ref["hist"]) <= 1e-9
    assert relerr(r["x"], ref["x"]) <= 1e-9
    bn = bc.copy()
    bn[3] = np.nan
    assert gpu_solve(mc, bn, 2)["status"] == oracle.bicgstab_l(mc, bn, ell=2)["status"] == "NONFINITE"
    with pytest.raises(zk.ZkError) as e:
        gpu_solve(mc, np.zeros(mc["n"], np.complex128), 2)
    assert e.value.code == -8


@pytest.mark.parametrize("mode", ["2", "3"])
def test_bicgstab_l_loop_modes_bitwise_identical(mode, monkeypatch):
    m = gen.make_matrix("C2")
    b = gen.make_rhs(m)
    monkeypatch.setenv("ZK_LOOP_MODE", "1")
    base = gpu_solve(m, b, 4, tol=1e-8)
    monkeypatch.setenv("ZK_LOOP_MODE", mode)
    r = gpu_solve(m, b, 4, tol=1e-8)
    assert r["loop_mode"] == int(mode)
    assert r["iters"] == base["iters"] and np.array_equal(r["x"], base["x"])
    assert np.array_equal(r["hist"], base["hist"])


def test_bicgstab_l_deterministic_and_ell_switch():
    """Repeated solves are bitwise identical; switching ℓ on one handle rebuilds the loop graph."""
    m = gen.make_matrix("C2")
    b = gen.make_rhs(m)
    A = zk.csr_create(m["row_ptr"], m["col_idx"], m["values"], m["n"])
    B = cuda(b)
    r1 = zk.solve(A, B, method="bicgstab_l", ell=2)
    x1 = r1["x"].cpu().numpy()
    r8 = zk.solve(A, B, method="bicgstab_l", ell=8)
    r2 = zk.solve(A, B, method="bicgstab_l", ell=2)
    assert np.array_equal(x1, r2["x"].cpu().numpy()) and np.array_equal(r1["hist"], r2["hist"])
    assert r8["iters"] == oracle.bicgstab_l(m, b, ell=8)["iters"]


def test_bicgstab_l_single_rank_comm(monkeypatch):
    """The row-partitioned BiCGStab(ℓ) path (halo before every S1/S2 SpMV, allreduce of each
    reduction point and of the Gram totals, replicated Cholesky) on a 1-rank NCCL communicator
    is bitwise the local split-schedule solve (same kernels, identity allreduces)."""
    m = gen.make_matrix("C2")
    b = gen.make_rhs(m)
    monkeypatch.setenv("ZK_LOOP_MODE", "3")
    monkeypatch.setenv("ZK_SPLIT_RED", "1")
    base = gpu_solve(m, b, 4, tol=1e-8)
    monkeypatch.delenv("ZK_LOOP_MODE")
    comm = zk.Comm(zk.Comm.unique_id(), 1, 0, 0)
    A = zk.csr_create(m["row_ptr"], m["col_idx"], m["values"], m["n"], comm=comm, row_begin=0)
    r = zk.solve(A, cuda(b), method="bicgstab_l", ell=4)
    assert r["loop_mode"] == 3 and r["iters"] == base["iters"]
    assert np.array_equal(r["x"].cpu().numpy(), base["x"]) and np.array_equal(r["hist"], base["hist"])
    A.close()
    comm.close()


@pytest.mark.parametrize("ell", [2, 8])
def test_bicgstab_l_c4_vs_golden(ell):
    """C4 (8M rows) against the oracle's full BiCGStab(ℓ) solves (tests/golden/
    c4_oracle_bicgstab_l.json, tools/make_golden_c4.py --bl; seq / rev / block-256 orders): cycle
    count within [0.95·min, 1.05·max] of the orders, the first 3 cycles' history to HTOL[ℓ], and
    the seeded x sample within 4× the orders' own spread (and within 2κ·tol)."""
    import json
    import os
    with open(os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "c4_oracle_bicgstab_l.json")) as f:
        G = json.load(f)
    spec = gen.CONFIGS["C4"]
    m = gen.make_matrix(spec)
    b = gen.make_rhs(m)
    A = zk.csr_create(cuda(m["row_ptr"]), cuda(m["col_idx"]), cuda(m["values"]), m["n"], borrow=True)
    r = zk.solve(A, cuda(b), tol=1e-8, maxit=300, method="bicgstab_l", ell=ell)
    refs = {o: G["results"][f"bicgstab_l{ell}/{o}"] for o in ("seq", "rev", "block256")}
    its = [q["iters"] for q in refs.values()]
    assert r["status"] == "CONVERGED" and 0.95 * min(its) <= r["iters"] <= 1.05 * max(its), (r["iters"], its)
    h0 = np.array(refs["seq"]["hist"])
    assert np.max(np.abs(r["hist"][:4] - h0[:4]) / h0[:4]) <= htol(ell)

    def xs(g):
        return np.array(g["x_sample_re"]) + 1j * np.array(g["x_sample_im"])
    x0 = xs(refs["seq"])
    spread = max(relerr(xs(refs[o]), x0) for o in ("rev", "block256"))
    got = r["x"].cpu().numpy()[np.array(G["sample_idx"])]
    assert relerr(got, x0) <= max(4 * spread, 1e-9) and relerr(got, x0) <= 2 * cf.box_kappa(spec, gen.ETA) * 1e-8


def test_bicgstab_l8_c4_full_size():
    """C4 (8M rows), ℓ = 8 as the paper's P-BiCGSTAB(8): closed-form forward error, true residual,
    and the first cycle's residual against the oracle (one oracle cycle = 16 SpMVs)."""
    spec = gen.CONFIGS["C4"]
    m = gen.make_matrix(spec)
    b = gen.make_rhs(m)
    A = zk.csr_create(cuda(m["row_ptr"]), cuda(m["col_idx"]), cuda(m["values"]), m["n"], borrow=True)
    r = zk.solve(A, cuda(b), tol=1e-8, maxit=300, method="bicgstab_l", ell=8)
    assert r["status"] == "CONVERGED" and r["true_relres"] <= 1e-7
    xe = cf.box_solve(spec, b, gen.ETA)
    assert relerr(r["x"].cpu().numpy(), xe) <= 2 * cf.box_kappa(spec, gen.ETA) * 1e-8
    ref = oracle.bicgstab_l(m, b, tol=1e-8, maxit=1, ell=8)
    assert abs(r["hist"][1] - ref["hist"][1]) / ref["hist"][1] <= 1e-3


@pytest.mark.parametrize("split", ["0", "1"])
@pytest.mark.parametrize("ell", [1, 3])
def test_bicgstab_l_split_schedule(split, ell, monkeypatch):
    """Both BiCGStab(ℓ) schedules (fused SpMV reductions; split: SpMV stores, a vector pass reduces —
    the default from 2^18 rows) against the oracle on C2 in the WHILE-graph loop."""
    monkeypatch.setenv("ZK_LOOP_MODE", "1")  # the WHILE-graph kernels (C2 would take the cluster solver)
    monkeypatch.setenv("ZK_SPLIT_RED", split)
    m = gen.make_matrix("C2")
    b = gen.make_rhs(m)
    r = gpu_solve(m, b, ell, tol=1e-8)
    refs = [oracle.bicgstab_l(m, b, tol=1e-8, ell=ell, order=o) for o in ORDERS]
    its = [q["iters"] for q in refs]
    assert r["status"] == "CONVERGED" and 0.95 * min(its) <= r["iters"] <= 1.05 * max(its)
    k = min(6, r["iters"]) + 1
    assert np.max(np.abs(r["hist"][:k] - refs[0]["hist"][:k]) / refs[0]["hist"][:k]) <= htol(ell)
    assert relerr(r["x"], refs[0]["x"]) <= 1e-6


@pytest.mark.parametrize("variant", ["auto", "w1", "w8", "gval"])
@pytest.mark.parametrize("ell", [1, 2, 4, 8])
@pytest.mark.parametrize("cfg", ["C1", "C2", "T0"])
def test_bicgstab_l_cluster_parity(cfg, ell, variant, monkeypatch):
    """Loop mode 5 for BiCGStab(ℓ) (the default up to 16384 rows): the whole cycle loop in one
    thread-block cluster, Gram matrix reduced over DSMEM, Cholesky replicated per CTA; the bars of
    test_bicgstab_l_parity; deterministic."""
    monkeypatch.setenv("ZK_LOOP_MODE", "5")
    if variant.startswith("w"):
        monkeypatch.setenv("ZK_CLUSTER_W", variant[1:])
    if variant == "gval":
        monkeypatch.setenv("ZK_CLUSTER_VS", "0")
    m = gen.make_matrix(cfg)
    b = gen.make_rhs(m)
    r = gpu_solve(m, b, ell, tol=1e-8, maxit=1000)
    # own rows of the 2ℓ+4 vectors must fit in shared memory: C2 at ℓ = 8 falls back to the graph
    fits = not (cfg == "C2" and ell == 8)
    assert r["loop_mode"] == (5 if fits else 1) and (r["gpu_launches"] == 1 or not fits)
    refs = [oracle.bicgstab_l(m, b, tol=1e-8, ell=ell, order=o) for o in ORDERS]
    its = [q["iters"] for q in refs]
    assert r["status"] == "CONVERGED" and 0.95 * min(its) <= r["iters"] <= 1.05 * max(its), (r["iters"], its)
    k = min(6, r["iters"], refs[0]["iters"]) + 1
    assert np.max(np.abs(r["hist"][:k] - refs[0]["hist"][:k]) / refs[0]["hist"][:k]) <= htol(ell)
    assert relerr(r["x"], refs[0]["x"]) <= 1e-6
    assert r["true_relres"] <= 10 * 1e-8
    r2 = gpu_solve(m, b, ell, tol=1e-8, maxit=1000)
    assert np.array_equal(r["x"], r2["x"]) and np.array_equal(r["hist"], r2["hist"])


@pytest.mark.parametrize("ell", [2, 8])
def test_bicgstab_l_cluster_exits(ell, monkeypatch):
    """Mode 5 BiCGStab(ℓ) exits: MAXIT after 1..3 cycles with the oracle's history and x; a
    mid-cycle convergence (B2 exit) on A = cI."""
    monkeypatch.setenv("ZK_LOOP_MODE", "5")
    m = gen.make_matrix("C1")
    b = gen.make_rhs(m)
    for k in ((1, 2, 3) if ell == 2 else (1,)):  # ℓ = 8 reaches the 1e-14 rounding floor in cycle 2
        r = gpu_solve(m, b, ell, tol=1e-14, maxit=k)
        ref = oracle.bicgstab_l(m, b, tol=1e-14, ell=ell, maxit=k)
        assert r["loop_mode"] == 5 and r["status"] == ref["status"] == "MAXIT" and r["iters"] == k
        assert np.max(np.abs(r["hist"] - ref["hist"]) / ref["hist"]) <= htol(ell)
        assert relerr(r["x"], ref["x"]) <= (1e-10 if ell <= 2 else 1e-6)
    d = diag(np.full(300, 0.3 - 2j))
    bb = gen.rand_vector(300, 1)
    q = gpu_solve(d, bb, ell, tol=1e-12)
    qr = oracle.bicgstab_l(d, bb, tol=1e-12, ell=ell)
    assert q["loop_mode"] == 5 and q["status"] == qr["status"] == "CONVERGED" and q["iters"] == qr["iters"]
    assert np.max(np.abs(q["x"] - bb / (0.3 - 2j))) <= 1e-14 * np.max(np.abs(bb))
