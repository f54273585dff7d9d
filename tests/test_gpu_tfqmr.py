"""GPU parity of the device-resident TFQMR (NEXT-2; zk_solve method ZK_TFQMR) against oracle.tfqmr.

Bars (as BiCGStab's, SURVEY.md §8(c) L11/L12 — TFQMR is a two-sided Lanczos method whose counts
move with rounding order like BiCGStab's):
  * iteration count within [0.95·min, 1.05·max] of the oracle's counts under its summation
    orders (seq, rev, block-256); the quasi-residual histories agree to 1e-10 relative over the
    first 12 iterations; solutions to 1e-6 relative (C1/C2/T0);
  * the true residual never exceeds the quasi-residual bound it stopped on (S:388 allows 10·tol);
  * C4 (bench shape): forward error within 2κ·tol of the DST-I closed-form solution, first
    iterations' history against the oracle;
  * outcomes (CONVERGED at either half step / MAXIT / BREAKDOWN_SIGMA / NONFINITE / ZERO_RHS)
    match the oracle's; loop modes and the distributed code path are bitwise identical."""
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


def gpu_solve(m, b, **kw):
    A = zk.csr_create(m["row_ptr"], m["col_idx"], m["values"], m["n"])
    x0 = kw.pop("x0", None)
    r = zk.solve(A, cuda(b), None if x0 is None else cuda(x0), method="tfqmr", **kw)
    r["x"] = r["x"].cpu().numpy()
    return r


def relerr(a, b):
    return np.linalg.norm(a - b) / np.linalg.norm(b)


def diag(n, c):
    return dict(row_ptr=np.arange(n + 1, dtype=np.int64), col_idx=np.arange(n, dtype=np.int32),
                values=np.full(n, c, np.complex128), n=n)


@pytest.mark.parametrize("spmv_mode", ["0", "3"])
@pytest.mark.parametrize("cfg", ["C1", "C2", "T0"])
def test_tfqmr_parity(cfg, spmv_mode, monkeypatch):
    monkeypatch.setenv("ZK_SPMV_MODE", spmv_mode)
    monkeypatch.setenv("ZK_LOOP_MODE", "1")  # the WHILE-graph kernels with each SpMV mapping
    m = gen.make_matrix(cfg)
    b = gen.make_rhs(m)
    r = gpu_solve(m, b, tol=1e-8, maxit=1000)
    refs = [oracle.tfqmr(m, b, tol=1e-8, order=o) for o in ORDERS]
    its = [q["iters"] for q in refs]
    assert r["status"] == "CONVERGED" and all(q["status"] == "CONVERGED" for q in refs)
    assert 0.95 * min(its) <= r["iters"] <= 1.05 * max(its), (r["iters"], its)
    k = min(12, r["iters"], refs[0]["iters"]) + 1
    assert np.max(np.abs(r["hist"][:k] - refs[0]["hist"][:k]) / refs[0]["hist"][:k]) <= 1e-10
    assert relerr(r["x"], refs[0]["x"]) <= 1e-6
    assert r["hist"][-1] <= 1e-8 and r["true_relres"] <= 10 * 1e-8
    assert r["loop_mode"] == 1


@pytest.mark.parametrize("c", [2.0, -1.0, 1j, 0.3 - 2j])
def test_tfqmr_scalar_identity(c):
    """A = cI: the first half step gives w = 0 and x = b/c; exit at half step 1."""
    n = 1000
    b = gen.rand_vector(n, 1)
    r = gpu_solve(diag(n, c), b, tol=1e-12)
    ref = oracle.tfqmr(diag(n, c), b, tol=1e-12)
    assert r["status"] == ref["status"] == "CONVERGED" and r["iters"] == ref["iters"] == 1
    assert np.max(np.abs(r["x"] - b / c)) <= 1e-15 * np.max(np.abs(b / c))


def test_tfqmr_outcomes_match_oracle():
    # BREAKDOWN_SIGMA: σ = ⟨r̃, A r0⟩ = 0 on a real skew matrix
    m = dict(row_ptr=np.array([0, 1, 2]), col_idx=np.array([1, 0], np.int32),
             values=np.array([1, -1], np.complex128), n=2)
    b = np.array([1, 0], np.complex128)
    assert gpu_solve(m, b)["status"] == oracle.tfqmr(m, b)["status"] == "BREAKDOWN_SIGMA"
    # MAXIT from an x0, with the history of every iteration
    mc = gen.make_matrix("C2")
    bc = gen.make_rhs(mc)
    x0 = gen.rand_vector(mc["n"], 5)
    r = gpu_solve(mc, bc, x0=x0, tol=1e-14, maxit=7)
    ref = oracle.tfqmr(mc, bc, x0=x0, tol=1e-14, maxit=7)
    assert r["status"] == ref["status"] == "MAXIT" and r["iters"] == ref["iters"] == 7
    assert np.max(np.abs(r["hist"] - ref["hist"]) / ref["hist"]) <= 1e-10
    # the x of a MAXIT exit includes both half steps' updates of the last iteration
    assert relerr(r["x"], ref["x"]) <= 1e-9
    # NONFINITE input
    bn = bc.copy()
    bn[3] = np.nan
    assert gpu_solve(mc, bn)["status"] == oracle.tfqmr(mc, bn)["status"] == "NONFINITE"
    # ZERO_RHS is an error
    with pytest.raises(zk.ZkError) as e:
        gpu_solve(mc, np.zeros(mc["n"], np.complex128))
    assert e.value.code == -8


def test_tfqmr_maxit_each_exit_point():
    """maxit = 1..4 on C1: every early exit leaves x equal to the oracle's (the pending x update
    of the last half step is applied by the next kernel)."""
    m = gen.make_matrix("C1")
    b = gen.make_rhs(m)
    for k in range(1, 5):
        r = gpu_solve(m, b, tol=1e-14, maxit=k)
        ref = oracle.tfqmr(m, b, tol=1e-14, maxit=k)
        assert r["status"] == ref["status"] == "MAXIT" and r["iters"] == k
        assert relerr(r["x"], ref["x"]) <= 1e-11, k


def test_tfqmr_x0_restart_and_alias():
    m = gen.make_matrix("C1")
    b = gen.make_rhs(m)
    A = zk.csr_create(m["row_ptr"], m["col_idx"], m["values"], m["n"])
    B = cuda(b)
    r = zk.solve(A, B, tol=1e-8, method="tfqmr")
    x = r["x"]
    r2 = zk.solve(A, B, x0=x, x=x, tol=1e-7, method="tfqmr")            # x may alias x0
    assert r2["status"] == "CONVERGED" and r2["iters"] == 0
    x0 = cuda(gen.rand_vector(m["n"], 3))
    r3 = zk.solve(A, B, x0=x0, tol=1e-8, method="tfqmr")
    ref = oracle.tfqmr(m, b, x0=x0.cpu().numpy(), tol=1e-8)
    assert abs(r3["iters"] - ref["iters"]) <= max(1, 0.05 * ref["iters"])
    assert np.max(np.abs(r3["hist"][:8] - ref["hist"][:8]) / ref["hist"][:8]) <= 1e-10


@pytest.mark.parametrize("mode", ["2", "3"])
def test_tfqmr_loop_modes_bitwise_identical(mode, monkeypatch):
    m = gen.make_matrix("C2")
    b = gen.make_rhs(m)
    monkeypatch.setenv("ZK_LOOP_MODE", "1")
    base = gpu_solve(m, b, tol=1e-8)
    monkeypatch.setenv("ZK_LOOP_MODE", mode)
    r = gpu_solve(m, b, tol=1e-8)
    assert r["loop_mode"] == int(mode)
    assert r["iters"] == base["iters"] and np.array_equal(r["x"], base["x"])
    assert np.array_equal(r["hist"], base["hist"])


def test_tfqmr_deterministic():
    m = gen.make_matrix("C2")
    b = gen.make_rhs(m)
    A = zk.csr_create(m["row_ptr"], m["col_idx"], m["values"], m["n"])
    ws = zk.alloc_workspace(A, "tfqmr", 1000)
    B = cuda(b)
    r1 = zk.solve(A, B, workspace=ws, method="tfqmr")
    x1 = r1["x"].cpu().numpy()
    r2 = zk.solve(A, B, workspace=ws, method="tfqmr")
    assert np.array_equal(x1, r2["x"].cpu().numpy()) and np.array_equal(r1["hist"], r2["hist"])


def test_tfqmr_distributed_path_single_rank_comm(monkeypatch):
    m = gen.make_matrix("C2")
    b = gen.make_rhs(m)
    monkeypatch.setenv("ZK_LOOP_MODE", "3")
    monkeypatch.setenv("ZK_SPLIT_RED", "1")  # a distributed solve always runs the split schedule
    monkeypatch.setenv("ZK_SPLIT_TAIL", "0")  # ... with separate reduction passes
    base = gpu_solve(m, b, tol=1e-8)
    monkeypatch.delenv("ZK_LOOP_MODE")
    comm = zk.Comm(zk.Comm.unique_id(), 1, 0, 0)
    A = zk.csr_create(m["row_ptr"], m["col_idx"], m["values"], m["n"], comm=comm, row_begin=0)
    r = zk.solve(A, cuda(b), tol=1e-8, method="tfqmr")
    assert r["loop_mode"] == 3
    assert r["iters"] == base["iters"] and np.array_equal(r["x"].cpu().numpy(), base["x"])
    assert np.array_equal(r["hist"], base["hist"])
    A.close()
    comm.close()


def test_tfqmr_c4_full_size():
    """C4 (8M rows): closed-form forward error, true residual, first iterations vs the oracle."""
    spec = gen.CONFIGS["C4"]
    m = gen.make_matrix(spec)
    b = gen.make_rhs(m)
    A = zk.csr_create(cuda(m["row_ptr"]), cuda(m["col_idx"]), cuda(m["values"]), m["n"], borrow=True)
    r = zk.solve(A, cuda(b), tol=1e-8, maxit=2000, method="tfqmr")
    assert r["status"] == "CONVERGED" and r["true_relres"] <= 1e-7
    xe = cf.box_solve(spec, b, gen.ETA)
    assert relerr(r["x"].cpu().numpy(), xe) <= 2 * cf.box_kappa(spec, gen.ETA) * 1e-8
    ref = oracle.tfqmr(m, b, tol=1e-8, maxit=3)
    assert np.max(np.abs(r["hist"][:4] - ref["hist"][:4]) / ref["hist"][:4]) <= 1e-10


@pytest.mark.parametrize("split", ["0", "1", "tail"])
def test_tfqmr_split_schedule(split, monkeypatch):
    """The TFQMR schedules (fused epilogues; split: T2/T4 store A·y and vector passes finish; tail:
    T2/T4 run those passes as their own tails — the default from 2^18 rows) against the oracle on
    C2 in the WHILE-graph loop, and their MAXIT exits."""
    monkeypatch.setenv("ZK_LOOP_MODE", "1")
    monkeypatch.setenv("ZK_SPLIT_RED", "0" if split == "0" else "1")
    monkeypatch.setenv("ZK_SPLIT_TAIL", "1" if split == "tail" else "0")
    m = gen.make_matrix("C2")
    b = gen.make_rhs(m)
    r = gpu_solve(m, b, tol=1e-8)
    refs = [oracle.tfqmr(m, b, tol=1e-8, order=o) for o in ORDERS]
    its = [q["iters"] for q in refs]
    assert r["status"] == "CONVERGED" and 0.95 * min(its) <= r["iters"] <= 1.05 * max(its)
    k = min(12, r["iters"]) + 1
    assert np.max(np.abs(r["hist"][:k] - refs[0]["hist"][:k]) / refs[0]["hist"][:k]) <= 1e-10
    assert relerr(r["x"], refs[0]["x"]) <= 1e-6
    for kk in (1, 2, 5):
        q = gpu_solve(m, b, tol=1e-14, maxit=kk)
        ref = oracle.tfqmr(m, b, tol=1e-14, maxit=kk)
        assert q["status"] == "MAXIT" and relerr(q["x"], ref["x"]) <= 1e-11


@pytest.mark.parametrize("variant", ["auto", "w1", "w2", "w4", "w8", "gval"])
@pytest.mark.parametrize("cfg", ["C1", "C2", "T0"])
def test_tfqmr_cluster_parity(cfg, variant, monkeypatch):
    """Loop mode 5 for TFQMR (the default up to 16384 rows): the whole loop in one thread-block
    cluster, own rows in shared memory; every lane-count instantiation and the values-in-global
    variant, against the oracle with the bars of test_tfqmr_parity; deterministic."""
    monkeypatch.setenv("ZK_LOOP_MODE", "5")
    if variant.startswith("w"):
        monkeypatch.setenv("ZK_CLUSTER_W", variant[1:])
    if variant == "gval":
        monkeypatch.setenv("ZK_CLUSTER_VS", "0")
    m = gen.make_matrix(cfg)
    b = gen.make_rhs(m)
    r = gpu_solve(m, b, tol=1e-8, maxit=1000)
    assert r["loop_mode"] == 5 and r["gpu_launches"] == 1  # init and K0 inside the cluster kernel
    refs = [oracle.tfqmr(m, b, tol=1e-8, order=o) for o in ORDERS]
    its = [q["iters"] for q in refs]
    assert r["status"] == "CONVERGED" and 0.95 * min(its) <= r["iters"] <= 1.05 * max(its), (r["iters"], its)
    k = min(12, r["iters"], refs[0]["iters"]) + 1
    assert np.max(np.abs(r["hist"][:k] - refs[0]["hist"][:k]) / refs[0]["hist"][:k]) <= 1e-10
    assert relerr(r["x"], refs[0]["x"]) <= 1e-6
    assert r["hist"][-1] <= 1e-8 and r["true_relres"] <= 10 * 1e-8
    r2 = gpu_solve(m, b, tol=1e-8, maxit=1000)
    assert np.array_equal(r["x"], r2["x"]) and np.array_equal(r["hist"], r2["hist"])


def test_tfqmr_cluster_exits(monkeypatch):
    """Mode 5 exits inside an iteration: MAXIT after each of the first 6 iterations (x equal to the
    oracle's, including the pending half-step updates), and convergence at either half step."""
    monkeypatch.setenv("ZK_LOOP_MODE", "5")
    m = gen.make_matrix("T0")
    b = gen.make_rhs(m)
    for k in range(1, 7):
        r = gpu_solve(m, b, tol=1e-14, maxit=k)
        ref = oracle.tfqmr(m, b, tol=1e-14, maxit=k)
        assert r["loop_mode"] == 5 and r["status"] == ref["status"] == "MAXIT" and r["iters"] == k
        assert relerr(r["x"], ref["x"]) <= 1e-11, k
        assert np.max(np.abs(r["hist"] - ref["hist"]) / ref["hist"]) <= 1e-10
    for tol in (3e-3, 1e-3, 3e-4, 1e-4):  # stops land on both half steps
        r = gpu_solve(m, b, tol=tol)
        ref = oracle.tfqmr(m, b, tol=tol)
        assert r["status"] == ref["status"] == "CONVERGED" and r["iters"] == ref["iters"]
        assert relerr(r["x"], ref["x"]) <= 1e-9
