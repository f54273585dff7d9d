"""GPU parity of the device-resident BiCGStab / CG (zk_solve) against the CPU oracle.

Bars (north star):
  * CG: iteration count within ±5 % of the oracle's.
  * BiCGStab: count within [0.95·min, 1.05·max] of the oracle's counts under its summation
    orders (seq, rev, block-256) — rounding order alone moves BiCGStab counts (App. B4) — and
    the residual histories agree to 1e-10 relative over the first 12 iterations.
  * Final solutions agree to 1e-6 relative (C1/C2); on larger shapes both sides satisfy
    ‖x − x_exact‖/‖x_exact‖ ≤ 2κ·tol with x_exact and κ in closed form (DST-I).
  * Outcomes (CONVERGED / MAXIT / breakdowns / NOT_HPD / ZERO_RHS) match the oracle's."""
import json
import os

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
    r = zk.solve(A, cuda(b), None if x0 is None else cuda(x0), **kw)
    r["x"] = r["x"].cpu().numpy()
    return r


def relerr(a, b):
    return np.linalg.norm(a - b) / np.linalg.norm(b)


@pytest.mark.parametrize("spmv_mode", ["0", "3"])
@pytest.mark.parametrize("cfg", ["C1", "C2", "T0"])
def test_bicgstab_parity(cfg, spmv_mode, monkeypatch):
    monkeypatch.setenv("ZK_SPMV_MODE", spmv_mode)
    monkeypatch.setenv("ZK_LOOP_MODE", "1")  # the WHILE-graph path with each SpMV mapping
    m = gen.make_matrix(cfg)
    b = gen.make_rhs(m)
    r = gpu_solve(m, b, tol=1e-8, maxit=1000, method="bicgstab")
    refs = [oracle.bicgstab(m, b, tol=1e-8, order=o) for o in ORDERS]
    its = [q["iters"] for q in refs]
    assert r["status"] == "CONVERGED" and all(q["status"] == "CONVERGED" for q in refs)
    assert 0.95 * min(its) <= r["iters"] <= 1.05 * max(its), (r["iters"], its)
    k = min(12, r["iters"], refs[0]["iters"]) + 1
    assert np.max(np.abs(r["hist"][:k] - refs[0]["hist"][:k]) / refs[0]["hist"][:k]) <= 1e-10
    assert relerr(r["x"], refs[0]["x"]) <= 1e-6
    assert r["true_relres"] <= 2e-8 and abs(r["true_relres"] - r["hist"][-1]) <= 1e-8
    assert r["loop_mode"] == 1                          # device-resident WHILE graph


@pytest.mark.parametrize("spmv_mode", ["0", "3"])
@pytest.mark.parametrize("cfg", ["C1", "C2", "T0"])
def test_cg_parity_twisted_hpd(cfg, spmv_mode, monkeypatch):
    monkeypatch.setenv("ZK_SPMV_MODE", spmv_mode)
    monkeypatch.setenv("ZK_LOOP_MODE", "1")  # the WHILE-graph kernels with each SpMV mapping
    mg = gen.make_matrix(cfg, eta=0.0, twist_seed=gen.SEED_TWIST)
    b = np.exp(1j * mg["phase"]) * gen.make_rhs(mg)
    r = gpu_solve(mg, b, tol=1e-8, method="cg")
    ref = oracle.cg(mg, b, tol=1e-8)
    assert r["status"] == ref["status"] == "CONVERGED"
    assert abs(r["iters"] - ref["iters"]) <= 0.05 * ref["iters"], (r["iters"], ref["iters"])
    k = min(12, r["iters"]) + 1
    assert np.max(np.abs(r["hist"][:k] - ref["hist"][:k]) / ref["hist"][:k]) <= 1e-10
    assert relerr(r["x"], ref["x"]) <= 1e-6


@pytest.mark.parametrize("cfg", ["C3", "C3T"])
def test_bicgstab_paper_largest_shapes(cfg):
    """PAPER.md T1's largest levels: counts within the oracle's order envelope, forward error
    within 2κ·tol of the DST-I exact solution (L12)."""
    spec = gen.CONFIGS[cfg]
    m = gen.make_matrix(spec)
    b = gen.make_rhs(m)
    r = gpu_solve(m, b, tol=1e-8, method="bicgstab")
    refs = [oracle.bicgstab(m, b, tol=1e-8, order=o) for o in ORDERS]
    its = [q["iters"] for q in refs]
    assert 0.95 * min(its) <= r["iters"] <= 1.05 * max(its), (r["iters"], its)
    xe = cf.box_solve(spec, b, gen.ETA)
    bound = 2 * cf.box_kappa(spec, gen.ETA) * 1e-8
    assert relerr(r["x"], xe) <= bound and relerr(refs[0]["x"], xe) <= bound
    assert np.max(np.abs(r["hist"][:13] - refs[0]["hist"][:13]) / refs[0]["hist"][:13]) <= 1e-10


GOLD_DIR = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def _golden(name):
    """tests/golden/c4_oracle*.json, written by tools/make_golden_c4.py from oracle/ only."""
    with open(os.path.join(GOLD_DIR, name)) as f:
        return json.load(f)


def _xs(g):
    return np.array(g["x_sample_re"]) + 1j * np.array(g["x_sample_im"])


@pytest.fixture(scope="module")
def c4_system():
    m = gen.make_matrix("C4")
    b = gen.make_rhs(m)
    A = zk.csr_create(cuda(m["row_ptr"]), cuda(m["col_idx"]), cuda(m["values"]), m["n"])
    yield m, b, A
    A.close()


def _check_golden_envelope(r, G, meth, orders=("seq", "rev", "block256"), hist_k=12):
    """L11 against the oracle's own full-size solves: count within [0.95·min, 1.05·max] of its
    summation orders, history prefix to 1e-10, and the seeded x sample within 4× the spread of
    the oracle's orders (which is itself ≪ the 2κ·tol forward-error bound, L12)."""
    refs = {o: G["results"][f"{meth}/{o}"] for o in orders if f"{meth}/{o}" in G["results"]}
    its = [q["iters"] for q in refs.values()]
    assert r["status"] == "CONVERGED" and all(q["status"] == "CONVERGED" for q in refs.values())
    assert 0.95 * min(its) <= r["iters"] <= 1.05 * max(its), (r["iters"], its)
    h0 = np.array(refs["seq"]["hist"])
    k = min(hist_k, r["iters"], len(h0) - 1) + 1
    assert np.max(np.abs(r["hist"][:k] - h0[:k]) / h0[:k]) <= 1e-10
    idx = np.array(G["sample_idx"])
    x0 = _xs(refs["seq"])
    got = r["x"].cpu().numpy()[idx] if isinstance(r["x"], torch.Tensor) else r["x"][idx]
    spread = max([relerr(_xs(q), x0) for o, q in refs.items() if o != "seq"] + [1e-12])
    err = relerr(got, x0)
    return err, spread


def test_bicgstab_c4_full_size(c4_system):
    """C4 (8M rows) exactly as bench.py runs it, against the oracle's full C4 solves
    (tests/golden/c4_oracle.json: seq / rev / block-256 orders, VERDICT r1 "Next" 2): iteration
    count envelope, 12-iteration history prefix, x sample; plus the closed-form forward error
    and the true residual."""
    m, b, A = c4_system
    spec = gen.CONFIGS["C4"]
    r = zk.solve(A, cuda(b), tol=1e-8, maxit=1000, method="bicgstab")
    G = _golden("c4_oracle.json")
    err, spread = _check_golden_envelope(r, G, "bicgstab")
    kappa = cf.box_kappa(spec, gen.ETA)
    assert err <= 4 * spread and err <= 2 * kappa * 1e-8, (err, spread)
    x = r["x"].cpu().numpy()
    xe = cf.box_solve(spec, b, gen.ETA)
    assert relerr(x, xe) <= 2 * kappa * 1e-8
    assert r["true_relres"] <= 2e-8


def test_bicgstab_c4_tol1e10_solution(c4_system):
    """L12's optional mode at full size: both sides at tol 1e-10 agree on x to 1e-6
    (tests/golden/c4_oracle_tol1e-10.json, oracle orders seq / rev), with the 12-iteration history
    prefix to 1e-10.  The count envelope (L11) is asserted at the north star's tol 1e-8 above: below
    1e-8 BiCGStab's count is set by rounding-driven stagnation steps (GPU 346 vs the oracle's 323 /
    326 at 1e-10, while at 1e-8 every order lands in 271-295)."""
    m, b, A = c4_system
    G = _golden("c4_oracle_tol1e-10.json")
    r = zk.solve(A, cuda(b), tol=1e-10, maxit=1000, method="bicgstab")
    assert r["status"] == "CONVERGED" and r["true_relres"] <= 2e-10
    h0 = np.array(G["results"]["bicgstab/seq"]["hist"])
    assert np.max(np.abs(r["hist"][:13] - h0[:13]) / h0[:13]) <= 1e-10
    got = r["x"].cpu().numpy()[np.array(G["sample_idx"])]
    for o in ("seq", "rev"):
        assert relerr(got, _xs(G["results"][f"bicgstab/{o}"])) <= 1e-6


@pytest.mark.parametrize("method", ["tfqmr", "cocg"])
def test_tfqmr_cocg_c4_full_size(c4_system, method):
    m, b, A = c4_system
    G = _golden("c4_oracle.json")
    r = zk.solve(A, cuda(b), tol=1e-8, maxit=2000, method=method)
    err, spread = _check_golden_envelope(r, G, method)
    assert err <= 4 * spread and err <= 2 * cf.box_kappa(gen.CONFIGS["C4"], gen.ETA) * 1e-8, (err, spread)


def test_cg_c4_twisted_hpd_full_size():
    """CG at 8M rows (A7 at scale, split schedule): the gauge-twisted HPD C4 against the oracle's
    full solves — strict ±5 % count (L11 (i); the oracle's three orders give the same count),
    12-iteration history to 1e-10, x sample to 1e-6."""
    mg = gen.make_matrix("C4", eta=0.0, twist_seed=gen.SEED_TWIST)
    bg = np.exp(1j * mg["phase"]) * gen.make_rhs(mg)
    A = zk.csr_create(cuda(mg["row_ptr"]), cuda(mg["col_idx"]), cuda(mg["values"]), mg["n"])
    r = zk.solve(A, cuda(bg), tol=1e-8, maxit=3000, method="cg")
    G = _golden("c4_oracle.json")
    ref = G["results"]["cg_twisted_hpd/seq"]
    assert r["status"] == ref["status"] == "CONVERGED"
    assert abs(r["iters"] - ref["iters"]) <= 0.05 * ref["iters"], (r["iters"], ref["iters"])
    h0 = np.array(ref["hist"])
    assert np.max(np.abs(r["hist"][:13] - h0[:13]) / h0[:13]) <= 1e-10
    got = r["x"].cpu().numpy()[np.array(G["sample_idx"])]
    assert relerr(got, _xs(ref)) <= 1e-6
    assert r["true_relres"] <= 2e-8


@pytest.mark.parametrize("mode", ["1", "2", "3"])
def test_loop_modes_bitwise_identical(mode, monkeypatch):
    """WHILE graph, chunked graphs and direct launches run the same kernels: identical results."""
    m = gen.make_matrix("C2")
    b = gen.make_rhs(m)
    monkeypatch.setenv("ZK_LOOP_MODE", "1")
    base = gpu_solve(m, b, tol=1e-8)
    monkeypatch.setenv("ZK_LOOP_MODE", mode)
    r = gpu_solve(m, b, tol=1e-8)
    assert r["loop_mode"] == int(mode)
    assert r["iters"] == base["iters"] and np.array_equal(r["x"], base["x"])
    assert np.array_equal(r["hist"], base["hist"])


def test_solve_deterministic_and_workspace_reuse():
    m = gen.make_matrix("C2")
    b = gen.make_rhs(m)
    A = zk.csr_create(m["row_ptr"], m["col_idx"], m["values"], m["n"])
    ws = zk.alloc_workspace(A, "bicgstab", 1000)
    B = cuda(b)
    r1 = zk.solve(A, B, workspace=ws)
    x1 = r1["x"].cpu().numpy()
    r2 = zk.solve(A, B, workspace=ws)
    assert np.array_equal(x1, r2["x"].cpu().numpy()) and np.array_equal(r1["hist"], r2["hist"])


@pytest.mark.parametrize("c", [2.0, -1.0, 1j])
def test_bicgstab_scalar_identity(c):
    n = 1000
    m = dict(row_ptr=np.arange(n + 1, dtype=np.int64), col_idx=np.arange(n, dtype=np.int32),
             values=np.full(n, c, np.complex128), n=n)
    b = gen.rand_vector(n, 1)
    r = gpu_solve(m, b, tol=1e-12)
    assert r["status"] == "CONVERGED" and r["iters"] == 1         # half-step exit (L6)
    assert np.max(np.abs(r["x"] - b / c)) <= 1e-15 * np.max(np.abs(b / c))


def test_outcomes_match_oracle():
    # BREAKDOWN_SIGMA on a real skew matrix
    m = dict(row_ptr=np.array([0, 1, 2]), col_idx=np.array([1, 0], np.int32),
             values=np.array([1, -1], np.complex128), n=2)
    b = np.array([1, 0], np.complex128)
    assert gpu_solve(m, b)["status"] == oracle.bicgstab(m, b)["status"] == "BREAKDOWN_SIGMA"
    # MAXIT with the history of the first maxit iterations
    m = gen.make_matrix("C2")
    b = gen.make_rhs(m)
    r = gpu_solve(m, b, tol=1e-14, maxit=5)
    ref = oracle.bicgstab(m, b, tol=1e-14, maxit=5)
    assert r["status"] == ref["status"] == "MAXIT" and r["iters"] == 5
    assert np.max(np.abs(r["hist"] - ref["hist"]) / ref["hist"]) <= 1e-10
    # NOT_HPD for CG on a negative definite matrix
    n = 64
    neg = dict(row_ptr=np.arange(n + 1, dtype=np.int64), col_idx=np.arange(n, dtype=np.int32),
               values=np.full(n, -2.0, np.complex128), n=n)
    assert gpu_solve(neg, gen.rand_vector(n, 2), method="cg")["status"] == "NOT_HPD"
    # ZERO_RHS is an error
    with pytest.raises(zk.ZkError) as e:
        gpu_solve(neg, np.zeros(n, np.complex128))
    assert e.value.code == -8


def test_x0_restart_and_alias():
    m = gen.make_matrix("C1")
    b = gen.make_rhs(m)
    A = zk.csr_create(m["row_ptr"], m["col_idx"], m["values"], m["n"])
    B = cuda(b)
    r = zk.solve(A, B, tol=1e-8)
    x = r["x"]
    r2 = zk.solve(A, B, x0=x, x=x, tol=1e-7)                       # x may alias x0
    assert r2["status"] == "CONVERGED" and r2["iters"] == 0
    x0 = cuda(gen.rand_vector(m["n"], 3))
    r3 = zk.solve(A, B, x0=x0, tol=1e-8)
    ref = oracle.bicgstab(m, b, x0=x0.cpu().numpy(), tol=1e-8)
    assert abs(r3["iters"] - ref["iters"]) <= max(1, 0.05 * ref["iters"])
    assert np.max(np.abs(r3["hist"][:8] - ref["hist"][:8]) / ref["hist"][:8]) <= 1e-10
    with pytest.raises(zk.ZkError) as e:
        zk.solve(A, B, x=B)
    assert e.value.code == -7


def test_distributed_path_single_rank_comm(monkeypatch):
    """The row-partitioned code path (NCCL comm, halo plan, allreduce + finish kernels, direct
    launches) on a 1-rank communicator gives bitwise the same solve as the local path running the
    same per-iteration kernels."""
    m = gen.make_matrix("C2")
    b = gen.make_rhs(m)
    monkeypatch.setenv("ZK_LOOP_MODE", "3")
    monkeypatch.setenv("ZK_SPLIT_RED", "1")  # a distributed solve always runs the split schedule
    monkeypatch.setenv("ZK_SPLIT_TAIL", "0")  # ... with separate reduction passes
    base = gpu_solve(m, b, tol=1e-8)
    monkeypatch.delenv("ZK_LOOP_MODE")
    comm = zk.Comm(zk.Comm.unique_id(), 1, 0, 0)
    A = zk.csr_create(m["row_ptr"], m["col_idx"], m["values"], m["n"], comm=comm, row_begin=0)
    assert A.info["nranks"] == 1 and A.info["n_halo"] == 0
    r = zk.solve(A, cuda(b), tol=1e-8)
    assert r["loop_mode"] == 3
    assert r["iters"] == base["iters"] and np.array_equal(r["x"].cpu().numpy(), base["x"])
    x = cuda(gen.rand_vector(m["n"], 4))
    y = torch.empty_like(x)
    zk.zcsrmv(A, 1, x, 0, y)
    y_local = torch.empty_like(x)
    zk.zcsrmv(zk.csr_create(m["row_ptr"], m["col_idx"], m["values"], m["n"]), 1, x, 0, y_local)
    assert torch.equal(y, y_local)
    d = zk.zdotc(x, y, comm=comm).cpu().numpy()[0]
    assert d == zk.zdotc(x, y).cpu().numpy()[0]
    A.close()
    comm.close()


# ------------------------------------------------------------------ Jacobi P-BiCGStab (NEXT-1)
def row_scaled(m, seed=5):
    rng = np.random.default_rng(seed)
    ds = np.exp(rng.uniform(-3, 3, m["n"])) * np.exp(1j * rng.uniform(0, 2 * np.pi, m["n"]))
    rows = np.repeat(np.arange(m["n"]), np.diff(m["row_ptr"]))
    return dict(m, values=m["values"] * ds[rows]), ds


@pytest.mark.parametrize("cfg", ["C1", "C2", "T0"])
def test_bicgstab_jacobi_parity(cfg):
    """P-BiCGStab (M = diag A) on the row-scaled system against the oracle's Templates recurrences:
    count within the order envelope, hist prefix, solution 1e-6 (L11/L12)."""
    m0 = gen.make_matrix(cfg)
    m, ds = row_scaled(m0)
    b = ds * gen.make_rhs(m0)
    r = gpu_solve(m, b, tol=1e-8, method="bicgstab_jacobi")
    refs = [oracle.bicgstab_jacobi(m, b, tol=1e-8, order=o) for o in ORDERS]
    its = [q["iters"] for q in refs]
    assert r["status"] == "CONVERGED" and all(q["status"] == "CONVERGED" for q in refs)
    assert 0.95 * min(its) <= r["iters"] <= 1.05 * max(its), (r["iters"], its)
    k = min(12, r["iters"], refs[0]["iters"]) + 1
    assert np.max(np.abs(r["hist"][:k] - refs[0]["hist"][:k]) / refs[0]["hist"][:k]) <= 1e-10
    assert relerr(r["x"], refs[0]["x"]) <= 1e-6
    assert r["true_relres"] <= 2e-8


def test_bicgstab_jacobi_cases():
    # diagonal: one iteration
    n = 500
    d = gen.rand_vector(n, 9) + 2.0
    m = dict(row_ptr=np.arange(n + 1, dtype=np.int64), col_idx=np.arange(n, dtype=np.int32), values=d, n=n)
    b = gen.rand_vector(n, 10)
    r = gpu_solve(m, b, tol=1e-12, method="bicgstab_jacobi")
    assert r["status"] == "CONVERGED" and r["iters"] == 1
    assert np.max(np.abs(r["x"] - b / d)) <= 1e-14 * np.max(np.abs(b / d))
    # x0 path (u0 = M x0) against the oracle
    m0 = gen.make_matrix("C1")
    ms, ds = row_scaled(m0, 3)
    bb = ds * gen.make_rhs(m0)
    x0 = gen.rand_vector(m0["n"], 4)
    r = gpu_solve(ms, bb, x0=x0, tol=1e-8, method="bicgstab_jacobi")
    ref = oracle.bicgstab_jacobi(ms, bb, x0=x0, tol=1e-8)
    assert abs(r["iters"] - ref["iters"]) <= max(1, 0.05 * ref["iters"])
    assert np.max(np.abs(r["hist"][:8] - ref["hist"][:8]) / ref["hist"][:8]) <= 1e-10
    # missing diagonal → ZK_ERR_INVALID_CSR naming the row
    skew = dict(row_ptr=np.array([0, 1, 2]), col_idx=np.array([1, 0], np.int32),
                values=np.array([1, -1], np.complex128), n=2)
    with pytest.raises(zk.ZkError) as e:
        gpu_solve(skew, np.array([1, 0], np.complex128), method="bicgstab_jacobi")
    assert e.value.code == -2 and "row 0" in str(e.value)


def test_bicgstab_jacobi_c4():
    """C4 in the bench configuration: Jacobi P-BiCGStab converges to the DST-I exact solution."""
    spec = gen.CONFIGS["C4"]
    m = gen.make_matrix(spec)
    b = gen.make_rhs(m)
    A = zk.csr_create(cuda(m["row_ptr"]), cuda(m["col_idx"]), cuda(m["values"]), m["n"], borrow=True)
    r = zk.solve(A, cuda(b), tol=1e-8, maxit=2000, method="bicgstab_jacobi")
    assert r["status"] == "CONVERGED" and r["true_relres"] <= 2e-8
    xe = cf.box_solve(spec, b, gen.ETA)
    assert relerr(r["x"].cpu().numpy(), xe) <= 2 * cf.box_kappa(spec, gen.ETA) * 1e-8


# ------------------------------------------------------------------ COCG (NEXT-4)
@pytest.mark.parametrize("cfg", ["C1", "C2", "T0"])
def test_cocg_parity(cfg):
    """COCG on the absorbing complex-symmetric Helmholtz matrices: ±5 % of the oracle's count
    (like CG, the recurrences are order-insensitive), hist prefix, solution 1e-6."""
    m = gen.make_matrix(cfg)
    b = gen.make_rhs(m)
    r = gpu_solve(m, b, tol=1e-8, method="cocg")
    ref = oracle.cocg(m, b, tol=1e-8)
    assert r["status"] == ref["status"] == "CONVERGED"
    assert abs(r["iters"] - ref["iters"]) <= 0.05 * ref["iters"], (r["iters"], ref["iters"])
    k = min(12, r["iters"]) + 1
    assert np.max(np.abs(r["hist"][:k] - ref["hist"][:k]) / ref["hist"][:k]) <= 1e-10
    assert relerr(r["x"], ref["x"]) <= 1e-6
    assert r["true_relres"] <= 2e-8


def test_cocg_cases():
    n = 200
    c = 0.3 - 2j
    m = dict(row_ptr=np.arange(n + 1, dtype=np.int64), col_idx=np.arange(n, dtype=np.int32),
             values=np.full(n, c, np.complex128), n=n)
    b = gen.rand_vector(n, 1)
    r = gpu_solve(m, b, tol=1e-12, method="cocg")
    assert r["status"] == "CONVERGED" and r["iters"] == 1
    # quasi-null start bᵀb = 0 → BREAKDOWN_SIGMA, as the oracle
    m2 = dict(row_ptr=np.arange(3, dtype=np.int64), col_idx=np.arange(2, dtype=np.int32),
              values=np.ones(2, np.complex128), n=2)
    bb = np.array([1, 1j])
    assert gpu_solve(m2, bb, method="cocg")["status"] == oracle.cocg(m2, bb)["status"] == "BREAKDOWN_SIGMA"
    # x0 path and MAXIT history against the oracle
    mc = gen.make_matrix("C2")
    bc = gen.make_rhs(mc)
    x0 = gen.rand_vector(mc["n"], 5)
    r = gpu_solve(mc, bc, x0=x0, tol=1e-14, maxit=7, method="cocg")
    ref = oracle.cocg(mc, bc, x0=x0, tol=1e-14, maxit=7)
    assert r["status"] == ref["status"] == "MAXIT" and r["iters"] == 7
    assert np.max(np.abs(r["hist"] - ref["hist"]) / ref["hist"]) <= 1e-10


def test_cocg_c4():
    spec = gen.CONFIGS["C4"]
    m = gen.make_matrix(spec)
    b = gen.make_rhs(m)
    A = zk.csr_create(cuda(m["row_ptr"]), cuda(m["col_idx"]), cuda(m["values"]), m["n"], borrow=True)
    r = zk.solve(A, cuda(b), tol=1e-8, maxit=2000, method="cocg")
    assert r["status"] == "CONVERGED" and r["true_relres"] <= 2e-8
    xe = cf.box_solve(spec, b, gen.ETA)
    assert relerr(r["x"].cpu().numpy(), xe) <= 2 * cf.box_kappa(spec, gen.ETA) * 1e-8


@pytest.mark.parametrize("tail", ["0", "1"])
@pytest.mark.parametrize("method", ["bicgstab", "cg", "cocg"])
def test_split_reductions_parity(method, tail, monkeypatch):
    """The split-reduction schedule (SpMV stores only; the dot products come from a vector pass
    (tail=0) or from the SpMV kernel's own tail over the rows it just produced (tail=1) — the
    default from 2^18 rows) forced on C2 against the oracle, and against the fused schedule."""
    monkeypatch.setenv("ZK_SPLIT_TAIL", tail)
    if method == "cg":
        m = gen.make_matrix("C2", eta=0.0, twist_seed=gen.SEED_TWIST)
        b = np.exp(1j * m["phase"]) * gen.make_rhs(m)
        ref = oracle.cg(m, b, tol=1e-8)
    else:
        m = gen.make_matrix("C2")
        b = gen.make_rhs(m)
        ref = (oracle.bicgstab if method == "bicgstab" else oracle.cocg)(m, b, tol=1e-8)
    monkeypatch.setenv("ZK_LOOP_MODE", "1")
    monkeypatch.setenv("ZK_SPLIT_RED", "1")
    r = gpu_solve(m, b, tol=1e-8, method=method)
    monkeypatch.setenv("ZK_SPLIT_RED", "0")
    f = gpu_solve(m, b, tol=1e-8, method=method)
    assert r["status"] == f["status"] == ref["status"] == "CONVERGED"
    assert abs(r["iters"] - ref["iters"]) <= max(1, 0.05 * ref["iters"])
    k = min(12, r["iters"], ref["iters"]) + 1
    assert np.max(np.abs(r["hist"][:k] - ref["hist"][:k]) / ref["hist"][:k]) <= 1e-10
    assert relerr(r["x"], ref["x"]) <= 1e-6 and relerr(f["x"], ref["x"]) <= 1e-6
    if tail == "0":
        assert r["gpu_launches"] > f["gpu_launches"]      # + the reduction passes
    else:
        assert r["gpu_launches"] == f["gpu_launches"]     # reductions in the SpMV kernels' tails


def test_bicgstab_irregular_rows_stress():
    """NEXT-4 stress input (C2 with 2 % of its rows grown to 39 entries, Twingo's max): the
    default mapping falls back to the CSR kernel (padding > 10 %) and BiCGStab matches the oracle."""
    m = gen.add_long_rows(gen.make_matrix("C2"))
    b = gen.make_rhs(m)
    A = zk.csr_create(m["row_ptr"], m["col_idx"], m["values"], m["n"])
    assert A.info["spmv_mode"] == 0
    r = zk.solve(A, cuda(b), tol=1e-8, method="bicgstab")
    refs = [oracle.bicgstab(m, b, tol=1e-8, order=o) for o in ORDERS]
    its = [q["iters"] for q in refs]
    assert r["status"] == "CONVERGED" and 0.95 * min(its) <= r["iters"] <= 1.05 * max(its)
    assert relerr(r["x"].cpu().numpy(), refs[0]["x"]) <= 1e-6


@pytest.mark.parametrize("method", ["bicgstab", "bicgstab_jacobi"])
@pytest.mark.parametrize("cfg", ["C1", "C2", "T0"])
def test_cluster_solver_parity(cfg, method, monkeypatch):
    """Loop mode 5 (the default up to 16384 rows when the rows fit the cluster's shared memory): the whole
    loop in one thread-block cluster, reductions over distributed shared memory, scalar steps
    replicated per CTA."""
    if cfg != "C1":
        monkeypatch.setenv("ZK_LOOP_MODE", "5")
    m = gen.make_matrix(cfg)
    b = gen.make_rhs(m)
    r = gpu_solve(m, b, tol=1e-8, method=method)
    # BiCGStab from x0 = 0: ONE launch (the cluster kernel does the init); Jacobi: + x = M⁻¹u, k_true
    assert r["loop_mode"] == 5 and r["gpu_launches"] == (1 if method == "bicgstab" else 3)
    fn = oracle.bicgstab if method == "bicgstab" else oracle.bicgstab_jacobi
    refs = [fn(m, b, tol=1e-8, order=o) for o in ORDERS]
    its = [q["iters"] for q in refs]
    assert r["status"] == "CONVERGED" and 0.95 * min(its) <= r["iters"] <= 1.05 * max(its), (r["iters"], its)
    k = min(12, r["iters"], refs[0]["iters"]) + 1
    assert np.max(np.abs(r["hist"][:k] - refs[0]["hist"][:k]) / refs[0]["hist"][:k]) <= 1e-10
    assert relerr(r["x"], refs[0]["x"]) <= 1e-6 and r["true_relres"] <= 2e-8
    r2 = gpu_solve(m, b, tol=1e-8, method=method)                  # deterministic
    assert np.array_equal(r["x"], r2["x"]) and np.array_equal(r["hist"], r2["hist"])


def test_cluster_solver_outcomes(monkeypatch):
    """Mode 5 exits: MAXIT with the oracle's history, half-step exit (cI), breakdown."""
    monkeypatch.setenv("ZK_LOOP_MODE", "5")
    m = gen.make_matrix("C2")
    b = gen.make_rhs(m)
    r = gpu_solve(m, b, tol=1e-14, maxit=9)
    ref = oracle.bicgstab(m, b, tol=1e-14, maxit=9)
    assert r["loop_mode"] == 5 and r["status"] == ref["status"] == "MAXIT" and r["iters"] == 9
    assert np.max(np.abs(r["hist"] - ref["hist"]) / ref["hist"]) <= 1e-10
    assert relerr(r["x"], ref["x"]) <= 1e-10
    n = 3000
    c = 0.3 - 2j
    d = dict(row_ptr=np.arange(n + 1, dtype=np.int64), col_idx=np.arange(n, dtype=np.int32),
             values=np.full(n, c, np.complex128), n=n)
    bb = gen.rand_vector(n, 1)
    q = gpu_solve(d, bb, tol=1e-12)
    assert q["loop_mode"] == 5 and q["status"] == "CONVERGED" and q["iters"] == 1
    assert np.max(np.abs(q["x"] - bb / c)) <= 1e-15 * np.max(np.abs(bb / c))
    sk = dict(row_ptr=np.array([0, 1, 2]), col_idx=np.array([1, 0], np.int32),
              values=np.array([1, -1], np.complex128), n=2)
    assert gpu_solve(sk, np.array([1, 0], np.complex128))["status"] == "BREAKDOWN_SIGMA"


@pytest.mark.parametrize("w", ["1", "2", "4", "8"])
@pytest.mark.parametrize("vs", ["0", "1"])
@pytest.mark.parametrize("cfg", ["C1", "T0"])
def test_cluster_solver_lane_variants(cfg, w, vs, monkeypatch):
    """Every instantiation of the cluster solver (W lanes per row, values in shared memory or in
    global memory) against the oracle: same parity bar as test_cluster_solver_parity."""
    monkeypatch.setenv("ZK_LOOP_MODE", "5")
    monkeypatch.setenv("ZK_CLUSTER_W", w)
    monkeypatch.setenv("ZK_CLUSTER_VS", vs)
    m = gen.make_matrix(cfg)
    b = gen.make_rhs(m)
    r = gpu_solve(m, b, tol=1e-8)
    assert r["loop_mode"] == 5
    refs = [oracle.bicgstab(m, b, tol=1e-8, order=o) for o in ORDERS]
    its = [q["iters"] for q in refs]
    assert r["status"] == "CONVERGED" and 0.95 * min(its) <= r["iters"] <= 1.05 * max(its), (r["iters"], its)
    k = min(12, r["iters"], refs[0]["iters"]) + 1
    assert np.max(np.abs(r["hist"][:k] - refs[0]["hist"][:k]) / refs[0]["hist"][:k]) <= 1e-10
    assert relerr(r["x"], refs[0]["x"]) <= 1e-6 and r["true_relres"] <= 2e-8


@pytest.mark.parametrize("variant", ["auto", "w1", "w2", "w4", "w8", "gval"])
@pytest.mark.parametrize("cfg", ["C1", "C2", "T0"])
@pytest.mark.parametrize("method", ["cg", "cocg"])
def test_cg_cocg_cluster_parity(method, cfg, variant, monkeypatch):
    """Loop mode 5 for CG (gauge-twisted HPD variant, L9) and COCG (the absorbing complex-symmetric
    matrices): every lane-count instantiation and the values-in-global variant against the oracle
    (±5 % iterations, hist prefix 1e-10, solution 1e-6); deterministic."""
    monkeypatch.setenv("ZK_LOOP_MODE", "5")
    if variant.startswith("w"):
        monkeypatch.setenv("ZK_CLUSTER_W", variant[1:])
    if variant == "gval":
        monkeypatch.setenv("ZK_CLUSTER_VS", "0")
    if method == "cg":
        m = gen.make_matrix(cfg, eta=0.0, twist_seed=gen.SEED_TWIST)
        b = np.exp(1j * m["phase"]) * gen.make_rhs(m)
        ref = oracle.cg(m, b, tol=1e-8)
    else:
        m = gen.make_matrix(cfg)
        b = gen.make_rhs(m)
        ref = oracle.cocg(m, b, tol=1e-8)
    r = gpu_solve(m, b, tol=1e-8, method=method)
    assert r["loop_mode"] == 5 and r["gpu_launches"] == 1  # the cluster kernel starts from x0 = 0 itself
    assert r["status"] == ref["status"] == "CONVERGED"
    assert abs(r["iters"] - ref["iters"]) <= 0.05 * ref["iters"], (r["iters"], ref["iters"])
    k = min(12, r["iters"]) + 1
    assert np.max(np.abs(r["hist"][:k] - ref["hist"][:k]) / ref["hist"][:k]) <= 1e-10
    assert relerr(r["x"], ref["x"]) <= 1e-6 and r["true_relres"] <= 2e-8
    r2 = gpu_solve(m, b, tol=1e-8, method=method)
    assert np.array_equal(r["x"], r2["x"]) and np.array_equal(r["hist"], r2["hist"])


def test_cg_cluster_outcomes(monkeypatch):
    """Mode 5 CG exits: MAXIT with the oracle's history and x, NOT_HPD on an indefinite matrix."""
    monkeypatch.setenv("ZK_LOOP_MODE", "5")
    m = gen.make_matrix("T0", eta=0.0, twist_seed=gen.SEED_TWIST)
    b = np.exp(1j * m["phase"]) * gen.make_rhs(m)
    r = gpu_solve(m, b, tol=1e-14, maxit=9, method="cg")
    ref = oracle.cg(m, b, tol=1e-14, maxit=9)
    assert r["loop_mode"] == 5 and r["status"] == ref["status"] == "MAXIT" and r["iters"] == 9
    assert np.max(np.abs(r["hist"] - ref["hist"]) / ref["hist"]) <= 1e-10
    assert relerr(r["x"], ref["x"]) <= 1e-10
    n = 500
    vals = np.where(np.arange(n) % 2 == 0, 1.0, -1.0).astype(np.complex128)
    d = dict(row_ptr=np.arange(n + 1, dtype=np.int64), col_idx=np.arange(n, dtype=np.int32), values=vals, n=n)
    bb = np.ones(n, np.complex128)
    q = gpu_solve(d, bb, tol=1e-10, method="cg")
    assert q["loop_mode"] == 5 and q["status"] == oracle.cg(d, bb, tol=1e-10)["status"] == "NOT_HPD"


def test_bicgstab_c5_full_size_closed_form():
    """C5 (BASELINE.json configs[4], unit-cube interior 400^3: 64M rows, 1.72G nonzeros) on ONE
    B200 — the system the row-partitioned runs split: BiCGStab to 1e-8 through zk_solve, the
    forward error against the DST-I exact solution within 2κ·tol (L12; κ = 2.4e4 closed form),
    the true residual, and the first 2 iterations' history against the oracle (one oracle
    iteration at 64M rows is ~11 s of single-thread SpMV)."""
    spec = gen.CONFIGS["C5"]
    m = gen.make_matrix(spec)
    b = gen.make_rhs(m)
    A = zk.csr_create(cuda(m["row_ptr"]), cuda(m["col_idx"]), cuda(m["values"]), m["n"], borrow=True)
    assert A.info["spmv_mode"] == 3 and A.info["nnz"] == 1_719_374_392
    r = zk.solve(A, cuda(b), tol=1e-8, maxit=2000, method="bicgstab")
    assert r["status"] == "CONVERGED" and r["true_relres"] <= 2e-8
    x = r["x"].cpu().numpy()
    hist = r["hist"]
    del r
    A.close()
    torch.cuda.empty_cache()
    oracle.use_all_cores(True)  # the bit-identical OpenMP build (test_oracle_openmp_build_is_bitwise_identical)
    try:
        ref = oracle.bicgstab(m, b, tol=1e-8, maxit=2)
    finally:
        oracle.use_all_cores(False)
    assert np.max(np.abs(hist[:3] - ref["hist"][:3]) / ref["hist"][:3]) <= 1e-10
    del m
    xe = cf.box_solve(spec, b, gen.ETA)
    assert relerr(x, xe) <= 2 * cf.box_kappa(spec, gen.ETA) * 1e-8


@pytest.mark.parametrize("init", ["0", "1"])
def test_cluster_fused_init(init, monkeypatch):
    """The fused x0 = 0 start of the BiCGStab cluster kernel (init=1: one launch per solve) and the
    k_set_ctx + k_init_zero start (init=0: three launches) both match the oracle, deterministically."""
    monkeypatch.setenv("ZK_LOOP_MODE", "5")
    monkeypatch.setenv("ZK_CLUSTER_INIT", init)
    m = gen.make_matrix("C1")
    b = gen.make_rhs(m)
    r, r2 = gpu_solve(m, b, tol=1e-8), gpu_solve(m, b, tol=1e-8)
    assert r["gpu_launches"] == (1 if init == "1" else 3)
    assert np.array_equal(r["x"], r2["x"]) and np.array_equal(r["hist"], r2["hist"])
    ref = oracle.bicgstab(m, b, tol=1e-8)
    assert abs(r["iters"] - ref["iters"]) <= 1
    assert np.max(np.abs(r["hist"][:13] - ref["hist"][:13]) / ref["hist"][:13]) <= 1e-10
    assert relerr(r["x"], ref["x"]) <= 1e-6


@pytest.mark.parametrize("keep", ["0", "1"])
def test_dropped_csr_values_jacobi_and_update(keep, monkeypatch):
    """Copied handles above 16384 rows keep only the SELL copy of the values (the library's CSR value
    copy is dropped; ZK_KEEP_CSR_VALUES=1 keeps it): Jacobi-BiCGStab then takes its diagonal from
    the SELL copy and zk_csr_update_values refills the SELL copy from a temporary.  Both ways give
    the oracle's results, and bitwise the same solves."""
    monkeypatch.setenv("ZK_KEEP_CSR_VALUES", keep)
    m = gen.make_matrix("A3")                      # Audi3D-3 shape, 85,001 rows
    b = gen.make_rhs(m)
    A = zk.csr_create(m["row_ptr"], m["col_idx"], m["values"], m["n"])
    assert A.info["spmv_mode"] == 3 and A.info["csr_values_kept"] == int(keep)
    r = zk.solve(A, cuda(b), tol=1e-8, method="bicgstab_jacobi")
    refs = [oracle.bicgstab_jacobi(m, b, tol=1e-8, order=o) for o in ORDERS]
    its = [q["iters"] for q in refs]
    assert r["status"] == "CONVERGED" and 0.95 * min(its) <= r["iters"] <= 1.05 * max(its), (r["iters"], its)
    assert relerr(r["x"].cpu().numpy(), refs[0]["x"]) <= 1e-6
    m2 = gen.make_matrix("A3", k=2 * np.pi / 2.5)
    A.update_values(m2["values"])
    x = gen.rand_vector(m["n"], 3)
    y = torch.empty(m["n"], dtype=torch.complex128, device=DEV)
    zk.zcsrmv(A, 1, cuda(x), 0, y)
    want = oracle.zcsrmv(m2, x)
    scale = np.add.reduceat(np.abs(m2["values"]) * np.abs(x[m2["col_idx"]]), m2["row_ptr"][:-1])
    assert np.all(np.abs(y.cpu().numpy() - want) <= 1e-13 * scale)
    r2 = zk.solve(A, cuda(b), tol=1e-8, method="bicgstab_jacobi")
    ref2 = oracle.bicgstab_jacobi(m2, b, tol=1e-8)
    assert r2["status"] == "CONVERGED" and relerr(r2["x"].cpu().numpy(), ref2["x"]) <= 1e-6


def test_dropped_csr_values_bitwise(monkeypatch):
    m = gen.make_matrix("A3")
    b = gen.make_rhs(m)
    out = []
    for keep in ("0", "1"):
        monkeypatch.setenv("ZK_KEEP_CSR_VALUES", keep)
        A = zk.csr_create(m["row_ptr"], m["col_idx"], m["values"], m["n"])
        out.append(zk.solve(A, cuda(b), tol=1e-8, method="bicgstab_jacobi"))
    assert out[0]["iters"] == out[1]["iters"] and torch.equal(out[0]["x"], out[1]["x"])


@pytest.mark.parametrize("cfg", ["C1", "T1"])
def test_create_solve_destroy_loop_on_side_stream(cfg):
    """The e2e pattern (bench.py e2e_step) on a torch side stream: pinned host CSR → create →
    solve → x back → destroy, many times with no other handle alive and with one alive.  The
    library's small scratch comes from its stream-ordered pool and its pinned readback staging
    from a process-wide free list (no cudaMalloc / cudaFree / cudaFreeHost on this path): every
    round must give the same iterations and the same x bits as the first."""
    m = gen.make_matrix(cfg)
    rp, ci, va = (torch.from_numpy(a).pin_memory() for a in (m["row_ptr"], m["col_idx"], m["values"]))
    b_pin = torch.from_numpy(gen.make_rhs(m)).pin_memory()
    x_h = torch.empty(m["n"], dtype=torch.complex128).pin_memory()
    side = torch.cuda.Stream()
    ref = None
    keep = None
    for rnd in range(12):
        if rnd == 6:  # second half: another handle stays alive (the pool is not trimmed between rounds)
            keep = zk.csr_create(m["row_ptr"], m["col_idx"], m["values"], m["n"])
        with torch.cuda.stream(side):
            A = zk.csr_create(rp, ci, va, m["n"], stream=side)
            bd = b_pin.to(DEV, non_blocking=True)
            # maxit varies: the readback staging grows, old buffers go back to the free list
            r = zk.solve(A, bd, tol=1e-8, maxit=500 + 100 * rnd, method="bicgstab", stream=side)
            x_h.copy_(r["x"], non_blocking=True)
            A.close()
        side.synchronize()
        got = (r["iters"], r["status"], x_h.numpy().copy())
        if ref is None:
            ref = got
        assert got[0] == ref[0] and got[1] == ref[1] == "CONVERGED"
        assert np.array_equal(got[2], ref[2]), f"round {rnd}: x differs"
    keep.close()



@pytest.mark.parametrize("method", ["cg", "cocg", "tfqmr", "bicgstab_l2", "bicgstab_l8"])
@pytest.mark.parametrize("cfg", ["C1", "T0"])
def test_cluster_fused_init_all_solvers(cfg, method, monkeypatch):
    """Every cluster solver starts from x0 = 0 inside its kernel (OpInitZero's rows and sums, the
    method's fin_init step; TFQMR also its K0 SpMV and σ): one launch per solve instead of
    k_set_ctx + k_init_zero (+ k0_tfqmr) + the cluster kernel.  Both starts against the oracle (the
    per-method bars of the cluster parity tests) and against each other (same count ±1, histories
    to 1e-9 — 1e-3 for BiCGStab(8), R20 — only the init reductions' order differs)."""
    monkeypatch.setenv("ZK_LOOP_MODE", "5")
    ell = int(method[-1]) if method.startswith("bicgstab_l") else 8
    meth = "bicgstab_l" if method.startswith("bicgstab_l") else method
    if method == "cg":
        m = gen.make_matrix(cfg, eta=0.0, twist_seed=gen.SEED_TWIST)
        b = np.exp(1j * m["phase"]) * gen.make_rhs(m)
        refs = [oracle.cg(m, b, tol=1e-8, order=o) for o in ORDERS]
    else:
        m = gen.make_matrix(cfg)
        b = gen.make_rhs(m)
        fn = {"cocg": oracle.cocg, "tfqmr": oracle.tfqmr,
              "bicgstab_l": lambda mm, bb, **kw: oracle.bicgstab_l(mm, bb, ell=ell, **kw)}[meth]
        refs = [fn(m, b, tol=1e-8, order=o) for o in ORDERS]
    its = [q["iters"] for q in refs]
    out = {}
    for init in ("0", "1"):
        monkeypatch.setenv("ZK_CLUSTER_INIT", init)
        r = gpu_solve(m, b, tol=1e-8, maxit=1000, method=meth, ell=ell)
        extra = 1 if (meth == "tfqmr" and init == "0") else 0
        assert r["loop_mode"] == 5 and r["gpu_launches"] == (1 if init == "1" else 3 + extra)
        assert r["status"] == "CONVERGED" and 0.95 * min(its) - 1 <= r["iters"] <= 1.05 * max(its) + 1, (r["iters"], its)
        assert r["true_relres"] <= 10 * 1e-8
        out[init] = r
    a, f = out["0"], out["1"]
    assert abs(a["iters"] - f["iters"]) <= 1
    k = min(a["iters"], f["iters"], 8) + 1
    # BiCGStab(8)'s normal-equations step amplifies rounding-order differences (R20: the
    # oracle's own summation orders spread by 9.2e-5 at ℓ = 8, bar 1e-3); 1e-9 elsewhere
    bar = 1e-3 if method == "bicgstab_l8" else 1e-9
    assert np.max(np.abs(a["hist"][:k] - f["hist"][:k]) / a["hist"][:k]) <= bar


def test_jacobi_cache_without_csr_values():
    """Above 16384 rows a copied handle keeps A·M⁻¹ only in its SELL copy (csr_values_kept = 0):
    Jacobi-BiCGStab builds it once per handle — repeated solves allocate no device memory and give
    the same bits — and zk_csr_update_values invalidates it (regression: the cache was keyed on the
    CSR copy and A·M⁻¹ was rebuilt and leaked on every solve)."""
    m = gen.make_matrix("T1")
    assert m["n"] > 16384
    A = zk.csr_create(m["row_ptr"], m["col_idx"], m["values"], m["n"])
    assert A.info["csr_values_kept"] == 0 and A.info["spmv_mode"] == 3
    b = cuda(gen.make_rhs(m))
    x = torch.empty_like(b)
    ws = zk.alloc_workspace(A, "bicgstab_jacobi", 1000)
    r0 = zk.solve(A, b, tol=1e-8, method="bicgstab_jacobi", workspace=ws, x=x)
    x0 = x.cpu()  # (host-side comparisons: no torch kernel is loaded lazily inside the measured loop)
    torch.cuda.synchronize()
    free0 = torch.cuda.mem_get_info()[0]
    for _ in range(6):
        r = zk.solve(A, b, tol=1e-8, method="bicgstab_jacobi", workspace=ws, x=x)
        assert r["iters"] == r0["iters"] and torch.equal(x.cpu(), x0)
    torch.cuda.synchronize()
    assert free0 - torch.cuda.mem_get_info()[0] < (4 << 20)   # one A·M⁻¹ SELL copy is ≈ 27 MB
    its = [oracle.bicgstab_jacobi(m, gen.make_rhs(m), tol=1e-8, order=o)["iters"] for o in ORDERS]
    assert r0["status"] == "CONVERGED" and 0.95 * min(its) <= r0["iters"] <= 1.05 * max(its), (r0["iters"], its)
    # new values on the same pattern: A·M⁻¹ rebuilt from them.  For 2·A every step of the scaling
    # is exact (powers of two), so A·M⁻¹ and the iterates are bitwise the same and x is exactly x0 / 2
    A.update_values(2.0 * m["values"])
    r2 = zk.solve(A, b, tol=1e-8, method="bicgstab_jacobi", workspace=ws, x=x)
    assert r2["status"] == "CONVERGED" and r2["iters"] == r0["iters"]
    assert torch.equal(2.0 * x.cpu(), x0)
    A.close()


def test_concurrent_solves_on_two_streams():
    """Two host threads, each with its own handle and torch stream, solving at the same time (a
    cluster solve on C1 and a WHILE-graph solve on T1, plus zdotc / dznrm2 on each stream): every
    result equals the one computed alone (per-handle staging, per-stream reduction scratch, the
    process-wide pinned free list and memory pool are shared safely)."""
    import threading
    cases = []
    for cfg in ("C1", "T1"):
        m = gen.make_matrix(cfg)
        A = zk.csr_create(m["row_ptr"], m["col_idx"], m["values"], m["n"])
        b = cuda(gen.make_rhs(m))
        alone = zk.solve(A, b, tol=1e-8, maxit=1000)
        cases.append((A, b, alone["x"].cpu(), alone["iters"], float(zk.dznrm2(b).cpu()[0])))
    errors = []

    def work(A, b, x_ref, it_ref, nb_ref):
        st = torch.cuda.Stream()
        try:
            with torch.cuda.stream(st):
                for _ in range(15):
                    r = zk.solve(A, b, tol=1e-8, maxit=1000, stream=st)
                    nb = zk.dznrm2(b, stream=st)
                    d = zk.zdotc(b, b, stream=st)
                    st.synchronize()
                    if r["iters"] != it_ref or not torch.equal(r["x"].cpu(), x_ref):
                        errors.append("solve differs")
                    if float(nb.cpu()[0]) != nb_ref or abs(float(d.cpu()[0].real) - nb_ref ** 2) > 1e-12 * nb_ref ** 2:
                        errors.append("reduction differs")
        except Exception as e:  # noqa: BLE001 — reported below
            errors.append(repr(e))

    th = [threading.Thread(target=work, args=c) for c in cases]
    for t in th:
        t.start()
    for t in th:
        t.join()
    assert not errors, errors[:3]
    for c in cases:
        c[0].close()


@pytest.mark.parametrize("method", ["bicgstab", "cg", "tfqmr", "bicgstab_l2"])
def test_while_body_exits_at_every_position(method, monkeypatch):
    """The WHILE graph runs four iterations per body (solve.cu kWhileUnroll): a solve that stops
    after k iterations (MAXIT, k = 1..6, and the converged count) must give the bits of the direct-
    launch loop (one iteration per host step), whatever the exit's position inside a body."""
    ell = 2 if method == "bicgstab_l2" else 8
    meth = "bicgstab_l" if method == "bicgstab_l2" else method
    if method == "cg":
        m = gen.make_matrix("T1", eta=0.0, twist_seed=gen.SEED_TWIST)
        b = np.exp(1j * m["phase"]) * gen.make_rhs(m)
    else:
        m = gen.make_matrix("T1")
        b = gen.make_rhs(m)
    A = zk.csr_create(m["row_ptr"], m["col_idx"], m["values"], m["n"])
    bd = cuda(b)
    for maxit in (1, 2, 3, 4, 5, 6, 1000):
        out = {}
        for mode in ("1", "3"):
            monkeypatch.setenv("ZK_LOOP_MODE", mode)
            r = zk.solve(A, bd, tol=1e-8, maxit=maxit, method=meth, ell=ell)
            assert r["loop_mode"] == int(mode)
            out[mode] = r
        a, d = out["1"], out["3"]
        assert a["status"] == d["status"] and a["iters"] == d["iters"], (maxit, a["status"], a["iters"], d["iters"])
        assert (a["status"] == "MAXIT") == (maxit < 1000) and a["iters"] <= maxit
        assert torch.equal(a["x"], d["x"]) and np.array_equal(a["hist"], d["hist"])
        assert a["true_relres"] == d["true_relres"]
    A.close()
