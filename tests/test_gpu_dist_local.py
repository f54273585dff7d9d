"""Row-partitioned path with REAL multi-rank halos on one GPU.

The ranks are threads of this process joined by libzk's LOCAL transport (zk_local_group_create +
zk_comm_create_local, include/zk.h): the same dist.cu halo plan, pack kernel, grouped send/recv
exchange and distributed reduction finish that run over NCCL on 2-8 GPUs, with the bytes moved by
stream-ordered device copies instead (NCCL refuses two ranks on one GPU).  Every call goes through
the C-ABI; the results are compared with the CPU oracle on the global system:

  * distributed zk_zcsrmv: elementwise 1e-13 (row scale, L4) against the oracle, and bitwise equal
    to the 1-rank result (the renumbered rows sum the same entries in the same order);
  * zk_zdotc / zk_dznrm2 with a comm: 1e-12 (L5);
  * BiCGStab / CG / COCG / TFQMR with n_halo > 0 on every rank: count within the oracle envelope
    (L11), history prefix to 1e-10, x to 1e-6 (L12), identical outcome on every rank.
"""
import threading

import numpy as np
import pytest
import torch

import gen
import oracle
from paper_2112_11880_b200 import zk

pytestmark = pytest.mark.gpu
DEV = 0
ORDERS = (oracle.ORD_SEQ, oracle.ORD_REV, oracle.ORD_BLOCK256)


def run_ranks(n, fn):
    """Run fn(rank, comm, stream) on n threads of one LOCAL group; return the per-rank results."""
    group = zk.LocalGroup(n)
    out, errs = [None] * n, [None] * n

    def body(r):
        try:
            torch.cuda.set_device(DEV)
            s = torch.cuda.Stream()
            with torch.cuda.stream(s):
                comm = zk.Comm.local(group, r, DEV)
                try:
                    out[r] = fn(r, comm, s)
                finally:
                    torch.cuda.synchronize()
            comm.close()
        except BaseException as e:  # noqa: BLE001 — re-raised in the main thread
            errs[r] = e

    th = [threading.Thread(target=body, args=(r,)) for r in range(n)]
    for t in th:
        t.start()
    for t in th:
        t.join(timeout=600)
    group.close()
    for e in errs:
        if e is not None:
            raise e
    return out


def block(m, off, r):
    """Rows [off[r], off[r+1]) of a global CSR dict, global column ids."""
    lo, hi = int(off[r]), int(off[r + 1])
    rp = m["row_ptr"]
    a, b = int(rp[lo]), int(rp[hi])
    return rp[lo:hi + 1] - a, m["col_idx"][a:b], m["values"][a:b], lo, hi


def offsets(m, n):
    return zk.partition_rows(m["row_ptr"], n)


def dist_csr(m, off, r, comm, s, **kw):
    rp, ci, va, lo, hi = block(m, off, r)
    return zk.csr_create(rp, ci, va, m["n"], comm=comm, row_begin=lo, stream=s, **kw)


def interior_run(m, off, r):
    """Rows of the longest run of 32-row slices of rank r's block referencing only its own rows."""
    _, ci, _, lo, hi = block(m, off, r)
    rp = m["row_ptr"][lo:hi + 1] - m["row_ptr"][lo]
    ext = (ci < lo) | (ci >= hi)
    best = (0, 0)
    run = 0
    ns = (hi - lo + 31) // 32
    for s in range(ns + 1):
        ok = s < ns and not ext[rp[32 * s]:rp[min(32 * s + 32, hi - lo)]].any()
        if ok:
            run += 1
        else:
            if run > best[1] - best[0]:
                best = (s - run, s)
            run = 0
    return min(best[1] * 32, hi - lo) - best[0] * 32 if best[1] > best[0] else 0


def cuda(a):
    return torch.from_numpy(np.ascontiguousarray(a)).to(f"cuda:{DEV}")


def row_scale(m, x):
    rp, ci, va = m["row_ptr"], m["col_idx"], m["values"]
    t = np.abs(va) * np.abs(x[ci])
    return np.add.reduceat(t, rp[:-1]) * (np.diff(rp) > 0)


@pytest.mark.parametrize("overlap", ["1", "0"])
@pytest.mark.parametrize("nranks", [2, 3, 4])
@pytest.mark.parametrize("cfg", ["C1", "C2", "random"])
def test_local_zcsrmv_halo(cfg, nranks, overlap, monkeypatch):
    """ZK_DIST_OVERLAP=1 (default): interior slices run while the exchange is in flight, boundary
    slices after it; 0: blocking exchange, then the whole SpMV."""
    monkeypatch.setenv("ZK_DIST_OVERLAP", overlap)
    m = gen.random_csr(3000, 5, max_len=40) if cfg == "random" else gen.make_matrix(cfg)
    n = m["n"]
    x = gen.rand_vector(n, 11)
    y0 = gen.rand_vector(n, 12)
    off = offsets(m, nranks)
    A1 = zk.csr_create(m["row_ptr"], m["col_idx"], m["values"], n)
    y1 = cuda(y0)
    zk.zcsrmv(A1, 1.0, cuda(x), 0.0, y1)
    y1 = y1.cpu().numpy()

    def fn(r, comm, s):
        A = dist_csr(m, off, r, comm, s)
        lo, hi = int(off[r]), int(off[r + 1])
        xl = cuda(x[lo:hi])
        y = cuda(y0[lo:hi])
        zk.zcsrmv(A, 1.0, xl, 0.0, y)
        y2 = cuda(y0[lo:hi])
        zk.zcsrmv(A, 0.5 - 2j, xl, 1.5j, y2)  # beta != 0 reads y
        torch.cuda.current_stream().synchronize()
        return A.info, y.cpu().numpy(), y2.cpu().numpy()

    res = run_ranks(nranks, fn)
    for r, (info, _, _) in enumerate(res):
        assert info["nranks"] == nranks and info["n_global"] == n and info["row_begin"] == off[r]
        assert info["n_halo"] > 0, f"rank {r} has no halo"
        if overlap == "0" or info["spmv_mode"] != 3:
            assert info["interior_rows"] == 0
        else:  # the longest run of 32-row slices whose rows reference no off-rank column
            assert info["interior_rows"] == interior_run(m, off, r), info
    y = np.concatenate([q[1] for q in res])
    y2 = np.concatenate([q[2] for q in res])
    ref = oracle.zcsrmv(m, x)
    ref2 = oracle.zcsrmv(m, x, alpha=0.5 - 2j, beta=1.5j, y=y0)
    sc = row_scale(m, x)
    assert np.all(np.abs(y - ref) <= 1e-13 * sc + 1e-300)
    assert np.all(np.abs(y2 - ref2) <= 1e-13 * (sc * abs(0.5 - 2j) + 1.5 * np.abs(y0)))
    # same mapping (SELL-32) on every rank as on one GPU: each row sums the same entries in the
    # same order, so the bits agree (a rank whose SELL padding exceeds 10 % takes the CSR
    # sub-warp kernel, whose lane-split sums round differently)
    if all(q[0]["spmv_mode"] == A1.info["spmv_mode"] == 3 for q in res):
        assert np.array_equal(y, y1), "distributed SpMV must equal the 1-rank SpMV bitwise"


@pytest.mark.parametrize("nranks", [2, 4])
def test_local_dot_norm(nranks):
    n = 100_003
    x, y = gen.rand_vector(n, 1), gen.rand_vector(n, 2)
    off = np.linspace(0, n, nranks + 1).astype(np.int64)

    def fn(r, comm, s):
        lo, hi = off[r], off[r + 1]
        d = zk.zdotc(cuda(x[lo:hi]), cuda(y[lo:hi]), comm=comm)
        nr = zk.dznrm2(cuda(x[lo:hi]), comm=comm)
        return complex(d.cpu().numpy()[0]), float(nr.cpu().numpy()[0])

    res = run_ranks(nranks, fn)
    dref, nref = oracle.zdotc(x, y), oracle.dznrm2(x)
    for d, nr in res:
        assert d == res[0][0] and nr == res[0][1], "every rank holds the same bits"
        assert abs(d - dref) <= 1e-12 * oracle.dznrm2(x) * oracle.dznrm2(y)
        assert abs(nr - nref) <= 1e-12 * nref


def _solve_ranks(m, b, off, nranks, method, tol=1e-8, maxit=1000):
    def fn(r, comm, s):
        A = dist_csr(m, off, r, comm, s)
        lo, hi = int(off[r]), int(off[r + 1])
        out = zk.solve(A, cuda(b[lo:hi]), tol=tol, maxit=maxit, method=method)
        out["x"] = out["x"].cpu().numpy()
        out["n_halo"] = A.info["n_halo"]
        return out

    return run_ranks(nranks, fn)


def _check_ranks(res, nranks):
    for q in res:
        assert q["n_halo"] > 0
        assert q["status"] == res[0]["status"] and q["iters"] == res[0]["iters"]
        assert np.array_equal(q["hist"], res[0]["hist"]), "every rank takes the same branches"
        assert q["loop_mode"] == 3
    return np.concatenate([q["x"] for q in res])


def relerr(a, b):
    return np.linalg.norm(a - b) / np.linalg.norm(b)


@pytest.mark.parametrize("overlap", ["1", "0"])
@pytest.mark.parametrize("nranks", [2, 4])
@pytest.mark.parametrize("method", ["bicgstab", "tfqmr"])
@pytest.mark.parametrize("cfg", ["C1", "C2"])
def test_local_bicgstab_tfqmr(cfg, method, nranks, overlap, monkeypatch):
    monkeypatch.setenv("ZK_DIST_OVERLAP", overlap)
    m = gen.make_matrix(cfg)
    b = gen.make_rhs(m)
    res = _solve_ranks(m, b, offsets(m, nranks), nranks, method)
    x = _check_ranks(res, nranks)
    r = res[0]
    fn = oracle.bicgstab if method == "bicgstab" else oracle.tfqmr
    refs = [fn(m, b, tol=1e-8, order=o) for o in ORDERS]
    its = [q["iters"] for q in refs]
    assert r["status"] == "CONVERGED" and all(q["status"] == "CONVERGED" for q in refs)
    assert 0.95 * min(its) <= r["iters"] <= 1.05 * max(its), (r["iters"], its)
    k = min(12, r["iters"], refs[0]["iters"]) + 1
    assert np.max(np.abs(r["hist"][:k] - refs[0]["hist"][:k]) / refs[0]["hist"][:k]) <= 1e-10
    assert relerr(x, refs[0]["x"]) <= 1e-6
    assert r["true_relres"] <= (2e-8 if method == "bicgstab" else 1e-7)


@pytest.mark.parametrize("nranks", [2, 4])
@pytest.mark.parametrize("cfg", ["C1", "C2"])
def test_local_cg_cocg(cfg, nranks):
    mg = gen.make_matrix(cfg, eta=0.0, twist_seed=gen.SEED_TWIST)
    bg = np.exp(1j * mg["phase"]) * gen.make_rhs(mg)
    res = _solve_ranks(mg, bg, offsets(mg, nranks), nranks, "cg")
    x = _check_ranks(res, nranks)
    ref = oracle.cg(mg, bg, tol=1e-8)
    assert res[0]["status"] == ref["status"] == "CONVERGED"
    assert abs(res[0]["iters"] - ref["iters"]) <= 0.05 * ref["iters"]
    k = min(12, res[0]["iters"]) + 1
    assert np.max(np.abs(res[0]["hist"][:k] - ref["hist"][:k]) / ref["hist"][:k]) <= 1e-10
    assert relerr(x, ref["x"]) <= 1e-6

    m = gen.make_matrix(cfg)
    b = gen.make_rhs(m)
    res = _solve_ranks(m, b, offsets(m, nranks), nranks, "cocg")
    x = _check_ranks(res, nranks)
    ref = oracle.cocg(m, b, tol=1e-8)
    assert res[0]["status"] == ref["status"] == "CONVERGED"
    assert abs(res[0]["iters"] - ref["iters"]) <= max(1, 0.05 * ref["iters"])
    assert relerr(x, ref["x"]) <= 1e-6


def test_local_ranks_match_single_gpu_counts():
    """The same system on 1, 2 and 4 ranks: CG counts identical (L11 (i)), x within 1e-6."""
    mg = gen.make_matrix("C2", eta=0.0, twist_seed=gen.SEED_TWIST)
    bg = np.exp(1j * mg["phase"]) * gen.make_rhs(mg)
    xs, its = [], []
    for nr in (1, 2, 4):
        def fn(r, comm, s, nr=nr):
            A = dist_csr(mg, offsets(mg, nr), r, comm, s)
            lo, hi = int(offsets(mg, nr)[r]), int(offsets(mg, nr)[r + 1])
            o = zk.solve(A, cuda(bg[lo:hi]), tol=1e-8, method="cg")
            return o["iters"], o["x"].cpu().numpy()
        res = run_ranks(nr, fn)
        its.append(res[0][0])
        xs.append(np.concatenate([q[1] for q in res]))
    assert its[0] == its[1] == its[2], its
    assert relerr(xs[1], xs[0]) <= 1e-6 and relerr(xs[2], xs[0]) <= 1e-6


def test_local_validation_agreement():
    """A rank whose block fails validation makes every rank fail (no rank is left blocked in the
    halo-plan collectives)."""
    m = gen.make_matrix("C1")
    off = offsets(m, 2)

    def fn(r, comm, s):
        rp, ci, va, lo, hi = block(m, off, r)
        if r == 1:
            ci = ci.copy()
            ci[5] = m["n"] + 3  # column out of range on rank 1 only
        try:
            zk.csr_create(rp, ci, va, m["n"], comm=comm, row_begin=lo, stream=s)
        except zk.ZkError as e:
            return str(e)
        return "ok"

    res = run_ranks(2, fn)
    assert "another rank" in res[0], res
    assert "out of range" in res[1], res


@pytest.mark.parametrize("ell", [1, 2, 4])
@pytest.mark.parametrize("nranks", [2, 4])
def test_local_bicgstab_l(nranks, ell):
    """BiCGStab(ℓ) row-partitioned: halo before every S1/S2 SpMV, each reduction point and the
    (ℓ+1)² Gram totals allreduced, the Cholesky replicated on every rank; against the oracle's
    envelope, the history to HTOL[ℓ] and x to 1e-6."""
    from tests.test_gpu_bicgstab_l import HTOL
    m = gen.make_matrix("C2")
    b = gen.make_rhs(m)

    def fn(r, comm, s):
        off = offsets(m, nranks)
        A = dist_csr(m, off, r, comm, s)
        lo, hi = int(off[r]), int(off[r + 1])
        out = zk.solve(A, cuda(b[lo:hi]), tol=1e-8, method="bicgstab_l", ell=ell)
        out["x"] = out["x"].cpu().numpy()
        out["n_halo"] = A.info["n_halo"]
        return out

    res = run_ranks(nranks, fn)
    x = _check_ranks(res, nranks)
    refs = [oracle.bicgstab_l(m, b, tol=1e-8, ell=ell, order=o) for o in ORDERS]
    its = [q["iters"] for q in refs]
    r = res[0]
    assert r["status"] == "CONVERGED" and 0.95 * min(its) <= r["iters"] <= 1.05 * max(its), (r["iters"], its)
    k = min(6, r["iters"], refs[0]["iters"]) + 1
    assert np.max(np.abs(r["hist"][:k] - refs[0]["hist"][:k]) / refs[0]["hist"][:k]) <= HTOL[ell]
    assert relerr(x, refs[0]["x"]) <= 1e-6 and r["true_relres"] <= 1e-7


def test_local_c4_zslabs_two_ranks_vs_golden():
    """The bench's strong-scaling partition at full size: C4 (8M rows) split into 2 z-slabs of
    100 planes (one halo plane of 40,000 entries per rank, interior = every slice but the
    boundary plane's), BiCGStab through the LOCAL transport with the exchange overlapped, against
    the oracle's full C4 solves (tests/golden/c4_oracle.json): count within the L11 envelope of
    the three orders, 12-iteration history to 1e-10, x sample within 4x the orders' spread."""
    import json
    import os
    with open(os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "c4_oracle.json")) as f:
        G = json.load(f)
    spec = gen.CONFIGS["C4"]
    plane = spec.nx * spec.ny
    off = np.array([0, 100 * plane, 200 * plane], dtype=np.int64)
    idx = np.array(G["sample_idx"])

    def fn(r, comm, s):
        m = gen.make_matrix(spec, row_range=(off[r], off[r + 1]))
        b = gen.make_rhs(m)
        A = zk.csr_create(m["row_ptr"], m["col_idx"], m["values"], spec.n, comm=comm, row_begin=off[r], stream=s)
        del m
        out = zk.solve(A, cuda(b), tol=1e-8, maxit=1000, method="bicgstab")
        out["x"] = out["x"].cpu().numpy()
        out["info"] = A.info
        A.close()
        return out

    res = run_ranks(2, fn)
    for q in res:
        assert q["info"]["n_halo"] == plane and q["info"]["interior_rows"] >= 99 * plane - 32
        assert q["iters"] == res[0]["iters"] and np.array_equal(q["hist"], res[0]["hist"])
    r = res[0]
    its = [G["results"][f"bicgstab/{o}"]["iters"] for o in ("seq", "rev", "block256")]
    assert r["status"] == "CONVERGED" and 0.95 * min(its) <= r["iters"] <= 1.05 * max(its), (r["iters"], its)
    h0 = np.array(G["results"]["bicgstab/seq"]["hist"])
    assert np.max(np.abs(r["hist"][:13] - h0[:13]) / h0[:13]) <= 1e-10
    x = np.concatenate([q["x"] for q in res])[idx]

    def xs(g):
        return np.array(g["x_sample_re"]) + 1j * np.array(g["x_sample_im"])
    x0 = xs(G["results"]["bicgstab/seq"])
    spread = max(relerr(xs(G["results"][f"bicgstab/{o}"]), x0) for o in ("rev", "block256"))
    assert relerr(x, x0) <= 4 * spread


@pytest.mark.parametrize("nranks", [2, 4])
def test_local_jacobi_bicgstab(nranks):
    """The paper's P-Bi-CGSTAB (Jacobi right preconditioning, NEXT-1) on a row-partitioned matrix:
    the ranks exchange 1/a_jj of their halo columns once (dist_halo on dinv), then the distributed
    BiCGStab loop runs on A·M⁻¹; against oracle.bicgstab_jacobi's envelope, history and solution."""
    m = gen.make_matrix("C2")
    b = gen.make_rhs(m)
    res = _solve_ranks(m, b, offsets(m, nranks), nranks, "bicgstab_jacobi")
    x = _check_ranks(res, nranks)
    refs = [oracle.bicgstab_jacobi(m, b, tol=1e-8, order=o) for o in ORDERS]
    its = [q["iters"] for q in refs]
    r = res[0]
    assert r["status"] == "CONVERGED" and 0.95 * min(its) <= r["iters"] <= 1.05 * max(its), (r["iters"], its)
    k = min(12, r["iters"], refs[0]["iters"]) + 1
    assert np.max(np.abs(r["hist"][:k] - refs[0]["hist"][:k]) / refs[0]["hist"][:k]) <= 1e-10
    assert relerr(x, refs[0]["x"]) <= 1e-6 and r["true_relres"] <= 2e-8
