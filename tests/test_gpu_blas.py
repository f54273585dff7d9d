"""GPU parity of ZSpMV and BLAS-1 (libzk through the C-ABI) against the CPU oracle.

Tolerances (north star): SpMV and axpy elementwise relative 1e-13, read
as |Δy_i| ≤ 1e-13·Σ_j|a_ij||x_j| (the row's absolute scale); dot and norm relative 1e-12,
|Δ| ≤ 1e-12·‖x‖‖y‖.  Integer-exact inputs and exact scalars must match bitwise."""
import os

import numpy as np
import pytest
import scipy.sparse as sp
import torch

import gen
import oracle
from paper_2112_11880_b200 import zk
from tests import closed_form as cf

pytestmark = pytest.mark.gpu
DEV = "cuda:0"


def cuda(a):
    return torch.from_numpy(np.ascontiguousarray(a)).to(DEV)


def row_scale(m, x):
    n = len(m["row_ptr"]) - 1
    A = sp.csr_matrix((np.abs(m["values"]), m["col_idx"], m["row_ptr"]), shape=(n, m.get("n_cols", m["n"])))
    return A @ np.abs(x)


MAPPINGS = [(0, 2, None), (0, 4, None), (0, 8, None), (0, 16, None), (0, 32, None), (3, 32, None)]
MAP_NAMES = {0: "subwarp", 3: "sell32"}
MAP_IDS = [f"{MAP_NAMES[m]}-W{w}" for m, w, c in MAPPINGS]


def make_csr(m, W=None, mode=None, tma=None, **kw):
    """csr_create with the SpMV mapping forced through the env overrides read at create."""
    env = {}
    if W is not None:
        env["ZK_SPMV_W"] = str(W)
    if mode is not None:
        env["ZK_SPMV_MODE"] = str(mode)
    old = {k: os.environ.get(k) for k in env}
    os.environ.update(env)
    try:
        return zk.csr_create(m["row_ptr"], m["col_idx"], m["values"], m.get("n_cols", m["n"]), **kw)
    finally:
        for k, v in old.items():
            if v is None:
                del os.environ[k]
            else:
                os.environ[k] = v


# ------------------------------------------------------------------ ZSpMV
@pytest.mark.parametrize("mapping", MAPPINGS, ids=MAP_IDS)
@pytest.mark.parametrize("alpha,beta", [(1, 0), (0.5 - 2j, 0), (1j, -0.25 + 1j)])
def test_zcsrmv_random(mapping, alpha, beta):
    """Random CSR with empty rows, 1-nnz rows and rows > 32 nnz; ragged n spanning many tiles."""
    mode, W, tma = mapping
    m = gen.random_csr(5003, seed=W + 10 * mode, max_len=70)
    x, y0 = gen.rand_vector(5003, 1), gen.rand_vector(5003, 2)
    A = make_csr(m, W, mode, tma)
    assert A.info["lanes_per_row"] == W and A.info["spmv_mode"] == mode
    y = cuda(y0)
    zk.zcsrmv(A, alpha, cuda(x), beta, y)
    want = oracle.zcsrmv(m, x, alpha, beta, y0)
    tol = 1e-13 * (abs(alpha) * row_scale(m, x) + abs(beta) * np.abs(y0)) + 1e-300
    assert np.all(np.abs(y.cpu().numpy() - want) <= tol)


@pytest.mark.parametrize("mapping", MAPPINGS, ids=MAP_IDS)
def test_zcsrmv_integer_exact_bitwise(mapping):
    mode, W, tma = mapping
    m = gen.random_csr(3001, seed=11, max_len=40, integer=True)
    x = gen.int_vector(3001, 3)
    A = make_csr(m, W, mode, tma)
    y = torch.empty(3001, dtype=torch.complex128, device=DEV)
    zk.zcsrmv(A, 1, cuda(x), 0, y)
    assert np.array_equal(y.cpu().numpy(), oracle.zcsrmv(m, x))


def test_zcsrmv_beta_zero_ignores_nan_and_empty_rows():
    m = gen.random_csr(777, seed=5)
    x = gen.rand_vector(777, 1)
    y = torch.full((777,), complex(np.nan, np.nan), dtype=torch.complex128, device=DEV)
    zk.zcsrmv(make_csr(m), 1, cuda(x), 0, y)
    got = y.cpu().numpy()
    assert np.all(np.isfinite(got))
    assert np.all(got[np.diff(m["row_ptr"]) == 0] == 0)


@pytest.mark.parametrize("mode", [0, 3])
@pytest.mark.parametrize("cfg", ["C1", "C2", "C3", "C3T"])
def test_zcsrmv_paper_shapes(cfg, mode):
    m = gen.make_matrix(cfg)
    x = gen.rand_vector(m["n"], 7)
    A = make_csr(m, mode=mode)
    y = torch.empty(m["n"], dtype=torch.complex128, device=DEV)
    zk.zcsrmv(A, 1, cuda(x), 0, y)
    got = y.cpu().numpy()
    want = oracle.zcsrmv(m, x)
    assert np.all(np.abs(got - want) <= 1e-13 * row_scale(m, x) + 1e-300)
    ident = m["free_mask"] == 0                                  # identity rows exact (pin (3))
    assert np.array_equal(got[ident], want[ident])


@pytest.mark.parametrize("mode", ["0", "3"])
def test_zcsrmv_c4_full_size_sampled(mode, monkeypatch):
    """C4 (8M rows, 214M nnz) in the bench's launch configuration: sampled rows against the
    oracle computed row by row, and the closed-form eigenvector identity A·v = λ·v on all rows."""
    monkeypatch.setenv("ZK_SPMV_MODE", mode)
    spec = gen.CONFIGS["C4"]
    m = gen.make_matrix(spec)
    n = m["n"]
    A = zk.csr_create(cuda(m["row_ptr"]), cuda(m["col_idx"]), cuda(m["values"]), n, borrow=False)
    x = gen.rand_vector(n, 9)
    y = torch.empty(n, dtype=torch.complex128, device=DEV)
    zk.zcsrmv(A, 1, cuda(x), 0, y)
    got = y.cpu().numpy()
    # 4000 seeded rows spread over the whole matrix (+ the first, middle and last rows), checked
    # in ONE oracle call on the sub-CSR of exactly those rows (same entries, same stored order)
    rows = np.unique(np.concatenate([np.random.default_rng(0).integers(0, n, 4000), [0, 1, n // 2, n - 2, n - 1]]))
    assert rows.max() == n - 1 and (rows > n // 2).sum() > 1500        # not biased to the first rows
    rp = m["row_ptr"]
    lens = rp[rows + 1] - rp[rows]
    take = np.concatenate([np.arange(rp[i], rp[i + 1]) for i in rows])
    sub = dict(row_ptr=np.concatenate([[0], np.cumsum(lens)]).astype(np.int64), col_idx=m["col_idx"][take],
               values=m["values"][take], n=n)
    want = oracle.zcsrmv(sub, x)
    scale = np.add.reduceat(np.abs(sub["values"]) * np.abs(x[sub["col_idx"]]), sub["row_ptr"][:-1])
    assert np.all(np.abs(got[rows] - want) <= 1e-13 * scale)
    lam = cf.box_eigs(spec, gen.ETA)
    v = cf.sine_mode(spec, 2, 5, 199)
    zk.zcsrmv(A, 1, cuda(v), 0, y)
    err = np.abs(y.cpu().numpy() - lam[198, 4, 1] * v)
    assert np.all(err <= 1e-13 * row_scale(m, v) + 1e-300)


def test_zcsrmv_errors():
    m = gen.random_csr(50, seed=1)
    A = make_csr(m)
    x = cuda(gen.rand_vector(50, 1))
    with pytest.raises(zk.ZkError) as e:
        zk.zcsrmv(A, 1, x, 0, x)
    assert e.value.code == -7                                     # ZK_ERR_ALIAS


@pytest.mark.parametrize("where", ["host", "device"])
def test_csr_create_validation(where):
    m = gen.random_csr(200, seed=2)
    conv = (lambda a: a) if where == "host" else cuda
    bad = m["col_idx"].copy()
    r = int(np.argmax(np.diff(m["row_ptr"]) > 3))
    p = m["row_ptr"][r]
    bad[p], bad[p + 1] = bad[p + 1], bad[p]                      # unsorted row r
    with pytest.raises(zk.ZkError) as e:
        zk.csr_create(conv(m["row_ptr"]), conv(bad), conv(m["values"]), 200)
    assert e.value.code == -2 and f"row {r}" in str(e.value)
    bad = m["col_idx"].copy()
    bad[5] = 200                                                  # out of range
    with pytest.raises(zk.ZkError) as e:
        zk.csr_create(conv(m["row_ptr"]), conv(bad), conv(m["values"]), 200)
    assert e.value.code == -2
    v = m["values"].copy()
    v[3] = np.inf
    with pytest.raises(zk.ZkError) as e:
        zk.csr_create(conv(m["row_ptr"]), conv(m["col_idx"]), conv(v), 200)
    assert e.value.code == -3
    rp = m["row_ptr"].copy()
    rp[-1] += 1
    with pytest.raises(zk.ZkError):
        zk.csr_create(conv(rp), conv(m["col_idx"]), conv(m["values"]), 200)


def test_csr_borrow_and_empty():
    m = gen.random_csr(300, seed=3)
    rp, ci, va = cuda(m["row_ptr"]), cuda(m["col_idx"]), cuda(m["values"])
    A = zk.csr_create(rp, ci, va, 300, borrow=True)
    assert A.info["borrowed"] == 1
    x = gen.rand_vector(300, 4)
    y = torch.empty(300, dtype=torch.complex128, device=DEV)
    zk.zcsrmv(A, 1, cuda(x), 0, y)
    assert np.all(np.abs(y.cpu().numpy() - oracle.zcsrmv(m, x)) <= 1e-13 * row_scale(m, x) + 1e-300)
    E = zk.csr_create(np.zeros(1, np.int64), np.zeros(0, np.int32), np.zeros(0, np.complex128), 0)
    assert E.n_rows == 0


# ------------------------------------------------------------------ zdotc / dznrm2
@pytest.mark.parametrize("n", [1, 7, 1000, 1 << 20, (1 << 22) + 13])
def test_zdotc_dznrm2_random(n):
    x, y = gen.rand_vector(n, 1), gen.rand_vector(n, 2)
    X, Y = cuda(x), cuda(y)
    d = zk.zdotc(X, Y).cpu().numpy()[0]
    ref = oracle.zdotc(x, y)
    nx, ny = oracle.dznrm2(x), oracle.dznrm2(y)
    assert abs(d - ref) <= 1e-12 * nx * ny
    nr = zk.dznrm2(X).cpu().numpy()[0]
    assert abs(nr - nx) <= 1e-12 * nx
    # non-cancelling inputs: literally relative 1e-12 (L5)
    xp, yp = np.abs(x.real) + 1j * np.abs(x.imag), np.abs(y.real) + 1j * np.abs(y.imag)
    d = zk.zdotc(cuda(xp), cuda(yp)).cpu().numpy()[0]
    ref = oracle.zdotc(xp, yp)
    assert abs(d.real - ref.real) <= 1e-12 * abs(ref.real)


def test_dot_norm_exact_and_deterministic():
    one_i = cuda(np.array([1j]))
    assert zk.zdotc(one_i, one_i).cpu().numpy()[0] == 1 + 0j       # conj first
    assert zk.dznrm2(cuda(np.array([3 + 4j]))).cpu().numpy()[0] == 5.0
    n = 3_000_017
    x, y = gen.int_vector(n, 1, -90, 90), gen.int_vector(n, 2, -90, 90)
    X, Y = cuda(x), cuda(y)
    d = zk.zdotc(X, Y).cpu().numpy()[0]
    assert d == oracle.zdotc(x, y, oracle.ORD_SEQ)                  # exact integer sums: bitwise
    assert zk.dznrm2(X).cpu().numpy()[0] == oracle.dznrm2(x, oracle.ORD_SEQ)
    # determinism: fixed grid + fixed-order last-block finish
    r = gen.rand_vector(n, 5)
    R = cuda(r)
    vals = {complex(zk.zdotc(R, Y).cpu().numpy()[0]) for _ in range(5)}
    assert len(vals) == 1
    # conjugate symmetry and ‖x‖² = Re⟨x,x⟩
    assert abs(zk.zdotc(Y, R).cpu().numpy()[0] - np.conj(zk.zdotc(R, Y).cpu().numpy()[0])) <= 1e-13 * n
    e = zk.zdotc(torch.empty(0, dtype=torch.complex128, device=DEV), torch.empty(0, dtype=torch.complex128, device=DEV))
    assert e.cpu().numpy()[0] == 0


# ------------------------------------------------------------------ zaxpy / zscal
@pytest.mark.parametrize("n", [1, 1023, 1 << 20, 5_000_011])
def test_zaxpy_zscal_random(n):
    x, y = gen.rand_vector(n, 3), gen.rand_vector(n, 4)
    a = 0.3 - 1.7j
    Y = cuda(y)
    zk.zaxpy(a, cuda(x), Y)
    want = oracle.zaxpy(a, x, y)
    assert np.all(np.abs(Y.cpu().numpy() - want) <= 1e-13 * (abs(a) * np.abs(x) + np.abs(y)))
    X = cuda(x)
    zk.zscal(a, X)
    assert np.all(np.abs(X.cpu().numpy() - oracle.zscal(a, x)) <= 1e-13 * abs(a) * np.abs(x))


def test_zaxpy_zscal_exact_alphas():
    x, y = gen.rand_vector(100_003, 3), gen.rand_vector(100_003, 4)
    for a in (0, 1, -1, 1j, 0.25, -8):
        Y = cuda(y)
        zk.zaxpy(a, cuda(x), Y)
        assert np.array_equal(Y.cpu().numpy(), oracle.zaxpy(a, x, y)), a
        X = cuda(x)
        zk.zscal(a, X)
        assert np.array_equal(X.cpu().numpy(), oracle.zscal(a, x)), a
    xi, yi = gen.int_vector(50_000, 5), gen.int_vector(50_000, 6)
    Y = cuda(yi)
    zk.zaxpy(3 - 2j, cuda(xi), Y)
    assert np.array_equal(Y.cpu().numpy(), oracle.zaxpy(3 - 2j, xi, yi))


# ------------------------------------------------------------------ ZASSIGN / ZAXMY (NEXT-4)
def test_zassign_zaxmy():
    x = torch.empty(1_000_003, dtype=torch.complex128, device=DEV)
    zk.zassign(1.5 - 2j, x)
    assert np.array_equal(x.cpu().numpy(), oracle.zassign(1_000_003, 1.5 - 2j))
    a, b = gen.rand_vector(1 << 20, 1), gen.rand_vector(1 << 20, 2)
    Y = cuda(b)
    zk.zaxmy(cuda(a), Y)
    want = oracle.zaxmy(a, b)
    assert np.all(np.abs(Y.cpu().numpy() - want) <= 1e-15 * np.abs(a) * np.abs(b))
    ai, bi = gen.int_vector(100_001, 3), gen.int_vector(100_001, 4)
    Y = cuda(bi)
    zk.zaxmy(cuda(ai), Y)
    assert np.array_equal(Y.cpu().numpy(), oracle.zaxmy(ai, bi))    # integer-exact: bitwise
    one_i = cuda(np.array([1j]))
    zk.zaxmy(one_i, one_i)
    assert one_i.cpu().numpy()[0] == -1


def test_sell_default_and_padding_fallback(monkeypatch):
    """The sliced-ELL copy is the default for regular FE rows (C2: 6.5 % padding) and is dropped
    for irregular rows (random lengths 0-70: padding far above 10 %), falling back to the CSR
    sub-warp kernel; both give the oracle's product."""
    monkeypatch.delenv("ZK_SPMV_MODE", raising=False)
    m = gen.make_matrix("C2")
    A = zk.csr_create(m["row_ptr"], m["col_idx"], m["values"], m["n"])
    assert A.info["spmv_mode"] == 3 and m["nnz"] <= A.info["sell_entries"] <= 1.1 * m["nnz"]
    r = gen.random_csr(4099, seed=5, max_len=70)
    B = zk.csr_create(r["row_ptr"], r["col_idx"], r["values"], 4099)
    assert B.info["spmv_mode"] == 0 and B.info["sell_entries"] == 0
    for mat, M in ((m, A), (r, B)):
        x = gen.rand_vector(mat["n"], 4)
        y = torch.empty(mat["n"], dtype=torch.complex128, device=DEV)
        zk.zcsrmv(M, 1, cuda(x), 0, y)
        assert np.all(np.abs(y.cpu().numpy() - oracle.zcsrmv(mat, x)) <= 1e-13 * row_scale(mat, x) + 1e-300)


@pytest.mark.parametrize("mode", ["0", "3"])
def test_zcsrmv_irregular_rows_stress(mode, monkeypatch):
    """NEXT-4: Twingo-like irregular rows (2 % of the rows of the Twingo3D-0 shape grown to 39 entries)
    through the CSR sub-warp kernel and the (heavily padded, forced) sliced-ELL kernel."""
    monkeypatch.setenv("ZK_SPMV_MODE", mode)
    m = gen.add_long_rows(gen.make_matrix("T0"))
    A = zk.csr_create(m["row_ptr"], m["col_idx"], m["values"], m["n"])
    assert A.info["spmv_mode"] == int(mode) and A.info["max_row_len"] == 39
    x = gen.rand_vector(m["n"], 8)
    y = torch.empty(m["n"], dtype=torch.complex128, device=DEV)
    zk.zcsrmv(A, 1, cuda(x), 0, y)
    assert np.all(np.abs(y.cpu().numpy() - oracle.zcsrmv(m, x)) <= 1e-13 * row_scale(m, x) + 1e-300)


def test_handle_memory_reused_across_create_destroy():
    """Per-handle device arrays come from the stream-ordered pool (zk_host.h dev_alloc): creating
    and destroying the same-size handle repeatedly must not grow device memory use."""
    m = gen.make_matrix("C2")
    torch.cuda.synchronize()
    A = zk.csr_create(m["row_ptr"], m["col_idx"], m["values"], m["n"])
    A.close()
    free0, _ = torch.cuda.mem_get_info()
    for _ in range(20):
        A = zk.csr_create(m["row_ptr"], m["col_idx"], m["values"], m["n"])
        A.close()
    free1, _ = torch.cuda.mem_get_info()
    assert free0 - free1 <= 64 << 20, (free0, free1)


def test_plain_cudamalloc_path_subprocess():
    """ZK_POOL=0 (plain cudaMalloc/cudaFree) in a fresh process: create, SpMV against the oracle,
    a solve, destroy."""
    import subprocess
    import sys
    import os
    code = (
        "import numpy as np, torch, gen, oracle\n"
        "from paper_2112_11880_b200 import zk\n"
        "m = gen.make_matrix('C1'); x = gen.rand_vector(m['n'], 1)\n"
        "A = zk.csr_create(m['row_ptr'], m['col_idx'], m['values'], m['n'])\n"
        "y = torch.empty(m['n'], dtype=torch.complex128, device='cuda')\n"
        "zk.zcsrmv(A, 1.0, torch.from_numpy(x).cuda(), 0.0, y)\n"
        "ref = oracle.zcsrmv(m, x)\n"
        "assert np.max(np.abs(y.cpu().numpy() - ref)) <= 1e-13 * np.abs(ref).max()\n"
        "r = zk.solve(A, torch.from_numpy(gen.make_rhs(m)).cuda(), tol=1e-8)\n"
        "assert r['status'] == 'CONVERGED'\n"
        "A.close(); print('ok')\n")
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = dict(os.environ, ZK_POOL="0", PYTHONPATH=root)
    out = subprocess.run([sys.executable, "-c", code], env=env, cwd=root, capture_output=True, text=True, timeout=600)
    assert out.returncode == 0 and out.stdout.strip().endswith("ok"), out.stderr[-2000:]


@pytest.mark.parametrize("where", ["host", "device", "borrow"])
def test_csr_update_values_frequency_sweep(where):
    """zk_csr_update_values: same pattern, new values — the C2 mesh at another
    wavelength (a Helmholtz frequency sweep, §2).  The SELL copy is refilled and the
    Jacobi cache rebuilt: SpMV and Jacobi-BiCGStab match the oracle on the NEW matrix."""
    m1 = gen.make_matrix("C2")
    m2 = gen.make_matrix("C2", k=2 * np.pi / 2.5)
    assert np.array_equal(m1["col_idx"], m2["col_idx"]) and not np.array_equal(m1["values"], m2["values"])
    b = gen.make_rhs(m1)
    x = gen.rand_vector(m1["n"], 6)
    if where == "borrow":
        vals = cuda(m1["values"])
        A = zk.csr_create(cuda(m1["row_ptr"]), cuda(m1["col_idx"]), vals, m1["n"], borrow=True)
    else:
        A = zk.csr_create(m1["row_ptr"], m1["col_idx"], m1["values"], m1["n"])
    y = torch.empty(m1["n"], dtype=torch.complex128, device=DEV)
    r1 = zk.solve(A, cuda(b), method="bicgstab_jacobi")                # builds the Jacobi cache of m1
    assert r1["status"] == "CONVERGED"
    if where == "borrow":
        vals.copy_(cuda(m2["values"]))
        A.update_values(None)
    else:
        A.update_values(m2["values"] if where == "host" else cuda(m2["values"]))
    zk.zcsrmv(A, 1, cuda(x), 0, y)
    assert np.all(np.abs(y.cpu().numpy() - oracle.zcsrmv(m2, x)) <= 1e-13 * row_scale(m2, x) + 1e-300)
    r2 = zk.solve(A, cuda(b), method="bicgstab_jacobi")
    ref = oracle.bicgstab_jacobi(m2, b)
    assert r2["status"] == ref["status"] == "CONVERGED"
    assert np.linalg.norm(r2["x"].cpu().numpy() - ref["x"]) <= 1e-6 * np.linalg.norm(ref["x"])
    bad = m2["values"].copy()
    bad[17] = np.nan
    if where != "borrow":
        with pytest.raises(zk.ZkError) as e:
            A.update_values(bad)
        assert e.value.code == -3 and "value 17" in str(e.value)
