#!/usr/bin/env python
"""Kernel microbenchmarks on one GPU (CUDA events on the launching stream, inputs > L2).

  python tools/microbench.py spmv   [--config C4] [--ws 4,8,16,32] [--reps 50]
  python tools/microbench.py blas1  [--n 268435456]
  python tools/microbench.py ncu-spmv [--config C4]     (few launches, for ncu --set full)

Prints one JSON object per measurement.  Counted bytes follow paper_2112_11880_b200/metrics.py.
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import gen  # noqa: E402
from paper_2112_11880_b200 import metrics as M  # noqa: E402
from paper_2112_11880_b200 import zk  # noqa: E402


def timeit(fn, reps, warm=3):
    for _ in range(warm):
        fn()
    s = torch.cuda.current_stream()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    a.record(s)
    for _ in range(reps):
        fn()
    b.record(s)
    torch.cuda.synchronize()
    return 1e3 * a.elapsed_time(b) / reps  # µs


def load_matrix(cfg):
    m = gen.make_matrix(cfg)
    d = "cuda"
    return m, torch.from_numpy(m["row_ptr"]).to(d), torch.from_numpy(m["col_idx"]).to(d), torch.from_numpy(m["values"]).to(d)


def spmv(a):
    m, rp, ci, va = load_matrix(a.config)
    n, nnz = m["n"], m["nnz"]
    x = torch.from_numpy(gen.rand_vector(n, 1)).cuda()
    y = torch.empty_like(x)
    for spec in a.maps.split(","):                      # mode:W  (mode 0 CSR sub-warp, 3 SELL-32)
        f = spec.split(":")
        os.environ.update({"ZK_SPMV_MODE": f[0], "ZK_SPMV_W": f[1]})
        A = zk.csr_create(rp, ci, va, n, borrow=True)
        us = timeit(lambda: zk.zcsrmv(A, 1.0, x, a.beta, y), a.reps)
        gbs = M.spmv_bytes(n, nnz, a.beta != 0) / (us * 1e-6) / 1e9
        print(json.dumps({"kernel": "zcsrmv", "config": a.config, "map": spec, "info": A.info, "us": us,
                          "gbs": gbs, "gflops": M.spmv_flops(nnz) / (us * 1e-6) / 1e9}), flush=True)
        A.close()


def blas1(a):
    n = a.n
    x = torch.ones(n, dtype=torch.complex128, device="cuda")
    y = torch.ones(n, dtype=torch.complex128, device="cuda")
    z = torch.empty(n, dtype=torch.complex128, device="cuda")
    for name, fn, byts in [
        ("dznrm2 (read-only stream)", lambda: zk.dznrm2(x), 16 * n),
        ("zdotc", lambda: zk.zdotc(x, y), 32 * n),
        ("zaxpy", lambda: zk.zaxpy(1e-30, x, y), 48 * n),
        ("zscal", lambda: zk.zscal(1.0, y), 32 * n),
        ("torch copy (reference)", lambda: z.copy_(x), 32 * n),
    ]:
        us = timeit(fn, a.reps)
        print(json.dumps({"kernel": name, "n": n, "us": us, "gbs": byts / (us * 1e-6) / 1e9}), flush=True)


def ncu_spmv(a):
    m, rp, ci, va = load_matrix(a.config)
    n = m["n"]
    if a.maps.count(",") == 0:
        f = a.maps.split(":")
        os.environ.update({"ZK_SPMV_MODE": f[0], "ZK_SPMV_W": f[1]})
    A = zk.csr_create(rp, ci, va, n, borrow=True)
    x = torch.from_numpy(gen.rand_vector(n, 1)).cuda()
    y = torch.empty_like(x)
    for _ in range(4):
        zk.zcsrmv(A, 1.0, x, 0.0, y)
    torch.cuda.synchronize()


def solve(a):
    """One BiCGStab solve of the config (for the ncu launch list run it with ZK_LOOP_MODE=3:
    ncu cannot profile kernel nodes inside graphs that contain conditional nodes)."""
    m, rp, ci, va = load_matrix(a.config)
    A = zk.csr_create(rp, ci, va, m["n"], borrow=True)
    b = torch.from_numpy(gen.make_rhs(m)).cuda()
    r = zk.solve(A, b, tol=1e-8, maxit=2000)
    print(json.dumps({k: v for k, v in r.items() if k not in ("x", "hist")}), flush=True)


if __name__ == "__main__":
    p = argparse.ArgumentParser()
    p.add_argument("what", choices=["spmv", "blas1", "ncu-spmv", "solve"])
    p.add_argument("--config", default="C4")
    p.add_argument("--maps", default="0:4,0:8,3:32")
    p.add_argument("--reps", type=int, default=50)
    p.add_argument("--beta", type=float, default=0.0)
    p.add_argument("--n", type=int, default=1 << 28)
    a = p.parse_args()
    {"spmv": spmv, "blas1": blas1, "ncu-spmv": ncu_spmv, "solve": solve}[a.what](a)
