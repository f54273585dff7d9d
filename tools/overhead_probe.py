#!/usr/bin/env python
"""Fixed cost of one zk_solve on a tiny system: host wall time of the Python call vs the device
time between the solve's first and last enqueued work (info.solve_ms).  python tools/overhead_probe.py"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import gen  # noqa: E402
from paper_2112_11880_b200 import zk  # noqa: E402

for cfg in ("C1",):
    m = gen.make_matrix(cfg)
    A = zk.csr_create(m["row_ptr"], m["col_idx"], m["values"], m["n"])
    b = torch.from_numpy(gen.make_rhs(m)).cuda()
    for method in ("bicgstab", "cocg"):
        ws = zk.alloc_workspace(A, method, 64)
        x = torch.empty_like(b)
        for maxit in (1, 16):
            for _ in range(5):
                r = zk.solve(A, b, tol=1e-300, maxit=maxit, method=method, workspace=ws, x=x)
            torch.cuda.synchronize()
            t = time.perf_counter()
            N = 50
            dev = 0.0
            for _ in range(N):
                r = zk.solve(A, b, tol=1e-300, maxit=maxit, method=method, workspace=ws, x=x)
                dev += r["solve_ms"]
            wall = (time.perf_counter() - t) / N * 1e6
            print(f"{cfg} {method} maxit={maxit}: wall {wall:.1f} us, device (ev0->ev1) {1e3 * dev / N:.1f} us, "
                  f"mode {r['loop_mode']}", flush=True)
