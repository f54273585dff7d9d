#!/usr/bin/env python
"""Where the end-to-end C4 step goes: pinned H2D of the CSR arrays alone (torch), zk_csr_create
from pinned host arrays, zk_csr_destroy, and the solve.   python tools/e2e_probe.py"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import gen  # noqa: E402
from paper_2112_11880_b200 import zk  # noqa: E402

m = gen.make_matrix("C4")
n = m["n"]
rp = torch.from_numpy(m["row_ptr"]).pin_memory()
ci = torch.from_numpy(m["col_idx"]).pin_memory()
va = torch.from_numpy(m["values"]).pin_memory()
s = torch.cuda.current_stream()


def ev(fn, reps=2):
    fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t = time.perf_counter()
    a.record()
    for _ in range(reps):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / reps, (time.perf_counter() - t) * 1e3 / reps


d_rp = torch.empty_like(rp, device="cuda")
d_ci = torch.empty_like(ci, device="cuda")
d_va = torch.empty_like(va, device="cuda")


def h2d():
    d_rp.copy_(rp, non_blocking=True)
    d_ci.copy_(ci, non_blocking=True)
    d_va.copy_(va, non_blocking=True)


print("h2d only (ms dev, ms wall):", ev(h2d))


def create_close():
    A = zk.csr_create(rp, ci, va, n)
    A.close()


print("csr_create+close from pinned host:", ev(create_close))


def create_borrow_close():
    h2d()
    A = zk.csr_create(d_rp, d_ci, d_va, n, borrow=True)
    A.close()


print("h2d + csr_create(borrow)+close:", ev(create_borrow_close))
