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

b = torch.from_numpy(gen.make_rhs(m)).pin_memory()
x_h = torch.empty(n, dtype=torch.complex128).pin_memory()
A0 = zk.csr_create(rp, ci, va, n)
ws = zk.alloc_workspace(A0, "bicgstab", 1000)
for step in range(3):
    t0 = time.perf_counter()
    A = zk.csr_create(rp, ci, va, n)
    torch.cuda.synchronize()
    t1 = time.perf_counter()
    bd = b.to("cuda", non_blocking=True)
    r = zk.solve(A, bd, None, 1e-8, 1000, "bicgstab", workspace=ws)
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    x_h.copy_(r["x"], non_blocking=True)
    torch.cuda.synchronize()
    t3 = time.perf_counter()
    A.close()
    torch.cuda.synchronize()
    t4 = time.perf_counter()
    print(f"step {step}: create {1e3*(t1-t0):.1f} ms, solve {1e3*(t2-t1):.1f} ms (device {r['solve_ms']:.1f}, "
          f"iters {r['iters']}, mode {r['loop_mode']}), x D2H {1e3*(t3-t2):.1f}, close {1e3*(t4-t3):.1f}", flush=True)

# the bench's e2e loop verbatim (non-default stream, no host syncs between steps)
stream = torch.cuda.Stream()
with torch.cuda.stream(stream):
    for reps in (2, 2):
        torch.cuda.synchronize()
        f0, f1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        t = time.perf_counter()
        f0.record(stream)
        for _ in range(reps):
            h0 = time.perf_counter()
            Ah = zk.csr_create(rp, ci, va, n, stream=stream)
            h1 = time.perf_counter()
            bd = b.to("cuda", non_blocking=True)
            re = zk.solve(Ah, bd, None, 1e-8, 1000, "bicgstab", workspace=ws, stream=stream)
            h2 = time.perf_counter()
            x_h.copy_(re["x"], non_blocking=True)
            Ah.close()
            h3 = time.perf_counter()
            print(f"  host: create {1e3*(h1-h0):.1f} solve {1e3*(h2-h1):.1f} (device {re['solve_ms']:.1f}) "
                  f"copy+close {1e3*(h3-h2):.1f} ms", flush=True)
        f1.record(stream)
        torch.cuda.synchronize()
        print(f"bench-style e2e: {f0.elapsed_time(f1) / reps:.1f} ms/step (events), "
              f"{(time.perf_counter() - t) * 1e3 / reps:.1f} ms/step (wall), last solve: mode {re['loop_mode']} "
              f"iters {re['iters']} device {re['solve_ms']:.1f} ms", flush=True)
