#!/usr/bin/env python
"""Why is the in-loop ZSpMV slower than the standalone one?  C4, one GPU.

Times (CUDA events, µs per launch): zk_zcsrmv alone; zk_zcsrmv after a 128 MB vector write
(dirty L2 lines, as in the solver loop); and BiCGStab's in-loop SpMV classes (device timers)
under each loop mode / PDL setting given.   python tools/inloop_probe.py [--modes 1,3]"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import gen  # noqa: E402
from paper_2112_11880_b200 import zk  # noqa: E402

p = argparse.ArgumentParser()
p.add_argument("--cfg", default="C4")
p.add_argument("--modes", default="")
p.add_argument("--reps", type=int, default=30)
a = p.parse_args()


def ev_time(fn, reps):
    for _ in range(3):
        fn()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return 1e3 * e0.elapsed_time(e1) / reps


m = gen.make_matrix(a.cfg)
n = m["n"]
A = zk.csr_create(m["row_ptr"], m["col_idx"], m["values"], n)
x = torch.from_numpy(gen.rand_vector(n, 1)).cuda()
y = torch.empty_like(x)
z = torch.empty_like(x)
w = torch.empty_like(x)
out = {}
out["spmv_alone_us"] = ev_time(lambda: zk.zcsrmv(A, 1.0, x, 0.0, y), a.reps)
out["copy_alone_us"] = ev_time(lambda: z.copy_(w), a.reps)


def pair():
    z.copy_(w)
    zk.zcsrmv(A, 1.0, x, 0.0, y)


out["copy_then_spmv_us"] = ev_time(pair, a.reps)


def pair2():
    x.mul_(1.0)  # x itself freshly written (dirty in L2), as p / s in the loop
    zk.zcsrmv(A, 1.0, x, 0.0, y)


out["scale_x_alone_us"] = ev_time(lambda: x.mul_(1.0), a.reps)
out["scale_x_then_spmv_us"] = ev_time(pair2, a.reps)
def seq(*fs):
    def run():
        for f in fs:
            f()
    return run


spmv = lambda: zk.zcsrmv(A, 1.0, x, 0.0, y)  # noqa: E731
nrm_x = lambda: zk.dznrm2(x)  # noqa: E731
nrm_w = lambda: zk.dznrm2(w)  # noqa: E731
scal_x = lambda: zk.zscal(1.0, x)  # noqa: E731
copy_xw = lambda: w.copy_(x)  # noqa: E731
for name, fs in [("nrm_x", [nrm_x]), ("nrm_w", [nrm_w]), ("scal_x", [scal_x]), ("copy_x_to_w", [copy_xw]),
                 ("scal_x+nrm_x", [scal_x, nrm_x]), ("scal_x+nrm_w", [scal_x, nrm_w])]:
    base = ev_time(seq(*fs), a.reps)
    out[f"{name}_alone_us"] = base
    out[f"spmv_after_{name}_us"] = ev_time(seq(*fs, spmv), a.reps) - base
b = torch.from_numpy(gen.make_rhs(m)).cuda()
ws = zk.alloc_workspace(A, "bicgstab", 2000)
for mode in [md for md in a.modes.split(",") if md]:
    for pdl in ("1", "0"):
        os.environ["ZK_LOOP_MODE"] = mode
        os.environ["ZK_PDL"] = pdl
        r = zk.solve(A, b, maxit=2000, method="bicgstab", workspace=ws)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        r = zk.solve(A, b, maxit=2000, method="bicgstab", workspace=ws)
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1)
        km = r["kernel_ms"]
        ln = r["kernel_launches"]
        out[f"solve_mode{mode}_pdl{pdl}"] = {"iters": r["iters"], "us_per_iter": 1e3 * ms / r["iters"],
                                            "class_us": [round(1e3 * k / max(l, 1), 1) for k, l in zip(km, ln)],
                                            "launches": ln}
out["spmv_alone_after_us"] = ev_time(lambda: zk.zcsrmv(A, 1.0, x, 0.0, y), a.reps)
print(json.dumps(out, indent=1))
