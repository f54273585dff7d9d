"""Time one libzk build (env ZK_LIB, default the in-tree libzk.so): standalone zk_zcsrmv and the
BiCGStab / CG / TFQMR solves (WHILE graph) on the given configs, CUDA events, medians.
Usage: ZK_LIB=... python tools/ab_lib.py C3 C4"""
import os
import statistics
import sys

sys.path.insert(0, os.getcwd())
import numpy as np  # noqa: E402
import torch  # noqa: E402

import gen  # noqa: E402
from paper_2112_11880_b200 import zk  # noqa: E402

tag = os.path.basename(os.environ.get("ZK_LIB", "libzk.so"))


def med(fn, reps):
    ts = []
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        out = fn()
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    return statistics.median(ts), out


for cfg in sys.argv[1:] or ["C3"]:
    m = gen.make_matrix(cfg)
    A = zk.csr_create(torch.from_numpy(m["row_ptr"]).cuda(), torch.from_numpy(m["col_idx"]).cuda(),
                      torch.from_numpy(m["values"]).cuda(), m["n"])
    b = torch.from_numpy(gen.make_rhs(m)).cuda()
    y = torch.empty_like(b)
    zk.zcsrmv(A, 1, b, 0, y)
    t, _ = med(lambda: zk.zcsrmv(A, 1, b, 0, y), 20)
    res = [f"zcsrmv {1e3 * t:7.1f} us"]
    mg = gen.make_matrix(cfg, eta=0.0, twist_seed=gen.SEED_TWIST)
    Ag = zk.csr_create(torch.from_numpy(mg["row_ptr"]).cuda(), torch.from_numpy(mg["col_idx"]).cuda(),
                       torch.from_numpy(mg["values"]).cuda(), mg["n"])
    bg = torch.from_numpy(np.exp(1j * mg["phase"]) * gen.make_rhs(mg)).cuda()
    del m, mg
    for meth in os.environ.get("AB_METHODS", "bicgstab,cg,tfqmr").split(","):
        AA, bb = (Ag, bg) if meth == "cg" else (A, b)
        ws = zk.alloc_workspace(AA, meth, 2000)
        zk.solve(AA, bb, tol=1e-8, maxit=2000, method=meth, workspace=ws)
        t, r = med(lambda: zk.solve(AA, bb, tol=1e-8, maxit=2000, method=meth, workspace=ws), 5)
        res.append(f"{meth} {1e3 * t / r['iters']:7.1f} us/it ({r['iters']})")
    print(tag, cfg, " | ".join(res), flush=True)
    A.close()
    Ag.close()
