"""A/B of the split-schedule variants on one GPU: ms per iteration of BiCGStab / CG / TFQMR on the
given configs under ZK_SPLIT_TAIL=0 (separate reduction pass) and =1 (reduction in the SpMV kernel's
tail), WHILE-graph loop, CUDA events, median of 5 solves.  Usage: python tools/ab_split.py C3 C4"""
import os
import statistics
import sys

sys.path.insert(0, os.getcwd())
import numpy as np  # noqa: E402
import torch  # noqa: E402

import gen  # noqa: E402
from paper_2112_11880_b200 import zk  # noqa: E402


def timed(A, b, meth, reps=5):
    ws = zk.alloc_workspace(A, meth, 2000)
    r = zk.solve(A, b, tol=1e-8, maxit=2000, method=meth, workspace=ws)
    ts = []
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        r = zk.solve(A, b, tol=1e-8, maxit=2000, method=meth, workspace=ws)
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    return statistics.median(ts) / r["iters"], r["iters"], r["hist"][-1]


for cfg in sys.argv[1:] or ["C3"]:
    m = gen.make_matrix(cfg)
    A = zk.csr_create(torch.from_numpy(m["row_ptr"]).cuda(), torch.from_numpy(m["col_idx"]).cuda(),
                      torch.from_numpy(m["values"]).cuda(), m["n"])
    b = torch.from_numpy(gen.make_rhs(m)).cuda()
    mg = gen.make_matrix(cfg, eta=0.0, twist_seed=gen.SEED_TWIST)
    Ag = zk.csr_create(torch.from_numpy(mg["row_ptr"]).cuda(), torch.from_numpy(mg["col_idx"]).cuda(),
                       torch.from_numpy(mg["values"]).cuda(), mg["n"])
    bg = torch.from_numpy(np.exp(1j * mg["phase"]) * gen.make_rhs(mg)).cuda()
    del m, mg
    for meth in ("bicgstab", "cg", "tfqmr"):
        row = []
        for tail in os.environ.get("AB_TAILS", "0,1").split(","):
            os.environ["ZK_SPLIT_TAIL"] = tail
            AA, bb = (Ag, bg) if meth == "cg" else (A, b)
            ms, it, h = timed(AA, bb, meth)
            row.append(f"tail={tail}: {1e3 * ms:8.1f} us/iter ({it} it, {h:.2e})")
        print(cfg, f"{meth:9s}", " | ".join(row), flush=True)
    A.close()
    Ag.close()
