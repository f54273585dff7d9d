#!/usr/bin/env python
"""Per-iteration time of the solver loop modes on the paper's shapes (and C4):
   python tools/loopmodes.py [--cfgs C1,C2,C3] [--modes 1,4] [--method tfqmr|bicgstab_l --ell 8]"""
import argparse, json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import gen
from paper_2112_11880_b200 import zk

p = argparse.ArgumentParser()
p.add_argument("--cfgs", default="C1,C2,C3")
p.add_argument("--modes", default="1,4")
p.add_argument("--method", default="bicgstab")
p.add_argument("--ell", type=int, default=8)
a = p.parse_args()
for cfg in a.cfgs.split(","):
    m = gen.make_matrix(cfg)
    A = zk.csr_create(m["row_ptr"], m["col_idx"], m["values"], m["n"])
    b = torch.from_numpy(gen.make_rhs(m)).cuda()
    ws = zk.alloc_workspace(A, a.method, 2000, ell=a.ell)
    for mode in a.modes.split(","):
        os.environ["ZK_LOOP_MODE"] = mode
        for _ in range(2):
            r = zk.solve(A, b, maxit=2000, method=a.method, workspace=ws, ell=a.ell)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(5):
            r = zk.solve(A, b, maxit=2000, method=a.method, workspace=ws, ell=a.ell)
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / 5
        print(json.dumps({"cfg": cfg, "mode": r["loop_mode"], "iters": r["iters"], "ms": round(ms, 4),
                          "us_per_iter": round(1e3 * ms / r["iters"], 2), "kernel_ms": [round(v, 3) for v in r["kernel_ms"]],
                          "launches": r["kernel_launches"]}), flush=True)
