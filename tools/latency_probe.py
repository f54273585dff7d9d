#!/usr/bin/env python
"""Fixed per-solve cost vs per-iteration cost on the latency-bound paper shapes:
   time zk_solve (CUDA events, mean of 20) at maxit = 1, 2, 4, 8, 16 (tol tiny so every run hits
   maxit) for each loop mode.   python tools/latency_probe.py [--cfgs C1,C2] [--modes 1,5]"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import gen  # noqa: E402
from paper_2112_11880_b200 import zk  # noqa: E402

p = argparse.ArgumentParser()
p.add_argument("--cfgs", default="C1,C2")
p.add_argument("--modes", default="1,5")
p.add_argument("--method", default="bicgstab")
a = p.parse_args()
for cfg in a.cfgs.split(","):
    m = gen.make_matrix(cfg)
    A = zk.csr_create(m["row_ptr"], m["col_idx"], m["values"], m["n"])
    b = torch.from_numpy(gen.make_rhs(m)).cuda()
    ws = zk.alloc_workspace(A, a.method, 64)
    for mode in a.modes.split(","):
        os.environ["ZK_LOOP_MODE"] = mode
        row = {"cfg": cfg, "mode": mode}
        for mi in (1, 2, 4, 8, 16):
            for _ in range(3):
                r = zk.solve(A, b, tol=1e-300, maxit=mi, method=a.method, workspace=ws)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            for _ in range(20):
                r = zk.solve(A, b, tol=1e-300, maxit=mi, method=a.method, workspace=ws)
            e1.record()
            torch.cuda.synchronize()
            row[f"maxit{mi}_us"] = round(1e3 * e0.elapsed_time(e1) / 20, 1)
        row["loop_mode_used"] = r["loop_mode"]
        row["marginal_us_per_iter"] = round((row["maxit16_us"] - row["maxit8_us"]) / 8, 2)
        print(json.dumps(row), flush=True)
