#!/usr/bin/env python
"""Device free memory (cudaMemGetInfo) after each of N repeated solves on one handle: a solve that
allocates (or leaks) device memory shows up as a falling line.  python tools/mem_probe.py [cfg] [method...]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import gen  # noqa: E402
from paper_2112_11880_b200 import zk  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "T1"
m = gen.make_matrix(cfg)
A = zk.csr_create(m["row_ptr"], m["col_idx"], m["values"], m["n"])
b = torch.from_numpy(gen.make_rhs(m)).cuda()
x = torch.empty_like(b)
for meth in sys.argv[2:] or ["bicgstab", "bicgstab_jacobi"]:
    ws = zk.alloc_workspace(A, meth, 1000)
    free = []
    for _ in range(8):
        r = zk.solve(A, b, tol=1e-8, method=meth, workspace=ws, x=x)
        torch.cuda.synchronize()
        free.append(torch.cuda.mem_get_info()[0] >> 20)
    print(cfg, meth, "loop", r["loop_mode"], "free MiB after each solve:", free, flush=True)
