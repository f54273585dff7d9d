#!/usr/bin/env python
"""Per-phase cycle totals of the BiCGStab cluster kernel (CTA 0, thread 0; the kernel prints them).
Needs a -DZK_CLUSTER_PROF=1 build:  python -m paper_2112_11880_b200.build --out paper_2112_11880_b200/variants/cprof.so -D ZK_CLUSTER_PROF=1
then  ZK_LIB=paper_2112_11880_b200/variants/cprof.so python tools/cluster_phase_probe.py C1 T0 C2"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import gen  # noqa: E402
from paper_2112_11880_b200 import zk  # noqa: E402

for cfg in sys.argv[1:] or ["C1", "T0", "C2"]:
    m = gen.make_matrix(cfg)
    A = zk.csr_create(m["row_ptr"], m["col_idx"], m["values"], m["n"])
    b = torch.from_numpy(gen.make_rhs(m)).cuda()
    ws = zk.alloc_workspace(A, "bicgstab", 64)
    for _ in range(3):
        r = zk.solve(A, b, tol=1e-300, maxit=int(os.environ.get("MAXIT", "20")), method="bicgstab", workspace=ws)
    torch.cuda.synchronize()
    print(cfg, "n", m["n"], "W", A.info.get("lanes_per_row"), "loop_mode", r["loop_mode"], "solve_ms", r["solve_ms"], flush=True)
