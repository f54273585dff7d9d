#!/usr/bin/env python
"""In-loop time split of a solve (device global timer, zk_solve_info.kernel_ms): SpMV kernels (with
their fused reductions), the vector kernels that carry a reduction, and the rest (kernels without a
reduction such as BiCGStab K5, launch gaps), per iteration.  python tools/inloop_split.py C3 C3T C4"""
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import gen  # noqa: E402
from paper_2112_11880_b200 import zk  # noqa: E402

meths = os.environ.get("METHODS", "bicgstab").split(",")
for cfg in sys.argv[1:] or ["C3"]:
    m = gen.make_matrix(cfg)
    A = zk.csr_create(m["row_ptr"], m["col_idx"], m["values"], m["n"])
    b = torch.from_numpy(gen.make_rhs(m)).cuda()
    for meth in meths:
        ws = zk.alloc_workspace(A, meth, 2000)
        zk.solve(A, b, tol=1e-8, maxit=2000, method=meth, workspace=ws)
        rows = []
        for _ in range(5):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            r = zk.solve(A, b, tol=1e-8, maxit=2000, method=meth, workspace=ws)
            e1.record()
            torch.cuda.synchronize()
            it = r["iters"]
            rows.append((1e3 * e0.elapsed_time(e1) / it, 1e3 * r["kernel_ms"][0] / it, 1e3 * r["kernel_ms"][1] / it,
                         r["kernel_launches"][0] / it, r["kernel_launches"][1] / it))
        med = [statistics.median(x[k] for x in rows) for k in range(5)]
        print(f"{cfg} {meth} iters {it}: total {med[0]:.1f} us/it | spmv {med[1]:.1f} ({med[3]:.0f}/it) | "
              f"vec-red {med[2]:.1f} ({med[4]:.0f}/it) | rest {med[0] - med[1] - med[2]:.1f}", flush=True)
    A.close()
