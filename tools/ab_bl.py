"""A/B of the BiCGStab(l) split schedule at C4: ZK_SPLIT_TAIL=1 (S1/S2 store only + reduction pass)
vs 2 (S1/S2 with per-slice warp-reduced fused dot products).  ms per cycle, median of 3 solves."""
import os
import statistics
import sys

sys.path.insert(0, os.getcwd())
import torch  # noqa: E402

import gen  # noqa: E402
from paper_2112_11880_b200 import zk  # noqa: E402

m = gen.make_matrix(sys.argv[1] if len(sys.argv) > 1 else "C4")
A = zk.csr_create(torch.from_numpy(m["row_ptr"]).cuda(), torch.from_numpy(m["col_idx"]).cuda(),
                  torch.from_numpy(m["values"]).cuda(), m["n"])
b = torch.from_numpy(gen.make_rhs(m)).cuda()
for ell in (2, 8):
    row = []
    for tail in ("1", "2"):
        os.environ["ZK_SPLIT_TAIL"] = tail
        ws = zk.alloc_workspace(A, "bicgstab_l", 300, ell=ell)
        zk.solve(A, b, tol=1e-8, maxit=300, method="bicgstab_l", ell=ell, workspace=ws)
        ts = []
        for _ in range(3):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            r = zk.solve(A, b, tol=1e-8, maxit=300, method="bicgstab_l", ell=ell, workspace=ws)
            e1.record()
            torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1))
        row.append(f"tail={tail}: {statistics.median(ts) / r['iters']:.3f} ms/cycle ({r['iters']} cycles)")
        del ws
    print(f"BiCGStab({ell})", " | ".join(row), flush=True)
