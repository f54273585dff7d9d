"""ncu / sanitizer target: solve one config with one method a few times (default C3 BiCGStab,
maxit 10) in the default loop mode.  Usage: python tools/solve_target.py [cfg] [method] [maxit] [reps]"""
import os
import sys

sys.path.insert(0, os.getcwd())
import torch  # noqa: E402

import gen  # noqa: E402
from paper_2112_11880_b200 import zk  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "C3"
meth = sys.argv[2] if len(sys.argv) > 2 else "bicgstab"
maxit = int(sys.argv[3]) if len(sys.argv) > 3 else 10
reps = int(sys.argv[4]) if len(sys.argv) > 4 else 2
m = gen.make_matrix(cfg)
A = zk.csr_create(m["row_ptr"], m["col_idx"], m["values"], m["n"])
b = torch.from_numpy(gen.make_rhs(m)).cuda()
ws = zk.alloc_workspace(A, meth, maxit)
for _ in range(reps):
    r = zk.solve(A, b, tol=1e-12, maxit=maxit, method=meth, workspace=ws)
torch.cuda.synchronize()
print(cfg, meth, r["iters"], r["status"], "loop", r["loop_mode"], "ms", r["solve_ms"])
