"""One solve of C4 with the given method (for ncu: run with ZK_LOOP_MODE=3, since kernels inside
graphs with conditional nodes cannot be profiled).  python tools/debug/solve_one.py tfqmr [ell]"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch, gen
from paper_2112_11880_b200 import zk
meth = sys.argv[1] if len(sys.argv) > 1 else "bicgstab"
ell = int(sys.argv[2]) if len(sys.argv) > 2 else 8
m = gen.make_matrix(os.environ.get("CFG", "C4"))
A = zk.csr_create(torch.from_numpy(m["row_ptr"]).cuda(), torch.from_numpy(m["col_idx"]).cuda(),
                  torch.from_numpy(m["values"]).cuda(), m["n"], borrow=True)
b = torch.from_numpy(gen.make_rhs(m)).cuda()
r = zk.solve(A, b, tol=1e-8, maxit=int(os.environ.get("MAXIT", "30")), method=meth, ell=ell)
torch.cuda.synchronize()
print(meth, r["iters"], r["status"])
