import os, sys
sys.path.insert(0, os.getcwd())
import torch, gen
from paper_2112_11880_b200 import zk
os.environ["ZK_LOOP_MODE"] = "5"
m = gen.make_matrix(sys.argv[1])
A = zk.csr_create(m["row_ptr"], m["col_idx"], m["values"], m["n"])
b = torch.from_numpy(gen.make_rhs(m)).cuda()
for _ in range(2):
    r = zk.solve(A, b, tol=1e-8, maxit=200)
torch.cuda.synchronize()
print(r["iters"], r["loop_mode"])
