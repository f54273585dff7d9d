"""Debug: TFQMR from a random x0 on C1, fresh vs reused handle, GPU hist vs oracle."""
import numpy as np, torch, gen, oracle
from paper_2112_11880_b200 import zk
m = gen.make_matrix("C1"); b = gen.make_rhs(m); x0 = gen.rand_vector(m["n"], 3)
ref = oracle.tfqmr(m, b, x0=x0, tol=1e-8)
print("oracle", ref["iters"], ref["hist"])
for reuse in (False, True):
    A = zk.csr_create(m["row_ptr"], m["col_idx"], m["values"], m["n"])
    B = torch.from_numpy(b).cuda()
    if reuse:
        zk.solve(A, B, tol=1e-8, method="tfqmr")
    r = zk.solve(A, B, x0=torch.from_numpy(x0).cuda(), tol=1e-8, method="tfqmr")
    print("gpu reuse=%s" % reuse, r["iters"], r["hist"])
for mode in ("3",):
    import os; os.environ["ZK_LOOP_MODE"] = mode
    A = zk.csr_create(m["row_ptr"], m["col_idx"], m["values"], m["n"])
    r = zk.solve(A, torch.from_numpy(b).cuda(), x0=torch.from_numpy(x0).cuda(), tol=1e-8, method="tfqmr")
    print("gpu mode", mode, r["iters"], r["hist"])
