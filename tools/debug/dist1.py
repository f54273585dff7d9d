import sys, os
sys.path.insert(0, os.getcwd())
import numpy as np, torch, gen
from paper_2112_11880_b200 import zk
m = gen.make_matrix("C2"); b = gen.make_rhs(m)
A0 = zk.csr_create(m["row_ptr"], m["col_idx"], m["values"], m["n"])
B = torch.from_numpy(b).cuda()
r0 = zk.solve(A0, B, tol=1e-8)
os.environ["ZK_LOOP_MODE"] = "3"
r3 = zk.solve(A0, B, tol=1e-8)
del os.environ["ZK_LOOP_MODE"]
comm = zk.Comm(zk.Comm.unique_id(), 1, 0, 0)
A = zk.csr_create(m["row_ptr"], m["col_idx"], m["values"], m["n"], comm=comm, row_begin=0)
r = zk.solve(A, B, tol=1e-8)
for name, q in [("mode3", r3), ("dist", r)]:
    dx = (q["x"] - r0["x"]).abs().max().item()
    dh = np.max(np.abs(q["hist"] - r0["hist"]))
    print(name, q["iters"], q["status"], "max|dx|", dx, "max|dhist|", dh, "first hist diff idx",
          np.nonzero(q["hist"] != r0["hist"])[0][:5], q["true_relres"], r0["true_relres"], q["kernel_launches"], r0["kernel_launches"])
