"""Small workload for compute-sanitizer (memcheck / racecheck / synccheck / initcheck): every
solver on C1 (and T0) in the WHILE-graph loop (mode 1), the direct-launch loop (mode 3), the
cluster solver (mode 5), the split-reduction schedule forced, plus the standalone ZSpMV and
BLAS-1 calls.  Usage: python tools/sanitize_target.py [cfg ...]   (default C1)."""
import os
import sys

sys.path.insert(0, os.getcwd())
import numpy as np  # noqa: E402
import torch  # noqa: E402

import gen  # noqa: E402
from paper_2112_11880_b200 import zk  # noqa: E402

MAXIT = int(os.environ.get("SAN_MAXIT", "60"))
METHODS = [("bicgstab", 8), ("cg", 8), ("cocg", 8), ("tfqmr", 8), ("bicgstab_jacobi", 8),
           ("bicgstab_l", 2), ("bicgstab_l", 8)]


def main(cfgs):
    dev = torch.device("cuda:0")
    for cfg in cfgs:
        m = gen.make_matrix(cfg)
        mg = gen.make_matrix(cfg, eta=0.0, twist_seed=gen.SEED_TWIST)
        A = zk.csr_create(m["row_ptr"], m["col_idx"], m["values"], m["n"])
        Ag = zk.csr_create(mg["row_ptr"], mg["col_idx"], mg["values"], mg["n"])
        b = torch.from_numpy(gen.make_rhs(m)).to(dev)
        bg = torch.from_numpy(np.exp(1j * mg["phase"]) * gen.make_rhs(mg)).to(dev)
        x = torch.from_numpy(gen.rand_vector(m["n"], 1)).to(dev)
        y = torch.empty_like(x)
        zk.zcsrmv(A, 1.0, x, 0.0, y)
        zk.zcsrmv(A, 0.5j, x, 2.0, y)
        zk.zdotc(x, y)
        zk.dznrm2(y)
        zk.zaxpy(1 - 1j, x, y)
        zk.zscal(2j, y)
        zk.zassign(1j, y)
        zk.zaxmy(x, y)
        for mode in os.environ.get("SAN_MODES", "1,3,5").split(","):
            for split in os.environ.get("SAN_SPLIT", "0,1").split(","):
                os.environ["ZK_LOOP_MODE"] = mode
                os.environ["ZK_SPLIT_RED"] = split
                for meth, ell in METHODS:
                    M, rhs = (Ag, bg) if meth == "cg" else (A, b)
                    r = zk.solve(M, rhs, tol=1e-8, maxit=MAXIT, method=meth, ell=ell)
                    print(cfg, "mode", mode, "split", split, meth, ell, r["status"], r["iters"],
                          "loop", r["loop_mode"], flush=True)
        r = zk.solve(A, b, x0=x, tol=1e-8, maxit=60)  # x0 path
        print(cfg, "x0", r["status"], r["iters"])
    torch.cuda.synchronize()
    print("sanitize target done")


if __name__ == "__main__":
    main(sys.argv[1:] or ["C1"])
