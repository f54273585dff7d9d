#!/usr/bin/env python
"""ncu target: zk_zcsrmv after a kernel that rewrites x (dirty L2) vs after one that only reads it.
   ncu --cache-control none --clock-control none -k regex:zcsrmv python tools/dirty_probe.py"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import gen  # noqa: E402
from paper_2112_11880_b200 import zk  # noqa: E402

m = gen.make_matrix(sys.argv[1] if len(sys.argv) > 1 else "C4")
A = zk.csr_create(m["row_ptr"], m["col_idx"], m["values"], m["n"])
x = torch.from_numpy(gen.rand_vector(m["n"], 1)).cuda()
y = torch.empty_like(x)
for _ in range(3):  # launches 1-3: after a read of x; 4-6: after a rewrite of x
    zk.dznrm2(x)
    zk.zcsrmv(A, 1.0, x, 0.0, y)
for _ in range(3):
    zk.zscal(1.0, x)
    zk.zcsrmv(A, 1.0, x, 0.0, y)
torch.cuda.synchronize()
