#!/usr/bin/env python
"""Host cost of one small solve (C1, BiCGStab, maxit 1): the Python binding (zk.solve), the bare
ctypes call with every argument prepared, and the device time (info.solve_ms).  With ZK_TRACE=1
libzk prints its own host phases.   python tools/host_overhead.py"""
import ctypes
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import gen  # noqa: E402
from paper_2112_11880_b200 import zk  # noqa: E402

m = gen.make_matrix("C1")
A = zk.csr_create(m["row_ptr"], m["col_idx"], m["values"], m["n"])
b = torch.from_numpy(gen.make_rhs(m)).cuda()
x = torch.empty_like(b)
maxit = int(os.environ.get("MAXIT", "1"))
ws = zk.alloc_workspace(A, "bicgstab", maxit)
N = 200
for _ in range(20):
    zk.solve(A, b, tol=1e-300, maxit=maxit, workspace=ws, x=x)
torch.cuda.synchronize()
t = time.perf_counter()
for _ in range(N):
    r = zk.solve(A, b, tol=1e-300, maxit=maxit, workspace=ws, x=x)
t_py = (time.perf_counter() - t) / N * 1e6
lib = zk.lib()
it = ctypes.c_int32(0)
hist = np.full(maxit + 1, np.nan)
info = zk.zk_solve_info()
st = torch.cuda.current_stream().cuda_stream
args = (A.handle, b.data_ptr(), None, 1e-300, maxit, zk.method_code("bicgstab"), x.data_ptr(), ctypes.byref(it),
        hist.ctypes.data, ctypes.byref(info), ws.data_ptr(), ws.numel(), st)
t = time.perf_counter()
for _ in range(N):
    lib.zk_solve(*args)
t_c = (time.perf_counter() - t) / N * 1e6
print(f"C1 bicgstab maxit={maxit}: zk.solve {t_py:.1f} us, bare ctypes call {t_c:.1f} us, device {1e3 * info.solve_ms:.1f} us, "
      f"mode {info.loop_mode}", flush=True)
