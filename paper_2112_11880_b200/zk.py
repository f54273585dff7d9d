"""Python binding of libzk (include/zk.h) — argument marshalling only.

Every step of the path runs in libzk's sm_100a kernels; this module only turns torch tensors
(device memory, streams) and numpy arrays (host CSR) into the C-ABI's pointers and sizes.
There is no CPU fallback: if libzk.so is missing or CUDA is unusable the calls raise.
Function names follow the ABI: csr_create, zcsrmv, zdotc, dznrm2, zaxpy, zscal, solve.
"""
from __future__ import annotations

import ctypes
import os

import numpy as np
import torch

_PKG = os.path.dirname(os.path.abspath(__file__))
SO_PATH = os.path.join(_PKG, "libzk.so")

ZK_PTRS_HOST, ZK_PTRS_DEVICE, ZK_PTRS_DEVICE_BORROW, ZK_SKIP_VALIDATE = 0, 1, 2, 4
ZK_BICGSTAB, ZK_CG = 0, 1
ZK_BICGSTAB_JACOBI, ZK_COCG, ZK_TFQMR = 2, 3, 4
METHODS = {"bicgstab": ZK_BICGSTAB, "cg": ZK_CG, "bicgstab_jacobi": ZK_BICGSTAB_JACOBI, "cocg": ZK_COCG, "tfqmr": ZK_TFQMR}


def ZK_BICGSTAB_L(ell: int) -> int:
    """Method code of BiCGStab(l), 1 <= l <= 8 (zk.h ZK_BICGSTAB_L)."""
    return 16 + int(ell)


def method_code(method: str, ell: int = 8) -> int:
    """"bicgstab", "cg", "bicgstab_jacobi", "cocg", "tfqmr" or "bicgstab_l" (with ell)."""
    if method == "bicgstab_l":
        return ZK_BICGSTAB_L(ell)
    return METHODS[method]
OUTCOMES = {0: "CONVERGED", 1: "MAXIT", 2: "BREAKDOWN_RHO", 3: "BREAKDOWN_SIGMA", 4: "BREAKDOWN_OMEGA",
            5: "NOT_HPD", 6: "NONFINITE"}


class ZkError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"{msg} (status {code})")
        self.code = code


class zk_z(ctypes.Structure):
    _fields_ = [("re", ctypes.c_double), ("im", ctypes.c_double)]


class zk_csr_info_t(ctypes.Structure):
    _fields_ = [("n_rows", ctypes.c_int64), ("n_cols", ctypes.c_int64), ("nnz", ctypes.c_int64),
                ("row_begin", ctypes.c_int64), ("n_global", ctypes.c_int64),
                ("max_row_len", ctypes.c_int32), ("lanes_per_row", ctypes.c_int32),
                ("mean_row_len", ctypes.c_double), ("n_halo", ctypes.c_int64),
                ("borrowed", ctypes.c_int32), ("nranks", ctypes.c_int32), ("spmv_mode", ctypes.c_int32),
                ("sell_entries", ctypes.c_int64),
                ("interior_rows", ctypes.c_int64), ("csr_values_kept", ctypes.c_int32)]


class zk_solve_info(ctypes.Structure):
    _fields_ = [("status", ctypes.c_int32), ("iters", ctypes.c_int32), ("true_relres", ctypes.c_double),
                ("n_spmv", ctypes.c_int64), ("solve_ms", ctypes.c_double), ("loop_mode", ctypes.c_int32),
                ("gpu_launches", ctypes.c_int32), ("kernel_ms", ctypes.c_double * 4),
                ("kernel_launches", ctypes.c_int32 * 4)]


# (name, restype, argtypes) of every symbol include/zk.h declares
P, I32, I64, U32, D, SZ = ctypes.c_void_p, ctypes.c_int32, ctypes.c_int64, ctypes.c_uint32, ctypes.c_double, ctypes.c_size_t
SIGNATURES = {
    "zk_last_error": (ctypes.c_char_p, []),
    "zk_status_string": (ctypes.c_char_p, [I32]),
    "zk_version": (I32, []),
    "zk_comm_get_unique_id": (I32, [P]),
    "zk_comm_create": (I32, [ctypes.POINTER(P), P, I32, I32, I32]),
    "zk_comm_destroy": (I32, [P]),
    "zk_local_group_create": (I32, [ctypes.POINTER(P), I32]),
    "zk_local_group_destroy": (I32, [P]),
    "zk_comm_create_local": (I32, [ctypes.POINTER(P), P, I32, I32]),
    "zk_csr_create": (I32, [ctypes.POINTER(P), I64, I64, I64, P, P, P, U32, P, I64, P]),
    "zk_csr_destroy": (I32, [P]),
    "zk_csr_update_values": (I32, [P, P, U32, P]),
    "zk_csr_info": (I32, [P, ctypes.POINTER(zk_csr_info_t)]),
    "zk_zcsrmv": (I32, [P, zk_z, P, zk_z, P, P]),
    "zk_zdotc": (I32, [I64, P, P, P, P, P]),
    "zk_dznrm2": (I32, [I64, P, P, P, P]),
    "zk_zaxpy": (I32, [I64, zk_z, P, P, P]),
    "zk_zscal": (I32, [I64, zk_z, P, P]),
    "zk_zassign": (I32, [I64, zk_z, P, P]),
    "zk_zaxmy": (I32, [I64, P, P, P]),
    "zk_solve_workspace_size": (SZ, [P, I32, I32]),
    "zk_solve": (I32, [P, P, P, D, I32, I32, P, ctypes.POINTER(I32), P, ctypes.POINTER(zk_solve_info), P, SZ, P]),
    # include/zk_dist.h (host-only)
    "zk_partition_rows": (I32, [I64, P, I32, P]),
    "zk_halo_plan": (I32, [I64, P, I32, I32, P, ctypes.POINTER(I64), P, P]),
    "zk_halo_renumber": (I32, [I64, P, I64, I64, I64, P, P]),
}

_lib = None


def lib():
    """Load libzk.so (built by __graft_entry__.build() / paper_2112_11880_b200/build.py). Fails loudly."""
    global _lib
    if _lib is None:
        path = os.environ.get("ZK_LIB", SO_PATH)  # A/B builds of libzk (tools), default in-tree
        if not os.path.exists(path):
            raise ImportError(f"libzk.so not built at {path}: run `python __graft_entry__.py build` "
                              "(no CPU fallback exists)")
        h = ctypes.CDLL(path)
        for name, (res, args) in SIGNATURES.items():
            f = getattr(h, name)
            f.restype, f.argtypes = res, args
        _lib = h
    return _lib


def _check(code: int):
    if code != 0:
        raise ZkError(code, lib().zk_last_error().decode())


def _z(a) -> zk_z:
    a = complex(a)
    return zk_z(a.real, a.imag)


_raw_stream = getattr(torch._C, "_cuda_getCurrentRawStream", None)


def _stream(stream) -> int:
    if stream is None:  # torch's current stream (the raw handle: no Stream object per call)
        if _raw_stream is not None:
            return _raw_stream(torch.cuda.current_device())
        return torch.cuda.current_stream().cuda_stream
    return stream.cuda_stream if hasattr(stream, "cuda_stream") else int(stream)


def _dev_c128(t: torch.Tensor, name: str) -> int:
    if isinstance(t, torch.Tensor) and t.is_cuda and t.dtype is torch.complex128 and t.is_contiguous():
        return t.data_ptr()  # (the common case: one combined test)
    if not isinstance(t, torch.Tensor) or not t.is_cuda:
        raise TypeError(f"{name} must be a CUDA tensor")
    if t.dtype != torch.complex128:
        raise TypeError(f"{name} must be complex128")
    raise ValueError(f"{name} must be contiguous")


class Comm:
    """Communicator owned by libzk (one per rank): NCCL (one process per GPU, zk_comm_create) or
    LOCAL (ranks are threads of this process, zk_comm_create_local; see Comm.local)."""

    def __init__(self, id_bytes: bytes, nranks: int, rank: int, device: int):
        h = P()
        buf = ctypes.create_string_buffer(bytes(id_bytes), 128)
        _check(lib().zk_comm_create(ctypes.byref(h), buf, nranks, rank, device))
        self.handle, self.nranks, self.rank = h, nranks, rank

    @classmethod
    def local(cls, group: "LocalGroup", rank: int, device: int) -> "Comm":
        """zk_comm_create_local: every rank calls this concurrently from its own thread."""
        self = cls.__new__(cls)
        h = P()
        _check(lib().zk_comm_create_local(ctypes.byref(h), group.handle, int(rank), int(device)))
        self.handle, self.nranks, self.rank = h, group.nranks, int(rank)
        self.group = group
        return self

    @staticmethod
    def unique_id() -> bytes:
        buf = ctypes.create_string_buffer(128)
        _check(lib().zk_comm_get_unique_id(buf))
        return buf.raw

    def close(self):
        if self.handle:
            lib().zk_comm_destroy(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class LocalGroup:
    """zk_local_group_create: a group of `nranks` in-process ranks (threads), see include/zk.h."""

    def __init__(self, nranks: int):
        h = P()
        _check(lib().zk_local_group_create(ctypes.byref(h), int(nranks)))
        self.handle, self.nranks = h, int(nranks)

    def close(self):
        if self.handle:
            lib().zk_local_group_destroy(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def _as_ptr_array(a, dtype, name):
    """Return (pointer, keepalive, where) for a numpy array / CPU tensor (host) or CUDA tensor."""
    if isinstance(a, torch.Tensor):
        if a.is_cuda:
            if not a.is_contiguous():
                raise ValueError(f"{name} must be contiguous")
            return a.data_ptr(), a, "device"
        a = a.numpy()
    arr = np.ascontiguousarray(a, dtype=dtype)
    return arr.ctypes.data, arr, "host"


class Csr:
    """A zk_csr handle (zk_csr_create / zk_csr_destroy)."""

    def __init__(self, row_ptr, col_idx, values, n_cols: int | None = None, *, borrow: bool = False,
                 validate: bool = True, comm: Comm | None = None, row_begin: int = 0, stream=None):
        rp, k1, w1 = _as_ptr_array(row_ptr, np.int64, "row_ptr")
        ci, k2, w2 = _as_ptr_array(col_idx, np.int32, "col_idx")
        va, k3, w3 = _as_ptr_array(values, np.complex128, "values")
        if len({w1, w2, w3}) != 1:
            raise ValueError("row_ptr, col_idx and values must all be host or all be CUDA")
        for k, want in ((k1, (np.int64, torch.int64)), (k2, (np.int32, torch.int32)), (k3, (np.complex128, torch.complex128))):
            if getattr(k, "dtype", None) not in want:
                raise TypeError(f"bad dtype {k.dtype}")
        n_rows = int(k1.shape[0]) - 1
        nnz = int(k2.shape[0])
        if n_cols is None:
            n_cols = n_rows
        flags = ZK_PTRS_HOST if w1 == "host" else (ZK_PTRS_DEVICE_BORROW if borrow else ZK_PTRS_DEVICE)
        if not validate:
            flags |= ZK_SKIP_VALIDATE
        h = P()
        _check(lib().zk_csr_create(ctypes.byref(h), n_rows, int(n_cols), nnz, rp, ci, va, flags,
                                   comm.handle if comm else None, int(row_begin), _stream(stream)))
        self.handle = h
        self._keep = (k1, k2, k3) if (w1 == "device" and borrow) else None
        self.comm = comm
        info = zk_csr_info_t()
        _check(lib().zk_csr_info(h, ctypes.byref(info)))
        self.info = {f: getattr(info, f) for f, _ in zk_csr_info_t._fields_}
        self.n_rows, self.n_cols, self.nnz = info.n_rows, info.n_cols, info.nnz

    def update_values(self, values=None, stream=None, validate: bool = True):
        """zk_csr_update_values: new values for the same pattern (host / CUDA array in the original
        CSR order), or None after changing a borrowed values array in place."""
        flags = 0 if validate else ZK_SKIP_VALIDATE
        ptr, keep = None, None
        if values is not None:
            ptr, keep, where = _as_ptr_array(values, np.complex128, "values")
            flags |= ZK_PTRS_HOST if where == "host" else ZK_PTRS_DEVICE
        _check(lib().zk_csr_update_values(self.handle, ptr, flags, _stream(stream)))
        return self

    def close(self):
        if self.handle:
            lib().zk_csr_destroy(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def csr_create(row_ptr, col_idx, values, n_cols=None, **kw) -> Csr:
    return Csr(row_ptr, col_idx, values, n_cols, **kw)


def zcsrmv(A: Csr, alpha, x: torch.Tensor, beta, y: torch.Tensor, stream=None) -> torch.Tensor:
    """y ← αAx + βy (zk_zcsrmv)."""
    px, py = _dev_c128(x, "x"), _dev_c128(y, "y")
    _check(lib().zk_zcsrmv(A.handle, _z(alpha), px, _z(beta), py, _stream(stream)))
    return y


def zdotc(x: torch.Tensor, y: torch.Tensor, result: torch.Tensor | None = None, comm: Comm | None = None,
          stream=None) -> torch.Tensor:
    """Σ conj(x_i) y_i into a 1-element complex128 device tensor (zk_zdotc)."""
    if x.numel() != y.numel():
        raise ValueError("length mismatch")
    if result is None:
        result = torch.empty(1, dtype=torch.complex128, device=x.device)
    _check(lib().zk_zdotc(x.numel(), _dev_c128(x, "x"), _dev_c128(y, "y"), _dev_c128(result, "result"),
                          comm.handle if comm else None, _stream(stream)))
    return result


def dznrm2(x: torch.Tensor, result: torch.Tensor | None = None, comm: Comm | None = None, stream=None) -> torch.Tensor:
    """‖x‖₂ into a 1-element float64 device tensor (zk_dznrm2)."""
    if result is None:
        result = torch.empty(1, dtype=torch.float64, device=x.device)
    if result.dtype != torch.float64 or not result.is_cuda:
        raise TypeError("result must be a float64 CUDA tensor")
    _check(lib().zk_dznrm2(x.numel(), _dev_c128(x, "x"), result.data_ptr(), comm.handle if comm else None,
                           _stream(stream)))
    return result


def zaxpy(alpha, x: torch.Tensor, y: torch.Tensor, stream=None) -> torch.Tensor:
    """y ← αx + y (zk_zaxpy)."""
    if x.numel() != y.numel():
        raise ValueError("length mismatch")
    _check(lib().zk_zaxpy(x.numel(), _z(alpha), _dev_c128(x, "x"), _dev_c128(y, "y"), _stream(stream)))
    return y


def zscal(alpha, x: torch.Tensor, stream=None) -> torch.Tensor:
    """x ← αx (zk_zscal)."""
    _check(lib().zk_zscal(x.numel(), _z(alpha), _dev_c128(x, "x"), _stream(stream)))
    return x


def zassign(alpha, x: torch.Tensor, stream=None) -> torch.Tensor:
    """x ← α (zk_zassign; the paper's ZASSIGN fill)."""
    _check(lib().zk_zassign(x.numel(), _z(alpha), _dev_c128(x, "x"), _stream(stream)))
    return x


def zaxmy(x: torch.Tensor, y: torch.Tensor, stream=None) -> torch.Tensor:
    """y ← x ⊙ y (zk_zaxmy; the paper's ZAXMY / EWProduct)."""
    if x.numel() != y.numel():
        raise ValueError("length mismatch")
    _check(lib().zk_zaxmy(x.numel(), _dev_c128(x, "x"), _dev_c128(y, "y"), _stream(stream)))
    return y


def workspace_size(A: Csr, method: str = "bicgstab", maxit: int = 1000, ell: int = 8) -> int:
    return int(lib().zk_solve_workspace_size(A.handle, method_code(method, ell), int(maxit)))


def alloc_workspace(A: Csr, method: str = "bicgstab", maxit: int = 1000, device=None, ell: int = 8) -> torch.Tensor:
    nbytes = workspace_size(A, method, maxit, ell)
    # torch's caching allocator returns 512-B aligned blocks
    return torch.empty(nbytes, dtype=torch.uint8, device=device or "cuda")


def solve(A: Csr, b: torch.Tensor, x0: torch.Tensor | None = None, tol: float = 1e-8, maxit: int = 1000,
          method: str = "bicgstab", x: torch.Tensor | None = None, workspace: torch.Tensor | None = None,
          stream=None, ell: int = 8) -> dict:
    """zk_solve: returns dict(x, iters, hist, status, true_relres, n_spmv, solve_ms, loop_mode).
    method "bicgstab_l" runs BiCGStab(ell) (iters/hist count outer cycles)."""
    m = method_code(method, ell)
    pb = _dev_c128(b, "b")
    if x is None:
        x = torch.empty_like(b)
    px = _dev_c128(x, "x")
    px0 = _dev_c128(x0, "x0") if x0 is not None else None
    if workspace is None:
        workspace = alloc_workspace(A, method, maxit, b.device, ell)
    iters = I32(0)
    hist = np.empty(maxit + 1)  # (entries past iters are unspecified, zk.h; only hist[:iters+1] is returned)
    info = zk_solve_info()
    _check(lib().zk_solve(A.handle, pb, px0, float(tol), int(maxit), m, px, ctypes.byref(iters),
                          hist.ctypes.data, ctypes.byref(info), workspace.data_ptr(), workspace.numel(),
                          _stream(stream)))
    it = iters.value
    return dict(x=x, iters=it, hist=hist[: it + 1].copy(), status=OUTCOMES.get(info.status, str(info.status)),
                true_relres=info.true_relres, n_spmv=info.n_spmv, solve_ms=info.solve_ms,
                loop_mode=info.loop_mode, gpu_launches=info.gpu_launches,
                kernel_ms=list(info.kernel_ms), kernel_launches=list(info.kernel_launches))


# ---------------------------------------------------------------- include/zk_dist.h (host-only)
def partition_rows(row_ptr: np.ndarray, nranks: int) -> np.ndarray:
    """nnz-balanced contiguous row blocks: offsets[nranks+1] (zk_partition_rows)."""
    rp = np.ascontiguousarray(row_ptr, dtype=np.int64)
    off = np.zeros(nranks + 1, dtype=np.int64)
    _check(lib().zk_partition_rows(len(rp) - 1, rp.ctypes.data, nranks, off.ctypes.data))
    return off


def halo_plan(col: np.ndarray, nranks: int, rank: int, offsets: np.ndarray):
    """(sorted distinct off-rank columns, count per owner rank) of one rank's block (zk_halo_plan)."""
    c = np.ascontiguousarray(col, dtype=np.int32)
    off = np.ascontiguousarray(offsets, dtype=np.int64)
    n_ext = I64(0)
    _check(lib().zk_halo_plan(len(c), c.ctypes.data, nranks, rank, off.ctypes.data, ctypes.byref(n_ext), None, None))
    ext = np.zeros(max(n_ext.value, 1), dtype=np.int32)
    cnt = np.zeros(nranks, dtype=np.int64)
    _check(lib().zk_halo_plan(len(c), c.ctypes.data, nranks, rank, off.ctypes.data, ctypes.byref(n_ext),
                              ext.ctypes.data, cnt.ctypes.data))
    return ext[: n_ext.value], cnt


def halo_renumber(col: np.ndarray, row_begin: int, n_rows: int, ext: np.ndarray) -> np.ndarray:
    """Columns renumbered to [local rows | halo slots] (zk_halo_renumber)."""
    c = np.ascontiguousarray(col, dtype=np.int32)
    e = np.ascontiguousarray(ext, dtype=np.int32)
    out = np.empty_like(c)
    _check(lib().zk_halo_renumber(len(c), c.ctypes.data, int(row_begin), int(n_rows), len(e),
                                  e.ctypes.data if len(e) else None, out.ctypes.data))
    return out
