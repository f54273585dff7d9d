"""Work and byte models used for reporting (no arithmetic of the method itself).

Flop conventions (per element / per nonzero) are the paper's own, recovered from every row of
PAPER.md Tables 2-8 as Gflops × time / h:
assign 1, scal 6, axpy 8, ewp 6, dot 8, norm 5, SpMV 8 per nnz.  Pinned by
tests/test_metrics.py against tests/golden/paper_flop_tables.json.

Algorithmic bytes: complex128 = 16 B, col_idx int32 = 4 B, row_ptr int64 = 8 B.
"""
FLOPS_PER_ELEM = {"zassign": 1, "zscal": 6, "zaxpy": 8, "zaxmy": 6, "zdotc": 8, "dznrm2": 5}
FLOPS_PER_NNZ_SPMV = 8

Z = 16  # bytes per complex128


def csr_bytes(n: int, nnz: int) -> int:
    """Mat = 20·nnz + 8·(n+1): values + int32 col_idx + int64 row_ptr."""
    return 20 * nnz + 8 * (n + 1)


def spmv_bytes(n: int, nnz: int, beta_nonzero: bool = False) -> int:
    """ZSpMV y ← αAx + βy: Mat + x once + y written (+ y read if β ≠ 0)."""
    return csr_bytes(n, nnz) + Z * n + Z * n + (Z * n if beta_nonzero else 0)


def blas1_bytes(op: str, n: int) -> int:
    """Algorithmic bytes of one BLAS-1 call: read x (and y), write the output vector."""
    return {"zdotc": 2 * Z * n, "dznrm2": Z * n, "zaxpy": 3 * Z * n, "zscal": 2 * Z * n,
            "zassign": Z * n, "zaxmy": 3 * Z * n}[op]


def bicgstab_iter_bytes(n: int, nnz: int) -> int:
    """Schedule F: 2·Mat + 304n (19 complex vector passes)."""
    return 2 * csr_bytes(n, nnz) + 19 * Z * n


def cg_iter_bytes(n: int, nnz: int) -> int:
    """Mat + 176n (11 vector passes)."""
    return csr_bytes(n, nnz) + 11 * Z * n


def cocg_iter_bytes(n: int, nnz: int) -> int:
    """COCG (NEXT-4) runs CG's schedule with unconjugated products: Mat + 176n."""
    return cg_iter_bytes(n, nnz)


def tfqmr_iter_bytes(n: int, nnz: int) -> int:
    """TFQMR (NEXT-2), kernels T1-T4 of solve.cu: 2·Mat + 400n (25 complex vector passes:
    T1 6, T2 5 incl. the gathered y2, T3 8, T4 6 incl. the gathered y1)."""
    return 2 * csr_bytes(n, nnz) + 25 * Z * n


def bicgstab_l_cycle_bytes(n: int, nnz: int, ell: int) -> int:
    """BiCGStab(ℓ) (NEXT-3), one outer cycle of solve.cu's bl_* kernels: 2ℓ·Mat + (3ℓ² + 15ℓ + 7)
    complex vector passes — BiCG step j: B1 3(j+1), S1 3, B2 6 + 3j, S2 3 (2 for j = ℓ−1);
    Gram ℓ+1; update 2ℓ + 7.  ℓ = 8: 319 passes."""
    return 2 * ell * csr_bytes(n, nnz) + (3 * ell * ell + 15 * ell + 7) * Z * n


def spmv_flops(nnz: int) -> int:
    return FLOPS_PER_NNZ_SPMV * nnz
