/*
 * zk.h — C-ABI of libzk, the B200 (sm_100a) hot path of arXiv 2112.11880:
 * complex-double CSR SpMV (ZSpMV), the BLAS-1 kernels a Krylov iteration needs
 * (zdotc, dznrm2, zaxpy, zscal) and device-resident BiCGStab / CG solves.
 *
 * Citations: P:L = PAPER.md line L (the paper), S:L = SPEC.md line L,
 * SURVEY.md §8(b) is the boundary table this header implements.
 *
 * Conventions (all calls):
 *  - Complex numbers are zk_z {double re, im}, layout-identical to
 *    cuDoubleComplex and to one element of a torch.complex128 tensor.
 *  - Vector/matrix pointers passed to compute calls are DEVICE pointers on
 *    the current CUDA device, owned by the caller; alignment 16 B for zk_z.
 *  - `zk_stream` is a cudaStream_t (NULL = legacy default stream).  Compute
 *    calls are asynchronous and stream-ordered unless stated otherwise.
 *  - Return value: ZK_OK (0) or a negative zk_status error; the thread-local
 *    message is available from zk_last_error().  Solver *outcomes* (MAXIT,
 *    breakdowns, ...) are not errors: they come back in zk_solve_info.
 *  - A zk_csr handle owns reduction scratch, its solve graphs and its pinned
 *    readback staging (which small cluster solves write directly from the
 *    device): do not use one handle on two streams, or from two host threads,
 *    concurrently.  Different handles may solve concurrently.  The standalone reductions (zk_zdotc, zk_dznrm2)
 *    use a scratch per (device, stream), allocated on the first call on that
 *    stream (128 KB, kept for the process lifetime): calls on different streams
 *    (or host threads) may run concurrently; calls on one stream are serialised.
 *  - No CPU fallback: every call runs in libzk's sm_100a kernels; without a
 *    usable device the calls fail with ZK_ERR_CUDA.
 */
#ifndef ZK_H
#define ZK_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct { double re, im; } zk_z;
typedef struct zk_csr_s* zk_csr;
typedef struct zk_comm_s* zk_comm;
typedef int32_t zk_status;
typedef void* zk_stream; /* cudaStream_t */

/* ---- status codes (errors are negative) ---- */
enum {
    ZK_OK = 0,
    ZK_ERR_INVALID_VALUE = -1, /* NULL pointer, bad size, bad flag, tol <= 0, maxit < 1, ws too small */
    ZK_ERR_INVALID_CSR = -2,   /* row_ptr not 0..nnz monotone, column out of range / unsorted / duplicate */
    ZK_ERR_NONFINITE = -3,     /* non-finite matrix value at create */
    ZK_ERR_DIM = -4,           /* dimension mismatch (e.g. solve on a non-square matrix) */
    ZK_ERR_OOM = -5,           /* device allocation failed */
    ZK_ERR_CUDA = -6,          /* CUDA runtime error (message names it) */
    ZK_ERR_ALIAS = -7,         /* forbidden aliasing (x == y in zcsrmv; b == x in solve) */
    ZK_ERR_ZERO_RHS = -8,      /* ||b|| = 0 */
    ZK_ERR_NCCL = -9,          /* NCCL error (multi-GPU) */
    ZK_ERR_UNSUPPORTED = -10   /* feature not built / not available */
};

/* ---- zk_csr_create flags ---- */
enum {
    ZK_PTRS_HOST = 0,          /* arrays are host memory: copied to the device (H2D inside the call) */
    ZK_PTRS_DEVICE = 1,        /* arrays are device memory: copied device-to-device */
    ZK_PTRS_DEVICE_BORROW = 2, /* arrays are device memory and are used in place; they must outlive A (the
                                  SpMV may also keep a library-owned sliced-ELL copy, see spmv_mode) */
    ZK_SKIP_VALIDATE = 4       /* trust the input (no validation pass) */
};

/* ---- solver methods and outcomes ---- */
enum {
    ZK_BICGSTAB = 0,        /* unpreconditioned BiCGStab (O6) */
    ZK_CG = 1,              /* CG, A Hermitian positive definite (O7) */
    ZK_BICGSTAB_JACOBI = 2, /* Jacobi (M = diag A) right-preconditioned BiCGStab, the paper's P-Bi-CGSTAB
                               (P:308); also row-partitioned (the ranks exchange 1/a_jj of their halo
                               columns once); a zero/missing diagonal fails with ZK_ERR_INVALID_CSR */
    ZK_COCG = 3,            /* COCG: CG with the unconjugated form rᵀr for complex SYMMETRIC A (Aᵀ = A, the
                               absorbing Helmholtz matrices); 1 SpMV per iteration */
    ZK_TFQMR = 4            /* TFQMR (Freund 1993, two half-steps per iteration), the paper's P-TFQMR
                               without preconditioner; 2 SpMV per iteration; the convergence test
                               is the quasi-residual bound tau*sqrt(m+1)/||b|| */
};
/* BiCGStab(l) (Sleijpen & Fokkema 1993), the paper's "P-BiCGSTAB parametered (l)" / P-BiCGSTAB(8)
 * without preconditioner (T9/T10): method code ZK_BICGSTAB_L(l), 1 <= l <= 8.  One iteration
 * (iters, hist[j]) is one outer cycle of l BiCG steps + the l-dimensional minimal-residual step,
 * 2l SpMVs; the BiCG part also tests ||r||/||b|| after every step.  Row-partitioned too: the Gram
 * totals ((l+1)² doubles) are allreduced and every rank solves the same l×l system. */
#define ZK_BICGSTAB_L(l) (16 + (l))
enum {
    ZK_CONVERGED = 0, ZK_MAXIT = 1, ZK_BREAKDOWN_RHO = 2, ZK_BREAKDOWN_SIGMA = 3,
    ZK_BREAKDOWN_OMEGA = 4, ZK_NOT_HPD = 5, ZK_NONFINITE = 6
};

typedef struct {
    int64_t n_rows;        /* local rows (this rank) */
    int64_t n_cols;        /* global columns */
    int64_t nnz;           /* local nonzeros */
    int64_t row_begin;     /* first global row of this rank (0 on one GPU) */
    int64_t n_global;      /* global rows (sum over ranks) */
    int32_t max_row_len;
    int32_t lanes_per_row; /* SpMV mapping chosen at create: sub-warp width W */
    double mean_row_len;
    int64_t n_halo;        /* off-rank x entries received per SpMV (0 on one GPU) */
    int32_t borrowed;      /* 1 if the arrays are borrowed (ZK_PTRS_DEVICE_BORROW) */
    int32_t nranks;
    int32_t spmv_mode;     /* 0 = CSR, a sub-warp of lanes_per_row lanes per row; 3 = sliced ELL (SELL-32
                              copy of the matrix, the default unless its padding exceeds 10 % of nnz; a
                              library-owned copy, also for borrowed arrays) */
    int64_t sell_entries;  /* mode 3: stored entries incl. padding (slices of 32 rows, each padded to
                              its longest row); 0 otherwise */
    int64_t interior_rows; /* distributed: rows whose SpMV runs while the halo exchange is in flight
                              (the longest run of 32-row slices referencing no halo column; the
                              boundary rows follow the exchange); 0 on one GPU or with
                              ZK_DIST_OVERLAP=0 (blocking exchange, then the whole SpMV) */
    int32_t csr_values_kept; /* 1 if the library keeps its CSR copy of the values; 0 when the SELL copy
                              is the only one (copied handles above 16384 rows with spmv_mode 3: the
                              library's matrix memory drops from 2× to ≈ 1.2× the CSR input;
                              ZK_KEEP_CSR_VALUES=1 keeps it) */
} zk_csr_info_t;

typedef struct {
    int32_t status;        /* ZK_CONVERGED, ZK_MAXIT, ZK_BREAKDOWN_*, ZK_NOT_HPD, ZK_NONFINITE */
    int32_t iters;         /* completed loop passes (a BiCGStab half-step exit counts as one) */
    double true_relres;    /* ||b - A x|| / ||b|| recomputed at exit */
    int64_t n_spmv;        /* SpMV applications performed (incl. initial residual and final check) */
    double solve_ms;       /* device time of the solve (CUDA events, entry to final check) */
    int32_t loop_mode;     /* 1 = CUDA graph WHILE node, 2 = chunked graph launches, 3 = per-iteration launches
                              (distributed matrices), 5 = the whole loop in one thread-block cluster (small
                              systems); env ZK_LOOP_MODE forces 1, 2, 3 or 5 */
    int32_t gpu_launches;  /* libzk kernels launched by this solve */
    /* in-loop kernel timing from the device global timer (first block start -> last block end),
     * summed over launches: [0] SpMV kernels (BiCGStab K1+K3 / CG K1), [1] fused vector kernels
     * with reductions (BiCGStab K2+K4 / CG K2), [2] init, [3] final true-residual SpMV */
    double kernel_ms[4];
    int32_t kernel_launches[4];
} zk_solve_info;

/* ---- diagnostics ---- */
const char* zk_last_error(void);            /* thread-local message of the last failing call */
const char* zk_status_string(zk_status s);  /* name of a status / outcome code */
int32_t zk_version(void);                   /* 100*major + minor */

/* ---- multi-GPU communicator (row-partitioned runs) ----
 * zk_comm_get_unique_id writes a 128-byte NCCL unique id (rank 0 calls it and
 * broadcasts the bytes, e.g. with torch.distributed).  zk_comm_create wraps
 * ncclCommInitRank on `device`.  A NULL zk_comm everywhere means one GPU.
 * Errors: ZK_ERR_NCCL, ZK_ERR_INVALID_VALUE. The library owns the communicator. */
zk_status zk_comm_get_unique_id(void* id128);
zk_status zk_comm_create(zk_comm* out, const void* id128, int32_t nranks, int32_t rank, int32_t device);
zk_status zk_comm_destroy(zk_comm c);

/* ---- in-process communicator (LOCAL transport): the ranks are host threads of one process ----
 * Same row-partitioned semantics as the NCCL communicator (halo exchange before each SpMV, sums of
 * the reduction partials in RANK ORDER, bitwise identical on every rank), with the data moved by
 * stream-ordered device copies and a rank-order sum kernel, ordered with CUDA events; no device
 * spinning, so several ranks may share ONE GPU (NCCL refuses that): this is how the multi-rank path
 * runs with real halos on a single B200, and how one process can drive several GPUs.
 * zk_local_group_create: a group of nranks (1..16) ranks; the caller owns one reference.
 * zk_comm_create_local: called by EVERY rank concurrently (one host thread each; it rendezvouses
 *   with the other ranks before returning), `device` = the rank's GPU.  Every later collective
 *   call (zk_csr_create/zk_zcsrmv/zk_zdotc/zk_dznrm2/zk_solve with this comm) must likewise be made
 *   by all ranks, each on its own stream; a rank that does not arrive within ZK_LOCAL_TIMEOUT_S
 *   seconds (default 120) makes the others fail with ZK_ERR_NCCL.
 * zk_local_group_destroy drops the caller's reference (the group lives until its comms are gone).
 * Errors: ZK_ERR_INVALID_VALUE (bad rank / count, rank joined twice), ZK_ERR_CUDA, ZK_ERR_NCCL. */
typedef struct zk_local_group_s* zk_local_group;
zk_status zk_local_group_create(zk_local_group* out, int32_t nranks);
zk_status zk_local_group_destroy(zk_local_group g);
zk_status zk_comm_create_local(zk_comm* out, zk_local_group g, int32_t rank, int32_t device);

/* ---- CSR create / upload ("Compressed Sparse Row (CSR)";
 *      upload once before the iterations; invariants S:38-44) ----
 * A          out: new handle.
 * n_rows     rows held by this caller (all rows on one GPU; the rank's block otherwise).
 * n_cols     global number of columns (== global rows for a square operator).
 * nnz        nonzeros in these rows.
 * row_ptr    int64[n_rows+1], row_ptr[0] = 0, non-decreasing, row_ptr[n_rows] = nnz (local).
 * col_idx    int32[nnz], GLOBAL column ids in [0, n_cols), strictly increasing within a row.
 * values     zk_z[nnz]; explicit zeros allowed (structural zeros of the 27-point pattern, L21).
 * flags      ZK_PTRS_HOST | ZK_PTRS_DEVICE | ZK_PTRS_DEVICE_BORROW, optionally | ZK_SKIP_VALIDATE.
 * comm       NULL for one GPU; else this rank's communicator (rows [row_begin, row_begin+n_rows)).
 * row_begin  first global row of this rank (0 on one GPU).
 * s          stream for the copies / validation; the call synchronises s before returning.
 * Errors: ZK_ERR_INVALID_CSR (message names the first bad row), ZK_ERR_NONFINITE,
 *         ZK_ERR_INVALID_VALUE, ZK_ERR_OOM, ZK_ERR_CUDA, ZK_ERR_NCCL.
 * The library owns its device copies (not borrowed arrays) and its scratch; zk_csr_destroy frees them.
 * The large copies come from libzk's own stream-ordered memory pool on the device (not the device's
 * default pool): memory freed by zk_csr_destroy stays reserved for the next zk_csr_create while any
 * handle lives, and the pool is trimmed back to the driver when the last handle is destroyed
 * (environment ZK_POOL=0: plain cudaMalloc/cudaFree).
 * Borrowed arrays (ZK_PTRS_DEVICE_BORROW): the SpMV reads the library's sliced-ELL copy of the values
 * (and ZK_BICGSTAB_JACOBI its cached A·M⁻¹), both built from the borrowed arrays; after changing the
 * values in place call zk_csr_update_values, or the handle keeps using the old values. */
zk_status zk_csr_create(zk_csr* A, int64_t n_rows, int64_t n_cols, int64_t nnz, const int64_t* row_ptr,
                        const int32_t* col_idx, const zk_z* values, uint32_t flags, zk_comm comm,
                        int64_t row_begin, zk_stream s);
zk_status zk_csr_destroy(zk_csr A);
/* New values, same sparsity pattern (e.g. a Helmholtz frequency sweep on one mesh: A = K − k²M for
 * several k, §2):
 *   owned handle (ZK_PTRS_HOST / ZK_PTRS_DEVICE at create): `values` = zk_z[nnz] in the original
 *     CSR order (this rank's rows on >1 GPU), host or device per `flags`, copied into the library;
 *   borrowed handle: update the borrowed values array in place, then call with values = NULL (or
 *     the borrowed pointer itself).
 * The sliced-ELL copy is refilled and the cached Jacobi A·M⁻¹ dropped (rebuilt by the next
 * ZK_BICGSTAB_JACOBI solve).  Values are checked for finiteness unless flags has ZK_SKIP_VALIDATE.
 * Errors: ZK_ERR_NONFINITE (names the first bad entry; the handle then holds the rejected values —
 * call again with finite ones before the next SpMV or solve), ZK_ERR_INVALID_VALUE, ZK_ERR_CUDA.
 * Synchronises s. */
zk_status zk_csr_update_values(zk_csr A, const zk_z* values, uint32_t flags, zk_stream s);
zk_status zk_csr_info(zk_csr A, zk_csr_info_t* info);

/* ---- ZSpMV: y <- alpha*A*x + beta*y (§3, Table 8 "SpMV CSR") ----
 * x: zk_z[n_cols] on one GPU, or this rank's zk_z[n_rows] block (halo exchanged internally).
 * y: zk_z[n_rows].  beta == 0 => y is not read (NaN-safe).  Rows without entries give beta*y.
 * Errors: ZK_ERR_INVALID_VALUE (NULL), ZK_ERR_ALIAS (x == y). Asynchronous on s. */
zk_status zk_zcsrmv(zk_csr A, zk_z alpha, const zk_z* x, zk_z beta, zk_z* y, zk_stream s);

/* ---- zdotc: *result = sum_i conj(x_i) * y_i ("ZDOT"; conjugates the
 *      FIRST argument) ----
 * result is a DEVICE pointer (one zk_z).  Deterministic: fixed grid, fixed-order
 * last-block finish.  With a comm the result is summed over ranks.  n >= 0 (n = 0 gives 0). */
zk_status zk_zdotc(int64_t n, const zk_z* x, const zk_z* y, zk_z* result, zk_comm comm, zk_stream s);

/* ---- dznrm2: *result = sqrt(sum_i re_i^2 + im_i^2) ("ZNORM"; plain sum of
 *      squares, no overflow scaling: inputs must satisfy |x_i| < 1e150, L3) ----
 * result is a DEVICE pointer (one double). With a comm the sum of squares is over all ranks. */
zk_status zk_dznrm2(int64_t n, const zk_z* x, double* result, zk_comm comm, zk_stream s);

/* ---- zaxpy: y <- alpha*x + y; zscal: x <- alpha*x in place ---- */
zk_status zk_zaxpy(int64_t n, zk_z alpha, const zk_z* x, zk_z* y, zk_stream s);
zk_status zk_zscal(int64_t n, zk_z alpha, zk_z* x, zk_stream s);

/* ---- NEXT-4: the paper's remaining BLAS-1 operations ----
 * zk_zassign: x_i <- alpha for i < n ("assign of a vector", §3, Table 2; a fill —
 *             the table's bytes per element imply a write-only pass).
 * zk_zaxmy:   y_i <- x_i * y_i (element-wise product "EWProduct"/ZAXMY, Table 5; the
 *             listing's unused alpha is dropped, L17).  x and y device zk_z[n]; may alias. */
zk_status zk_zassign(int64_t n, zk_z alpha, zk_z* x, zk_stream s);
zk_status zk_zaxmy(int64_t n, const zk_z* x, zk_z* y, zk_stream s);

/* ---- solve(A, b, x0, tol, maxit) (§4: Krylov solve with residual
 *      tolerance, initial guess, maximum iterations) ----
 * method     ZK_BICGSTAB (unpreconditioned BiCGStab, O6), ZK_CG (Hermitian positive definite A, O7) or
 *            ZK_BICGSTAB_JACOBI (P-BiCGStab with M = diag(A); the first call builds A·M⁻¹ in the handle)
 *            or ZK_COCG (complex symmetric A; breakdowns: μ = pᵀAp = 0 → BREAKDOWN_SIGMA,
 *            ρ = rᵀr ≈ 0 → BREAKDOWN_RHO) or ZK_TFQMR (σ = ⟨r̃,v⟩ = 0 → BREAKDOWN_SIGMA,
 *            ρ = ⟨r̃,w⟩ ≈ 0 → BREAKDOWN_RHO; hist[j] is the quasi-residual bound τ_m·sqrt(m+1)/||b||
 *            after the second half step m = 2j, or after the first m = 2j−1 when that converges)
 *            or ZK_BICGSTAB_L(l) (γ = ⟨r̃,Aû⟩ ≈ 0 → BREAKDOWN_SIGMA, ρ ≈ 0 → BREAKDOWN_RHO, a singular
 *            l×l minimal-residual system or ω ≈ 0 → BREAKDOWN_OMEGA).
 * b          device zk_z[n_rows]; must not alias x.
 * x0         device zk_z[n_rows] initial guess, or NULL for zero; may alias x.
 * tol        stop when the recurrence residual ||r_j||/||b|| <= tol (BiCGStab also tests the
 *            half step ||s||/||b||, L6); tol > 0.
 * maxit      >= 1.
 * x          device zk_z[n_rows] output.
 * iters      host int32 out: completed loop passes.
 * resid_hist host double[maxit+1] out: hist[j] = ||r_j||/||b||, hist[0] = ||r_0||/||b||;
 *            entries beyond iters are unspecified.
 * info       host out (may be NULL): outcome status, true relres, SpMV count, device time.
 * workspace  device buffer of >= zk_solve_workspace_size(A, method, maxit) bytes, 256-B aligned.
 * The loop runs device-resident (scalars on the device, no per-iteration host sync);
 * the call synchronises s once at the end and returns.
 * Errors: ZK_ERR_ZERO_RHS, ZK_ERR_INVALID_VALUE, ZK_ERR_DIM, ZK_ERR_ALIAS, ZK_ERR_CUDA, ZK_ERR_NCCL. */
size_t zk_solve_workspace_size(zk_csr A, int32_t method, int32_t maxit);
zk_status zk_solve(zk_csr A, const zk_z* b, const zk_z* x0, double tol, int32_t maxit, int32_t method,
                   zk_z* x, int32_t* iters, double* resid_hist, zk_solve_info* info, void* workspace,
                   size_t ws_bytes, zk_stream s);

#ifdef __cplusplus
}
#endif
#endif /* ZK_H */
