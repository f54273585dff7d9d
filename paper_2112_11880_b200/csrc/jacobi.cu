// jacobi.cu — NEXT-1: Jacobi (diagonal) right preconditioning for BiCGStab, the paper's
// "P-Bi-CGSTAB" (§4; SPEC S:296-322 reads the unnamed preconditioner as Jacobi).
// Right preconditioning with M = diag(A) is BiCGStab on A' = A·M⁻¹ with x = M⁻¹u (the Templates
// P-BiCGSTAB recurrences, scalar for scalar), so instead of two extra vector passes per
// iteration (p̂ = M⁻¹p, ŝ = M⁻¹s) the column scaling is folded into a copy of the values once at
// setup (cached in the handle) and the fused BiCGStab kernels run unchanged on A'.
#include "spmv.cuh"
#include "zk_host.h"

namespace zk {

// diag_i = a_ii (stored entry with col == i), dinv_i = 1/diag_i written out as the oracle does
__global__ void jacobi_diag_kernel(const int64_t* __restrict__ row_ptr, const int* __restrict__ col,
                                   const double2* __restrict__ val, int64_t n, double2* __restrict__ diag,
                                   double2* __restrict__ dinv, unsigned long long* first_bad) {
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
        double2 d = make_double2(0.0, 0.0);
        for (int64_t p = row_ptr[i]; p < row_ptr[i + 1]; p++)
            if (col[p] == i) d = val[p];
        if (d.x == 0.0 && d.y == 0.0) {
            atomicMin(first_bad, (unsigned long long)i);
            d = make_double2(1.0, 0.0);
        }
        diag[i] = d;
        dinv[i] = cdiv(make_double2(1.0, 0.0), d);
    }
}

// the same from the SELL copy (handles that dropped their CSR value copy): row r = slice r/32, lane
// r%32, entry k at sl_ptr[r/32] + 32k + r%32
__global__ void jacobi_diag_sell_kernel(const int64_t* __restrict__ sl_ptr, const int* __restrict__ sl_col,
                                        const double2* __restrict__ sl_val, int64_t n, double2* __restrict__ diag,
                                        double2* __restrict__ dinv, unsigned long long* first_bad) {
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
        const int64_t base = sl_ptr[i >> 5], width = (sl_ptr[(i >> 5) + 1] - base) >> 5;
        double2 d = make_double2(0.0, 0.0);
        for (int64_t k = 0; k < width; k++) {
            const int64_t q = base + 32 * k + (i & 31);
            if (sl_col[q] == i) d = sl_val[q];
        }
        if (d.x == 0.0 && d.y == 0.0) {
            atomicMin(first_bad, (unsigned long long)i);
            d = make_double2(1.0, 0.0);
        }
        diag[i] = d;
        dinv[i] = cdiv(make_double2(1.0, 0.0), d);
    }
}

// a'_ij = a_ij · dinv_j
__global__ void jacobi_scale_kernel(const int* __restrict__ col, const double2* __restrict__ val,
                                    const double2* __restrict__ dinv, int64_t nnz, double2* __restrict__ out) {
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; p < nnz; p += stride) {
        const int c = col[p];
        out[p] = c >= 0 ? cmul(val[p], __ldg(dinv + c)) : make_double2(0.0, 0.0);  // c < 0: SELL padding
    }
}

// out_i = d_i · in_i (x0 → u0 = M x0, u → x = M⁻¹ u); out may alias in
__global__ void cscale_kernel(const double2* __restrict__ d, const double2* in, double2* out, int64_t n) {
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) out[i] = cmul(d[i], in[i]);
}

int64_t dist_gather_len(const zk_csr_s* A);                                         // dist.cu
zk_status dist_halo(const zk_csr_s* A, double2* xg, cudaStream_t s);                // dist.cu
zk_status dist_agree_failed(zk_comm_s* c, bool failed, cudaStream_t s, int* any_failed);  // dist.cu

// Build A·M⁻¹ (CSR values and the SELL copy) once per handle.  On a row-partitioned matrix the
// column scaling needs 1/a_jj of the halo columns too: the ranks exchange their dinv entries once
// through the SpMV's halo plan (dinv is laid out like a gathered vector: [local rows | halo slots]),
// after agreeing on whether any rank lacks a diagonal (so no rank is left in the exchange).
zk_status jacobi_prepare(zk_csr_s* A, cudaStream_t s) {
    // built already?  (jac_diag, not jac_val: a handle whose CSR value copy was dropped keeps A·M⁻¹
    // only in the SELL copy, jac_val stays NULL — keying on it rebuilt, and leaked, A·M⁻¹ on every
    // Jacobi solve above 16384 rows)
    if (A->jac_diag) return ZK_OK;
    const int64_t n = A->n_rows, nnz = A->nnz;
    const int64_t glen = A->dist ? dist_gather_len(A) : n;
    double2 *val = nullptr, *diag = nullptr, *dinv = nullptr;
    unsigned long long* bad = nullptr;
    auto release = [&] {
        dev_free(val);
        dev_free(diag);
        dev_free(dinv);
        dev_free(A->jac_sl_val);
        A->jac_sl_val = nullptr;
    };
    const bool csr_vals = A->val != nullptr;  // false: the SELL copy is the only value array
    cudaError_t e = csr_vals ? dev_alloc(&val, sizeof(double2) * (nnz > 0 ? nnz : 1), s) : cudaSuccess;
    if (e == cudaSuccess) e = dev_alloc(&diag, sizeof(double2) * (n > 0 ? n : 1), s);
    if (e == cudaSuccess) e = dev_alloc(&dinv, sizeof(double2) * (glen > 0 ? glen : 1), s);
    if (e == cudaSuccess) e = scratch_alloc(&bad, sizeof(unsigned long long), s);
    if (e == cudaSuccess) e = cudaMemsetAsync(bad, 0xff, sizeof(unsigned long long), s);
    if (e == cudaSuccess && n > 0) {
        if (csr_vals)
            jacobi_diag_kernel<<<grid_for(n, kBlock, A->dev.num_sms * 8), kBlock, 0, s>>>(A->row_ptr, A->col, A->val, n,
                                                                                         diag, dinv, bad);
        else
            jacobi_diag_sell_kernel<<<grid_for(n, kBlock, A->dev.num_sms * 8), kBlock, 0, s>>>(
                A->sl_ptr, A->sl_col, A->sl_val, n, diag, dinv, bad);
        e = cudaGetLastError();
    }
    unsigned long long hbad = ~0ull;
    if (e == cudaSuccess) e = cudaMemcpyAsync(&hbad, bad, sizeof hbad, cudaMemcpyDeviceToHost, s);
    if (e == cudaSuccess) e = cudaStreamSynchronize(s);
    scratch_free(bad, s);
    bool failed = e != cudaSuccess || hbad != ~0ull;
    if (A->dist) {
        int any = 0;
        const zk_status st = dist_agree_failed(A->comm, failed, s, &any);
        if (st != ZK_OK) {
            release();
            return st;
        }
        if (any && !failed) {
            release();
            return fail(ZK_ERR_INVALID_CSR, "another rank has a row without a stored diagonal (Jacobi preconditioner)");
        }
    }
    if (failed) {
        release();
        if (e != cudaSuccess) return cuda_fail(e, "jacobi_prepare", __FILE__, __LINE__);
        char buf[160];
        snprintf(buf, sizeof buf, "row %lld has no nonzero stored diagonal (Jacobi preconditioner)",
                 (long long)hbad + (long long)A->row_begin);
        return fail(ZK_ERR_INVALID_CSR, buf);
    }
    if (A->dist) {
        const zk_status st = dist_halo(A, dinv, s);  // 1/a_jj of the halo columns
        if (st != ZK_OK) {
            release();
            return st;
        }
    }
    if (nnz > 0 && csr_vals) {
        jacobi_scale_kernel<<<grid_for(nnz, kBlock, A->dev.num_sms * 8), kBlock, 0, s>>>(A->col, A->val, dinv, nnz,
                                                                                        val);
        e = cudaGetLastError();
    }
    if (e == cudaSuccess && A->sl_val) {  // the same scaling of the sliced-ELL copy (SpMV mode 3)
        e = dev_alloc(&A->jac_sl_val, sizeof(double2) * (size_t)(A->sl_nnz > 0 ? A->sl_nnz : 1), s);
        if (e == cudaSuccess && A->sl_nnz > 0) {
            jacobi_scale_kernel<<<grid_for(A->sl_nnz, kBlock, A->dev.num_sms * 8), kBlock, 0, s>>>(
                A->sl_col, A->sl_val, dinv, A->sl_nnz, A->jac_sl_val);
            e = cudaGetLastError();
        }
    }
    if (e == cudaSuccess) e = cudaStreamSynchronize(s);  // pool memory: usable from any stream afterwards
    if (e != cudaSuccess) {
        release();
        return cuda_fail(e, "jacobi_prepare", __FILE__, __LINE__);
    }
    A->jac_val = val;
    A->jac_diag = diag;
    A->jac_dinv = dinv;
    return ZK_OK;
}

zk_status cscale(const zk_csr_s* A, const double2* d, const double2* in, double2* out, cudaStream_t s) {
    if (A->n_rows == 0) return ZK_OK;
    cscale_kernel<<<grid_for(A->n_rows, kBlock, A->dev.num_sms * 8), kBlock, 0, s>>>(d, in, out, A->n_rows);
    ZK_CUDA(cudaGetLastError());
    return ZK_OK;
}

void jacobi_destroy(zk_csr_s* A, bool synced) {
    dev_free(A->jac_val, synced);
    dev_free(A->jac_diag, synced);
    dev_free(A->jac_dinv, synced);
    dev_free(A->jac_sl_val, synced);  // (the SELL copy's A·M⁻¹ values: stale after zk_csr_update_values)
    A->jac_val = A->jac_diag = A->jac_dinv = A->jac_sl_val = nullptr;
}

}  // namespace zk
