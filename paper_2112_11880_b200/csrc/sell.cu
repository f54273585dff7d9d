// sell.cu — the sliced-ELL (SELL-32) copy of a CSR matrix used by SpMV mode 3 (spmv.cuh
// spmv_body_sell).  The ABI stays CSR (§3); this is an internal HBM layout
// chosen at zk_csr_create: slices of 32 consecutive rows, each padded to its longest row and
// stored column-major, so a warp's loads of values / columns are contiguous 512 / 128-byte runs
// and its epilogue touches 32 consecutive rows.  Built on the device from the (validated,
// renumbered on >1 GPU) CSR arrays; padding = col −1, value 0 (skipped by the kernel).
#include <vector>

#include "spmv.cuh"
#include "zk_host.h"

namespace zk {

// width of each slice = its longest row
__global__ void sell_width_kernel(const int64_t* __restrict__ row_ptr, int64_t n, int64_t n_sl, int* __restrict__ w) {
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t s = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; s < n_sl; s += stride) {
        int m = 0;
        const int64_t r1 = (s + 1) * 32 < n ? (s + 1) * 32 : n;
        for (int64_t r = s * 32; r < r1; r++) {
            const int len = (int)(row_ptr[r + 1] - row_ptr[r]);
            m = len > m ? len : m;
        }
        w[s] = m;
    }
}

// thread per (padded) row: entry k of row r goes to sl_ptr[r/32] + k·32 + r%32
__global__ void sell_fill_kernel(const int64_t* __restrict__ row_ptr, const int* __restrict__ col,
                                 const double2* __restrict__ val, int64_t n, int64_t n_sl,
                                 const int64_t* __restrict__ sl_ptr, int* __restrict__ sl_col,
                                 double2* __restrict__ sl_val) {
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; r < n_sl * 32; r += stride) {
        const int64_t s = r >> 5, lane = r & 31;
        const int64_t base = sl_ptr[s];
        const int width = (int)((sl_ptr[s + 1] - base) >> 5);
        const int64_t rs = r < n ? row_ptr[r] : 0;
        const int len = r < n ? (int)(row_ptr[r + 1] - rs) : 0;
        for (int k = 0; k < width; k++) {
            const int64_t d = base + (int64_t)k * 32 + lane;
            if (k < len) {
                sl_col[d] = col[rs + k];
                sl_val[d] = val[rs + k];
            } else {
                sl_col[d] = -1;
                sl_val[d] = make_double2(0.0, 0.0);
            }
        }
    }
}

void sell_destroy(zk_csr_s* A, bool synced) {
    dev_free(A->sl_ptr, synced);
    dev_free(A->sl_col, synced);
    dev_free(A->sl_val, synced);
    dev_free(A->jac_sl_val, synced);
    A->sl_ptr = nullptr;
    A->sl_col = nullptr;
    A->sl_val = nullptr;
    A->jac_sl_val = nullptr;
    A->n_slices = A->sl_nnz = 0;
}

// Build the SELL-32 copy of A (its current CSR arrays).  Returns ZK_OK and leaves A->sl_* set.
zk_status sell_build(zk_csr_s* A, cudaStream_t s) {
    sell_destroy(A);
    const int64_t n = A->n_rows;
    const int64_t n_sl = (n + 31) / 32;
    A->n_slices = n_sl;
    int* w = nullptr;
    cudaError_t e = dev_alloc(&A->sl_ptr, sizeof(int64_t) * (size_t)(n_sl + 1), s);
    if (e == cudaSuccess) e = scratch_alloc(&w, sizeof(int) * (size_t)(n_sl > 0 ? n_sl : 1), s);
    if (e != cudaSuccess) {
        scratch_free(w, s);
        sell_destroy(A);
        return cuda_fail(e, "sell_build alloc", __FILE__, __LINE__);
    }
    const int grid = A->dev.num_sms * 8;
    if (n_sl > 0) sell_width_kernel<<<grid_for(n_sl, kBlock, grid), kBlock, 0, s>>>(A->row_ptr, n, n_sl, w);
    std::vector<int> hw((size_t)n_sl);
    std::vector<int64_t> hp((size_t)n_sl + 1);
    if (n_sl > 0) e = cudaMemcpyAsync(hw.data(), w, sizeof(int) * (size_t)n_sl, cudaMemcpyDeviceToHost, s);
    if (e == cudaSuccess) e = cudaStreamSynchronize(s);
    scratch_free(w, s);
    if (e != cudaSuccess) {
        sell_destroy(A);
        return cuda_fail(e, "sell_build widths", __FILE__, __LINE__);
    }
    hp[0] = 0;
    for (int64_t i = 0; i < n_sl; i++) hp[(size_t)i + 1] = hp[(size_t)i] + 32 * (int64_t)hw[(size_t)i];
    A->sl_nnz = hp[(size_t)n_sl];
    e = cudaMemcpyAsync(A->sl_ptr, hp.data(), sizeof(int64_t) * (size_t)(n_sl + 1), cudaMemcpyHostToDevice, s);
    if (e == cudaSuccess) e = dev_alloc(&A->sl_col, sizeof(int) * (size_t)(A->sl_nnz > 0 ? A->sl_nnz : 1), s);
    if (e == cudaSuccess) e = dev_alloc(&A->sl_val, sizeof(double2) * (size_t)(A->sl_nnz > 0 ? A->sl_nnz : 1), s);
    if (e == cudaSuccess && n_sl > 0) {
        sell_fill_kernel<<<grid_for(n_sl * 32, kBlock, grid), kBlock, 0, s>>>(A->row_ptr, A->col, A->val, n, n_sl,
                                                                           A->sl_ptr, A->sl_col, A->sl_val);
        e = cudaGetLastError();
    }
    if (e == cudaSuccess) e = cudaStreamSynchronize(s);  // hp is host memory of this frame
    if (e != cudaSuccess) {
        sell_destroy(A);
        return cuda_fail(e, "sell_build", __FILE__, __LINE__);
    }
    return ZK_OK;
}

// Re-fill the SELL values (and columns) from the CSR arrays after zk_csr_update_values: same
// pattern, so the slice layout (sl_ptr) is unchanged.
zk_status sell_refill(zk_csr_s* A, const double2* val, cudaStream_t s) {
    const int64_t n_sl = A->n_slices;
    if (n_sl > 0) {
        sell_fill_kernel<<<grid_for(n_sl * 32, kBlock, A->dev.num_sms * 8), kBlock, 0, s>>>(
            A->row_ptr, A->col, val, A->n_rows, n_sl, A->sl_ptr, A->sl_col, A->sl_val);
        ZK_CUDA(cudaGetLastError());
    }
    return ZK_OK;
}

}  // namespace zk
