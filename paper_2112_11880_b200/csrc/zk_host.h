// zk_host.h — host-side internals of libzk: error plumbing, the zk_csr handle, device info.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include <string>

#include "../../include/zk.h"
#include "spmv.cuh"

namespace zk {

void set_error(const std::string& msg);
zk_status fail(zk_status code, const std::string& msg);
zk_status cuda_fail(cudaError_t e, const char* what, const char* file, int line);

#define ZK_CUDA(call)                                                        \
    do {                                                                     \
        cudaError_t _e = (call);                                             \
        if (_e != cudaSuccess) return ::zk::cuda_fail(_e, #call, __FILE__, __LINE__); \
    } while (0)

#define ZK_TRY(call)                      \
    do {                                  \
        zk_status _s = (call);            \
        if (_s != ZK_OK) return _s;       \
    } while (0)

struct DeviceInfo {
    int device = -1;
    int num_sms = 0;
};
zk_status current_device(DeviceInfo* out);

// cached blocks-per-SM for a kernel (occupancy API) at `smem` dynamic shared memory bytes; also
// raises the kernel's dynamic shared memory limit when smem > 48 KB
int blocks_per_sm(const void* kernel, int smem = 0);

struct GraphCache {
    const void* ws = nullptr;
    int method = -1;
    int mode = 0;
    int maxit = -1;  // the workspace layout (hist, partials, vectors) depends on maxit
    cudaGraphExec_t exec = nullptr;
    cudaGraph_t graph = nullptr;
    unsigned long long cond = 0;  // cudaGraphConditionalHandle
};

}  // namespace zk

struct zk_comm_s;

struct zk_csr_s {
    int64_t n_rows = 0, n_cols = 0, nnz = 0, row_begin = 0, n_global = 0;
    int64_t* row_ptr = nullptr;  // device
    int* col = nullptr;          // device (local column ids after the halo renumbering on >1 GPU)
    double2* val = nullptr;      // device
    bool owned = false;
    bool counted = false;        // included in the live-handle count (pool trim at zero)
    int W = 8;                   // SpMV lanes per row
    int spmv_mode = 0;           // 0 sub-warp CSR (spmv.cuh), 3 sliced ELL (sell.cu)
    // Jacobi right preconditioning (jacobi.cu), built on the first ZK_BICGSTAB_JACOBI solve
    double2* jac_val = nullptr;   // a_ij / a_jj
    double2* jac_diag = nullptr;  // a_ii
    double2* jac_dinv = nullptr;  // 1 / a_ii
    double2* jac_sl_val = nullptr;  // A·M⁻¹ in the sliced-ELL layout (SpMV mode 3)
    // sliced-ELL (SELL-32) copy of the matrix, SpMV mode 3 (sell.cu)
    int64_t* sl_ptr = nullptr;
    int* sl_col = nullptr;
    double2* sl_val = nullptr;
    int64_t n_slices = 0, sl_nnz = 0;
    int max_len = 0;
    double mean_len = 0.0;
    zk::DeviceInfo dev;
    // cluster solver (loop mode 5): the most nonzeros of one CTA's row block at cluster size cl_cs
    int cl_cs = 0;
    int64_t cl_nnz_max = -1;
    // zk_solve readback: pinned host staging for the context + residual history (one stream sync,
    // no pageable copies) and the two timing events, kept across solves
    void* pinned = nullptr;
    size_t pinned_bytes = 0;
    cudaEvent_t ev[2] = {nullptr, nullptr};
    cudaStream_t cap_stream = nullptr;  // private stream used for graph capture
    zk::GraphCache graph[8];            // per solver method code (ZK_BICGSTAB .. ZK_TFQMR)
    zk_comm_s* comm = nullptr;
    // distributed: halo plan (see dist.cu)
    void* dist = nullptr;
};

#include <cstdint>
#include <cstdlib>
#include <type_traits>

namespace zk {
// Big per-handle device arrays (CSR copy, SELL copy, Jacobi values) come from a PRIVATE
// stream-ordered memory pool per device (cudaMemPoolCreate; release threshold raised), so memory
// freed by one handle is reused by the next create instead of being unmapped and re-mapped (and
// re-cleared) by the driver: measured C4 (8.6 GB per handle), back-to-back create/destroy —
// zk_csr_create 88-772 ms and zk_csr_destroy 8-192 ms with cudaMalloc/cudaFree.  The pool is
// libzk's own (the device's default pool, which PyTorch and other libraries may use, keeps its
// settings), and it is trimmed back to the driver when the last handle is destroyed.
// ZK_POOL=0 restores cudaMalloc/cudaFree.
inline bool pool_enabled() {
    static int on = -1;
    if (on < 0) {
        const char* e = getenv("ZK_POOL");
        on = (e && atoi(e) == 0) ? 0 : 1;
    }
    return on == 1;
}
cudaMemPool_t dev_pool(int device);  // api.cu: libzk's pool on `device` (created on first use)
void handle_count(int delta);         // api.cu: live zk_csr handles; 0 → trim every pool
inline cudaError_t dev_alloc(void** p, size_t bytes, cudaStream_t s) {
    if (!pool_enabled()) return cudaMalloc(p, bytes);
    int dev = 0;
    cudaGetDevice(&dev);
    cudaMemPool_t pool = dev_pool(dev);
    if (!pool) return cudaMallocAsync(p, bytes, s);  // no private pool: the default pool
    return cudaMallocFromPoolAsync(p, bytes, pool, s);
}
template <class T>
inline cudaError_t dev_alloc(T** p, size_t bytes, cudaStream_t s) {
    return dev_alloc(reinterpret_cast<void**>(p), bytes, s);
}
// p must not be in use by pending work: the device is synchronised first, as cudaFree would,
// unless the caller already did (synced = true: zk_csr_destroy syncs once for all its arrays).
// (cudaFreeAsync returns a pool allocation to its own pool; a cudaMalloc'd one — ZK_POOL=0 or no
// pool support — is freed by cudaFree.)
inline void dev_free(void* p, bool synced = false) {
    if (!p) return;
    if (!pool_enabled()) {
        cudaFree(p);
        return;
    }
    if (!synced) cudaDeviceSynchronize();
    cudaFreeAsync(p, 0);
}
// After a batch of dev_free calls: wait until stream 0 has executed the frees, so the pool's
// opportunistic reuse hands the blocks to the next allocation on ANY stream.  Without it, a create
// on another (non-blocking) stream right after a destroy could not reuse them and the pool mapped
// fresh memory (measured C4: zk_csr_create 85 ms → 660-1420 ms on a torch side stream).
inline void dev_free_done() {
    if (pool_enabled()) cudaStreamSynchronize(0);
}
// Small per-call device scratch (validation flags, SELL widths, ...): a stream-ordered pool
// allocation on s, returned on s.  No cudaMalloc / cudaFree on the create / solve / destroy path:
// with GBs of pinned host memory in the process (torch pin_memory), cudaFree of a 16-byte buffer
// measured 2-580 ms and cudaFreeHost of the readback staging up to 474 ms (tools/e2e_probe.py
// with ZK_TRACE=1, profiles/r02_e2e_probe.txt) — the driver's free path, not the GPU.
template <class T>
inline cudaError_t scratch_alloc(T** p, size_t bytes, cudaStream_t s) {
    return dev_alloc(reinterpret_cast<void**>(p), bytes, s);
}
inline void scratch_free(void* p, cudaStream_t s) {
    if (!p) return;
    if (!pool_enabled()) {
        cudaFree(p);
        return;
    }
    cudaFreeAsync(p, s);
}
// Pinned host staging (zk_solve's context + history readback) from a process-wide free list:
// handles take a buffer at their first solve and give it back at destroy (no cudaMallocHost /
// cudaFreeHost per handle).  api.cu.
cudaError_t pinned_get(void** p, size_t bytes, size_t* got);
void pinned_put(void* p, size_t bytes);
void sell_destroy(zk_csr_s* A, bool synced = false);    // sell.cu  (synced: the device is already idle)
constexpr int64_t kCsrValuesKeepRows = 16384;           // ≤ this: the CSR value copy stays (cluster solver)
void jacobi_destroy(zk_csr_s* A, bool synced = false);  // jacobi.cu

// Call f(std::integral_constant<int, W>, std::integral_constant<int, MODE>) for the matrix's SpMV
// mapping (instantiated: SELL-32 (W = 32, MODE 3) and the CSR sub-warp kernel, W ∈ {2,4,8,16,32}).
template <class F>
zk_status with_spmv(const zk_csr_s* A, F&& f) {
    using std::integral_constant;
    if (A->spmv_mode == 3) return f(integral_constant<int, 32>{}, integral_constant<int, 3>{});
    switch (A->W) {
        case 2: return f(integral_constant<int, 2>{}, integral_constant<int, 0>{});
        case 4: return f(integral_constant<int, 4>{}, integral_constant<int, 0>{});
        case 8: return f(integral_constant<int, 8>{}, integral_constant<int, 0>{});
        case 16: return f(integral_constant<int, 16>{}, integral_constant<int, 0>{});
        default: return f(integral_constant<int, 32>{}, integral_constant<int, 0>{});
    }
}

inline CsrDev csr_dev(const zk_csr_s* A) {
    const int ns = (int)A->n_slices;
    return CsrDev{A->row_ptr, A->col, A->val, A->n_rows, A->nnz, A->sl_ptr, A->sl_col, A->sl_val, 0, ns, ns, 0, 1, 0, 0};
}

struct LaunchCfg {
    int grid;
    int smem;
};
// grid (and dynamic smem: none) of an SpMV kernel of A: at most one wave of resident CTAs
inline LaunchCfg spmv_cfg(const zk_csr_s* A, const void* kernel, int W, int mode) {
    int cap = A->dev.num_sms * blocks_per_sm(kernel, 0);
    if (cap > kMaxGrid) cap = kMaxGrid;
    if (mode == 3) return {grid_for(A->n_slices, kWarps, cap), 0};  // one warp per 32-row slice
    return {grid_for(A->n_rows, kBlock / W, cap), 0};
}
// SELL launch over the slice set of `a` (a partial range of a distributed SpMV)
inline LaunchCfg spmv_cfg_part(const zk_csr_s* A, const void* kernel, const CsrDev& a) {
    int cap = A->dev.num_sms * blocks_per_sm(kernel, 0);
    if (cap > kMaxGrid) cap = kMaxGrid;
    return {grid_for(a.sl_cnt > 0 ? a.sl_cnt : 1, kWarps, cap), 0};
}
}  // namespace zk
