// zk_host.h — host-side internals of libzk: error plumbing, the zk_csr handle, device info.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include <string>

#include "../../include/zk.h"
#include "spmv_tma.cuh"

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
    int W = 8;                   // SpMV lanes per row
    int spmv_mode = 0;           // 0 sub-warp CSR (spmv.cuh), 1 TMA-staged tiles, 2 blocked-4, 3 sliced ELL (sell.cu)
    zk::TmaPlan tma{};
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
// Big per-handle device arrays (CSR copy, SELL copy, Jacobi values) come from the device's
// stream-ordered memory pool with the release threshold raised, so memory freed by one handle is
// reused by the next create instead of being unmapped and re-mapped (and re-cleared) by the driver:
// measured C4 (8.6 GB per handle), back-to-back create/destroy — zk_csr_create 88-772 ms and
// zk_csr_destroy 8-192 ms with cudaMalloc/cudaFree.  ZK_POOL=0 restores cudaMalloc/cudaFree.
// The pool keeps the memory reserved for libzk after a handle is destroyed.
inline bool pool_enabled() {
    static int on = -1;
    if (on < 0) {
        const char* e = getenv("ZK_POOL");
        on = (e && atoi(e) == 0) ? 0 : 1;
    }
    return on == 1;
}
inline cudaError_t dev_alloc(void** p, size_t bytes, cudaStream_t s) {
    if (!pool_enabled()) return cudaMalloc(p, bytes);
    static int dev_done = -1;  // per process, first device used (multi-device processes: per create)
    int dev = 0;
    cudaGetDevice(&dev);
    if (dev_done != dev) {
        cudaMemPool_t pool;
        if (cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
            uint64_t thr = UINT64_MAX;
            cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
        }
        dev_done = dev;
    }
    return cudaMallocAsync(p, bytes, s);
}
template <class T>
inline cudaError_t dev_alloc(T** p, size_t bytes, cudaStream_t s) {
    return dev_alloc(reinterpret_cast<void**>(p), bytes, s);
}
// p must not be in use by pending work (the device is synchronised first, as cudaFree would)
inline void dev_free(void* p) {
    if (!p) return;
    if (!pool_enabled()) {
        cudaFree(p);
        return;
    }
    cudaDeviceSynchronize();
    cudaFreeAsync(p, 0);
}
// Call f(std::integral_constant<int, W>, std::integral_constant<int, MODE>) for the matrix's SpMV
// mapping (instantiated combinations: sub-warp W ∈ {2,4,8,16,32}, TMA W ∈ {4,8,16}).
template <class F>
zk_status with_spmv(const zk_csr_s* A, F&& f) {
    using std::integral_constant;
    if (A->spmv_mode == 3) return f(integral_constant<int, 32>{}, integral_constant<int, 3>{});
    if (A->spmv_mode == 2) {
        switch (A->W) {
            case 4: return f(integral_constant<int, 4>{}, integral_constant<int, 2>{});
            case 16: return f(integral_constant<int, 16>{}, integral_constant<int, 2>{});
            default: return f(integral_constant<int, 8>{}, integral_constant<int, 2>{});
        }
    }
    if (A->spmv_mode == 1) {
        switch (A->W) {
            case 4: return f(integral_constant<int, 4>{}, integral_constant<int, 1>{});
            case 16: return f(integral_constant<int, 16>{}, integral_constant<int, 1>{});
            default: return f(integral_constant<int, 8>{}, integral_constant<int, 1>{});
        }
    }
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
    return CsrDev{A->row_ptr, A->col, A->val, A->n_rows, A->nnz, A->sl_ptr, A->sl_col, A->sl_val, 0, ns, ns, 0, 1};
}

struct LaunchCfg {
    int grid;
    int smem;
};
// grid and dynamic smem for an SpMV kernel of A (TMA: one CTA per resident slot, ≤ n_tiles)
inline LaunchCfg spmv_cfg(const zk_csr_s* A, const void* kernel, int W, int mode) {
    if (mode == 1) {
        const int smem = A->tma.smem_bytes;
        int cap = A->dev.num_sms * blocks_per_sm(kernel, smem);
        if (cap > kMaxGrid) cap = kMaxGrid;
        int64_t g = A->tma.n_tiles < cap ? A->tma.n_tiles : cap;
        return {(int)(g < 1 ? 1 : g), smem};
    }
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
