// api.cu — libzk diagnostics, CSR create/upload/validate and ZSpMV (A2).
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <mutex>
#include <string>
#include <unordered_map>
#include <vector>

#include "spmv.cuh"
#include "zk_host.h"

// ------------------------------------------------------------------ diagnostics
namespace zk {
static thread_local std::string g_err;

void set_error(const std::string& msg) { g_err = msg; }
zk_status fail(zk_status code, const std::string& msg) {
    g_err = std::string(zk_status_string(code)) + ": " + msg;
    return code;
}
zk_status cuda_fail(cudaError_t e, const char* what, const char* file, int line) {
    char buf[512];
    snprintf(buf, sizeof buf, "%s failed: %s (%s:%d)", what, cudaGetErrorString(e), file, line);
    g_err = buf;
    return e == cudaErrorMemoryAllocation ? ZK_ERR_OOM : ZK_ERR_CUDA;
}

zk_status current_device(DeviceInfo* out) {
    ZK_CUDA(cudaGetDevice(&out->device));
    ZK_CUDA(cudaDeviceGetAttribute(&out->num_sms, cudaDevAttrMultiProcessorCount, out->device));
    return ZK_OK;
}

static std::mutex g_pool_mu;
static std::unordered_map<int, cudaMemPool_t> g_pools;
static int g_handles = 0;

cudaMemPool_t dev_pool(int device) {
    std::lock_guard<std::mutex> lk(g_pool_mu);
    auto it = g_pools.find(device);
    if (it != g_pools.end()) return it->second;
    cudaMemPoolProps props = {};
    props.allocType = cudaMemAllocationTypePinned;
    props.location.type = cudaMemLocationTypeDevice;
    props.location.id = device;
    cudaMemPool_t pool = nullptr;
    if (cudaMemPoolCreate(&pool, &props) != cudaSuccess) {
        cudaGetLastError();
        pool = nullptr;  // no pool support: cudaMalloc
    } else {
        uint64_t thr = UINT64_MAX;
        cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
    }
    g_pools[device] = pool;
    return pool;
}

static std::mutex g_pin_mu;
static std::vector<std::pair<void*, size_t>> g_pin_free;  // (buffer, bytes), reused across handles
constexpr size_t kPinMin = 64 * 1024, kPinKeep = 64;

cudaError_t pinned_get(void** p, size_t bytes, size_t* got) {
    {
        std::lock_guard<std::mutex> lk(g_pin_mu);
        size_t best = g_pin_free.size();
        for (size_t i = 0; i < g_pin_free.size(); i++)
            if (g_pin_free[i].second >= bytes && (best == g_pin_free.size() || g_pin_free[i].second < g_pin_free[best].second))
                best = i;
        if (best < g_pin_free.size()) {
            *p = g_pin_free[best].first;
            *got = g_pin_free[best].second;
            g_pin_free.erase(g_pin_free.begin() + (std::ptrdiff_t)best);
            return cudaSuccess;
        }
    }
    const size_t b = bytes > kPinMin ? bytes : kPinMin;
    cudaError_t e = cudaMallocHost(p, b);
    *got = e == cudaSuccess ? b : 0;
    return e;
}
void pinned_put(void* p, size_t bytes) {
    if (!p) return;
    {
        std::lock_guard<std::mutex> lk(g_pin_mu);
        if (g_pin_free.size() < kPinKeep) {
            g_pin_free.emplace_back(p, bytes);
            return;
        }
    }
    cudaFreeHost(p);
}

void handle_count(int delta) {
    std::lock_guard<std::mutex> lk(g_pool_mu);
    g_handles += delta;
    if (g_handles == 0)
        for (auto& kv : g_pools)
            if (kv.second) cudaMemPoolTrimTo(kv.second, 0);  // no live handle: give the memory back
}

int blocks_per_sm(const void* kernel, int smem) {
    static std::mutex mu;
    static std::unordered_map<const void*, std::pair<int, int>> cache;  // kernel → (smem, blocks)
    std::lock_guard<std::mutex> lk(mu);
    auto it = cache.find(kernel);
    if (it != cache.end() && it->second.first == smem) return it->second.second;
    if (smem > 48 * 1024) cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    int b = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b, kernel, kBlock, smem) != cudaSuccess || b < 1) b = 1;
    cache[kernel] = {smem, b};
    return b;
}
}  // namespace zk

extern "C" const char* zk_last_error(void) { return zk::g_err.c_str(); }

extern "C" int32_t zk_version(void) { return 200; }  // 2.0: zk_csr_info_t without the TMA fields, + interior_rows, csr_values_kept

extern "C" const char* zk_status_string(zk_status s) {
    switch (s) {
        case ZK_OK: return "ZK_OK";
        case ZK_ERR_INVALID_VALUE: return "ZK_ERR_INVALID_VALUE";
        case ZK_ERR_INVALID_CSR: return "ZK_ERR_INVALID_CSR";
        case ZK_ERR_NONFINITE: return "ZK_ERR_NONFINITE";
        case ZK_ERR_DIM: return "ZK_ERR_DIM";
        case ZK_ERR_OOM: return "ZK_ERR_OOM";
        case ZK_ERR_CUDA: return "ZK_ERR_CUDA";
        case ZK_ERR_ALIAS: return "ZK_ERR_ALIAS";
        case ZK_ERR_ZERO_RHS: return "ZK_ERR_ZERO_RHS";
        case ZK_ERR_NCCL: return "ZK_ERR_NCCL";
        case ZK_ERR_UNSUPPORTED: return "ZK_ERR_UNSUPPORTED";
        default: return "ZK_UNKNOWN_STATUS";
    }
}

// ------------------------------------------------------------------ validation
namespace zk {
enum : unsigned { V_OK = 0, V_ROWPTR = 1, V_COLRANGE = 2, V_COLORDER = 3, V_NONFINITE = 4 };

struct ValidateOut {
    unsigned long long first_bad;  // (row << 3) | code, min over offending rows
    unsigned int max_len;
};

__global__ void __launch_bounds__(kBlock) validate_kernel(const int64_t* __restrict__ row_ptr,
                                                         const int* __restrict__ col,
                                                         const double2* __restrict__ val, int64_t n_rows,
                                                         int64_t n_cols, int64_t nnz, int stats_only,
                                                         ValidateOut* out) {
    unsigned int my_max = 0;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n_rows; i += stride) {
        const int64_t rs = row_ptr[i], re = row_ptr[i + 1];
        unsigned code = V_OK;
        if (stats_only) {
            if (re - rs > (int64_t)my_max) my_max = (unsigned)(re - rs);
            continue;
        }
        if ((i == 0 && rs != 0) || re < rs || re > nnz || (i == n_rows - 1 && re != nnz)) {
            code = V_ROWPTR;
        } else {
            if ((uint64_t)(re - rs) > my_max) my_max = (unsigned)(re - rs);
            int prev = -1;
            for (int64_t p = rs; p < re; p++) {
                const int c = col[p];
                if (c < 0 || c >= n_cols) { code = V_COLRANGE; break; }
                if (c <= prev) { code = V_COLORDER; break; }
                prev = c;
                const double2 v = val[p];
                if (!isfinite(v.x) || !isfinite(v.y)) { code = V_NONFINITE; break; }
            }
        }
        if (code != V_OK) atomicMin(&out->first_bad, ((unsigned long long)i << 3) | code);
    }
    atomicMax(&out->max_len, my_max);
}

// first non-finite entry of a value array (zk_csr_update_values)
__global__ void __launch_bounds__(kBlock) nonfinite_kernel(const double2* __restrict__ val, int64_t nnz,
                                                          unsigned long long* first) {
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; p < nnz; p += stride) {
        const double2 v = val[p];
        if (!isfinite(v.x) || !isfinite(v.y)) atomicMin(first, (unsigned long long)p);
    }
}

// ------------------------------------------------------------------ ZSpMV kernel (zk_zcsrmv)
struct EpiAxpby {
    static constexpr int K = 0;
    using Pre = double2;
    double2 alpha, beta;
    double2* __restrict__ y;
    bool beta_zero;
    __device__ Pre pre(int64_t i) const { return beta_zero ? make_double2(0, 0) : y[i]; }
    __device__ void row(int64_t i, double2 s, const Pre& yo, double (&)[1]) {
        double2 r = cmul(alpha, s);
        if (!beta_zero) r = cadd(r, cmul(beta, yo));
        y[i] = r;
    }
    __device__ void finish(double (&)[1], int = 0, int = 0) {}
};

template <int W, int MODE>
__global__ void __launch_bounds__(kBlock, spmv_min_blocks(MODE)) zcsrmv_kernel(CsrDev A, const double2* __restrict__ x,
                                                                              EpiAxpby epi) {
    spmv_any<W, MODE>(A, x, epi);
}

zk_status zcsrmv_local(const zk_csr_s* A, double2 alpha, const double2* x, double2 beta, double2* y,
                       cudaStream_t s) {
    return with_spmv(A, [&](auto wc, auto mc) -> zk_status {
        constexpr int W = decltype(wc)::value, MODE = decltype(mc)::value;
        const void* k = (const void*)zcsrmv_kernel<W, MODE>;
        const LaunchCfg L = spmv_cfg(A, k, W, MODE);
        const CsrDev d = csr_dev(A);
        EpiAxpby e{alpha, beta, y, beta.x == 0.0 && beta.y == 0.0};
        zcsrmv_kernel<W, MODE><<<L.grid, kBlock, L.smem, s>>>(d, x, e);
        ZK_CUDA(cudaGetLastError());
        return ZK_OK;
    });
}

// one part (a slice set, CsrDev) of a SELL SpMV: the interior / boundary launches of dist.cu
zk_status zcsrmv_part(const zk_csr_s* A, double2 alpha, const double2* x, double2 beta, double2* y,
                      cudaStream_t s, const CsrDev& part) {
    const void* k = (const void*)zcsrmv_kernel<32, 3>;
    const LaunchCfg L = spmv_cfg_part(A, k, part);
    EpiAxpby e{alpha, beta, y, beta.x == 0.0 && beta.y == 0.0};
    zcsrmv_kernel<32, 3><<<L.grid, kBlock, 0, s>>>(part, x, e);
    ZK_CUDA(cudaGetLastError());
    return ZK_OK;
}

// SpMV mapping.  Default: the sliced-ELL copy (mode 3) — on C4 zk_zcsrmv 647 µs vs 812 µs for the
// best CSR mapping (profiles/r01_sell.md) — unless its padding exceeds kSellMaxPad of the nonzeros
// (checked after the build; then the CSR sub-warp kernel, mode 0, with W ≈ mean row length / 8
// lanes per row).  ZK_SPMV_MODE=0/3 forces a mapping, ZK_SPMV_W the lanes of mode 0.  (Round 1's
// TMA-staged and blocked-4 CSR mappings measured slower on every shape and were removed.)
constexpr double kSellMaxPad = 0.10;
static void choose_mapping(zk_csr_s* A, int force_mode = -1) {
    int mode = 3, w = -1;
    if (const char* e = getenv("ZK_SPMV_MODE")) mode = atoi(e) == 0 ? 0 : 3;
    if (force_mode >= 0) mode = force_mode;
    if (const char* e = getenv("ZK_SPMV_W")) w = atoi(e);
    A->spmv_mode = mode;
    if (mode == 3) {
        A->W = 32;  // a warp per 32-row slice (sell.cu)
        return;
    }
    if (!(w == 2 || w == 4 || w == 8 || w == 16 || w == 32)) {
        // ≈ 8 nonzeros per lane (two chunks of U = 4): W = 4 for the 27-point rows
        w = 2;
        while (w < 32 && 8.0 * w < A->mean_len) w *= 2;
    }
    A->W = w;
}

zk_status dist_setup(zk_csr_s* A, const int64_t* h_row_ptr, const int* h_col, cudaStream_t s);  // dist.cu
void dist_destroy(zk_csr_s* A);                                                                  // dist.cu
zk_status dist_zcsrmv(const zk_csr_s* A, double2 alpha, const double2* x, double2 beta, double2* y,
                      cudaStream_t s);                                                           // dist.cu
int64_t dist_n_halo(const zk_csr_s* A);                                                          // dist.cu
zk_status sell_build(zk_csr_s* A, cudaStream_t s);                                               // sell.cu
int dist_nranks(const zk_csr_s* A);                                                              // dist.cu
zk_status dist_agree_failed(zk_comm_s* c, bool failed, cudaStream_t s, int* any_failed);         // dist.cu
int64_t dist_interior_rows(const zk_csr_s* A);                                                   // dist.cu
}  // namespace zk

using namespace zk;

// everything of zk_csr_create that one rank does alone: argument checks, device arrays, validation,
// row statistics, SpMV mapping.  *outA is set as soon as a handle exists (the caller frees it on error).
static zk_status csr_create_local(zk_csr_s** outA, int64_t n_rows, int64_t n_cols, int64_t nnz,
                                  const int64_t* row_ptr, const int32_t* col_idx, const zk_z* values,
                                  uint32_t flags, zk_comm comm, int64_t row_begin, cudaStream_t s) {
    if (n_rows < 0 || n_cols < 0 || nnz < 0) return fail(ZK_ERR_INVALID_VALUE, "negative size");
    if (n_cols > INT32_MAX) return fail(ZK_ERR_INVALID_VALUE, "n_cols exceeds int32 column ids");
    if (n_rows >= INT32_MAX) return fail(ZK_ERR_INVALID_VALUE, "n_rows must be < 2^31 per matrix (rank)");
    if (!row_ptr || (nnz > 0 && (!col_idx || !values))) return fail(ZK_ERR_INVALID_VALUE, "NULL array");
    if (n_rows == 0 && nnz != 0) return fail(ZK_ERR_INVALID_CSR, "n_rows = 0 but nnz > 0");
    const uint32_t where = flags & 3u;
    if (where == 3u) return fail(ZK_ERR_INVALID_VALUE, "bad flags");
    if (comm && where == ZK_PTRS_DEVICE_BORROW)
        return fail(ZK_ERR_INVALID_VALUE, "distributed matrices are renumbered: use ZK_PTRS_HOST or ZK_PTRS_DEVICE");
    zk_csr_s* A = new zk_csr_s();
    *outA = A;
    auto cleanup = [&](zk_status st) { return st; };
    zk_status st = current_device(&A->dev);
    if (st != ZK_OK) return cleanup(st);
    A->n_rows = n_rows;
    A->n_cols = n_cols;
    A->nnz = nnz;
    A->row_begin = row_begin;
    A->n_global = n_rows;
    A->comm = comm;

    // ---- device arrays (copy or borrow); 16-B aligned by cudaMalloc
    if (where == ZK_PTRS_DEVICE_BORROW) {
        A->row_ptr = const_cast<int64_t*>(row_ptr);
        A->col = const_cast<int*>(col_idx);
        A->val = reinterpret_cast<double2*>(const_cast<zk_z*>(values));
        A->owned = false;
    } else {
        A->owned = true;
        cudaError_t e = dev_alloc(&A->row_ptr, sizeof(int64_t) * (n_rows + 1), s);
        if (e == cudaSuccess) e = dev_alloc(&A->col, sizeof(int) * (nnz > 0 ? nnz : 1), s);
        if (e == cudaSuccess) e = dev_alloc(&A->val, sizeof(double2) * (nnz > 0 ? nnz : 1), s);
        if (e != cudaSuccess) return cleanup(cuda_fail(e, "cudaMalloc(csr)", __FILE__, __LINE__));
        const cudaMemcpyKind kind = where == ZK_PTRS_HOST ? cudaMemcpyHostToDevice : cudaMemcpyDeviceToDevice;
        e = cudaMemcpyAsync(A->row_ptr, row_ptr, sizeof(int64_t) * (n_rows + 1), kind, s);
        if (e == cudaSuccess && nnz > 0) e = cudaMemcpyAsync(A->col, col_idx, sizeof(int) * nnz, kind, s);
        if (e == cudaSuccess && nnz > 0) e = cudaMemcpyAsync(A->val, values, sizeof(double2) * nnz, kind, s);
        if (e != cudaSuccess) return cleanup(cuda_fail(e, "cudaMemcpyAsync(csr)", __FILE__, __LINE__));
    }

    const bool trace = getenv("ZK_TRACE") != nullptr;
    auto now = [] { return std::chrono::steady_clock::now(); };
    auto ms = [](auto a, auto b) { return std::chrono::duration<double, std::milli>(b - a).count(); };
    const auto t0 = now();
    // ---- validation + row statistics on the device (one pass over the arrays)
    {
        ValidateOut h{~0ull, 0u}, *d = nullptr;
        cudaError_t e = scratch_alloc(&d, sizeof(ValidateOut), s);
        if (e == cudaSuccess) e = cudaMemcpyAsync(d, &h, sizeof h, cudaMemcpyHostToDevice, s);
        if (e != cudaSuccess) return cleanup(cuda_fail(e, "validate setup", __FILE__, __LINE__));
        if (n_rows > 0) {
            // ZK_SKIP_VALIDATE: statistics only (reads row_ptr, 8 B/row)
            const int G = grid_for(n_rows, kBlock, A->dev.num_sms * 8);
            validate_kernel<<<G, kBlock, 0, s>>>(A->row_ptr, A->col, A->val, n_rows, n_cols, nnz,
                                                 (flags & ZK_SKIP_VALIDATE) ? 1 : 0, d);
            e = cudaGetLastError();
        }
        if (e == cudaSuccess) e = cudaMemcpyAsync(&h, d, sizeof h, cudaMemcpyDeviceToHost, s);
        if (e == cudaSuccess) e = cudaStreamSynchronize(s);
        scratch_free(d, s);
        if (trace) fprintf(stderr, "  create: copies+validate %.2f ms\n", ms(t0, now()));
        if (e != cudaSuccess) return cleanup(cuda_fail(e, "validate", __FILE__, __LINE__));
        if (!(flags & ZK_SKIP_VALIDATE) && h.first_bad != ~0ull) {
            const long long row = (long long)(h.first_bad >> 3);
            const unsigned code = (unsigned)(h.first_bad & 7u);
            const char* what = code == V_ROWPTR     ? "row_ptr not 0..nnz non-decreasing"
                               : code == V_COLRANGE ? "column index out of range"
                               : code == V_COLORDER ? "columns not strictly increasing (unsorted or duplicate)"
                                                    : "non-finite value";
            char buf[256];
            snprintf(buf, sizeof buf, "row %lld: %s", row + (long long)row_begin, what);
            return cleanup(fail(code == V_NONFINITE ? ZK_ERR_NONFINITE : ZK_ERR_INVALID_CSR, buf));
        }
        A->max_len = (int)h.max_len;
    }
    A->mean_len = n_rows > 0 ? (double)nnz / (double)n_rows : 0.0;
    choose_mapping(A);
    if (cudaStreamCreateWithFlags(&A->cap_stream, cudaStreamNonBlocking) != cudaSuccess)
        return cleanup(fail(ZK_ERR_CUDA, "cudaStreamCreate"));
    return ZK_OK;
}

extern "C" zk_status zk_csr_create(zk_csr* out, int64_t n_rows, int64_t n_cols, int64_t nnz,
                                   const int64_t* row_ptr, const int32_t* col_idx, const zk_z* values,
                                   uint32_t flags, zk_comm comm, int64_t row_begin, zk_stream stream) {
    if (!out) return fail(ZK_ERR_INVALID_VALUE, "out is NULL");
    *out = nullptr;
    cudaStream_t s = (cudaStream_t)stream;
    zk_csr_s* A = nullptr;
    auto cleanup = [&](zk_status st) {
        zk_csr_destroy(A);
        return st;
    };
    const bool trace = getenv("ZK_TRACE") != nullptr;  // host-side phase times on stderr
    auto now = [] { return std::chrono::steady_clock::now(); };
    auto ms = [](auto a, auto b) { return std::chrono::duration<double, std::milli>(b - a).count(); };
    const auto t0 = now();
    zk_status st = csr_create_local(&A, n_rows, n_cols, nnz, row_ptr, col_idx, values, flags, comm, row_begin, s);
    const auto t1 = now();
    if (comm) {
        // every rank learns whether any rank failed before the setup collectives (a rank that
        // returned early would leave its peers blocked in the halo-plan allgather)
        const std::string mine = zk_last_error();
        int any = 0;
        const zk_status ast = dist_agree_failed(comm, st != ZK_OK, s, &any);
        if (ast != ZK_OK) return cleanup(ast);
        if (st != ZK_OK) {
            set_error(mine);
            return cleanup(st);
        }
        if (any) return cleanup(fail(ZK_ERR_INVALID_VALUE, "zk_csr_create failed on another rank"));
        st = dist_setup(A, nullptr, nullptr, s);
        if (st != ZK_OK) return cleanup(st);
    } else if (st != ZK_OK) {
        return cleanup(st);
    }
    const auto t2 = now();
    if (A->spmv_mode == 3) {  // after the halo renumbering: the copy holds the final column ids
        st = sell_build(A, s);
        if (st != ZK_OK) return cleanup(st);
        const char* forced = getenv("ZK_SPMV_MODE");
        if (!forced && (double)A->sl_nnz > (1.0 + kSellMaxPad) * (double)A->nnz) {
            sell_destroy(A);  // too much padding (irregular rows): CSR sub-warp kernel
            choose_mapping(A, 0);
        }
    }
    // The SELL copy carries the values the SpMV reads: the library's own CSR copy of the values
    // (16 B per nonzero, C4 3.4 GB, C5 27.5 GB) is dropped for systems above the cluster solver's
    // range (it reads CSR).  Row pointers and columns stay (Jacobi's diagonal comes from the SELL
    // copy, zk_csr_update_values refills it from a temporary).  ZK_KEEP_CSR_VALUES=1 keeps them.
    if (A->spmv_mode == 3 && A->owned && A->n_rows > kCsrValuesKeepRows &&
        !(getenv("ZK_KEEP_CSR_VALUES") && atoi(getenv("ZK_KEEP_CSR_VALUES")) != 0)) {
        cudaError_t e = cudaStreamSynchronize(s);  // the SELL fill read them
        if (e != cudaSuccess) return cleanup(cuda_fail(e, "zk_csr_create", __FILE__, __LINE__));
        dev_free(A->val, true);
        dev_free_done();
        A->val = nullptr;
    }
    const auto t3 = now();
    // the arrays may have come from the stream-ordered pool: usable from any stream after this
    {
        cudaError_t e = cudaStreamSynchronize(s);
        if (e != cudaSuccess) return cleanup(cuda_fail(e, "zk_csr_create", __FILE__, __LINE__));
    }
    if (trace)
        fprintf(stderr, "zk_csr_create: local (alloc, copy, validate) %.2f ms, dist %.2f ms, sell %.2f ms, sync %.2f ms\n",
                ms(t0, t1), ms(t1, t2), ms(t2, t3), ms(t3, now()));
    handle_count(+1);
    A->counted = true;
    *out = A;
    return ZK_OK;
}

extern "C" zk_status zk_csr_destroy(zk_csr A) {
    if (!A) return ZK_OK;
    const bool trace = getenv("ZK_TRACE") != nullptr;
    auto now = [] { return std::chrono::steady_clock::now(); };
    auto ms = [](auto a, auto b) { return std::chrono::duration<double, std::milli>(b - a).count(); };
    const auto t0 = now();
    cudaDeviceSynchronize();  // once: no array may be in use by pending work when it is freed
    const auto t1 = now();
    for (auto& g : A->graph) {
        if (g.exec) cudaGraphExecDestroy(g.exec);
        if (g.graph) cudaGraphDestroy(g.graph);
    }
    const auto t2 = now();
    if (A->dist) dist_destroy(A);
    jacobi_destroy(A, true);
    sell_destroy(A, true);
    if (A->owned) {
        dev_free(A->row_ptr, true);
        dev_free(A->col, true);
        dev_free(A->val, true);
    }
    dev_free_done();
    const auto t3 = now();
    if (A->cap_stream) cudaStreamDestroy(A->cap_stream);
    const auto t4 = now();
    pinned_put(A->pinned, A->pinned_bytes);
    const auto t5 = now();
    for (auto& e : A->ev)
        if (e) cudaEventDestroy(e);
    if (A->counted) handle_count(-1);
    delete A;
    if (trace)
        fprintf(stderr, "zk_csr_destroy: sync %.2f ms, graphs %.2f ms, frees %.2f ms, stream %.2f ms, pinned %.2f ms, rest %.2f ms\n",
                ms(t0, t1), ms(t1, t2), ms(t2, t3), ms(t3, t4), ms(t4, t5), ms(t5, now()));
    return ZK_OK;
}

namespace zk {
zk_status sell_refill(zk_csr_s* A, const double2* val, cudaStream_t s);  // sell.cu
}

extern "C" zk_status zk_csr_update_values(zk_csr A, const zk_z* values, uint32_t flags, zk_stream stream) {
    if (!A) return fail(ZK_ERR_INVALID_VALUE, "NULL handle");
    cudaStream_t s = (cudaStream_t)stream;
    const uint32_t where = flags & 3u;
    double2* tmp = nullptr;  // the new values when the handle dropped its CSR value copy
    if (A->owned) {
        if (!values && A->nnz > 0) return fail(ZK_ERR_INVALID_VALUE, "NULL values");
        if (where != ZK_PTRS_HOST && where != ZK_PTRS_DEVICE) return fail(ZK_ERR_INVALID_VALUE, "bad flags");
        if (!A->val && A->nnz > 0) ZK_CUDA(dev_alloc(&tmp, sizeof(double2) * A->nnz, s));
        if (A->nnz > 0)
            ZK_CUDA(cudaMemcpyAsync(tmp ? tmp : A->val, values, sizeof(double2) * A->nnz,
                                    where == ZK_PTRS_HOST ? cudaMemcpyHostToDevice : cudaMemcpyDeviceToDevice, s));
    } else if (values && (const void*)values != (const void*)A->val) {
        return fail(ZK_ERR_INVALID_VALUE, "borrowed handle: update the borrowed array in place, pass it or NULL");
    }
    if (!(flags & ZK_SKIP_VALIDATE) && A->nnz > 0) {  // finite values (the pattern is unchanged)
        unsigned long long h = ~0ull, *d = nullptr;
        ZK_CUDA(scratch_alloc(&d, sizeof h, s));
        cudaError_t e = cudaMemcpyAsync(d, &h, sizeof h, cudaMemcpyHostToDevice, s);
        if (e == cudaSuccess) {
            nonfinite_kernel<<<grid_for(A->nnz, kBlock, A->dev.num_sms * 8), kBlock, 0, s>>>(tmp ? tmp : A->val, A->nnz, d);
            e = cudaGetLastError();
        }
        if (e == cudaSuccess) e = cudaMemcpyAsync(&h, d, sizeof h, cudaMemcpyDeviceToHost, s);
        if (e == cudaSuccess) e = cudaStreamSynchronize(s);
        scratch_free(d, s);
        if (e != cudaSuccess) return cuda_fail(e, "zk_csr_update_values", __FILE__, __LINE__);
        if (h != ~0ull) {
            if (tmp) dev_free(tmp);
            char buf[128];
            snprintf(buf, sizeof buf, "value %llu (CSR order) is not finite", h);
            return fail(ZK_ERR_NONFINITE, buf);
        }
    }
    if (A->spmv_mode == 3) {
        const zk_status st = sell_refill(A, tmp ? tmp : A->val, s);
        if (tmp) {
            cudaStreamSynchronize(s);
            dev_free(tmp, true);
            dev_free_done();
        }
        ZK_TRY(st);
    }
    ZK_CUDA(cudaStreamSynchronize(s));
    for (auto& g : A->graph) {  // graphs bake the Jacobi values' address: rebuilt on the next solve
        if (g.exec) cudaGraphExecDestroy(g.exec);
        if (g.graph) cudaGraphDestroy(g.graph);
        g = GraphCache{};
    }
    jacobi_destroy(A, true);   // A·M⁻¹ is rebuilt from the new values on the next Jacobi solve
    return ZK_OK;
}

extern "C" zk_status zk_csr_info(zk_csr A, zk_csr_info_t* info) {
    if (!A || !info) return fail(ZK_ERR_INVALID_VALUE, "NULL argument");
    info->n_rows = A->n_rows;
    info->n_cols = A->n_cols;
    info->nnz = A->nnz;
    info->row_begin = A->row_begin;
    info->n_global = A->n_global;
    info->max_row_len = A->max_len;
    info->lanes_per_row = A->W;
    info->mean_row_len = A->mean_len;
    info->n_halo = dist_n_halo(A);
    info->borrowed = A->owned ? 0 : 1;
    info->nranks = dist_nranks(A);
    info->spmv_mode = A->spmv_mode;
    info->sell_entries = A->spmv_mode == 3 ? A->sl_nnz : 0;
    info->interior_rows = A->dist ? dist_interior_rows(A) : 0;
    info->csr_values_kept = A->val ? 1 : 0;
    return ZK_OK;
}

extern "C" zk_status zk_zcsrmv(zk_csr A, zk_z alpha, const zk_z* x, zk_z beta, zk_z* y, zk_stream s) {
    if (!A || !x || !y) return fail(ZK_ERR_INVALID_VALUE, "NULL argument");
    if ((const void*)x == (const void*)y) return fail(ZK_ERR_ALIAS, "x and y alias (S:244)");
    const double2 a = make_double2(alpha.re, alpha.im), b = make_double2(beta.re, beta.im);
    if (A->n_rows == 0) return ZK_OK;
    if (A->dist) return dist_zcsrmv(A, a, (const double2*)x, b, (double2*)y, (cudaStream_t)s);
    return zcsrmv_local(A, a, (const double2*)x, b, (double2*)y, (cudaStream_t)s);
}
