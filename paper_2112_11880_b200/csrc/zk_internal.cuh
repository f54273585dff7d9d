// zk_internal.cuh — device helpers shared by the libzk kernels (sm_100a only).
// Complex numbers are double2 {x = re, y = im} (layout of zk_z / torch.complex128).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/zk.h"

#if defined(__CUDA_ARCH__) && (__CUDA_ARCH__ < 1000)
#error "libzk targets sm_100a (B200) only"
#endif

namespace zk {

constexpr int kBlock = 256;      // threads per block for every libzk kernel
constexpr int kWarps = kBlock / 32;
constexpr int kMaxRed = 4;       // max doubles reduced by one kernel
constexpr int kMaxGrid = 4096;   // max blocks of a reducing kernel (partials capacity)

// ------------------------------------------------------------------ complex helpers
__device__ __forceinline__ double2 cmul(double2 a, double2 b) {
    return make_double2(fma(a.x, b.x, -a.y * b.y), fma(a.x, b.y, a.y * b.x));
}
// acc += a*b
__device__ __forceinline__ void cfma(double2& acc, double2 a, double2 b) {
    acc.x = fma(a.x, b.x, acc.x);
    acc.x = fma(-a.y, b.y, acc.x);
    acc.y = fma(a.x, b.y, acc.y);
    acc.y = fma(a.y, b.x, acc.y);
}
// conj(a)*b
__device__ __forceinline__ double2 cdotc1(double2 a, double2 b) {
    return make_double2(fma(a.x, b.x, a.y * b.y), fma(a.x, b.y, -a.y * b.x));
}
__device__ __forceinline__ double cabs2(double2 a) { return fma(a.x, a.x, a.y * a.y); }
__device__ __forceinline__ double2 cadd(double2 a, double2 b) { return make_double2(a.x + b.x, a.y + b.y); }
__device__ __forceinline__ double2 csub(double2 a, double2 b) { return make_double2(a.x - b.x, a.y - b.y); }
// (a+bi)/(c+di) written out as ((ac+bd) + (bc−ad)i)/(c²+d²) — same formula as the oracle (R7)
__device__ __forceinline__ double2 cdiv(double2 a, double2 b) {
    double den = b.x * b.x + b.y * b.y;
    return make_double2((a.x * b.x + a.y * b.y) / den, (a.y * b.x - a.x * b.y) / den);
}
__device__ __forceinline__ double cabs_(double2 a) { return sqrt(a.x * a.x + a.y * a.y); }
__device__ __forceinline__ bool cfinite(double2 a) { return isfinite(a.x) && isfinite(a.y); }

// ------------------------------------------------------------------ loads
// Streaming (read-once) loads: no L1 allocation.
__device__ __forceinline__ double2 ld_stream(const double2* p) {
    double2 v;
    asm volatile("ld.global.nc.L1::no_allocate.v2.f64 {%0, %1}, [%2];" : "=d"(v.x), "=d"(v.y) : "l"(p));
    return v;
}
__device__ __forceinline__ int ld_stream(const int* p) {
    int v;
    asm volatile("ld.global.nc.L1::no_allocate.b32 %0, [%1];" : "=r"(v) : "l"(p));
    return v;
}
// Matrix-stream loads with an explicit L2 eviction policy (createpolicy + .L2::cache_hint).
// LP 0: .L1::no_allocate alone (L2 treats it as evict-first: partially consumed sectors can be
// evicted before the neighbouring row asks for them, ncu showed 1.25x DRAM reads);
// LP 1: no L1 allocation, L2 evict_normal; LP 2: L2 evict_last; LP 3: plain read-only path.
// LP 4: no L1 allocation, explicit L2 evict_first (SELL: every load instruction consumes whole
// sectors, so nothing is re-fetched; the solver vectors keep their L2 lines)
template <int LP>
__device__ __forceinline__ uint64_t make_policy() {
    uint64_t pol = 0;
    if (LP == 1) asm volatile("createpolicy.fractional.L2::evict_normal.b64 %0, 1.0;" : "=l"(pol));
    if (LP == 2) asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol));
    if (LP == 4) asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
    return pol;
}
template <int LP>
__device__ __forceinline__ double2 ld_mat(const double2* p, uint64_t pol) {
    if constexpr (LP == 0) {
        return ld_stream(p);
    } else if constexpr (LP == 3) {
        return __ldg(p);
    } else {
        double2 v;
        asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.v2.f64 {%0, %1}, [%2], %3;"
                     : "=d"(v.x), "=d"(v.y) : "l"(p), "l"(pol));
        return v;
    }
}
template <int LP>
__device__ __forceinline__ int ld_mat(const int* p, uint64_t pol) {
    if constexpr (LP == 0) {
        return ld_stream(p);
    } else if constexpr (LP == 3) {
        return __ldg(p);
    } else {
        int v;
        asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.b32 %0, [%1], %2;" : "=r"(v) : "l"(p), "l"(pol));
        return v;
    }
}
// Streaming load of data this kernel also writes (coherent path, no L1 allocation).
#ifndef ZK_LD_CLOBBER
#define ZK_LD_CLOBBER : "memory"
#endif
#ifndef ZK_LDV_POLICY
#define ZK_LDV_POLICY 0
#endif
__device__ __forceinline__ double2 ld_stream_rw(const double2* p) {
    double2 v;
    if constexpr (ZK_LDV_POLICY == 1) {
        uint64_t pol;
        asm("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
        asm volatile("ld.global.L1::no_allocate.L2::cache_hint.v2.f64 {%0, %1}, [%2], %3;" : "=d"(v.x), "=d"(v.y) : "l"(p), "l"(pol) ZK_LD_CLOBBER);
    } else {
        asm volatile("ld.global.L1::no_allocate.v2.f64 {%0, %1}, [%2];" : "=d"(v.x), "=d"(v.y) : "l"(p) ZK_LD_CLOBBER);
    }
    return v;
}
// Gather through the read-only path (L1 + L2 reuse of x across neighbouring rows).
// Gather of x (ZK_GATHER_MODE): 2 (default) read-only path with an L2 evict_last policy; 0 plain
// __ldg; 1 coherent ld.global.  In the solver loops x (p, s, y1, ...) was written by the previous
// kernel and sits dirty in L2: with evict_normal gathers the matrix stream evicted x lines that
// were gathered again later (C4 zk_zcsrmv after a rewrite of x: 811 µs at mode 0, 656 µs at
// mode 2, 647 µs on a clean x either way; tools/inloop_probe.py).
#ifndef ZK_GATHER_MODE
#define ZK_GATHER_MODE 2
#endif
__device__ __forceinline__ double2 ld_gather(const double2* p) {
    if constexpr (ZK_GATHER_MODE == 1) {
        double2 v;
        asm volatile("ld.global.v2.f64 {%0, %1}, [%2];" : "=d"(v.x), "=d"(v.y) : "l"(p));
        return v;
    } else if constexpr (ZK_GATHER_MODE == 2) {
        double2 v;
        uint64_t pol;
        asm("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol));
        asm volatile("ld.global.nc.L2::cache_hint.v2.f64 {%0, %1}, [%2], %3;" : "=d"(v.x), "=d"(v.y) : "l"(p), "l"(pol));
        return v;
    } else {
        return __ldg(p);
    }
}
// Coherent loads for data written earlier in the SAME launch (the persistent solver phases,
// separated by grid-wide barriers whose gpu-scope fences invalidate L1): never .nc.
__device__ __forceinline__ double2 ld_gather_coh(const double2* p) {
    double2 v;
    asm volatile("ld.global.v2.f64 {%0, %1}, [%2];" : "=d"(v.x), "=d"(v.y) : "l"(p) ZK_LD_CLOBBER);
    return v;
}
__device__ __forceinline__ double2 ld_vec(const double2* p) { return ld_stream_rw(p); }
// Vector stores of the solver kernels.  ZK_ST_POLICY: 0 plain write-back; 1 .cs (streaming,
// evict-first); 2 L2::evict_first hint; 3 L2::evict_last hint.
#ifndef ZK_ST_POLICY
#define ZK_ST_POLICY 0
#endif
__device__ __forceinline__ void st_vec(double2* p, double2 v) {
    if constexpr (ZK_ST_POLICY == 1) {
        asm volatile("st.global.cs.v2.f64 [%0], {%1, %2};" :: "l"(p), "d"(v.x), "d"(v.y) : "memory");
    } else if constexpr (ZK_ST_POLICY == 4) {
        asm volatile("st.global.wt.v2.f64 [%0], {%1, %2};" :: "l"(p), "d"(v.x), "d"(v.y) : "memory");
    } else if constexpr (ZK_ST_POLICY == 2 || ZK_ST_POLICY == 3) {
        uint64_t pol;
        if constexpr (ZK_ST_POLICY == 2)
            asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
        else
            asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol));
        asm volatile("st.global.L1::no_allocate.L2::cache_hint.v2.f64 [%0], {%1, %2}, %3;" :: "l"(p), "d"(v.x), "d"(v.y), "l"(pol) : "memory");
    } else {
        *p = v;
    }
}
// Coherent L2 load (partials written by other blocks of the same launch).
__device__ __forceinline__ double ld_cg(const double* p) { return __ldcg(p); }

// ------------------------------------------------------------------ reductions
template <int K>
__device__ __forceinline__ void warp_sum(double (&v)[K]) {
#pragma unroll
    for (int k = 0; k < K; k++) {
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) v[k] += __shfl_xor_sync(0xffffffffu, v[k], o);
    }
}

// Block-wide sum of K doubles (fixed order). Result valid in thread 0. Uses `sm` (kWarps*K doubles).
template <int K>
__device__ __forceinline__ void block_sum(double (&v)[K], double* sm) {
    __syncwarp();  // reconverge the warp (row loops of different trip counts) before the shuffles/barrier
    warp_sum<K>(v);
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    if (lane == 0) {
#pragma unroll
        for (int k = 0; k < K; k++) sm[k * kWarps + warp] = v[k];
    }
    __syncthreads();
    if (warp == 0) {
#pragma unroll
        for (int k = 0; k < K; k++) v[k] = lane < kWarps ? sm[k * kWarps + lane] : 0.0;
        warp_sum<K>(v);
    }
}

// Deterministic grid reduction with a last-block finish (the paper's "two distinct tasks",
// P:199-200, fused into one pass).  Every block writes its partial; the block that takes the
// last ticket sums the partials in index order (fixed tree) and returns true, with the totals
// in `out` (valid in thread 0).  The ticket is reset by the last block, so the scratch is
// self-cleaning.  partials: [K][gridDim.x] doubles.
// off / total: a reduction spread over two launches of one SpMV (the interior and boundary slices
// of a distributed matrix, dist.cu): this launch's blocks are partials [off, off + gridDim.x) of
// `total`, one shared ticket, and only the block that takes the last of the `total` tickets — in the
// second launch — finishes.  total = 0: one launch.
template <int K>
__device__ __forceinline__ bool grid_sum(double (&v)[K], double* partials, unsigned int* ticket,
                                         double (&out)[K], int off = 0, int total = 0) {
    __shared__ double sm[kWarps * kMaxRed];
    __shared__ bool last;
    block_sum<K>(v, sm);
    const int G = total > 0 ? total : (int)gridDim.x;
    if (threadIdx.x == 0) {
#pragma unroll
        for (int k = 0; k < K; k++) partials[k * G + off + blockIdx.x] = v[k];
        __threadfence();
        unsigned int t = atomicAdd(ticket, 1u);
        last = (t == (unsigned)G - 1);
    }
    __syncthreads();
    if (!last) return false;
    __threadfence();
    double acc[K];
#pragma unroll
    for (int k = 0; k < K; k++) {
        acc[k] = 0.0;
        for (int i = threadIdx.x; i < G; i += kBlock) acc[k] += ld_cg(partials + k * G + i);
    }
    __syncthreads();  // sm reuse
    block_sum<K>(acc, sm);
    if (threadIdx.x == 0) {
#pragma unroll
        for (int k = 0; k < K; k++) out[k] = acc[k];
        *ticket = 0u;
    }
    return true;
}

// ------------------------------------------------------------------ CSR view
struct CsrDev {
    const int64_t* row_ptr;
    const int* col;
    const double2* val;
    int64_t n_rows;
    int64_t nnz;
    // sliced-ELL copy (SpMV mode 3, sell.cu): slice s of 32 rows holds its entries column-major at
    // [sl_ptr[s], sl_ptr[s+1]), width = (sl_ptr[s+1] − sl_ptr[s]) / 32; padding has col −1, val 0
    const int64_t* sl_ptr;
    const int* sl_col;
    const double2* sl_val;
    // slice set walked by the SELL kernel (distributed interior/boundary split, dist.cu): logical
    // slices t ∈ [0, sl_cnt) map to physical slices sl_lo + t (+ sl_gap for t ≥ sl_gap_at), i.e.
    // one contiguous run, or a prefix and a suffix around a skipped run.  The whole matrix:
    // sl_lo = 0, sl_cnt = n_slices, sl_gap_at = sl_cnt.  main_part = 0 on the second partial
    // launch of one SpMV (work that must happen once per SpMV is skipped there).
    int sl_lo, sl_cnt, sl_gap_at, sl_gap;
    int main_part;
    // the SpMV's fused reduction spans two launches (grid_sum off / total; 0 = one launch)
    int red_off, red_total;
};

}  // namespace zk
