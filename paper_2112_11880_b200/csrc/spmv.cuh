// spmv.cuh — the ZSpMV body (§3) and the BLAS-1 loop body,
// both as __device__ templates so the solver kernels can fuse their epilogues into them.
//
// ZSpMV mapping: a sub-warp of W lanes per row, W chosen at create from the mean
// row length (W = 4 for the 27-point FE rows: ≈ 7 nonzeros per lane).  A block of 256 threads owns 256/W consecutive
// rows per step and walks its tiles grid-stride (a fixed static schedule, so the fused
// reductions are deterministic).  Per row chunk of 4W nonzeros each lane issues 4 independent
// (value, column) loads before touching x, then the 4 gathers of x (read-only path; x stays
// L1/L2-resident across neighbouring rows), then 4 complex FMAs; the W partial sums are combined
// with xor-shuffles.  The row bounds of the NEXT tile are loaded while the current tile computes
// (one DRAM latency off each tile's dependency chain).  Matrix-stream loads carry an explicit
// L2 evict_normal policy (LP 1): with the default evict-first treatment of no-allocate loads,
// sectors shared by two row chunks were re-fetched (ncu: 1.25x DRAM reads; profiles/).
// No tensor cores: this is not a contraction (8 flops per 20+ bytes).
#pragma once
#include "zk_internal.cuh"

namespace zk {

// Epilogue concept:
//   static constexpr int K;                         // doubles reduced over the grid (0..4)
//   typename Pre; __device__ Pre pre(int64_t i);   // row i's own operands (loaded a tile ahead)
//   __device__ void row(int64_t i, double2 y, const Pre&, double (&acc)[K>0?K:1]);   // once per row
//   __device__ void finish(double (&acc)[K>0?K:1]); // called by every thread at the end
//   optional static constexpr int kPrePlace;        // SELL kernel: 0 / 1 / 2, see spmv_body_sell
//   optional static constexpr bool kAhead = false;  // load pre() at the start of the row's own tile
//                                                   // instead of one tile ahead (wide Pre: one copy
//                                                   // in registers instead of two)
#ifndef ZK_SELL_PRE
#define ZK_SELL_PRE 0
#endif
template <class E>
struct pre_place {
    template <class T> static constexpr int get(decltype(T::kPrePlace)*) { return T::kPrePlace; }
    template <class T> static constexpr int get(...) { return ZK_SELL_PRE; }
    static constexpr int value = get<E>(nullptr);
};
template <class E>
struct pre_ahead {
    template <class T> static constexpr bool get(decltype(T::kAhead)*) { return T::kAhead; }
    template <class T> static constexpr bool get(...) { return true; }
    static constexpr bool value = get<E>(nullptr);
};
#ifndef ZK_DEFAULT_LP
#define ZK_DEFAULT_LP 1
#endif
#ifndef ZK_SPMV_U
#define ZK_SPMV_U 4
#endif
// GCOH: gather x with coherent loads (x written earlier in the same launch: persistent solver)
template <int W, class Epi, int LP = ZK_DEFAULT_LP, bool GCOH = false>
__device__ __forceinline__ void spmv_body(const CsrDev& A, const double2* __restrict__ x, Epi& epi) {
    static_assert(W >= 1 && W <= 32 && (W & (W - 1)) == 0, "W must be a power of two <= 32");
    constexpr int RPB = kBlock / W;  // rows per block step
    constexpr int U = ZK_SPMV_U;     // nonzeros per lane per chunk
    constexpr int KA = Epi::K > 0 ? Epi::K : 1;
    constexpr bool AHEAD = pre_ahead<Epi>::value;
    const uint64_t pol = make_policy<LP>();
    double acc[KA];
#pragma unroll
    for (int k = 0; k < KA; k++) acc[k] = 0.0;

    // 32-bit row / in-row indices (n_rows < 2^31 is checked at create); nnz offsets stay 64-bit
    // only in the per-row base pointers, so each chunk costs one address computation.
    const int sub = threadIdx.x & (W - 1);
    const int grp = threadIdx.x / W;
    const int n = (int)A.n_rows;
    const int G = gridDim.x;
    int row = blockIdx.x * RPB + grp;
    int64_t rs = 0;
    int len = 0;
    typename Epi::Pre pre{};
    if (row < n) {
        rs = __ldg(A.row_ptr + row);
        len = (int)(__ldg(A.row_ptr + row + 1) - rs);
        if (AHEAD && sub == 0) pre = epi.pre(row);
    }
    for (int tile = blockIdx.x; tile * RPB < n; tile += G) {
        // bounds (and epilogue operands) of this lane's row in the next tile, used next iteration
        const int nrow = row + G * RPB;
        int64_t nrs = 0;
        int nlen = 0;
        typename Epi::Pre npre{};
        if (!AHEAD && sub == 0 && row < n) pre = epi.pre(row);
        if (nrow < n) {
            nrs = __ldg(A.row_ptr + nrow);
            nlen = (int)(__ldg(A.row_ptr + nrow + 1) - nrs);
            if (AHEAD && sub == 0) npre = epi.pre(nrow);
        }
        double2 sum = make_double2(0.0, 0.0);
        const double2* vr = A.val + rs;
        const int* cr = A.col + rs;
        for (int base = sub; base < len; base += U * W) {
            double2 v[U];
            int c[U];
#pragma unroll
            for (int u = 0; u < U; u++) {
                const int j = base + u * W;
                if (j < len) {
                    v[u] = ld_mat<LP>(vr + j, pol);
                    c[u] = ld_mat<LP>(cr + j, pol);
                } else {
                    v[u] = make_double2(0.0, 0.0);
                    c[u] = -1;
                }
            }
            double2 xv[U];
#pragma unroll
            for (int u = 0; u < U; u++)
                xv[u] = c[u] >= 0 ? (GCOH ? ld_gather_coh(x + c[u]) : ld_gather(x + c[u])) : make_double2(0.0, 0.0);
#pragma unroll
            for (int u = 0; u < U; u++) cfma(sum, v[u], xv[u]);
        }
#pragma unroll
        for (int o = W / 2; o > 0; o >>= 1) {
            sum.x += __shfl_xor_sync(0xffffffffu, sum.x, o, W);
            sum.y += __shfl_xor_sync(0xffffffffu, sum.y, o, W);
        }
        if (sub == 0 && row < n) epi.row(row, sum, pre, acc);
        row = nrow;
        rs = nrs;
        len = nlen;
        if (AHEAD) pre = npre;
    }
    epi.finish(acc);
}

// ---------------------------------------------------------------------------------------------
// Sliced-ELL mapping (MODE 3, built at create by sell.cu): one warp per slice of 32 consecutive
// rows, lane = row.  The slice's entries are stored column-major (entry k of the slice's rows at
// k·32 + lane), so every value / column load instruction of a warp reads 512 / 128 contiguous
// bytes, the gathers of x for neighbouring rows are adjacent, and the epilogue runs on all 32
// lanes with coalesced loads and stores.  Each lane sums its row's entries in stored order (the
// oracle's order).  U entries per lane are in flight per step; padding (col −1) is skipped.
#ifndef ZK_SELL_U
#define ZK_SELL_U 9
#endif
// Matrix-stream L2 policy of the SELL kernel: evict_first (LP 4).  Every SELL load instruction
// consumes whole sectors (nothing is re-requested), and the matrix stream no longer pushes the
// solver vectors out of L2: measured (tools/ab_lib.py, µs per iteration, evict_normal →
// evict_first) Audi3D-4 (C3) BiCGStab 164.3 → 150.2, CG 86.1 → 75.3, TFQMR 168.3 → 155.5;
// Twingo3D-2 130.1 → 117.3, 67.4 → 58.5, 131.4 → 118.7; C4 unchanged (1732 either way)
// (profiles/r02_sell_lp.txt).
#ifndef ZK_SELL_LP
#define ZK_SELL_LP 4
#endif
// elements in flight per thread of a vector Op (Op::U, default 4)
template <class Op>
struct vec_unroll {
    template <class T> static constexpr int get(decltype(T::U)*) { return T::U; }
    template <class T> static constexpr int get(...) { return 4; }
    static constexpr int value = get<Op>(nullptr);
};
// Per epilogue (Epi::kTail): after its slice loop the warp walks ITS slices once more and runs
// Epi::TailOp (built by epi.tail_op()) on its rows — a fused reduction pass over vectors the loop
// just wrote (each lane re-reads only what it stored itself), with no register pressure on the
// loop (neither the running sums nor the Op's operands are live there) and no extra launch.
template <class E>
struct sell_tail {
    template <class T> static constexpr bool get(decltype(T::kTail)*) { return T::kTail; }
    template <class T> static constexpr bool get(...) { return false; }
    static constexpr bool value = get<E>(nullptr);
};
// Per epilogue (Epi::kOrdered): the store-only epilogue of the split solver SpMVs needs it — left
// to itself the compiler schedules that kernel at 64 registers with 3 matrix loads in flight per
// gather batch instead of 9 (SASS; in-loop K1 708 µs vs 647 µs standalone at C4, ncu).
// Per epilogue (Epi::kWarpAcc): the epilogue's running sums are reduced over the warp after every
// slice and kept in a per-warp shared-memory slot (lane 0 adds), so no accumulator register is live
// across the slice loop (the fused-epilogue variant of the split schedule: the dot products come
// out of the SpMV itself, with no second pass over the vectors).
template <class E>
struct sell_warpacc {
    template <class T> static constexpr bool get(decltype(T::kWarpAcc)*) { return T::kWarpAcc; }
    template <class T> static constexpr bool get(...) { return false; }
    static constexpr bool value = get<E>(nullptr);
};
template <class E>
struct sell_ordered {
    template <class T> static constexpr bool get(decltype(T::kOrdered)*) { return T::kOrdered; }
    template <class T> static constexpr bool get(...) { return false; }
    static constexpr bool value = get<E>(nullptr);
};
// The rows of this warp's slices under the SELL body's static schedule (logical slices t0 + k·nw,
// physical slice as in spmv_body_sell with the same REV) — the rows the warp's SpMV wrote — with
// Op::U slices in flight: op.apply(row, op.load(row), acc) on each.  BACK walks the warp's slices
// in the reverse time order (its most recently written rows first).  The SpMV tail reductions and
// the phases of the phase-fused solver kernels run on it.
template <bool REV, bool BACK, class Op, int KA>
__device__ __forceinline__ void sell_walk_own(const CsrDev& A, const Op& op, double (&acc)[KA]) {
    constexpr int TU = vec_unroll<Op>::value;
    const int n = (int)A.n_rows;
    const int n_sl = A.sl_cnt;
    const int nw = gridDim.x * kWarps;
    const int lane = threadIdx.x & 31;
    const int t0 = blockIdx.x * kWarps + (threadIdx.x >> 5);
    const int cnt = t0 < n_sl ? (n_sl - 1 - t0) / nw + 1 : 0;
    for (int kb = 0; kb < cnt; kb += TU) {
        typename Op::In in[TU] = {};
        int rows[TU];
#pragma unroll
        for (int u = 0; u < TU; u++) {
            const int k = kb + u;
            const int t = t0 + (BACK ? cnt - 1 - k : k) * nw;
            const int q = REV ? n_sl - 1 - t : t;
            rows[u] = k < cnt ? (A.sl_lo + q + (q >= A.sl_gap_at ? A.sl_gap : 0)) * 32 + lane : n;
            if (rows[u] < n) in[u] = op.load(rows[u]);
        }
#pragma unroll
        for (int u = 0; u < TU; u++)
            if (rows[u] < n) op.apply(rows[u], in[u], acc);
    }
}

// REV: walk the slices last to first (opposite sweeps: the kernel starts on the rows
// its predecessor in the solver loop touched last, still in L2)
template <class Epi, int LP = ZK_SELL_LP, bool REV = false>
__device__ __forceinline__ void spmv_body_sell(const CsrDev& A, const double2* __restrict__ x, Epi& epi) {
    constexpr int U = ZK_SELL_U;
    constexpr int KA = Epi::K > 0 ? Epi::K : 1;
    // where the epilogue's row operands are loaded: 0 one slice ahead (registers held across the
    // whole slice), 1 with the slice's last batch of matrix loads, 2 after the row sums.  Per
    // epilogue (Epi::kPrePlace): wide epilogues (TFQMR T2/T4: 2-3 operands) measured faster at 2,
    // the one-operand BiCGStab epilogues at 0 (profiles/r01_sell.md)
    constexpr int PRE = pre_place<Epi>::value;
    constexpr bool ORD = sell_ordered<Epi>::value;
    constexpr bool AHEAD = PRE == 0 && pre_ahead<Epi>::value;
    constexpr bool WACC = sell_warpacc<Epi>::value;
    const uint64_t pol = make_policy<LP>();
    double acc[KA];
#pragma unroll
    for (int k = 0; k < KA; k++) acc[k] = 0.0;
    const int lane = threadIdx.x & 31;
    __shared__ double wacc[WACC ? kWarps : 1][KA];
    if constexpr (WACC) {
        if (lane == 0)
#pragma unroll
            for (int k = 0; k < KA; k++) wacc[threadIdx.x >> 5][k] = 0.0;
    }
    const int n = (int)A.n_rows;
    // logical slices t ∈ [0, sl_cnt) → physical slice phys(t) (the whole matrix, or one part of a
    // distributed SpMV split into interior / boundary slices, CsrDev)
    const int n_sl = A.sl_cnt;
    auto phys = [&](int t) {
        const int u = REV ? n_sl - 1 - t : t;
        return A.sl_lo + u + (u >= A.sl_gap_at ? A.sl_gap : 0);
    };
    const int nw = gridDim.x * kWarps;
    int t = blockIdx.x * kWarps + (threadIdx.x >> 5);
    int64_t base = 0;
    int width = 0;
    typename Epi::Pre pre{};
    if (t < n_sl) {
        const int s = phys(t);
        base = __ldg(A.sl_ptr + s);
        width = (int)((__ldg(A.sl_ptr + s + 1) - base) >> 5);
        if (AHEAD && s * 32 + lane < n) pre = epi.pre(s * 32 + lane);
    }
    for (; t < n_sl; t += nw) {
        const int row = phys(t) * 32 + lane;
        const int nt = t + nw;  // next slice: bounds and epilogue operands one step ahead
        int64_t nbase = 0;
        int nwidth = 0;
        typename Epi::Pre npre{};
        if (PRE == 0 && !AHEAD && row < n) pre = epi.pre(row);
        if (nt < n_sl) {
            const int ns = phys(nt);
            nbase = __ldg(A.sl_ptr + ns);
            nwidth = (int)((__ldg(A.sl_ptr + ns + 1) - nbase) >> 5);
            if (AHEAD && ns * 32 + lane < n) npre = epi.pre(ns * 32 + lane);
        }
        const double2* vr = A.sl_val + base + lane;
        const int* cr = A.sl_col + base + lane;
        double2 sum = make_double2(0.0, 0.0);
        for (int k0 = 0; k0 < width; k0 += U) {
            double2 v[U];
            int c[U];
#pragma unroll
            for (int u = 0; u < U; u++) {
                if (k0 + u < width) {
                    v[u] = ld_mat<LP>(vr + (k0 + u) * 32, pol);
                    c[u] = ld_mat<LP>(cr + (k0 + u) * 32, pol);
                } else {
                    v[u] = make_double2(0.0, 0.0);
                    c[u] = -1;
                }
            }
            if (PRE == 1 && k0 + U >= width && row < n) pre = epi.pre(row);
            // ORD: every gather address depends on ALL U column loads of the batch (an opaque 0
            // computed from their AND), so ptxas has to issue the whole batch of (value, column)
            // loads before the first gather — and cannot stall on one column at a time
            int dep = 0;
            if constexpr (ORD) {
                int m = c[0];
#pragma unroll
                for (int u = 1; u < U; u++) m &= c[u];
                asm("{.reg .pred q; setp.eq.s32 q, %1, 2147483647; selp.b32 %0, 1, 0, q;}" : "=r"(dep) : "r"(m));
            }
            double2 xv[U];
#pragma unroll
            for (int u = 0; u < U; u++) xv[u] = c[u] >= 0 ? ld_gather(x + (c[u] + dep)) : make_double2(0.0, 0.0);
#pragma unroll
            for (int u = 0; u < U; u++)
                if (c[u] >= 0) cfma(sum, v[u], xv[u]);
        }
        if (PRE == 1 && width == 0 && row < n) pre = epi.pre(row);
        if (PRE == 2 && row < n) pre = epi.pre(row);
        if constexpr (WACC) {
            double part[KA];
#pragma unroll
            for (int k = 0; k < KA; k++) part[k] = 0.0;
            if (row < n) epi.row(row, sum, pre, part);
            warp_sum<KA>(part);  // the slice is warp-uniform: every lane takes part
            if (lane == 0)
#pragma unroll
                for (int k = 0; k < KA; k++) wacc[threadIdx.x >> 5][k] += part[k];
        } else {
            if (row < n) epi.row(row, sum, pre, acc);
        }
        base = nbase;
        width = nwidth;
        if (AHEAD) pre = npre;
    }
    if constexpr (WACC) {
#pragma unroll
        for (int k = 0; k < KA; k++) acc[k] = lane == 0 ? wacc[threadIdx.x >> 5][k] : 0.0;
    }
    if constexpr (sell_tail<Epi>::value) {
        const auto op = epi.tail_op();
        sell_walk_own<REV, false>(A, op, acc);
        op.finish(acc, A.red_off, A.red_total);
    } else {
        epi.finish(acc, A.red_off, A.red_total);
    }
}

// The SpMV body of a mapping: MODE 3 sliced ELL (the default), MODE 0 CSR sub-warp rows
// (matrices whose SELL padding would exceed 10 %).
// (REV: SELL only; the CSR sub-warp body keeps its order)
template <int W, int MODE, bool REV = false, class Epi>
__device__ __forceinline__ void spmv_any(const CsrDev& A, const double2* __restrict__ x, Epi& epi) {
    static_assert(MODE == 0 || MODE == 3, "SpMV mappings: 0 (CSR sub-warp) and 3 (SELL-32)");
    if constexpr (sell_tail<Epi>::value && MODE != 3) {
        __trap();  // tail epilogues exist only in the SELL body (the host never launches this)
    } else if constexpr (MODE == 3) {
        spmv_body_sell<Epi, ZK_SELL_LP, REV>(A, x, epi);
    } else {
        spmv_body<W>(A, x, epi);
    }
}
// minimum resident CTAs per SM of an SpMV kernel (__launch_bounds__): 3 for SELL (80 registers,
// 9 entries in flight per lane), 4 for the CSR sub-warp kernel (64 registers)
__host__ __device__ constexpr int spmv_min_blocks(int mode) { return mode == 3 ? 3 : 4; }

// Grid-stride elementwise body with U elements in flight per thread.
//   Op::K, Op::In, In load(int64_t i), void apply(int64_t i, const In&, double (&acc)[K]), finish(acc)

// REV: element i is processed as n − 1 − i (a last-to-first sweep; warps stay coalesced)
template <bool REV = false, class Op>
__device__ __forceinline__ void vec_body(int64_t n, Op& op) {
    constexpr int U = vec_unroll<Op>::value;  // elements in flight per thread (Op::U, default 4)
    constexpr int KA = Op::K > 0 ? Op::K : 1;
    double acc[KA];
#pragma unroll
    for (int k = 0; k < KA; k++) acc[k] = 0.0;
    const int64_t step = (int64_t)gridDim.x * kBlock * U;
    for (int64_t base = (int64_t)blockIdx.x * kBlock * U + threadIdx.x; base < n; base += step) {
        typename Op::In in[U];
#pragma unroll
        for (int u = 0; u < U; u++) {
            const int64_t i = base + u * kBlock;
            if (i < n) in[u] = op.load(REV ? n - 1 - i : i);
        }
#pragma unroll
        for (int u = 0; u < U; u++) {
            const int64_t i = base + u * kBlock;
            if (i < n) op.apply(REV ? n - 1 - i : i, in[u], acc);
        }
    }
    op.finish(acc);
}

// number of blocks for a grid-stride kernel: enough to cover the work, at most `cap`
inline int grid_for(int64_t units, int64_t per_block, int cap) {
    int64_t g = (units + per_block - 1) / per_block;
    if (g < 1) g = 1;
    return (int)(g < cap ? g : cap);
}

}  // namespace zk
