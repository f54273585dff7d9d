// spmv_tma.cuh — ZSpMV with TMA bulk-copy staging (sm_100a), the default mapping for FE rows.
//
// Why: the sub-warp kernel (spmv.cuh) requests each 32-B sector of the value/column streams from
// several instructions (row chunks are not sector aligned); under the L2's evict-first policy for
// streaming loads the repeats miss and DRAM reads grew to 1.25× the algorithmic bytes (ncu,
// profiles/r01_*).  Here every row tile's [row_ptr[r0], row_ptr[r1]) value and column ranges are
// moved by ONE contiguous cp.async.bulk each (the TMA engine; no registers, no per-lane
// addresses), so each sector is fetched once, and the copies for the next S−1 tiles are in flight
// while the CTA computes the current one (mbarrier ring of S stages in shared memory).
//
// Tile t = rows [t·R, t·R+R), R even, R·max_row_len ≤ stage capacity.  CTA b of G walks tiles
// b, b+G, ... (static schedule: the fused reductions stay deterministic).  Thread 0 issues the
// copies of tile k+S right after the CTA finished reading stage k mod S, using row_ptr bounds it
// loaded one tile earlier (latency hidden behind a tile of compute).  Consumers: W lanes per row
// read values/columns from shared memory, gather x through L1/L2 (read-only path), 4 complex FMAs
// per nonzero, xor-shuffle reduce, then the epilogue (plain axpby or a fused solver step).
#pragma once
#include "spmv.cuh"

namespace zk {

struct TmaPlan {
    int R;             // rows per tile (even)
    int NV;            // value slots per stage (≥ R·max_row_len, multiple of 4)
    int S;             // pipeline stages
    int64_t n_tiles;
    int64_t nnz;
    int64_t nnz4;      // nnz rounded down to a multiple of 4 (column copies never read past it)
    int off_col;       // byte offsets inside a stage
    int off_rp;
    int stage_bytes;
    int smem_bytes;    // S · stage_bytes
};

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "ZK_WAIT_%=:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
        "@!p bra ZK_WAIT_%=;\n"
        "}\n" ::"r"(smem_u32(bar)),
        "r"(parity)
        : "memory");
}
// 1-D TMA bulk copy global → shared, completion counted in bytes on `bar`
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
            smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(bar))
        : "memory");
}

struct TileBounds {
    int64_t ps, pe;  // value range of the tile
};

// thread 0: issue the copies of tile t into `stage`
__device__ __forceinline__ void tma_issue(const CsrDev& A, const TmaPlan& T, int64_t t, TileBounds b, char* stage,
                                          uint64_t* bar) {
    const int64_t r0 = t * T.R;
    const int64_t r1 = min(r0 + (int64_t)T.R, A.n_rows);
    const int64_t cnt = r1 - r0 + 1;               // row_ptr entries the tile needs
    int64_t cpy = (cnt + 1) & ~(int64_t)1;         // even count → multiple of 16 B
    int64_t* srp = (int64_t*)(stage + T.off_rp);
    if (r0 + cpy > A.n_rows + 1) {                 // last tile: never read past row_ptr[n]
        cpy = cnt & ~(int64_t)1;
        srp[cnt - 1] = b.pe;                       // row_ptr[r1] = row_ptr[n]
    }
    const int64_t cs = b.ps & ~(int64_t)3;
    int64_t ce = min((b.pe + 3) & ~(int64_t)3, T.nnz4);
    if (ce < cs) ce = cs;
    const uint32_t vb = (uint32_t)((b.pe - b.ps) * 16), cb = (uint32_t)((ce - cs) * 4), rb = (uint32_t)(cpy * 8);
    mbar_expect_tx(bar, vb + cb + rb);
    if (rb) bulk_g2s(srp, A.row_ptr + r0, rb, bar);
    if (vb) bulk_g2s(stage, A.val + b.ps, vb, bar);
    if (cb) bulk_g2s(stage + T.off_col, A.col + cs, cb, bar);
}

__device__ __forceinline__ TileBounds tile_bounds(const CsrDev& A, const TmaPlan& T, int64_t t) {
    const int64_t r0 = t * T.R;
    const int64_t r1 = min(r0 + (int64_t)T.R, A.n_rows);
    return {__ldg(A.row_ptr + r0), __ldg(A.row_ptr + r1)};
}

__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}

// Warp-specialised pipeline: warp 0 is the producer (lane 0 issues the bulk copies of tile k into
// stage k mod S once the consumers released it), warps 1..7 are consumers (W lanes per row).
// "full" barriers: producer expect_tx + TMA complete_tx; "empty" barriers: one arrive per
// consumer warp.  No CTA-wide barrier inside the loop: a consumer warp only waits for its data.
template <int W, class Epi>
__device__ __forceinline__ void spmv_tma_body(const CsrDev& A, const TmaPlan& T, const double2* __restrict__ x,
                                              Epi& epi) {
    static_assert(W >= 2 && W <= 32 && (W & (W - 1)) == 0, "W must be a power of two");
    constexpr int U = 4;
    constexpr int CW = kWarps - 1;           // consumer warps
    constexpr int GROUPS = CW * 32 / W;      // rows in flight per pass
    constexpr int KA = Epi::K > 0 ? Epi::K : 1;
    constexpr int kMaxStages = 8;
    extern __shared__ __align__(128) char zk_dyn_smem[];
    __shared__ __align__(8) uint64_t full[kMaxStages];
    __shared__ __align__(8) uint64_t empty[kMaxStages];

    double acc[KA];
#pragma unroll
    for (int k = 0; k < KA; k++) acc[k] = 0.0;
    const int64_t G = gridDim.x;
    const int S = T.S;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

    if (threadIdx.x == 0) {
        for (int s = 0; s < S; s++) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], CW);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();

    if (warp == 0) {
        // ---------------- producer
        // lane j holds the bounds of tile batch + j·G; the next batch of 32 is loaded while the
        // current one is issued, so the row_ptr latency never sits on the issue path
        auto load_batch = [&](int64_t tb, int64_t& ps, int64_t& pe) {
            const int64_t t = tb + lane * G;
            if (t < T.n_tiles) {
                const TileBounds b = tile_bounds(A, T, t);
                ps = b.ps;
                pe = b.pe;
            }
        };
        int64_t cps = 0, cpe = 0, k = 0;
        load_batch(blockIdx.x, cps, cpe);
        for (int64_t tb = blockIdx.x; tb < T.n_tiles; tb += 32 * G) {
            int64_t nps = 0, npe = 0;
            load_batch(tb + 32 * G, nps, npe);
            for (int j = 0; j < 32; j++, k++) {
                const int64_t t = tb + j * G;
                if (t >= T.n_tiles) break;
                const TileBounds b{__shfl_sync(0xffffffffu, cps, j), __shfl_sync(0xffffffffu, cpe, j)};
                if (lane == 0) {
                    const int s = (int)(k % S);
                    if (k >= S) mbar_wait(&empty[s], (uint32_t)(((k / S) - 1) & 1));
                    tma_issue(A, T, t, b, zk_dyn_smem + s * T.stage_bytes, &full[s]);
                }
                __syncwarp();
            }
            cps = nps;
            cpe = npe;
        }
    } else {
        // ---------------- consumers (32-bit in-tile offsets; the ≤3 trailing columns past the
        // last 16-B aligned column copy exist only in the matrix's final tile: uniform branch)
        const int ct = threadIdx.x - 32;     // consumer thread id
        const int sub = ct & (W - 1);
        const int grp = ct / W;
        int k = 0;
        for (int t = blockIdx.x; t < T.n_tiles; t += (int)G, k++) {
            const int s = k % S;
            const char* stage = zk_dyn_smem + s * T.stage_bytes;
            mbar_wait(&full[s], (uint32_t)((k / S) & 1));
            const double2* sval = (const double2*)stage;
            const int64_t* srp = (const int64_t*)(stage + T.off_rp);
            const int r0 = t * T.R;
            const int rows = min(T.R, (int)A.n_rows - r0);
            const int64_t ps = srp[0];
            const int* scol = (const int*)(stage + T.off_col) + (int)(ps & 3);
            const bool tail = srp[rows] > T.nnz4;
            for (int lr0 = 0; lr0 < rows; lr0 += GROUPS) {  // all consumer lanes iterate together
                const int lr = lr0 + grp;
                double2 sum = make_double2(0.0, 0.0);
                if (lr < rows) {
                    const int rb = (int)(srp[lr] - ps);
                    const int len = (int)(srp[lr + 1] - srp[lr]);
                    const double2* sv = sval + rb;
                    const int* sc = scol + rb;
                    for (int j0 = sub; j0 < len; j0 += U * W) {
                        int c[U];
#pragma unroll
                        for (int u = 0; u < U; u++) {
                            const int j = j0 + u * W;
                            c[u] = j < len ? sc[j] : -1;
                            if (tail && j < len && ps + rb + j >= T.nnz4) c[u] = __ldg(A.col + ps + rb + j);
                        }
                        double2 xv[U];
#pragma unroll
                        for (int u = 0; u < U; u++) xv[u] = c[u] >= 0 ? ld_gather(x + c[u]) : make_double2(0.0, 0.0);
#pragma unroll
                        for (int u = 0; u < U; u++)
                            if (c[u] >= 0) cfma(sum, sv[j0 + u * W], xv[u]);
                    }
                }
#pragma unroll
                for (int o = W / 2; o > 0; o >>= 1) {
                    sum.x += __shfl_xor_sync(0xffffffffu, sum.x, o, W);
                    sum.y += __shfl_xor_sync(0xffffffffu, sum.y, o, W);
                }
                if (sub == 0 && lr < rows) epi.row(r0 + lr, sum, epi.pre(r0 + lr), acc);
            }
            __syncwarp();
            if ((threadIdx.x & 31) == 0) mbar_arrive(&empty[s]);
        }
    }
    epi.finish(acc);
}

// host: plan for a matrix (rows per tile from the max row length)
inline bool make_tma_plan(int64_t n_rows, int64_t nnz, int max_len, TmaPlan* P, int stages = 4,
                          int stage_nnz = 756) {
    if (n_rows <= 0 || max_len <= 0 || max_len > 128) return false;
    int R = stage_nnz / max_len;
    R &= ~1;
    if (R < 8) return false;
    if (R > 256) R = 256;
    P->R = R;
    P->NV = ((R * max_len + 3) & ~3);
    P->S = stages;
    P->n_tiles = (n_rows + R - 1) / R;
    P->nnz = nnz;
    P->nnz4 = nnz & ~(int64_t)3;
    const int vbytes = P->NV * 16;
    const int cbytes = ((P->NV + 8) * 4 + 15) & ~15;
    const int rbytes = (((R + 2) * 8) + 15) & ~15;
    P->off_col = vbytes;
    P->off_rp = vbytes + cbytes;
    P->stage_bytes = (vbytes + cbytes + rbytes + 127) & ~127;
    P->smem_bytes = P->stage_bytes * stages;
    return true;
}

}  // namespace zk

namespace zk {
// SpMV body selected at compile time: MODE 1 = TMA-staged tiles, MODE 0 = sub-warp kernel
template <int W, int MODE, class Epi>
__device__ __forceinline__ void spmv_any(const CsrDev& A, const TmaPlan& T, const double2* __restrict__ x, Epi& epi) {
    if constexpr (sell_tail<Epi>::value && MODE != 3) {
        __trap();  // tail epilogues exist only in the SELL body (the host never launches this)
    } else if constexpr (MODE == 1) {
        spmv_tma_body<W>(A, T, x, epi);
    } else if constexpr (MODE == 2) {
        spmv_body_b4<W>(A, x, epi);
    } else if constexpr (MODE == 3) {
        spmv_body_sell(A, x, epi);
    } else {
        spmv_body<W>(A, x, epi);
    }
}
}  // namespace zk

namespace zk {
// __launch_bounds__ min blocks per SM of SpMV kernels: the sub-warp kernel keeps its loads in
// registers (more registers = more bytes in flight, measured best uncapped); the TMA kernel
// keeps the stream in shared memory and wants many consumer warps (cap registers at 40).
#ifndef ZK_TMA_MINB
#define ZK_TMA_MINB 6
#endif
#ifndef ZK_SPMV_MINB
#define ZK_SPMV_MINB 4
#endif
#ifndef ZK_SELL_MINB
#define ZK_SELL_MINB 3  // 80 registers: U = 9 entries in flight per lane without spilling (C4: 647 vs 869 µs at 64)
#endif
__host__ __device__ constexpr int spmv_min_blocks(int mode) {
    return mode == 1 ? ZK_TMA_MINB : mode == 3 ? ZK_SELL_MINB : ZK_SPMV_MINB;
}
}  // namespace zk
