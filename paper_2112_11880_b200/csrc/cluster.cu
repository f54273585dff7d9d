// cluster.cu — loop mode 5: the whole Krylov loop of a small system in ONE thread-block cluster,
// every reduction over distributed shared memory, the scalar steps replicated per CTA
// (solve_ctx.cuh).  The paper's own matrices (PAPER.md T1 P:52-70: Audi3D-1..4, Twingo3D-0..2; the
// solvers of §4, T9 P:313-341) are 1.7k-650k rows: latency-bound on a B200, where a
// kernel boundary costs more than an iteration's arithmetic.  Same per-row arithmetic and scalar
// steps as the grid kernels of solve.cu (NEXT-1..4), parity-
// tested against the oracle in every instantiation.  DESIGN.md §7 "Solver loop".
#include <algorithm>
#include <cstdio>
#include <cstring>
#include <vector>

#include <cooperative_groups.h>

#include "solve_ctx.cuh"

namespace zk {
// ------------------------------------------------------------------ cluster solver (loop mode 5)
// Small systems (the paper's Audi/Twingo shapes) are latency-bound: a WHILE-graph iteration of 5
// kernels costs ≈ 34-36 µs there, mostly kernel boundaries and the dependent global-memory round
// trips of the grid reductions.  Mode 5 runs the whole BiCGStab loop in ONE thread-block cluster
// (16 CTAs × 512 threads, non-portable size; 8 if 16 cannot be scheduled):
//  * rows are split into CS contiguous blocks, one per CTA; the CTA keeps its rows' entries of
//    x, r, r̂, p, v, s, t in shared memory for the whole solve (only p and s, which other CTAs
//    gather, are also written to global memory), and copies its block's column indices and row
//    offsets — and its values too when they fit — into shared memory once at the start, so a
//    SpMV chunk costs one L2 round trip (the gathers, with the values alongside) instead of two;
//  * the SpMV phases give each row W lanes (W ∈ {8, 4, 2, 1}, chosen on the host to minimise
//    passes × chunks per lane), each lane issuing all its loads of a chunk before using them;
//    gathers read p / s (L1-cacheable weak loads) after the cluster barrier that published them;
//  * every reduction is a block reduction into a shared-memory slot, one cluster barrier, and a
//    fixed-order sum of the CS slots: lane r of warp 0 reads rank r's slot over distributed shared
//    memory (one round trip instead of CS), then a fixed xor tree.  Every CTA runs the scalar step
//    (the same fin_* functions) on its own shared-memory copy of the context — identical inputs in
//    identical order give identical scalars, so nothing is broadcast and the loop never touches
//    global memory for control.
#ifndef ZK_CBLOCK
#define ZK_CBLOCK 512
#endif
constexpr int kCBlock = ZK_CBLOCK;
constexpr int kCWarps = kCBlock / 32;
constexpr int kCMaxCta = 16;  // cluster size: 16 (non-portable), else 8
constexpr int kCVecs = 7;                        // BiCGStab: x r r̂ p v s t own rows in shared memory
constexpr int kCVecsTfqmr = 9;                   // TFQMR: x w y1 y2 u1 u2 v d r̃
constexpr int kCVecsCg = 4;                      // CG / COCG: x r p q
constexpr int kCSmemMax = 216 * 1024;            // dynamic shared memory: own rows + the block's matrix

// The solve context into / out of a cluster CTA's shared copy, 8-byte words over all threads (a
// struct assignment by one thread went through local memory: ~1.2 KB of STL/LDL in the prologue).
__device__ __forceinline__ void ctx_copy(SolveCtx* dst, const SolveCtx* src) {
    static_assert(sizeof(SolveCtx) % 8 == 0, "SolveCtx in 8-byte words");
    const unsigned long long* s = reinterpret_cast<const unsigned long long*>(src);
    unsigned long long* d = reinterpret_cast<unsigned long long*>(dst);
    for (int i = threadIdx.x; i < (int)(sizeof(SolveCtx) / 8); i += blockDim.x) d[i] = s[i];
}

// The x0 = 0 start inside a cluster kernel (init = 1: k_set_ctx and k_init_zero are not launched):
// OpInitZero's per-row sums {‖b‖², ‖r0‖², Re r0ᵀr0, Im r0ᵀr0} of one own row (r0 = b), and the
// workspace tickets cleared as k_set_ctx does (recycled workspace memory; CTA 0 only).
__device__ __forceinline__ void cl_init_row(const double2 bl, double (&acc)[4]) {
    const double bb = cabs2(bl);
    acc[0] += bb;
    acc[1] += bb;
    acc[2] = fma(bl.x, bl.x, fma(-bl.y, bl.y, acc[2]));
    acc[3] = fma(2.0 * bl.x, bl.y, acc[3]);
}
__device__ __forceinline__ void cl_init_tickets(const SolveCtx& cs) {
    namespace cg = cooperative_groups;
    if (cg::this_cluster().block_rank() == 0 && threadIdx.x == 0)
        for (int i = 0; i < kTickets; i++) cs.tickets[i] = 0u;
}

// The solve's results out of CTA 0: into the handle's pinned staging when zk_solve asked for the
// zero-copy readback (no D2H copy after the kernel), else into the workspace context.
__device__ __forceinline__ void ctx_out(SolveCtx* gctx, SolveCtx& cs) {
    if (cs.out_host) {
        ctx_copy(cs.out_host, &cs);
        const int nh = min(cs.iters, cs.maxit) + 1;
        for (int i = threadIdx.x; i < nh; i += blockDim.x) cs.hist_host[i] = cs.hist[i];
    } else {
        ctx_copy(gctx, &cs);
    }
}

struct ClusterRed {
    double slot[2][kCMaxCta][kMaxRed];  // every CTA's partial sums, pushed here by their owners (double-buffered)
    double warp_part[kMaxRed][kCWarps];
    double tot[kMaxRed];
    int parity;
};

// cluster-wide sum of K doubles; result in R.tot (valid after the caller's __syncthreads).  Warps
// → the CTA's partial (warp 0, lane 0's value), which lanes r < ncta PUSH into CTA r's slot array
// (st.shared::cluster) before the cluster barrier; after it every CTA adds the ncta slots of its
// own shared memory in rank order — identical totals in every CTA, and no remote load on the
// critical path (a DSMEM load is ≈ 215 cycles, B300_MICROARCH.md; the pull version read the ncta
// slots over DSMEM after the barrier).
template <int K>
__device__ __forceinline__ void cl_sum(double (&v)[K], ClusterRed& R) {
    namespace cg = cooperative_groups;
    cg::cluster_group cl = cg::this_cluster();
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    warp_sum<K>(v);
    if (lane == 0) {
#pragma unroll
        for (int k = 0; k < K; k++) R.warp_part[k][warp] = v[k];
    }
    __syncthreads();
    const int par = R.parity;
    const unsigned ncta = cl.num_blocks();
    if (warp == 0) {
        double w[K];
#pragma unroll
        for (int k = 0; k < K; k++) w[k] = lane < kCWarps ? R.warp_part[k][lane] : 0.0;
        warp_sum<K>(w);
#pragma unroll
        for (int k = 0; k < K; k++) w[k] = __shfl_sync(0xffffffffu, w[k], 0);  // lane 0's value, everywhere
        if ((unsigned)lane < ncta) {
            double* dst = cl.map_shared_rank(&R.slot[par][cl.block_rank()][0], lane);
#pragma unroll
            for (int k = 0; k < K; k++) dst[k] = w[k];
        }
    }
    cl.sync();  // release/acquire at cluster scope: the pushed slots (and this phase's global writes) visible
    if (warp == 0) {
        if (lane < K) {
            double t = 0.0;
            for (unsigned r = 0; r < ncta; r++) t += R.slot[par][r][lane];
            R.tot[lane] = t;
        }
        __syncwarp();  // R.tot for thread 0 (the caller's scalar step)
        if (lane == 0) R.parity = par ^ 1;
    }
}

// Gather of p / s inside the cluster solver: a weak load that may hit L1.  Correct because every
// phase that reads them starts after a cluster barrier (acquire at cluster scope, which also
// invalidates L1), and nothing writes them during the reading phase.  A CTA's rows gather from a
// window near its own block (FE bandwidth), which fits L1 next to the shared-memory carve-out.
__device__ __forceinline__ double2 ld_l1(const double2* p) {
    double2 v;
    asm volatile("ld.global.ca.v2.f64 {%0, %1}, [%2];" : "=d"(v.x), "=d"(v.y) : "l"(p));
    return v;
}

// Values in global memory (!VS) are loaded with L1::no_allocate: they are re-read from L2 every
// SpMV anyway (a CTA's block does not fit the L1 left beside the shared-memory carve-out), and
// allocating them evicted the gathered x window from L1.
#ifndef ZK_CL_VAL_NA
#define ZK_CL_VAL_NA 1
#endif
// own row l of A·x on W lanes (sub = lane within the row's group): columns (and values when VS)
// from the CTA's shared-memory copy, x gathered through L2.  valid == false: the lanes take part
// in the shuffles only.
template <int W, bool VS>
__device__ __forceinline__ double2 cl_row(const double2* __restrict__ gval, const double2* sval, const int* scol,
                                          const int* soff, const double2* x, int l, bool valid, int sub) {
    constexpr int U = 4;  // 8 spills at the 128-register cap of 512-thread CTAs (U = 8 at W = 2: 2.4 KB, 2x slower)
    double2 sum = make_double2(0.0, 0.0);
    if (valid) {
        const int rs = soff[l], re = soff[l + 1];
        for (int p0 = rs + sub; p0 < re; p0 += U * W) {
            double2 v[U], xv[U];
            int c[U];
#pragma unroll
            for (int u = 0; u < U; u++) c[u] = p0 + u * W < re ? scol[p0 + u * W] : -1;
#pragma unroll
            for (int u = 0; u < U; u++) {
                if (c[u] >= 0) {
                    v[u] = VS ? sval[p0 + u * W] : (ZK_CL_VAL_NA ? ld_stream(gval + p0 + u * W) : __ldg(gval + p0 + u * W));
                    xv[u] = ld_l1(x + c[u]);
                }
            }
#pragma unroll
            for (int u = 0; u < U; u++)
                if (c[u] >= 0) cfma(sum, v[u], xv[u]);
        }
    }
#pragma unroll
    for (int o = W / 2; o > 0; o >>= 1) {
        sum.x += __shfl_xor_sync(0xffffffffu, sum.x, o, W);
        sum.y += __shfl_xor_sync(0xffffffffu, sum.y, o, W);
    }
    return sum;
}

// The CTA's block of the matrix into shared memory (columns, row offsets relative to the block,
// values when VS); returns the block's first value in global memory (used when !VS).
template <bool VS>
__device__ __forceinline__ const double2* cl_stage(const CsrDev& A, int row0, int nr, double2* sval, int* scol,
                                                   int* soff) {
    const int64_t nz0 = nr > 0 ? A.row_ptr[row0] : 0;
    const int nnz_cta = nr > 0 ? (int)(A.row_ptr[row0 + nr] - nz0) : 0;
    for (int l = threadIdx.x; l <= nr; l += kCBlock) soff[l] = nr > 0 ? (int)(A.row_ptr[row0 + l] - nz0) : 0;
    for (int q = threadIdx.x; q < nnz_cta; q += kCBlock) {
        scol[q] = A.col[nz0 + q];
        if (VS) sval[q] = A.val[nz0 + q];
    }
    return A.val + nz0;
}

// The solve's exit check ‖b − A x‖/‖b‖ inside the cluster kernel (EpiTrue + fin_true; the host
// k_true launch is skipped).  The caller has written its rows of x to xg; the cluster barrier here
// publishes them for the gathers.
template <int W, bool VS>
__device__ __forceinline__ void cl_true(SolveCtx* c, ClusterRed& R, const double2* gval, const double2* sval,
                                        const int* scol, const int* soff, const double2* xg, int row0, int nr) {
    namespace cg = cooperative_groups;
    cg::this_cluster().sync();
    if (c->status == ST_ZERO_RHS) return;  // replicated state: the same branch in every CTA
    constexpr int RPP = kCBlock / W;
    const int sub = threadIdx.x & (W - 1), grp = threadIdx.x / W;
    const double2* bg = c->b;
    double acc[1] = {0.0};
    for (int b = 0; b < nr; b += RPP) {
        const int l = b + grp;
        const double2 y = cl_row<W, VS>(gval, sval, scol, soff, xg, l, l < nr, sub);
        if (sub == 0 && l < nr) acc[0] += cabs2(csub(bg[row0 + l], y));
    }
    cl_sum<1>(acc, R);
    if (threadIdx.x == 0) fin_true(c, R.tot);
    __syncthreads();
}

// init: the x0 = 0 start (x = 0, r = r̂ = p = b, ‖b‖, hist[0]) runs here from the context passed
// by value, instead of the k_set_ctx + k_init_zero launches (Audi3D-1: fixed cost of a solve
// 79.8 → 71.4 µs, tools/latency_probe.py).
// (Tried and removed, profiles/r02_cluster_latency.txt: (a) every CTA holding a shared-memory copy
// of the WHOLE SpMV input, filled over distributed shared memory before each publishing barrier —
// Audi3D-1 9.9 → 11.5 µs per iteration, the 16-way DSMEM broadcast costs more than the L2 round
// trips it removes; (b) 3 cluster barriers per iteration instead of 5, with p = r + β(p − ωv) and
// s = r − αv formed inside the SpMV gathers from the published r, p, v — 9.7 → 15.5 (C1), 24.2 →
// 53.3 (C2): the 2-3× L2 gathers cost far more than the two barriers.)
// dynamic shared memory: kCVecs × rpc vectors | [values nnz_max] | columns nnz_max | offsets rpc + 1
// ZK_CLUSTER_PROF (tools build only): per-phase SM-cycle totals of CTA 0's thread 0, printed at exit
#ifndef ZK_CLUSTER_PROF
#define ZK_CLUSTER_PROF 0
#endif
#define CPT(k)                                                                        \
    do {                                                                              \
        if (ZK_CLUSTER_PROF && threadIdx.x == 0 && cl.block_rank() == 0) pts_[k] = gtimer(); \
    } while (0)
#define CPROF(k)                                                            \
    do {                                                                    \
        if (ZK_CLUSTER_PROF && threadIdx.x == 0 && cl.block_rank() == 0) {  \
            const long long t_ = clock64();                                 \
            prof_[k] += t_ - prof_t_;                                       \
            prof_t_ = t_;                                                   \
        }                                                                   \
    } while (0)
template <int W, bool VS>
__global__ void __launch_bounds__(kCBlock, 1) k_cluster_bicg(SolveCtx* gctx, const __grid_constant__ SolveCtx hctx, const CsrDev A,
                                                             int nnz_max, int do_true, int init) {
    namespace cg = cooperative_groups;
    cg::cluster_group cl = cg::this_cluster();
    extern __shared__ double2 own[];
    __shared__ SolveCtx cs;
    __shared__ ClusterRed R;
    unsigned long long pts_[8] = {};  // ZK_CLUSTER_PROF: global-timer marks of the prologue / epilogue
    CPT(0);
    ctx_copy(&cs, init ? &hctx : gctx);
    if (threadIdx.x == 0) R.parity = 0;
    const int n = (int)A.n_rows;
    const int ncta = (int)cl.num_blocks();
    const int rpc = (n + ncta - 1) / ncta;
    const int row0 = (int)cl.block_rank() * rpc;
    const int nr = max(0, min(rpc, n - row0));
    double2 *X = own, *Rv = own + rpc, *RH = own + 2 * rpc, *P = own + 3 * rpc, *V = own + 4 * rpc,
            *S = own + 5 * rpc, *T = own + 6 * rpc;
    double2* sval = own + kCVecs * rpc;
    int* scol = (int*)(sval + (VS ? nnz_max : 0));
    int* soff = scol + nnz_max;
    __syncthreads();
    SolveCtx* c = &cs;
    double2 *xg = cs.x, *pg = cs.p, *sg = cs.s;
    if (init) {  // x0 = 0: x = 0 ; r = r̂ = p = b ; {‖b‖², ‖r‖², Re bᵀb, Im bᵀb} (OpInitZero, fin_init_bicg)
        const double2* bg = cs.b;
        double acc[4] = {0.0, 0.0, 0.0, 0.0};
        for (int l = threadIdx.x; l < nr; l += kCBlock) {
            const double2 bl = bg[row0 + l];
            X[l] = make_double2(0.0, 0.0);
            Rv[l] = RH[l] = P[l] = bl;
            pg[row0 + l] = bl;
            cl_init_row(bl, acc);
        }
        cl_init_tickets(cs);
        CPT(1);
        cl_sum<4>(acc, R);  // its cluster barrier also publishes p for the K1 gathers
        if (threadIdx.x == 0) fin_init_bicg(c, R.tot);
        __syncthreads();
        CPT(2);
    } else {
        for (int l = threadIdx.x; l < nr; l += kCBlock) {  // r0, r̂, p, x0 from the init kernel
            X[l] = xg[row0 + l];
            Rv[l] = cs.r[row0 + l];
            RH[l] = cs.rh[row0 + l];
            P[l] = pg[row0 + l];
        }
    }
    const double2* gval = cl_stage<VS>(A, row0, nr, sval, scol, soff);
    __syncthreads();
    CPT(3);
    constexpr int RPP = kCBlock / W;  // rows per SpMV pass
    const int sub = threadIdx.x & (W - 1);
    const int grp = threadIdx.x / W;
    int bodies = 0;
    long long prof_[13] = {}, prof_t_ = clock64();
    while (!c->done) {
        {   // K1: v = A p ; σ = ⟨r̂, v⟩, ‖v‖²
            double acc[3] = {0.0, 0.0, 0.0};
            for (int b = 0; b < nr; b += RPP) {
                const int l = b + grp;
                const double2 y = cl_row<W, VS>(gval, sval, scol, soff, pg, l, l < nr, sub);
                if (sub == 0 && l < nr) {
                    V[l] = y;
                    const double2 q = RH[l];
                    acc[0] = fma(q.x, y.x, fma(q.y, y.y, acc[0]));
                    acc[1] = fma(q.x, y.y, fma(-q.y, y.x, acc[1]));
                    acc[2] += cabs2(y);
                }
            }
            CPROF(0);
            cl_sum<3>(acc, R);
            CPROF(1);
            if (threadIdx.x == 0) fin_k1_bicg(c, R.tot);
            __syncthreads();
            CPROF(2);
            if (c->done) break;
        }
        {   // K2: s = r − α v ; ‖s‖²
            const double2 al = c->alpha;
            double acc[1] = {0.0};
            for (int l = threadIdx.x; l < nr; l += kCBlock) {
                const double2 vi = V[l];
                double2 o = Rv[l];
                o.x = fma(-al.x, vi.x, fma(al.y, vi.y, o.x));
                o.y = fma(-al.x, vi.y, fma(-al.y, vi.x, o.y));
                S[l] = o;
                sg[row0 + l] = o;
                acc[0] += cabs2(o);
            }
            CPROF(3);
            cl_sum<1>(acc, R);  // its cluster barrier also publishes s for the K3 gathers
            CPROF(4);
            if (threadIdx.x == 0) fin_k2_bicg(c, R.tot);
            __syncthreads();
            CPROF(5);
            if (c->done) {  // half-step exit: x += α p
                if (c->half) {
                    for (int l = threadIdx.x; l < nr; l += kCBlock) cfma(X[l], al, P[l]);
                    __syncthreads();
                    if (threadIdx.x == 0) c->half = 0;
                }
                break;
            }
        }
        {   // K3: t = A s ; ⟨t, s⟩, ‖t‖²
            double acc[3] = {0.0, 0.0, 0.0};
            for (int b = 0; b < nr; b += RPP) {
                const int l = b + grp;
                const double2 y = cl_row<W, VS>(gval, sval, scol, soff, sg, l, l < nr, sub);
                if (sub == 0 && l < nr) {
                    T[l] = y;
                    const double2 si = S[l];
                    acc[0] = fma(y.x, si.x, fma(y.y, si.y, acc[0]));
                    acc[1] = fma(y.x, si.y, fma(-y.y, si.x, acc[1]));
                    acc[2] += cabs2(y);
                }
            }
            CPROF(6);
            cl_sum<3>(acc, R);
            CPROF(7);
            if (threadIdx.x == 0) fin_k3_bicg(c, R.tot);
            __syncthreads();
            CPROF(8);
            if (c->done) break;
        }
        {   // K4: x += α p + ω s ; r = s − ω t ; ‖r‖², ⟨r̂, r⟩
            const double2 al = c->alpha, om = c->omega;
            double acc[3] = {0.0, 0.0, 0.0};
            for (int l = threadIdx.x; l < nr; l += kCBlock) {
                const double2 si = S[l], ti = T[l];
                double2 xi = X[l];
                cfma(xi, al, P[l]);
                cfma(xi, om, si);
                X[l] = xi;
                double2 rn = si;
                rn.x = fma(-om.x, ti.x, fma(om.y, ti.y, rn.x));
                rn.y = fma(-om.x, ti.y, fma(-om.y, ti.x, rn.y));
                Rv[l] = rn;
                const double2 q = RH[l];
                acc[0] += cabs2(rn);
                acc[1] = fma(q.x, rn.x, fma(q.y, rn.y, acc[1]));
                acc[2] = fma(q.x, rn.y, fma(-q.y, rn.x, acc[2]));
            }
            CPROF(9);
            cl_sum<3>(acc, R);
            CPROF(10);
            if (threadIdx.x == 0) fin_k4_bicg(c, R.tot);
            __syncthreads();
            CPROF(11);
            if (c->done) break;
        }
        {   // K5: p = r + β (p − ω v), then a cluster barrier (p is gathered by K1)
            const double2 be = c->beta, om = c->omega;
            for (int l = threadIdx.x; l < nr; l += kCBlock) {
                const double2 vi = V[l];
                double2 d = P[l];
                d.x = fma(-om.x, vi.x, fma(om.y, vi.y, d.x));
                d.y = fma(-om.x, vi.y, fma(-om.y, vi.x, d.y));
                double2 o = Rv[l];
                cfma(o, be, d);
                P[l] = o;
                pg[row0 + l] = o;
            }
            cl.sync();
            CPROF(12);
        }
        bodies++;
    }
    CPT(4);
    for (int l = threadIdx.x; l < nr; l += kCBlock) xg[row0 + l] = X[l];  // the solution leaves shared memory
    if (do_true) cl_true<W, VS>(c, R, gval, sval, scol, soff, xg, row0, nr);
    CPT(5);
    if (threadIdx.x == 0) cs.bodies = bodies;
    __syncthreads();
    if (cl.block_rank() == 0) ctx_out(gctx, cs);
    cl.sync();  // no CTA leaves while another may still read its reduction slots
    CPT(6);
    if (ZK_CLUSTER_PROF && threadIdx.x == 0 && cl.block_rank() == 0) {
        printf("cluster_prof bodies %d cycles: k1 %lld red %lld fin %lld | k2 %lld red %lld fin %lld | k3 %lld red %lld fin %lld | k4 %lld red %lld fin %lld | k5+sync %lld\n",
               bodies, prof_[0], prof_[1], prof_[2], prof_[3], prof_[4], prof_[5], prof_[6], prof_[7], prof_[8],
               prof_[9], prof_[10], prof_[11], prof_[12]);
        printf("cluster_prof ns: ctx+init rows %llu | init reduce %llu | stage %llu | loop %llu | x out + true %llu | ctx out %llu\n",
               pts_[1] - pts_[0], pts_[2] - pts_[1], pts_[3] - pts_[2], pts_[4] - pts_[3], pts_[5] - pts_[4],
               pts_[6] - pts_[5]);
    }
}

// TFQMR (NEXT-2) in one cluster: the per-row arithmetic of OpT1/EpiT2/OpT3/EpiT4 and the same
// scalar steps (fin_t1 / fin_t2 / fin_sigma), including the exits inside an iteration (half = 1:
// only x += η1·d1 remains; half = 2: T3's d and x updates without y1).  y1 and y2 are gathered by
// the SpMVs, so they are also written to global memory.
template <int W, bool VS>
__global__ void __launch_bounds__(kCBlock, 1) k_cluster_tfqmr(SolveCtx* gctx, const __grid_constant__ SolveCtx hctx,
                                                              const CsrDev A, int nnz_max, int do_true, int init) {
    namespace cg = cooperative_groups;
    cg::cluster_group cl = cg::this_cluster();
    extern __shared__ double2 own[];
    __shared__ SolveCtx cs;
    __shared__ ClusterRed R;
    ctx_copy(&cs, init ? &hctx : gctx);
    if (threadIdx.x == 0) R.parity = 0;
    const int n = (int)A.n_rows;
    const int ncta = (int)cl.num_blocks();
    const int rpc = (n + ncta - 1) / ncta;
    const int row0 = (int)cl.block_rank() * rpc;
    const int nr = max(0, min(rpc, n - row0));
    double2 *X = own, *Wv = own + rpc, *Y1 = own + 2 * rpc, *Y2 = own + 3 * rpc, *U1 = own + 4 * rpc,
            *U2 = own + 5 * rpc, *V = own + 6 * rpc, *D = own + 7 * rpc, *RT = own + 8 * rpc;
    double2* sval = own + kCVecsTfqmr * rpc;
    int* scol = (int*)(sval + (VS ? nnz_max : 0));
    int* soff = scol + nnz_max;
    __syncthreads();
    SolveCtx* c = &cs;
    double2 *xg = cs.x, *y1g = cs.y1, *y2g = cs.y2;
    double iacc[4] = {0.0, 0.0, 0.0, 0.0};
    if (init) {  // x0 = 0: x = 0 ; w = y1 = r̃ = b ; d = 0 (OpInitZero kind 4); y1 published for K0
        const double2* bg = cs.b;
        for (int l = threadIdx.x; l < nr; l += kCBlock) {
            const double2 bl = bg[row0 + l];
            X[l] = make_double2(0.0, 0.0);
            Wv[l] = Y1[l] = RT[l] = bl;
            y1g[row0 + l] = bl;
            D[l] = U1[l] = V[l] = make_double2(0.0, 0.0);
            U2[l] = Y2[l] = make_double2(0.0, 0.0);
            cl_init_row(bl, iacc);
        }
        cl_init_tickets(cs);
    } else {
        for (int l = threadIdx.x; l < nr; l += kCBlock) {  // state after the init kernel and K0
            const int i = row0 + l;
            X[l] = xg[i];
            Wv[l] = cs.w[i];
            Y1[l] = y1g[i];
            U1[l] = cs.u1[i];
            V[l] = cs.v[i];
            D[l] = cs.d[i];
            RT[l] = cs.rt[i];
            U2[l] = make_double2(0.0, 0.0);
            Y2[l] = make_double2(0.0, 0.0);
        }
    }
    const double2* gval = cl_stage<VS>(A, row0, nr, sval, scol, soff);
    __syncthreads();
    constexpr int RPP = kCBlock / W;
    const int sub = threadIdx.x & (W - 1);
    const int grp = threadIdx.x / W;
    if (init) {
        cl_sum<4>(iacc, R);  // its cluster barrier also publishes y1 for K0's gathers
        if (threadIdx.x == 0) fin_init_tfqmr(c, R.tot);
        __syncthreads();
        if (!c->done) {  // K0: u1 = v = A y1 ; σ = ⟨r̃, v⟩ (EpiT4Tfqmr<S_K0_TFQMR>, fin_sigma_tfqmr)
            double acc[2] = {0.0, 0.0};
            for (int b = 0; b < nr; b += RPP) {
                const int l = b + grp;
                const double2 y = cl_row<W, VS>(gval, sval, scol, soff, y1g, l, l < nr, sub);
                if (sub == 0 && l < nr) {
                    U1[l] = y;
                    V[l] = y;
                    const double2 q = RT[l];
                    acc[0] = fma(q.x, y.x, fma(q.y, y.y, acc[0]));
                    acc[1] = fma(q.x, y.y, fma(-q.y, y.x, acc[1]));
                }
            }
            cl_sum<2>(acc, R);
            if (threadIdx.x == 0) fin_sigma_tfqmr(c, R.tot);
            __syncthreads();
        }
    }
    int bodies = 0;
    while (!c->done) {
        {   // T1: y2 = y1 − α v ; w −= α u1 ; ‖w‖²
            const double2 al = c->alpha;
            double acc[1] = {0.0};
            for (int l = threadIdx.x; l < nr; l += kCBlock) {
                const double2 vv = V[l], uu = U1[l];
                double2 o = Y1[l];
                o.x = fma(-al.x, vv.x, fma(al.y, vv.y, o.x));
                o.y = fma(-al.x, vv.y, fma(-al.y, vv.x, o.y));
                Y2[l] = o;
                y2g[row0 + l] = o;
                double2 wn = Wv[l];
                wn.x = fma(-al.x, uu.x, fma(al.y, uu.y, wn.x));
                wn.y = fma(-al.x, uu.y, fma(-al.y, uu.x, wn.y));
                Wv[l] = wn;
                acc[0] += cabs2(wn);
            }
            cl_sum<1>(acc, R);  // also publishes y2 for the T2 gathers
            if (threadIdx.x == 0) fin_t1_tfqmr(c, R.tot);
            __syncthreads();
            if (c->done) {
                if (c->half == 1) {  // the first half step ended the loop: x += η1·d1, d1 = y1 + c1·d
                    const double2 eta = c->eta1, coef = c->coef1;
                    for (int l = threadIdx.x; l < nr; l += kCBlock) {
                        double2 d1 = Y1[l];
                        cfma(d1, coef, D[l]);
                        cfma(X[l], eta, d1);
                    }
                }
                break;
            }
        }
        {   // T2: u2 = A y2 ; w −= α u2 ; ‖w‖², ⟨r̃, w⟩
            const double2 al = c->alpha;
            double acc[3] = {0.0, 0.0, 0.0};
            for (int b = 0; b < nr; b += RPP) {
                const int l = b + grp;
                const double2 y = cl_row<W, VS>(gval, sval, scol, soff, y2g, l, l < nr, sub);
                if (sub == 0 && l < nr) {
                    U2[l] = y;
                    double2 wn = Wv[l];
                    wn.x = fma(-al.x, y.x, fma(al.y, y.y, wn.x));
                    wn.y = fma(-al.x, y.y, fma(-al.y, y.x, wn.y));
                    Wv[l] = wn;
                    const double2 q = RT[l];
                    acc[0] += cabs2(wn);
                    acc[1] = fma(q.x, wn.x, fma(q.y, wn.y, acc[1]));
                    acc[2] = fma(q.x, wn.y, fma(-q.y, wn.x, acc[2]));
                }
            }
            cl_sum<3>(acc, R);
            if (threadIdx.x == 0) fin_t2_tfqmr(c, R.tot);
            __syncthreads();
        }
        {   // T3: d1 = y1 + c1·d ; d = y2 + c2·d1 ; x += η1·d1 + η2·d ; y1 = w + β y2 (not on exit)
            const bool done = c->done != 0;
            if (done && c->half != 2) break;
            const double2 coef1 = c->coef1, coef2 = c->coef2, eta1 = c->eta1, eta2 = c->eta, be = c->beta;
            for (int l = threadIdx.x; l < nr; l += kCBlock) {
                double2 d1 = Y1[l];
                cfma(d1, coef1, D[l]);
                const double2 y2 = Y2[l];
                double2 d2 = y2;
                cfma(d2, coef2, d1);
                double2 xn = X[l];
                cfma(xn, eta1, d1);
                cfma(xn, eta2, d2);
                X[l] = xn;
                D[l] = d2;
                if (!done) {
                    double2 o = Wv[l];
                    cfma(o, be, y2);
                    Y1[l] = o;
                    y1g[row0 + l] = o;
                }
            }
            if (done) break;
            cl.sync();  // y1 complete for the T4 gathers
        }
        {   // T4: u1 = A y1 ; v = u1 + β(u2 + β v) ; σ = ⟨r̃, v⟩
            const double2 be = c->beta;
            double acc[2] = {0.0, 0.0};
            for (int b = 0; b < nr; b += RPP) {
                const int l = b + grp;
                const double2 y = cl_row<W, VS>(gval, sval, scol, soff, y1g, l, l < nr, sub);
                if (sub == 0 && l < nr) {
                    U1[l] = y;
                    double2 t = U2[l];
                    cfma(t, be, V[l]);
                    double2 vn = y;
                    cfma(vn, be, t);
                    V[l] = vn;
                    const double2 q = RT[l];
                    acc[0] = fma(q.x, vn.x, fma(q.y, vn.y, acc[0]));
                    acc[1] = fma(q.x, vn.y, fma(-q.y, vn.x, acc[1]));
                }
            }
            cl_sum<2>(acc, R);
            if (threadIdx.x == 0) fin_sigma_tfqmr(c, R.tot);
            __syncthreads();
        }
        bodies++;
    }
    __syncthreads();
    for (int l = threadIdx.x; l < nr; l += kCBlock) xg[row0 + l] = X[l];
    if (do_true) cl_true<W, VS>(c, R, gval, sval, scol, soff, xg, row0, nr);
    if (threadIdx.x == 0) {
        cs.half = 0;
        cs.bodies = bodies;
    }
    __syncthreads();
    if (cl.block_rank() == 0) ctx_out(gctx, cs);
    cl.sync();
}

// CG (conjugated products, real α/β) and COCG (NEXT-4: unconjugated, complex α/β) in one cluster:
// the per-row arithmetic of EpiK1Cg/OpK2Cg/OpK3Cg and EpiK1Cocg/OpK2Cocg/OpK3Cocg, the same
// scalar steps.  p is gathered by the SpMV, so it is also written to global memory.
template <int W, bool VS, bool COCG>
__global__ void __launch_bounds__(kCBlock, 1) k_cluster_cg(SolveCtx* gctx, const __grid_constant__ SolveCtx hctx,
                                                           const CsrDev A, int nnz_max, int do_true, int init) {
    namespace cg = cooperative_groups;
    cg::cluster_group cl = cg::this_cluster();
    extern __shared__ double2 own[];
    __shared__ SolveCtx cs;
    __shared__ ClusterRed R;
    ctx_copy(&cs, init ? &hctx : gctx);
    if (threadIdx.x == 0) R.parity = 0;
    const int n = (int)A.n_rows;
    const int ncta = (int)cl.num_blocks();
    const int rpc = (n + ncta - 1) / ncta;
    const int row0 = (int)cl.block_rank() * rpc;
    const int nr = max(0, min(rpc, n - row0));
    double2 *X = own, *Rv = own + rpc, *P = own + 2 * rpc, *Q = own + 3 * rpc;
    double2* sval = own + kCVecsCg * rpc;
    int* scol = (int*)(sval + (VS ? nnz_max : 0));
    int* soff = scol + nnz_max;
    __syncthreads();
    SolveCtx* c = &cs;
    double2 *xg = cs.x, *pg = cs.p;
    if (init) {  // x0 = 0: x = 0 ; r = p = b (OpInitZero kinds 1, 3) ; fin_init_cg / fin_init_cocg
        const double2* bg = cs.b;
        double acc[4] = {0.0, 0.0, 0.0, 0.0};
        for (int l = threadIdx.x; l < nr; l += kCBlock) {
            const double2 bl = bg[row0 + l];
            X[l] = make_double2(0.0, 0.0);
            Rv[l] = P[l] = bl;
            pg[row0 + l] = bl;
            cl_init_row(bl, acc);
        }
        cl_init_tickets(cs);
        cl_sum<4>(acc, R);  // its cluster barrier also publishes p for the K1 gathers
        if (threadIdx.x == 0) {
            if (COCG) fin_init_cocg(c, R.tot);
            else fin_init_cg(c, R.tot);
        }
        __syncthreads();
    } else {
        for (int l = threadIdx.x; l < nr; l += kCBlock) {
            X[l] = xg[row0 + l];
            Rv[l] = cs.r[row0 + l];
            P[l] = pg[row0 + l];
        }
    }
    const double2* gval = cl_stage<VS>(A, row0, nr, sval, scol, soff);
    __syncthreads();
    constexpr int RPP = kCBlock / W;
    const int sub = threadIdx.x & (W - 1);
    const int grp = threadIdx.x / W;
    int bodies = 0;
    while (!c->done) {
        {   // K1: q = A p ; CG δ = ⟨p, q⟩ / COCG μ = pᵀq
            double acc[2] = {0.0, 0.0};
            for (int b = 0; b < nr; b += RPP) {
                const int l = b + grp;
                const double2 y = cl_row<W, VS>(gval, sval, scol, soff, pg, l, l < nr, sub);
                if (sub == 0 && l < nr) {
                    Q[l] = y;
                    const double2 pi = P[l];
                    if (COCG) {
                        acc[0] = fma(pi.x, y.x, fma(-pi.y, y.y, acc[0]));
                        acc[1] = fma(pi.x, y.y, fma(pi.y, y.x, acc[1]));
                    } else {
                        acc[0] = fma(pi.x, y.x, fma(pi.y, y.y, acc[0]));
                        acc[1] = fma(pi.x, y.y, fma(-pi.y, y.x, acc[1]));
                    }
                }
            }
            cl_sum<2>(acc, R);
            if (threadIdx.x == 0) {
                if (COCG) fin_k1_cocg(c, R.tot);
                else fin_k1_cg(c, R.tot);
            }
            __syncthreads();
            if (c->done) break;
        }
        {   // K2: x += α p ; r −= α q ; ‖r‖² (COCG: and rᵀr)
            constexpr int K2 = COCG ? 3 : 1;
            double acc[K2];
#pragma unroll
            for (int k = 0; k < K2; k++) acc[k] = 0.0;
            for (int l = threadIdx.x; l < nr; l += kCBlock) {
                const double2 pi = P[l], qi = Q[l];
                if (COCG) {
                    const double2 al = c->alpha;
                    double2 xn = X[l];
                    cfma(xn, al, pi);
                    X[l] = xn;
                    double2 rn = Rv[l];
                    rn.x = fma(-al.x, qi.x, fma(al.y, qi.y, rn.x));
                    rn.y = fma(-al.x, qi.y, fma(-al.y, qi.x, rn.y));
                    Rv[l] = rn;
                    acc[0] += cabs2(rn);
                    acc[K2 > 1 ? 1 : 0] = fma(rn.x, rn.x, fma(-rn.y, rn.y, acc[K2 > 1 ? 1 : 0]));
                    acc[K2 > 2 ? 2 : 0] = fma(2.0 * rn.x, rn.y, acc[K2 > 2 ? 2 : 0]);
                } else {
                    const double al = c->alpha_cg;
                    const double2 xi = X[l], ri = Rv[l];
                    X[l] = make_double2(fma(al, pi.x, xi.x), fma(al, pi.y, xi.y));
                    const double2 rn = make_double2(fma(-al, qi.x, ri.x), fma(-al, qi.y, ri.y));
                    Rv[l] = rn;
                    acc[0] += cabs2(rn);
                }
            }
            cl_sum<K2>(acc, R);
            if (threadIdx.x == 0) {
                if (COCG) fin_k2_cocg(c, R.tot);
                else fin_k2_cg(c, R.tot);
            }
            __syncthreads();
            if (c->done) break;
        }
        {   // K3: p = r + β p, then a cluster barrier (p is gathered by K1)
            for (int l = threadIdx.x; l < nr; l += kCBlock) {
                double2 o;
                if (COCG) {
                    o = Rv[l];
                    cfma(o, c->beta, P[l]);
                } else {
                    const double be = c->beta_cg;
                    const double2 pi = P[l], ri = Rv[l];
                    o = make_double2(fma(be, pi.x, ri.x), fma(be, pi.y, ri.y));
                }
                P[l] = o;
                pg[row0 + l] = o;
            }
            cl.sync();
        }
        bodies++;
    }
    __syncthreads();
    for (int l = threadIdx.x; l < nr; l += kCBlock) xg[row0 + l] = X[l];
    if (do_true) cl_true<W, VS>(c, R, gval, sval, scol, soff, xg, row0, nr);
    if (threadIdx.x == 0) cs.bodies = bodies;
    __syncthreads();
    if (cl.block_rank() == 0) ctx_out(gctx, cs);
    cl.sync();
}

// BiCGStab(ℓ) (NEXT-3) in one cluster: one outer cycle = for j < ℓ: B1 (+ cluster barrier), S1
// (γ → α), B2 (exit test), S2 (ρ1 → β, j < ℓ−1); then the Gram matrix of r̂_0..ℓ and the update U —
// the per-element arithmetic of bl_b1 / EpiBl / bl_b2 / bl_gram / bl_u and the same scalar steps.
// The 2ℓ+2 vectors stay in global memory (L2-resident at these sizes); each thread owns the same
// elements in every phase, so only the SpMV gathers cross CTAs (after a cluster barrier).  The
// Gram matrix: ND ≤ 81 sums per CTA over its rows (6 threads per entry, fixed order), one slot
// per CTA, rank-ordered sum over DSMEM, Cholesky by fin_gram_bl<ℓ> in every CTA.
constexpr int kGramMax = 81;  // (ℓ+1) + ℓ(ℓ+1) doubles at ℓ = 8
constexpr int kGramSub = 6;   // threads per Gram entry
__device__ __noinline__ void fin_gram_any(SolveCtx* c, const double* g, int ell) {
    switch (ell) {
        case 1: fin_gram_bl<1>(c, g); break;
        case 2: fin_gram_bl<2>(c, g); break;
        case 3: fin_gram_bl<3>(c, g); break;
        case 4: fin_gram_bl<4>(c, g); break;
        case 5: fin_gram_bl<5>(c, g); break;
        case 6: fin_gram_bl<6>(c, g); break;
        case 7: fin_gram_bl<7>(c, g); break;
        default: fin_gram_bl<8>(c, g); break;
    }
}
template <int W, bool VS>
__global__ void __launch_bounds__(kCBlock, 1) k_cluster_bl(SolveCtx* gctx, const __grid_constant__ SolveCtx hctx,
                                                           const CsrDev A, int nnz_max, int do_true, int init) {
    namespace cg = cooperative_groups;
    cg::cluster_group cl = cg::this_cluster();
    extern __shared__ double2 own[];  // (2ℓ+4) × rpc: r̂_0..ℓ, û_0..ℓ, x, r̃ | [values] | columns | offsets
    __shared__ SolveCtx cs;
    __shared__ ClusterRed R;
    __shared__ double gpart[kGramMax][kGramSub];
    __shared__ double gslot[2][kGramMax];
    __shared__ double gtot[kGramMax];
    ctx_copy(&cs, init ? &hctx : gctx);
    if (threadIdx.x == 0) R.parity = 0;
    __syncthreads();
    const int n = (int)A.n_rows;
    const int ncta = (int)cl.num_blocks();
    const int rpc = (n + ncta - 1) / ncta;
    const int row0 = (int)cl.block_rank() * rpc;
    const int nr = max(0, min(rpc, n - row0));
    SolveCtx* c = &cs;
    const int ell = cs.ell;
    const int nd = (ell + 1) + ell * (ell + 1);
    double2* const Rs = own;                          // r̂_q at Rs + q·rpc
    double2* const Us = own + (ell + 1) * rpc;        // û_q at Us + q·rpc
    double2* const X = own + (2 * ell + 2) * rpc;
    double2* const RT = own + (2 * ell + 3) * rpc;
    double2* sval = own + (2 * ell + 4) * rpc;
    int* scol = (int*)(sval + (VS ? nnz_max : 0));
    int* soff = scol + nnz_max;
    double2* const* rl = cs.rl;  // global copies: only the SpMV inputs r̂_j / û_j are written through
    double2* const* ul = cs.ul;
    double2* xg = cs.x;
    if (init) {  // x0 = 0: r̂_0 = r̃ = b, û_0 = 0, x = 0 (OpInitZero kind 5) ; fin_init_bl
        const double2* bg = cs.b;
        double acc[4] = {0.0, 0.0, 0.0, 0.0};
        for (int l = threadIdx.x; l < nr; l += kCBlock) {
            const double2 bl = bg[row0 + l];
            for (int q = 0; q <= ell; q++) Rs[q * rpc + l] = Us[q * rpc + l] = make_double2(0.0, 0.0);
            Rs[l] = bl;
            Us[rpc + l] = bl;  // (the shared init's p = û_1 = r0; overwritten before use)
            X[l] = make_double2(0.0, 0.0);
            RT[l] = bl;
            cl_init_row(bl, acc);
        }
        cl_init_tickets(cs);
        cl_sum<4>(acc, R);
        if (threadIdx.x == 0) fin_init_bl(c, R.tot);
        __syncthreads();
    } else {
        for (int l = threadIdx.x; l < nr; l += kCBlock) {
            const int i = row0 + l;
            for (int q = 0; q <= ell; q++) {
                Rs[q * rpc + l] = rl[q][i];
                Us[q * rpc + l] = ul[q][i];
            }
            X[l] = xg[i];
            RT[l] = cs.rh[i];
        }
    }
    const double2* gval = cl_stage<VS>(A, row0, nr, sval, scol, soff);
    __syncthreads();
    constexpr int RPP = kCBlock / W;
    const int sub = threadIdx.x & (W - 1);
    const int grp = threadIdx.x / W;
    int gpar = 0;
    int bodies = 0;
    while (!c->done) {
        for (int j = 0; j < ell && !c->done; j++) {
            {   // B1: û_q = r̂_q − β û_q (q ≤ j); û_j written through, then a cluster barrier (S1 gathers it)
                const double2 be = c->beta;
                for (int l = threadIdx.x; l < nr; l += kCBlock) {
                    for (int q = 0; q <= j; q++) {
                        const double2 uv = Us[q * rpc + l];
                        double2 o = Rs[q * rpc + l];
                        o.x = fma(-be.x, uv.x, fma(be.y, uv.y, o.x));
                        o.y = fma(-be.x, uv.y, fma(-be.y, uv.x, o.y));
                        Us[q * rpc + l] = o;
                        if (q == j) ul[j][row0 + l] = o;
                    }
                }
                cl.sync();
            }
            {   // S1: û_{j+1} = A û_j ; γ = ⟨r̃, û_{j+1}⟩, ‖û_{j+1}‖²
                double acc[3] = {0.0, 0.0, 0.0};
                double2* out = Us + (j + 1) * rpc;
                for (int b = 0; b < nr; b += RPP) {
                    const int l = b + grp;
                    const double2 y = cl_row<W, VS>(gval, sval, scol, soff, ul[j], l, l < nr, sub);
                    if (sub == 0 && l < nr) {
                        out[l] = y;
                        const double2 q = RT[l];
                        acc[0] = fma(q.x, y.x, fma(q.y, y.y, acc[0]));
                        acc[1] = fma(q.x, y.y, fma(-q.y, y.x, acc[1]));
                        acc[2] += cabs2(y);
                    }
                }
                cl_sum<3>(acc, R);
                if (threadIdx.x == 0) fin_s1_bl(c, R.tot);
                __syncthreads();
                if (c->done) break;
            }
            {   // B2: r̂_0 −= α û_1 ; x += α û_0 ; ‖r̂_0‖² ; r̂_q −= α û_{q+1} (1 ≤ q ≤ j); r̂_j written through
                const double2 al = c->alpha;
                double acc[1] = {0.0};
                for (int l = threadIdx.x; l < nr; l += kCBlock) {
                    {
                        const double2 u1 = Us[rpc + l], u0 = Us[l];
                        double2 o = Rs[l];
                        o.x = fma(-al.x, u1.x, fma(al.y, u1.y, o.x));
                        o.y = fma(-al.x, u1.y, fma(-al.y, u1.x, o.y));
                        Rs[l] = o;
                        if (j == 0) rl[0][row0 + l] = o;
                        acc[0] += cabs2(o);
                        cfma(X[l], al, u0);
                    }
                    for (int q = 1; q <= j; q++) {
                        const double2 uv = Us[(q + 1) * rpc + l];
                        double2 o = Rs[q * rpc + l];
                        o.x = fma(-al.x, uv.x, fma(al.y, uv.y, o.x));
                        o.y = fma(-al.x, uv.y, fma(-al.y, uv.x, o.y));
                        Rs[q * rpc + l] = o;
                        if (q == j) rl[j][row0 + l] = o;
                    }
                }
                cl_sum<1>(acc, R);  // also publishes r̂_j for the S2 gathers
                if (threadIdx.x == 0) fin_b2_bl(c, R.tot);
                __syncthreads();
                if (c->done) break;
            }
            {   // S2: r̂_{j+1} = A r̂_j ; ρ1 = ⟨r̃, r̂_{j+1}⟩, ‖r̂_{j+1}‖² (j < ℓ−1)
                double acc[3] = {0.0, 0.0, 0.0};
                double2* out = Rs + (j + 1) * rpc;
                for (int b = 0; b < nr; b += RPP) {
                    const int l = b + grp;
                    const double2 y = cl_row<W, VS>(gval, sval, scol, soff, rl[j], l, l < nr, sub);
                    if (sub == 0 && l < nr) {
                        out[l] = y;
                        const double2 q = RT[l];
                        acc[0] = fma(q.x, y.x, fma(q.y, y.y, acc[0]));
                        acc[1] = fma(q.x, y.y, fma(-q.y, y.x, acc[1]));
                        acc[2] += cabs2(y);
                    }
                }
                if (j < ell - 1) {
                    cl_sum<3>(acc, R);
                    if (threadIdx.x == 0) fin_s2_bl(c, R.tot);
                }
                __syncthreads();
            }
        }
        if (c->done) break;
        {   // G: Gram matrix of r̂_0..ℓ (packed as GramPack), minimal-residual coefficients γ, ω
            const int k = threadIdx.x / kGramSub, sk = threadIdx.x % kGramSub;
            if (k < nd) {
                // entry k → (a, b): diag(a) = a + a(2(ℓ+1) − a − 1); off(a, b) = diag(a) + 1 + 2(b − a − 1)
                const int NV = ell + 1;
                int a = 0;
                while (a + 1 < NV && (a + 1) + (a + 1) * (2 * NV - (a + 1) - 1) <= k) a++;
                const int d = a + a * (2 * NV - a - 1);
                const bool dg = k == d;
                const int b = dg ? a : a + 1 + (k - d - 1) / 2;
                const bool im = !dg && ((k - d - 1) & 1);
                const double2* va = Rs + a * rpc;
                const double2* vb = Rs + b * rpc;
                double s = 0.0;
                for (int l = sk; l < nr; l += kGramSub) {
                    const double2 x1 = va[l];
                    if (dg) {
                        s += cabs2(x1);
                    } else {
                        const double2 x2 = vb[l];
                        s = im ? fma(x1.x, x2.y, fma(-x1.y, x2.x, s)) : fma(x1.x, x2.x, fma(x1.y, x2.y, s));
                    }
                }
                gpart[k][sk] = s;
            }
            __syncthreads();
            if (threadIdx.x < nd) {
                double t = 0.0;
                for (int q = 0; q < kGramSub; q++) t += gpart[threadIdx.x][q];
                gslot[gpar][threadIdx.x] = t;
            }
            cl.sync();
            if (threadIdx.x < nd) {
                double t = 0.0;
                for (int r = 0; r < ncta; r++) t += cl.map_shared_rank(&gslot[gpar][0], r)[threadIdx.x];
                gtot[threadIdx.x] = t;
            }
            gpar ^= 1;
            __syncthreads();
            if (threadIdx.x == 0) fin_gram_any(c, gtot, ell);
            __syncthreads();
            if (c->done) break;
        }
        {   // U: x += Σ γ_j r̂_{j−1} ; r̂_0 −= Σ γ_j r̂_j ; û_0 −= Σ γ_j û_j ; ‖r̂_0‖², ⟨r̃, r̂_0⟩
            double acc[3] = {0.0, 0.0, 0.0};
            for (int l = threadIdx.x; l < nr; l += kCBlock) {
                double2 xv = X[l], r0 = Rs[l], u0 = Us[l];
                double2 rprev = r0;
                for (int q = 1; q <= ell; q++) {  // oracle order: j ascending
                    const double2 g = c->gam[q];
                    const double2 rq = Rs[q * rpc + l], uq = Us[q * rpc + l];
                    cfma(xv, g, rprev);
                    r0.x = fma(-g.x, rq.x, fma(g.y, rq.y, r0.x));
                    r0.y = fma(-g.x, rq.y, fma(-g.y, rq.x, r0.y));
                    u0.x = fma(-g.x, uq.x, fma(g.y, uq.y, u0.x));
                    u0.y = fma(-g.x, uq.y, fma(-g.y, uq.x, u0.y));
                    rprev = rq;
                }
                X[l] = xv;
                Rs[l] = r0;
                Us[l] = u0;
                const double2 tv = RT[l];
                acc[0] += cabs2(r0);
                acc[1] = fma(tv.x, r0.x, fma(tv.y, r0.y, acc[1]));
                acc[2] = fma(tv.x, r0.y, fma(-tv.y, r0.x, acc[2]));
            }
            cl_sum<3>(acc, R);
            if (threadIdx.x == 0) fin_u_bl(c, R.tot);
            __syncthreads();
        }
        bodies++;
    }
    __syncthreads();
    for (int l = threadIdx.x; l < nr; l += kCBlock) xg[row0 + l] = X[l];  // the solution leaves shared memory
    if (do_true) cl_true<W, VS>(c, R, gval, sval, scol, soff, xg, row0, nr);
    if (threadIdx.x == 0) cs.bodies = bodies;
    __syncthreads();
    if (cl.block_rank() == 0) ctx_out(gctx, cs);
    cl.sync();
}

// lanes per row of the cluster SpMV: 8 when one pass of 512 threads covers the CTA's rows, else 4.
// Measured per BiCGStab iteration (µs, W = 1 / 2 / 4 / 8): Twingo3D-0 31.8 / 24.2 / 19.8 / 20.9,
// Audi3D-2 35.8 / 25.3 / 24.2 / 24.9; Audi3D-1 (108 rows per CTA) 10.5 at W = 8.
static int cluster_w(int64_t n, int cs, int /*max_len*/) {
    const int64_t rpc = (n + cs - 1) / cs;
    return rpc * 8 <= kCBlock ? 8 : 4;
}
// cluster solver kinds: 0 BiCGStab (and Jacobi-BiCGStab), 1 TFQMR, 2 CG, 3 COCG, 4 BiCGStab(ℓ)
int cluster_kind(int method) {
    return method == ZK_BICGSTAB ? 0 : method == ZK_TFQMR ? 1 : method == ZK_CG ? 2 : method == ZK_COCG ? 3
         : method == kBiCGStabL ? 4 : -1;
}
template <int W>
static const void* cluster_kernel(bool vs, int kind) {
    switch (kind) {
        case 1: return vs ? (const void*)k_cluster_tfqmr<W, true> : (const void*)k_cluster_tfqmr<W, false>;
        case 2: return vs ? (const void*)k_cluster_cg<W, true, false> : (const void*)k_cluster_cg<W, false, false>;
        case 3: return vs ? (const void*)k_cluster_cg<W, true, true> : (const void*)k_cluster_cg<W, false, true>;
        case 4: return vs ? (const void*)k_cluster_bl<W, true> : (const void*)k_cluster_bl<W, false>;
        default: return vs ? (const void*)k_cluster_bicg<W, true> : (const void*)k_cluster_bicg<W, false>;
    }
}
static const void* cluster_kernel(int w, bool vs, int kind = 0) {
    return w == 8 ? cluster_kernel<8>(vs, kind) : w == 4 ? cluster_kernel<4>(vs, kind)
         : w == 2 ? cluster_kernel<2>(vs, kind) : cluster_kernel<1>(vs, kind);
}
static int cluster_nvec(int kind, int ell) {
    return kind == 1 ? kCVecsTfqmr : kind == 4 ? 2 * ell + 4 : kind >= 2 ? kCVecsCg : kCVecs;
}
static size_t cluster_smem(int64_t n, int cs, int64_t nnz_max, bool vs, int kind, int ell) {
    const int64_t rpc = (n + cs - 1) / cs;
    return (size_t)(cluster_nvec(kind, ell) * 16 * rpc + (vs ? 16 : 0) * nnz_max + 4 * nnz_max + 4 * (rpc + 1));
}

// cluster size that can be launched on this device: 16 (non-portable), else 8, else 0
static int cluster_size_available() {
    static int cached = -1;  // per process
    if (cached < 0) {
        cached = 0;
        for (int w : {1, 2, 4, 8})
            for (bool vs : {false, true})
                for (int kind = 0; kind < 5; kind++) {
                    cudaFuncSetAttribute(cluster_kernel(w, vs, kind), cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
                    cudaFuncSetAttribute(cluster_kernel(w, vs, kind), cudaFuncAttributeMaxDynamicSharedMemorySize, kCSmemMax);
                }
        for (int cs : {16, 8}) {
            cudaLaunchConfig_t cfg;
            memset(&cfg, 0, sizeof cfg);
            cfg.gridDim = dim3(cs);
            cfg.blockDim = dim3(kCBlock);
            cfg.dynamicSmemBytes = kCSmemMax;
            cudaLaunchAttribute at[1];
            at[0].id = cudaLaunchAttributeClusterDimension;
            at[0].val.clusterDim.x = cs;
            at[0].val.clusterDim.y = 1;
            at[0].val.clusterDim.z = 1;
            cfg.attrs = at;
            cfg.numAttrs = 1;
            int nclusters = 0;
            if (cudaOccupancyMaxActiveClusters(&nclusters, cluster_kernel(1, false), &cfg) == cudaSuccess &&
                nclusters >= 1) {
                cached = cs;
                break;
            }
            cudaGetLastError();
        }
    }
    return cached;
}

// most nonzeros in one CTA's row block (one-off: CS + 1 row-pointer reads, cached in the handle)
static int64_t cluster_nnz_max(zk_csr_s* A, int cs, cudaStream_t s) {
    if (A->cl_cs == cs && A->cl_nnz_max >= 0) return A->cl_nnz_max;
    const int64_t n = A->n_rows, rpc = (n + cs - 1) / cs;
    std::vector<int64_t> rp(cs + 1, 0);
    for (int k = 0; k <= cs; k++) {
        const int64_t i = std::min<int64_t>((int64_t)k * rpc, n);
        if (cudaMemcpyAsync(&rp[k], A->row_ptr + i, sizeof(int64_t), cudaMemcpyDeviceToHost, s) != cudaSuccess) return -1;
    }
    if (cudaStreamSynchronize(s) != cudaSuccess) return -1;
    int64_t mx = 0;
    for (int k = 0; k < cs; k++) mx = std::max(mx, rp[k + 1] - rp[k]);
    A->cl_cs = cs;
    A->cl_nnz_max = mx;
    return mx;
}
// can the cluster solver hold this system (own rows + the block's columns in shared memory)?
bool cluster_fits(zk_csr_s* A, cudaStream_t s, int kind, int ell) {
    const int cs = cluster_size_available();
    if (kind < 0 || cs == 0 || A->n_rows == 0 || !A->val ||  // the cluster kernels stage the CSR values
        A->n_rows > (int64_t)cs * (kCSmemMax / (cluster_nvec(kind, ell) * 16 + 8)))
        return false;
    const int64_t nz = cluster_nnz_max(A, cs, s);
    return nz >= 0 && cluster_smem(A->n_rows, cs, nz, false, kind, ell) <= (size_t)kCSmemMax;
}

// launch the cluster solver on one cluster (A or A·M⁻¹ in av); false when unavailable.
// BiCGStab (kind 0): with `init` the kernel starts from x0 = 0 itself (context hc by value, no
// k_set_ctx / k_init_zero launches).
bool cluster_launch(zk_csr_s* A, SolveCtx* dc, const SolveCtx& hc, const CsrDev& av, cudaStream_t s,
                           int* out_cs, int kind, int ell, bool do_true, bool init) {
    const int cs = cluster_size_available();
    if (cs == 0) return false;
    const int64_t nz = cluster_nnz_max(A, cs, s);
    if (nz < 0) return false;
    bool vs = cluster_smem(av.n_rows, cs, nz, true, kind, ell) <= (size_t)kCSmemMax;
    int w = cluster_w(av.n_rows, cs, A->max_len);
    if (const char* e = getenv("ZK_CLUSTER_W")) {  // tests: force a lane count (1, 2, 4, 8)
        const int f = atoi(e);
        if (f == 1 || f == 2 || f == 4 || f == 8) w = f;
    }
    if (const char* e = getenv("ZK_CLUSTER_VS"))  // tests: 0 keeps the values in global memory
        vs = vs && atoi(e) != 0;
    cudaLaunchConfig_t cfg;
    memset(&cfg, 0, sizeof cfg);
    cfg.gridDim = dim3(cs);
    cfg.blockDim = dim3(kCBlock);
    cfg.dynamicSmemBytes = cluster_smem(av.n_rows, cs, nz, vs, kind, ell);
    cfg.stream = s;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = cs;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    int nzi = (int)nz;
    int dt = do_true ? 1 : 0;
    int in = init ? 1 : 0;
    cudaError_t e;
    {
        void* args[] = {(void*)&dc, (void*)&hc, (void*)&av, (void*)&nzi, (void*)&dt, (void*)&in};
        e = cudaLaunchKernelExC(&cfg, cluster_kernel(w, vs, kind), args);
    }
    if (e != cudaSuccess) {
        cudaGetLastError();
        return false;
    }
    *out_cs = cs;
    return true;
}

}  // namespace zk
