// solve.cu — device-resident BiCGStab and CG (§4; SURVEY.md §8(a) A6-A8,
// §8(c) O6/O7).  One iteration is a fixed schedule of fused kernels; every scalar (ρ, σ, α, ω,
// β, γ, δ) lives in a device SolveCtx and is computed by the last block of the kernel that
// finishes its reduction, so the loop needs no host synchronisation.  The loop itself runs as
// a CUDA graph with a conditional WHILE node (the last kernel of the body writes the
// condition); fallbacks: chunked graph launches or per-iteration launches with a device
// early-exit flag.
//
// BiCGStab schedule F (one iteration j):
//   K1  v = A p            ; σ = ⟨r̂,v⟩, ‖v‖²        → α = ρ/σ           (BREAKDOWN_SIGMA)
//   K2  s = r − α v        ; ‖s‖²                    → half-step exit test
//   K3  t = A s            ; ⟨t,s⟩, ⟨t,t⟩ = τ        → ω = ⟨t,s⟩/τ       (BREAKDOWN_OMEGA)
//   K4  x += αp + ωs ; r = s − ωt ; ‖r‖², ρ' = ⟨r̂,r⟩ → hist[j], tests, β = (ρ'/ρ)(α/ω)
//   K5  p = r + β(p − ωv)                             (writes the WHILE condition)
// CG: K1 q = A p ; δ = ⟨p,q⟩ → α = γ/Re δ (NOT_HPD) ; K2 x += αp ; r −= αq ; γ' → hist, β ;
//     K3 p = r + βp.
// TFQMR (NEXT-2; Freund 1993 in the two-half-step form of oracle_tfqmr), iteration k:
//   T1  y2 = y1 − αv ; w −= αu1 ; ‖w‖²                     → θ,c,τ,η1 (half step m = 2k−1), c2, test
//   T2  u2 = A y2 ; w −= αu2 ; ‖w‖², ⟨r̃,w⟩                 → half step m = 2k, hist[k], ρ', β
//   T3  d1 = y1 + c1·d ; d = y2 + c2·d1 ; x += η1·d1 + η2·d ; y1 = w + βy2
// The d recurrence and both x updates of an iteration are deferred to T3, which holds every
// operand they need (y1 before it is overwritten, y2, d): d and x are read and written once per
// iteration, and the SpMV epilogue of T2 carries 2 row operands.  2·Mat + 25 vector passes.
//   T4  u1 = A y1 ; v = u1 + β(u2 + βv) ; σ = ⟨r̃,v⟩        → α = ρ/σ, c1 (writes the WHILE condition)
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <algorithm>
#include <vector>

#include <cooperative_groups.h>

#include "spmv.cuh"
#include "zk_host.h"

#include "solve_ctx.cuh"

namespace zk {
enum Stage { S_INIT_BICG, S_K1_BICG, S_K2_BICG, S_K3_BICG, S_K4_BICG, S_INIT_CG, S_K1_CG, S_K2_CG, S_TRUE,
             S_INIT_COCG, S_K1_COCG, S_K2_COCG, S_INIT_TFQMR, S_K0_TFQMR, S_T1_TFQMR, S_T2_TFQMR,
             S_T4_TFQMR, S_INIT_BL, S_S1_BL, S_B2_BL, S_S2_BL, S_G_BL, S_U_BL, S_COUNT };
static_assert(S_COUNT <= kTickets, "one ticket per reduction stage");

// timer class of a stage: 0 SpMV in the loop, 1 fused vector kernels, 2 init, 3 true residual
__host__ __device__ constexpr int timer_of(int S) {
    return (S == S_K1_BICG || S == S_K3_BICG || S == S_K1_CG || S == S_K1_COCG || S == S_T2_TFQMR ||
            S == S_T4_TFQMR || S == S_S1_BL || S == S_S2_BL) ? 0
           : (S == S_K2_BICG || S == S_K4_BICG || S == S_K2_CG || S == S_K2_COCG || S == S_T1_TFQMR ||
              S == S_B2_BL || S == S_G_BL || S == S_U_BL) ? 1
           : (S == S_TRUE) ? 3 : 2;
}
template <int S>
__device__ __forceinline__ void stamp_start(SolveCtx* c) {
    if (threadIdx.x == 0) atomicMin(&c->t0[timer_of(S)], gtimer());
}

template <int S>
__device__ __forceinline__ void finish_stage(SolveCtx* c, const double* tot) {
    if (S == S_INIT_BICG) fin_init_bicg(c, tot);
    if (S == S_K1_BICG) fin_k1_bicg(c, tot);
    if (S == S_K2_BICG) fin_k2_bicg(c, tot);
    if (S == S_K3_BICG) fin_k3_bicg(c, tot);
    if (S == S_K4_BICG) fin_k4_bicg(c, tot);
    if (S == S_INIT_CG) fin_init_cg(c, tot);
    if (S == S_K1_CG) fin_k1_cg(c, tot);
    if (S == S_K2_CG) fin_k2_cg(c, tot);
    if (S == S_TRUE) fin_true(c, tot);
    if (S == S_INIT_COCG) fin_init_cocg(c, tot);
    if (S == S_K1_COCG) fin_k1_cocg(c, tot);
    if (S == S_K2_COCG) fin_k2_cocg(c, tot);
    if (S == S_INIT_TFQMR) fin_init_tfqmr(c, tot);
    if (S == S_K0_TFQMR || S == S_T4_TFQMR) fin_sigma_tfqmr(c, tot);
    if (S == S_T1_TFQMR) fin_t1_tfqmr(c, tot);
    if (S == S_T2_TFQMR) fin_t2_tfqmr(c, tot);
    if (S == S_INIT_BL) fin_init_bl(c, tot);
    if (S == S_S1_BL) fin_s1_bl(c, tot);
    if (S == S_B2_BL) fin_b2_bl(c, tot);
    if (S == S_S2_BL) fin_s2_bl(c, tot);
    if (S == S_U_BL) fin_u_bl(c, tot);
}

// grid reduction of K values, then (single GPU) the stage's scalar step in the last block, or
// (multi-GPU) publish the local sums in c->red for the allreduce + fin_kernel.
template <int S, int K>
__device__ __forceinline__ void reduce_finish(SolveCtx* c, double (&acc)[K], int off = 0, int total = 0) {
    double tot[K];
    if (grid_sum<K>(acc, c->partials, c->tickets + S, tot, off, total) && threadIdx.x == 0) {
        constexpr int T = timer_of(S);
        const unsigned long long st = atomicExch(&c->t0[T], ~0ull);
        c->tsum[T] += gtimer() - st;
        c->tcnt[T] += 1;
        if (c->dist) {
#pragma unroll
            for (int k = 0; k < K; k++) c->red[k] = tot[k];
        } else {
            finish_stage<S>(c, tot);
        }
    }
}

template <int S>
__global__ void fin_kernel(SolveCtx* c) {
    // the reducing kernel skipped its work (loop already finished): nothing to finish — the
    // chunked loop launches whole iterations past convergence (regression: tools/debug/dist1.py)
    if (S != S_TRUE && S != S_INIT_BICG && S != S_INIT_CG && S != S_INIT_COCG && S != S_INIT_TFQMR && S != S_INIT_BL && c->done) return;
    double tot[kMaxRed];
    for (int k = 0; k < kMaxRed; k++) tot[k] = c->red[k];
    finish_stage<S>(c, tot);
}

// ------------------------------------------------------------------ epilogues and vector ops
// Epilogues: pre(i) loads the row's own operands (issued one tile ahead by spmv_body, so the
// load is off the critical path); row(i, y, pre, acc) consumes them.  Pointers are cached from
// the SolveCtx at kernel start.
template <int S>
struct EpiInit {  // r = b − A x0 ; x = x0 ; r̂ = p = r ; {‖b‖², ‖r‖², Re rᵀr, Im rᵀr}
    static constexpr int K = 4;
    struct Pre { double2 b, x0; };
    SolveCtx* c;
    const double2* __restrict__ x0;
    const double2* __restrict__ b;
    double2 *r, *p, *rh, *x, *d;
    __device__ EpiInit(SolveCtx* c_, const double2* x0_, bool bicg)
        : c(c_), x0(x0_), b(c_->b), r(c_->r), p(c_->p), rh(bicg ? c_->rh : nullptr), x(c_->x), d(c_->d) {}
    __device__ Pre pre(int64_t i) const { return {ld_vec(b + i), x != x0 ? ld_gather_coh(x0 + i) : make_double2(0, 0)}; }
    __device__ void row(int64_t i, double2 y, const Pre& q, double (&acc)[4]) {
        const double2 rr = csub(q.b, y);
        st_vec(r + i, rr);
        st_vec(p + i, rr);
        if (rh) st_vec(rh + i, rr);
        if (x != x0) st_vec(x + i, q.x0);
        if (d) st_vec(d + i, make_double2(0.0, 0.0));
        acc[0] += cabs2(q.b);
        acc[1] += cabs2(rr);
        acc[2] = fma(rr.x, rr.x, fma(-rr.y, rr.y, acc[2]));  // rᵀr (COCG's ρ0)
        acc[3] = fma(2.0 * rr.x, rr.y, acc[3]);
    }
    __device__ void finish(double (&acc)[4], int off = 0, int tot = 0) { reduce_finish<S, 4>(c, acc, off, tot); }
};

struct EpiTrue {  // {‖b − A x‖²}
    static constexpr int K = 1;
    using Pre = double2;
    SolveCtx* c;
    const double2* __restrict__ b;
    __device__ explicit EpiTrue(SolveCtx* c_) : c(c_), b(c_->b) {}
    __device__ Pre pre(int64_t i) const { return ld_vec(b + i); }
    __device__ void row(int64_t, double2 y, const Pre& bi, double (&acc)[1]) { acc[0] += cabs2(csub(bi, y)); }
    __device__ void finish(double (&acc)[1], int off = 0, int tot = 0) { reduce_finish<S_TRUE, 1>(c, acc, off, tot); }
};

struct EpiK1Bicg {  // v = A p ; {σ = ⟨r̂, v⟩, ‖v‖²}
    static constexpr int K = 3;
    using Pre = double2;
    SolveCtx* c;
    double2* __restrict__ v;
    const double2* __restrict__ rh;
    __device__ explicit EpiK1Bicg(SolveCtx* c_) : c(c_), v(c_->v), rh(c_->rh) {}
    __device__ Pre pre(int64_t i) const { return ld_vec(rh + i); }
    __device__ void row(int64_t i, double2 y, const Pre& r, double (&acc)[3]) {
        st_vec(v + i, y);
        acc[0] = fma(r.x, y.x, fma(r.y, y.y, acc[0]));
        acc[1] = fma(r.x, y.y, fma(-r.y, y.x, acc[1]));
        acc[2] += cabs2(y);
    }
    __device__ void finish(double (&acc)[3], int off = 0, int tot = 0) { reduce_finish<S_K1_BICG, 3>(c, acc, off, tot); }
};

struct EpiK3Bicg {  // t = A s ; {⟨t, s⟩, ⟨t, t⟩}
    static constexpr int K = 3;
    using Pre = double2;
    SolveCtx* c;
    double2* __restrict__ t;
    const double2* __restrict__ s;
    __device__ explicit EpiK3Bicg(SolveCtx* c_) : c(c_), t(c_->t), s(c_->s) {}
    __device__ Pre pre(int64_t i) const { return ld_gather_coh(s + i); }
    __device__ void row(int64_t i, double2 y, const Pre& si, double (&acc)[3]) {
        st_vec(t + i, y);
        acc[0] = fma(y.x, si.x, fma(y.y, si.y, acc[0]));
        acc[1] = fma(y.x, si.y, fma(-y.y, si.x, acc[1]));
        acc[2] += cabs2(y);
    }
    __device__ void finish(double (&acc)[3], int off = 0, int tot = 0) { reduce_finish<S_K3_BICG, 3>(c, acc, off, tot); }
};

// Split reductions (large systems): the SpMV of BiCGStab K1/K3 and CG/COCG K1 only stores its
// product and a following vector pass (r1/r3/rq) forms the dot products.  The fused epilogue's
// operand load and running sums cost the SELL kernel ≈ 140 µs per launch on C4 (its batch of 18
// matrix loads gets interleaved with the gathers at the 80-register cap), the extra pass over
// two vectors ≈ 40 µs: BiCGStab 1.83 vs 1.90 ms per iteration.  Below kSplitRows the two extra
// launches per iteration cost more than they save (latency-bound sizes), so the fused kernels stay.
// At the paper's largest shapes the split wins too: Audi3D-4 (C3, 648,849 rows) BiCGStab 169 vs
// 176 µs per iteration, Twingo3D-2 (479,169 rows) 134 vs 137 µs (profiles/r01_c3_split.txt).
constexpr int64_t kSplitRows = 1 << 18;
#ifndef ZK_STORE_ORD
#define ZK_STORE_ORD 1
#endif
struct EpiStore {  // out = A x
    static constexpr int K = 0;
    static constexpr bool kOrdered = ZK_STORE_ORD;  // all 9 column loads of a batch before its gathers (spmv.cuh)
    using Pre = double2;
    double2* __restrict__ out;
    __device__ explicit EpiStore(double2* o) : out(o) {}
    __device__ Pre pre(int64_t) const { return make_double2(0.0, 0.0); }
    __device__ void row(int64_t i, double2 y, const Pre&, double (&)[1]) { st_vec(out + i, y); }
    __device__ void finish(double (&)[1], int = 0, int = 0) {}
};
struct OpRed1Bicg {  // {⟨r̂, v⟩, ‖v‖²}
    static constexpr int K = 3;
    struct In { double2 r, v; };
    SolveCtx* c;
    const double2 *__restrict__ rh, *__restrict__ v;
    __device__ explicit OpRed1Bicg(SolveCtx* c_) : c(c_), rh(c_->rh), v(c_->v) {}
    __device__ In load(int64_t i) const { return {ld_vec(rh + i), ld_vec(v + i)}; }
    __device__ void apply(int64_t, const In& in, double (&acc)[3]) const {
        acc[0] = fma(in.r.x, in.v.x, fma(in.r.y, in.v.y, acc[0]));
        acc[1] = fma(in.r.x, in.v.y, fma(-in.r.y, in.v.x, acc[1]));
        acc[2] += cabs2(in.v);
    }
    __device__ void finish(double (&acc)[3], int off = 0, int tot = 0) const { reduce_finish<S_K1_BICG, 3>(c, acc, off, tot); }
};
template <bool CONJ, int S>
struct OpRedPq {  // {⟨p, q⟩} (CG, CONJ) or {pᵀq} (COCG)
    static constexpr int K = 2;
    struct In { double2 p, q; };
    SolveCtx* c;
    const double2 *__restrict__ p, *__restrict__ q;
    __device__ explicit OpRedPq(SolveCtx* c_) : c(c_), p(c_->p), q(c_->q) {}
    __device__ In load(int64_t i) const { return {ld_vec(p + i), ld_vec(q + i)}; }
    __device__ void apply(int64_t, const In& in, double (&acc)[2]) const {
        if (CONJ) {
            acc[0] = fma(in.p.x, in.q.x, fma(in.p.y, in.q.y, acc[0]));
            acc[1] = fma(in.p.x, in.q.y, fma(-in.p.y, in.q.x, acc[1]));
        } else {
            acc[0] = fma(in.p.x, in.q.x, fma(-in.p.y, in.q.y, acc[0]));
            acc[1] = fma(in.p.x, in.q.y, fma(in.p.y, in.q.x, acc[1]));
        }
    }
    __device__ void finish(double (&acc)[2], int off = 0, int tot = 0) const { reduce_finish<S, 2>(c, acc, off, tot); }
};
struct OpRed3Bicg {  // {⟨t, s⟩, ‖t‖²}
    static constexpr int K = 3;
    struct In { double2 t, s; };
    SolveCtx* c;
    const double2 *__restrict__ t, *__restrict__ s;
    __device__ explicit OpRed3Bicg(SolveCtx* c_) : c(c_), t(c_->t), s(c_->s) {}
    __device__ In load(int64_t i) const { return {ld_vec(t + i), ld_vec(s + i)}; }
    __device__ void apply(int64_t, const In& in, double (&acc)[3]) const {
        acc[0] = fma(in.t.x, in.s.x, fma(in.t.y, in.s.y, acc[0]));
        acc[1] = fma(in.t.x, in.s.y, fma(-in.t.y, in.s.x, acc[1]));
        acc[2] += cabs2(in.t);
    }
    __device__ void finish(double (&acc)[3], int off = 0, int tot = 0) const { reduce_finish<S_K3_BICG, 3>(c, acc, off, tot); }
};

// Split schedule with a TAIL reduction (SPLIT = 2, SELL mapping on one GPU): the SpMV stores
// out = A x like EpiStore, then each warp runs Op (the r1/r3/rq/T2b/T4b pass) over the rows it
// just produced (spmv.cuh sell_tail) and the kernel's last block finishes the stage — the
// separate reduction launch, its ramp and tail disappear; the loop keeps the store-only schedule.
template <class Op>
struct EpiStoreTail {
    static constexpr int K = Op::K;
    static constexpr bool kOrdered = ZK_STORE_ORD;
    static constexpr bool kTail = true;
    using Pre = double2;
    using TailOp = Op;
    double2* __restrict__ out;
    SolveCtx* c;  // the Op (its pointers and scalars) is built only after the loop: nothing of it is live there
    __device__ EpiStoreTail(double2* o, SolveCtx* c_) : out(o), c(c_) {}
    __device__ Pre pre(int64_t) const { return make_double2(0.0, 0.0); }
    __device__ void row(int64_t i, double2 y, const Pre&, double (&)[K]) { st_vec(out + i, y); }
    __device__ Op tail_op() const { return Op(c); }
    __device__ void finish(double (&)[K], int = 0, int = 0) {}  // the tail's Op finishes the stage
};

// The fused epilogue with per-slice warp reductions (SPLIT = 3, SELL only): E's row() as is, its
// running sums kept in shared memory by the SELL body (sell_warpacc), its row operand loaded with
// the slice's last batch of matrix loads (kPrePlace 1), the store-only kernel's ordered loads.
template <class E, int PRE = 1>
struct WarpAcc : E {
    static constexpr bool kWarpAcc = true;
    static constexpr int kPrePlace = PRE;
    static constexpr bool kOrdered = ZK_STORE_ORD;
    using E::E;
};

struct EpiK1Cg {  // q = A p ; {δ = ⟨p, q⟩}
    static constexpr int K = 2;
    using Pre = double2;
    SolveCtx* c;
    double2* __restrict__ q;
    const double2* __restrict__ p;
    __device__ explicit EpiK1Cg(SolveCtx* c_) : c(c_), q(c_->q), p(c_->p) {}
    __device__ Pre pre(int64_t i) const { return ld_gather_coh(p + i); }
    __device__ void row(int64_t i, double2 y, const Pre& pi, double (&acc)[2]) {
        st_vec(q + i, y);
        acc[0] = fma(pi.x, y.x, fma(pi.y, y.y, acc[0]));
        acc[1] = fma(pi.x, y.y, fma(-pi.y, y.x, acc[1]));
    }
    __device__ void finish(double (&acc)[2], int off = 0, int tot = 0) { reduce_finish<S_K1_CG, 2>(c, acc, off, tot); }
};

// Vector ops: every pointer and scalar is copied out of the SolveCtx once per thread at kernel
// start (reading c->x inside the loop would force a reload after every store through a
// possibly-aliasing pointer).
struct OpInitZero {  // x0 = 0: x = 0 ; r = r̂ = p = b ; {‖b‖², ‖r‖², Re bᵀb, Im bᵀb}
    static constexpr int K = 4;
    struct In { double2 b; };
    SolveCtx* c;
    const double2* __restrict__ b;
    double2 *__restrict__ x, *__restrict__ r, *__restrict__ p, *__restrict__ rh, *__restrict__ d;
    int kind;  // 0 BiCGStab, 1 CG, 3 COCG, 4 TFQMR, 5 BiCGStab(ℓ)
    __device__ OpInitZero(SolveCtx* c_, int kind_)
        : c(c_), b(c_->b), x(c_->x), r(c_->r), p(c_->p), rh(c_->rh), d(c_->d), kind(kind_) {}
    __device__ In load(int64_t i) const { return {ld_vec(b + i)}; }
    __device__ void apply(int64_t i, const In& v, double (&acc)[4]) const {
        st_vec(x + i, make_double2(0.0, 0.0));
        st_vec(r + i, v.b);
        st_vec(p + i, v.b);
        if (kind == 0 || kind >= 4) st_vec(rh + i, v.b);
        if (kind >= 4) st_vec(d + i, make_double2(0.0, 0.0));
        const double bb = cabs2(v.b);
        acc[0] += bb;
        acc[1] += bb;
        acc[2] = fma(v.b.x, v.b.x, fma(-v.b.y, v.b.y, acc[2]));
        acc[3] = fma(2.0 * v.b.x, v.b.y, acc[3]);
    }
    __device__ void finish(double (&acc)[4], int off = 0, int tot = 0) const {
        if (kind == 0) reduce_finish<S_INIT_BICG, 4>(c, acc, off, tot);
        else if (kind == 1) reduce_finish<S_INIT_CG, 4>(c, acc, off, tot);
        else if (kind == 3) reduce_finish<S_INIT_COCG, 4>(c, acc, off, tot);
        else if (kind == 4) reduce_finish<S_INIT_TFQMR, 4>(c, acc, off, tot);
        else reduce_finish<S_INIT_BL, 4>(c, acc, off, tot);
    }
};

struct OpK2Bicg {  // s = r − α v ; {‖s‖²}
    static constexpr int K = 1;
    struct In { double2 r, v; };
    SolveCtx* c;
    const double2 *__restrict__ r, *__restrict__ v;
    double2* __restrict__ s;
    double2 alpha;
    __device__ explicit OpK2Bicg(SolveCtx* c_) : c(c_), r(c_->r), v(c_->v), s(c_->s), alpha(c_->alpha) {}
    __device__ In load(int64_t i) const { return {ld_vec(r + i), ld_vec(v + i)}; }
    __device__ void apply(int64_t i, const In& in, double (&acc)[1]) const {
        double2 o = in.r;
        o.x = fma(-alpha.x, in.v.x, fma(alpha.y, in.v.y, o.x));
        o.y = fma(-alpha.x, in.v.y, fma(-alpha.y, in.v.x, o.y));
        st_vec(s + i, o);
        acc[0] += cabs2(o);
    }
    __device__ void finish(double (&acc)[1], int off = 0, int tot = 0) const { reduce_finish<S_K2_BICG, 1>(c, acc, off, tot); }
};

struct OpK4Bicg {  // x += αp + ωs ; r = s − ωt ; {‖r‖², ⟨r̂, r⟩}   (half: x += αp only)
    static constexpr int K = 3;
    static constexpr int U = 1;  // 5 input streams: one element per thread per step keeps registers ≤ 64
    struct In { double2 x, p, s, t, rh; };
    SolveCtx* c;
    double2 *__restrict__ x, *__restrict__ r;
    const double2 *__restrict__ p, *__restrict__ s, *__restrict__ t, *__restrict__ rh;
    double2 alpha, omega;
    bool half;
    __device__ OpK4Bicg(SolveCtx* c_, bool half_)
        : c(c_), x(c_->x), r(c_->r), p(c_->p), s(c_->s), t(c_->t), rh(c_->rh), alpha(c_->alpha),
          omega(c_->omega), half(half_) {}
    __device__ In load(int64_t i) const {
        In v;
        v.x = ld_vec(x + i);
        v.p = ld_vec(p + i);
        if (!half) {
            v.s = ld_vec(s + i);
            v.t = ld_vec(t + i);
            v.rh = ld_vec(rh + i);
        }
        return v;
    }
    __device__ void apply(int64_t i, const In& in, double (&acc)[3]) const {
        double2 xn = in.x;
        cfma(xn, alpha, in.p);
        if (half) {
            st_vec(x + i, xn);
            return;
        }
        cfma(xn, omega, in.s);
        st_vec(x + i, xn);
        double2 rn = in.s;
        rn.x = fma(-omega.x, in.t.x, fma(omega.y, in.t.y, rn.x));
        rn.y = fma(-omega.x, in.t.y, fma(-omega.y, in.t.x, rn.y));
        st_vec(r + i, rn);
        acc[0] += cabs2(rn);
        acc[1] = fma(in.rh.x, rn.x, fma(in.rh.y, rn.y, acc[1]));
        acc[2] = fma(in.rh.x, rn.y, fma(-in.rh.y, rn.x, acc[2]));
    }
    __device__ void finish(double (&acc)[3], int off = 0, int tot = 0) const {
        if (half) return;  // no reduction on the half-step exit; K5 clears the flag
        reduce_finish<S_K4_BICG, 3>(c, acc, off, tot);
    }
};

struct OpK5Bicg {  // p = r + β(p − ω v)
    static constexpr int K = 0;
    static constexpr int U = 2;
    struct In { double2 r, p, v; };
    const double2 *__restrict__ r, *__restrict__ v;
    double2* __restrict__ p;
    double2 beta, omega;
    __device__ explicit OpK5Bicg(SolveCtx* c) : r(c->r), v(c->v), p(c->p), beta(c->beta), omega(c->omega) {}
    __device__ In load(int64_t i) const { return {ld_vec(r + i), ld_vec(p + i), ld_vec(v + i)}; }
    __device__ void apply(int64_t i, const In& in, double (&)[1]) const {
        double2 d = in.p;  // p − ω v
        d.x = fma(-omega.x, in.v.x, fma(omega.y, in.v.y, d.x));
        d.y = fma(-omega.x, in.v.y, fma(-omega.y, in.v.x, d.y));
        double2 o = in.r;
        cfma(o, beta, d);
        st_vec(p + i, o);
    }
    __device__ void finish(double (&)[1], int = 0, int = 0) const {}
};

struct OpK2Cg {  // x += α p ; r −= α q ; {‖r‖²}
    static constexpr int K = 1;
    static constexpr int U = 2;
    struct In { double2 x, p, r, q; };
    SolveCtx* c;
    double2 *__restrict__ x, *__restrict__ r;
    const double2 *__restrict__ p, *__restrict__ q;
    double alpha;
    __device__ explicit OpK2Cg(SolveCtx* c_) : c(c_), x(c_->x), r(c_->r), p(c_->p), q(c_->q), alpha(c_->alpha_cg) {}
    __device__ In load(int64_t i) const {
        return {ld_vec(x + i), ld_vec(p + i), ld_vec(r + i), ld_vec(q + i)};
    }
    __device__ void apply(int64_t i, const In& in, double (&acc)[1]) const {
        st_vec(x + i, make_double2(fma(alpha, in.p.x, in.x.x), fma(alpha, in.p.y, in.x.y)));
        const double2 rn = make_double2(fma(-alpha, in.q.x, in.r.x), fma(-alpha, in.q.y, in.r.y));
        st_vec(r + i, rn);
        acc[0] += cabs2(rn);
    }
    __device__ void finish(double (&acc)[1], int off = 0, int tot = 0) const { reduce_finish<S_K2_CG, 1>(c, acc, off, tot); }
};

struct OpK3Cg {  // p = r + β p
    static constexpr int K = 0;
    struct In { double2 r, p; };
    const double2* __restrict__ r;
    double2* __restrict__ p;
    double beta;
    __device__ explicit OpK3Cg(SolveCtx* c) : r(c->r), p(c->p), beta(c->beta_cg) {}
    __device__ In load(int64_t i) const { return {ld_vec(r + i), ld_vec(p + i)}; }
    __device__ void apply(int64_t i, const In& in, double (&)[1]) const {
        st_vec(p + i, make_double2(fma(beta, in.p.x, in.r.x), fma(beta, in.p.y, in.r.y)));
    }
    __device__ void finish(double (&)[1], int = 0, int = 0) const {}
};

struct EpiK1Cocg {  // q = A p ; {μ = pᵀ q} (unconjugated)
    static constexpr int K = 2;
    using Pre = double2;
    SolveCtx* c;
    double2* __restrict__ q;
    const double2* __restrict__ p;
    __device__ explicit EpiK1Cocg(SolveCtx* c_) : c(c_), q(c_->q), p(c_->p) {}
    __device__ Pre pre(int64_t i) const { return ld_gather_coh(p + i); }
    __device__ void row(int64_t i, double2 y, const Pre& pi, double (&acc)[2]) {
        st_vec(q + i, y);
        acc[0] = fma(pi.x, y.x, fma(-pi.y, y.y, acc[0]));
        acc[1] = fma(pi.x, y.y, fma(pi.y, y.x, acc[1]));
    }
    __device__ void finish(double (&acc)[2], int off = 0, int tot = 0) { reduce_finish<S_K1_COCG, 2>(c, acc, off, tot); }
};

struct OpK2Cocg {  // x += α p ; r −= α q ; {‖r‖², rᵀr}
    static constexpr int K = 3;
    static constexpr int U = 2;
    struct In { double2 x, p, r, q; };
    SolveCtx* c;
    double2 *__restrict__ x, *__restrict__ r;
    const double2 *__restrict__ p, *__restrict__ q;
    double2 alpha;
    __device__ explicit OpK2Cocg(SolveCtx* c_) : c(c_), x(c_->x), r(c_->r), p(c_->p), q(c_->q), alpha(c_->alpha) {}
    __device__ In load(int64_t i) const { return {ld_vec(x + i), ld_vec(p + i), ld_vec(r + i), ld_vec(q + i)}; }
    __device__ void apply(int64_t i, const In& in, double (&acc)[3]) const {
        double2 xn = in.x;
        cfma(xn, alpha, in.p);
        st_vec(x + i, xn);
        double2 rn = in.r;
        rn.x = fma(-alpha.x, in.q.x, fma(alpha.y, in.q.y, rn.x));
        rn.y = fma(-alpha.x, in.q.y, fma(-alpha.y, in.q.x, rn.y));
        st_vec(r + i, rn);
        acc[0] += cabs2(rn);
        acc[1] = fma(rn.x, rn.x, fma(-rn.y, rn.y, acc[1]));
        acc[2] = fma(2.0 * rn.x, rn.y, acc[2]);
    }
    __device__ void finish(double (&acc)[3], int off = 0, int tot = 0) const { reduce_finish<S_K2_COCG, 3>(c, acc, off, tot); }
};

struct OpK3Cocg {  // p = r + β p (complex β)
    static constexpr int K = 0;
    struct In { double2 r, p; };
    const double2* __restrict__ r;
    double2* __restrict__ p;
    double2 beta;
    __device__ explicit OpK3Cocg(SolveCtx* c) : r(c->r), p(c->p), beta(c->beta) {}
    __device__ In load(int64_t i) const { return {ld_vec(r + i), ld_vec(p + i)}; }
    __device__ void apply(int64_t i, const In& in, double (&)[1]) const {
        double2 o = in.r;
        cfma(o, beta, in.p);
        st_vec(p + i, o);
    }
    __device__ void finish(double (&)[1], int = 0, int = 0) const {}
};

// TFQMR epilogues and vector ops (the loops of oracle_tfqmr, fused per kernel T1..T4)
#ifndef ZK_TF_AHEAD
#define ZK_TF_AHEAD true
#endif
#ifndef ZK_T1_U
#define ZK_T1_U 1
#endif
// T2/T4 (SpMV + the TFQMR epilogues): 80 registers (3 CTAs/SM) measured 16 % faster on C4 than
// the 64 of the plain SpMV kernels (profiles/r01_tfqmr_variants.md)
#ifndef ZK_TF_MINB
#define ZK_TF_MINB ((MODE == 0 || MODE == 3) ? 3 : spmv_min_blocks(MODE))
#endif
struct OpT1Tfqmr {  // y2 = y1 − α v ; w −= α u1 ; {‖w‖²}
    static constexpr int K = 1;
    static constexpr int U = ZK_T1_U;
    struct In { double2 y1, v, w, u1; };
    SolveCtx* c;
    const double2 *__restrict__ y1, *__restrict__ v, *__restrict__ u1;
    double2 *__restrict__ y2, *__restrict__ w;
    double2 alpha;
    __device__ explicit OpT1Tfqmr(SolveCtx* c_)
        : c(c_), y1(c_->y1), v(c_->v), u1(c_->u1), y2(c_->y2), w(c_->w), alpha(c_->alpha) {}
    __device__ In load(int64_t i) const { return {ld_vec(y1 + i), ld_vec(v + i), ld_vec(w + i), ld_vec(u1 + i)}; }
    __device__ void apply(int64_t i, const In& in, double (&acc)[1]) const {
        double2 o = in.y1;
        o.x = fma(-alpha.x, in.v.x, fma(alpha.y, in.v.y, o.x));
        o.y = fma(-alpha.x, in.v.y, fma(-alpha.y, in.v.x, o.y));
        st_vec(y2 + i, o);
        double2 wn = in.w;
        wn.x = fma(-alpha.x, in.u1.x, fma(alpha.y, in.u1.y, wn.x));
        wn.y = fma(-alpha.x, in.u1.y, fma(-alpha.y, in.u1.x, wn.y));
        st_vec(w + i, wn);
        acc[0] += cabs2(wn);
    }
    __device__ void finish(double (&acc)[1], int off = 0, int tot = 0) const { reduce_finish<S_T1_TFQMR, 1>(c, acc, off, tot); }
};

struct EpiT2Tfqmr {  // u2 = A y2 ; w −= α u2 ; {‖w‖², ⟨r̃, w⟩}
    static constexpr int K = 3;
    static constexpr bool kAhead = ZK_TF_AHEAD;
    static constexpr int kPrePlace = 2;  // SELL: after the row sums (T2+T4 489 vs 547 ms on C4)
    struct Pre { double2 w, rt; };
    SolveCtx* c;
    double2 *__restrict__ u2, *__restrict__ w;
    const double2* __restrict__ rt;
    double2 alpha;
    __device__ explicit EpiT2Tfqmr(SolveCtx* c_) : c(c_), u2(c_->u2), w(c_->w), rt(c_->rt), alpha(c_->alpha) {}
    __device__ Pre pre(int64_t i) const { return {ld_vec(w + i), ld_vec(rt + i)}; }
    __device__ void row(int64_t i, double2 y, const Pre& q, double (&acc)[3]) {
        st_vec(u2 + i, y);
        double2 wn = q.w;
        wn.x = fma(-alpha.x, y.x, fma(alpha.y, y.y, wn.x));
        wn.y = fma(-alpha.x, y.y, fma(-alpha.y, y.x, wn.y));
        st_vec(w + i, wn);
        acc[0] += cabs2(wn);
        acc[1] = fma(q.rt.x, wn.x, fma(q.rt.y, wn.y, acc[1]));
        acc[2] = fma(q.rt.x, wn.y, fma(-q.rt.y, wn.x, acc[2]));
    }
    __device__ void finish(double (&acc)[3], int off = 0, int tot = 0) { reduce_finish<S_T2_TFQMR, 3>(c, acc, off, tot); }
};

// d1 = y1 + c1·d ; d = y2 + c2·d1 ; x += η1·d1 + η2·d ; y1 = w + β y2   (exit: no y1)
struct OpT3Tfqmr {
    static constexpr int K = 0;
    static constexpr int U = 1;  // 5 input streams
    struct In { double2 x, y1, d, w, y2; };
    double2 *__restrict__ x, *__restrict__ y1, *__restrict__ d;
    const double2 *__restrict__ w, *__restrict__ y2;
    double2 coef1, coef2, eta1, eta2, beta;
    bool exit_only;
    __device__ OpT3Tfqmr(SolveCtx* c, bool exit_only_)
        : x(c->x), y1(c->y1), d(c->d), w(c->w), y2(c->y2), coef1(c->coef1), coef2(c->coef2), eta1(c->eta1),
          eta2(c->eta), beta(c->beta), exit_only(exit_only_) {}
    __device__ In load(int64_t i) const {
        In v;
        v.x = ld_vec(x + i);
        v.y1 = ld_vec(y1 + i);
        v.d = ld_vec(d + i);
        v.y2 = ld_vec(y2 + i);
        if (!exit_only) v.w = ld_vec(w + i);
        return v;
    }
    __device__ void apply(int64_t i, const In& in, double (&)[1]) const {
        double2 d1 = in.y1;  // oracle order: d1, then d2 from d1, then (x + η1·d1) + η2·d2
        cfma(d1, coef1, in.d);
        double2 d2 = in.y2;
        cfma(d2, coef2, d1);
        double2 xn = in.x;
        cfma(xn, eta1, d1);
        cfma(xn, eta2, d2);
        st_vec(x + i, xn);
        st_vec(d + i, d2);
        if (exit_only) return;
        double2 o = in.w;
        cfma(o, beta, in.y2);
        st_vec(y1 + i, o);
    }
    __device__ void finish(double (&)[1], int = 0, int = 0) const {}
};

// split schedule (large systems): T2/T4 store A·y only, these passes do the rest
struct OpT2bTfqmr {  // w −= α u2 ; {‖w‖², ⟨r̃, w⟩}
    static constexpr int K = 3;
    static constexpr int U = 2;
    struct In { double2 w, u2, rt; };
    SolveCtx* c;
    double2* __restrict__ w;
    const double2 *__restrict__ u2, *__restrict__ rt;
    double2 alpha;
    __device__ explicit OpT2bTfqmr(SolveCtx* c_) : c(c_), w(c_->w), u2(c_->u2), rt(c_->rt), alpha(c_->alpha) {}
    __device__ In load(int64_t i) const { return {ld_vec(w + i), ld_vec(u2 + i), ld_vec(rt + i)}; }
    __device__ void apply(int64_t i, const In& in, double (&acc)[3]) const {
        double2 wn = in.w;
        wn.x = fma(-alpha.x, in.u2.x, fma(alpha.y, in.u2.y, wn.x));
        wn.y = fma(-alpha.x, in.u2.y, fma(-alpha.y, in.u2.x, wn.y));
        st_vec(w + i, wn);
        acc[0] += cabs2(wn);
        acc[1] = fma(in.rt.x, wn.x, fma(in.rt.y, wn.y, acc[1]));
        acc[2] = fma(in.rt.x, wn.y, fma(-in.rt.y, wn.x, acc[2]));
    }
    __device__ void finish(double (&acc)[3], int off = 0, int tot = 0) const { reduce_finish<S_T2_TFQMR, 3>(c, acc, off, tot); }
};
struct OpT4bTfqmr {  // v = u1 + β(u2 + β v) ; {σ = ⟨r̃, v⟩}
    static constexpr int K = 2;
    static constexpr int U = 1;
    struct In { double2 u1, u2, v, rt; };
    SolveCtx* c;
    double2* __restrict__ v;
    const double2 *__restrict__ u1, *__restrict__ u2, *__restrict__ rt;
    double2 beta;
    __device__ explicit OpT4bTfqmr(SolveCtx* c_) : c(c_), v(c_->v), u1(c_->u1), u2(c_->u2), rt(c_->rt), beta(c_->beta) {}
    __device__ In load(int64_t i) const { return {ld_vec(u1 + i), ld_vec(u2 + i), ld_vec(v + i), ld_vec(rt + i)}; }
    __device__ void apply(int64_t i, const In& in, double (&acc)[2]) const {
        double2 t = in.u2;
        cfma(t, beta, in.v);
        double2 vn = in.u1;
        cfma(vn, beta, t);
        st_vec(v + i, vn);
        acc[0] = fma(in.rt.x, vn.x, fma(in.rt.y, vn.y, acc[0]));
        acc[1] = fma(in.rt.x, vn.y, fma(-in.rt.y, vn.x, acc[1]));
    }
    __device__ void finish(double (&acc)[2], int off = 0, int tot = 0) const { reduce_finish<S_T4_TFQMR, 2>(c, acc, off, tot); }
};

template <int S>
struct EpiT4Tfqmr {  // u1 = A y1 ; v = u1 + β(u2 + β v) (first: v = u1) ; {σ = ⟨r̃, v⟩}
    static constexpr int K = 2;
    static constexpr bool kAhead = ZK_TF_AHEAD;
    static constexpr int kPrePlace = 2;
    struct Pre { double2 u2, v, rt; };
    SolveCtx* c;
    double2 *__restrict__ u1, *__restrict__ v;
    const double2 *__restrict__ u2, *__restrict__ rt;
    double2 beta;
    __device__ explicit EpiT4Tfqmr(SolveCtx* c_)
        : c(c_), u1(c_->u1), v(c_->v), u2(c_->u2), rt(c_->rt), beta(c_->beta) {}
    __device__ Pre pre(int64_t i) const {
        if (S == S_K0_TFQMR) return {make_double2(0, 0), make_double2(0, 0), ld_vec(rt + i)};
        return {ld_vec(u2 + i), ld_vec(v + i), ld_vec(rt + i)};
    }
    __device__ void row(int64_t i, double2 y, const Pre& q, double (&acc)[2]) {
        st_vec(u1 + i, y);
        double2 vn = y;
        if (S != S_K0_TFQMR) {
            double2 t = q.u2;
            cfma(t, beta, q.v);
            cfma(vn, beta, t);
        }
        st_vec(v + i, vn);
        acc[0] = fma(q.rt.x, vn.x, fma(q.rt.y, vn.y, acc[0]));
        acc[1] = fma(q.rt.x, vn.y, fma(-q.rt.y, vn.x, acc[1]));
    }
    __device__ void finish(double (&acc)[2], int off = 0, int tot = 0) { reduce_finish<S, 2>(c, acc, off, tot); }
};

// ------------------------------------------------------------------ kernels
#ifndef ZK_VEC_MINB
#define ZK_VEC_MINB 4  // fused vector kernels: ≤ 64 registers, 4 CTAs / 32 warps per SM
#endif
// The CSR view is copied into registers/locals once (not re-read from the ctx).
template <int W, int MODE, int S>
__global__ void __launch_bounds__(kBlock, spmv_min_blocks(MODE)) k_init_x0(SolveCtx* c, const double2* __restrict__ xg,
                                                                          int bicg) {
    stamp_start<S>(c);
    const CsrDev A = c->A;
    EpiInit<S> e(c, xg, bicg == 1);
    spmv_any<W, MODE>(A, xg, e);
}
__global__ void __launch_bounds__(kBlock, ZK_VEC_MINB) k_init_zero(SolveCtx* c, int kind) {
    stamp_start<S_INIT_BICG>(c);
    OpInitZero op(c, kind);
    vec_body(c->A.n_rows, op);
}
template <int W, int MODE>
__global__ void __launch_bounds__(kBlock, spmv_min_blocks(MODE)) k_true(SolveCtx* c, const double2* __restrict__ xg,
                                                                       CsrDev A) {
    // A: the ORIGINAL operator (the Jacobi path iterates on A·M⁻¹ but checks ‖b − A x‖)
    if (c->status == ST_ZERO_RHS) return;
    stamp_start<S_TRUE>(c);
    EpiTrue e(c);
    spmv_any<W, MODE>(A, xg, e);
}
// SPLIT: 0 fused epilogue; 1 products only (r1_bicg reduces); 2 products + tail reduction (SELL)
template <int W, int MODE, int SPLIT>
__global__ void __launch_bounds__(kBlock, spmv_min_blocks(MODE)) k1_bicg(SolveCtx* c, const CsrDev A) {
    pdl_enter();
    if (c->done) return;
    stamp_start<S_K1_BICG>(c);
    const double2* p = c->p;
        if constexpr (SPLIT == 3) {
        WarpAcc<EpiK1Bicg> e(c);
        spmv_any<W, MODE>(A, p, e);
    } else if constexpr (SPLIT == 2) {
        EpiStoreTail<OpRed1Bicg> e(c->v, c);
        spmv_any<W, MODE>(A, p, e);
    } else if constexpr (SPLIT == 1) {
        EpiStore e(c->v);
        spmv_any<W, MODE>(A, p, e);
    } else {
        EpiK1Bicg e(c);
        spmv_any<W, MODE>(A, p, e);
    }
}
__global__ void __launch_bounds__(kBlock, ZK_VEC_MINB) r1_bicg(SolveCtx* c) {
    pdl_enter();
    if (c->done) return;
    OpRed1Bicg op(c);
    vec_body(c->A.n_rows, op);
}
__global__ void __launch_bounds__(kBlock, ZK_VEC_MINB) r3_bicg(SolveCtx* c) {
    pdl_enter();
    if (c->done) return;
    OpRed3Bicg op(c);
    vec_body(c->A.n_rows, op);
}
__global__ void __launch_bounds__(kBlock, ZK_VEC_MINB) k2_bicg(SolveCtx* c) {
    pdl_enter();
    if (c->done) return;
    stamp_start<S_K2_BICG>(c);
    OpK2Bicg op(c);
    vec_body<kSweep>(c->A.n_rows, op);  // ←
}
template <int W, int MODE, int SPLIT>
__global__ void __launch_bounds__(kBlock, spmv_min_blocks(MODE)) k3_bicg(SolveCtx* c, const CsrDev A) {
    pdl_enter();
    if (c->done) return;
    stamp_start<S_K3_BICG>(c);
    const double2* s = c->s;
        if constexpr (SPLIT == 3) {
        WarpAcc<EpiK3Bicg> e(c);
        spmv_any<W, MODE>(A, s, e);
    } else if constexpr (SPLIT == 2) {
        EpiStoreTail<OpRed3Bicg> e(c->t, c);
        spmv_any<W, MODE>(A, s, e);
    } else if constexpr (SPLIT == 1) {
        EpiStore e(c->t);
        spmv_any<W, MODE>(A, s, e);
    } else {
        EpiK3Bicg e(c);
        spmv_any<W, MODE>(A, s, e);
    }
}
__global__ void __launch_bounds__(kBlock, ZK_VEC_MINB) k4_bicg(SolveCtx* c) {
    pdl_enter();
    const bool half = c->half != 0;
    if (c->done && !half) return;
    if (!half) stamp_start<S_K4_BICG>(c);
    OpK4Bicg op(c, half);
    vec_body<kSweep>(c->A.n_rows, op);  // ←
}
__global__ void __launch_bounds__(kBlock, ZK_VEC_MINB) k5_bicg(SolveCtx* c) {
    pdl_enter();
    if (c->done) {
        if (c->half && blockIdx.x == 0 && threadIdx.x == 0) c->half = 0;  // K4 applied x += αp
    } else {
        OpK5Bicg op(c);
        vec_body(c->A.n_rows, op);
    }
    set_cond(c);  // after the stream loop: the device-runtime call does not pressure its registers
}
template <int W, int MODE, int SPLIT>
__global__ void __launch_bounds__(kBlock, spmv_min_blocks(MODE)) k1_cocg(SolveCtx* c, const CsrDev A) {
    pdl_enter();
    if (c->done) return;
    stamp_start<S_K1_COCG>(c);
    const double2* p = c->p;
        if constexpr (SPLIT == 3) {
        WarpAcc<EpiK1Cocg> e(c);
        spmv_any<W, MODE>(A, p, e);
    } else if constexpr (SPLIT == 2) {
        EpiStoreTail<OpRedPq<false, S_K1_COCG>> e(c->q, c);
        spmv_any<W, MODE>(A, p, e);
    } else if constexpr (SPLIT == 1) {
        EpiStore e(c->q);
        spmv_any<W, MODE>(A, p, e);
    } else {
        EpiK1Cocg e(c);
        spmv_any<W, MODE>(A, p, e);
    }
}
__global__ void __launch_bounds__(kBlock, ZK_VEC_MINB) k2_cocg(SolveCtx* c) {
    pdl_enter();
    if (c->done) return;
    stamp_start<S_K2_COCG>(c);
    OpK2Cocg op(c);
    vec_body<kSweep>(c->A.n_rows, op);  // ←
}
__global__ void __launch_bounds__(kBlock, ZK_VEC_MINB) k3_cocg(SolveCtx* c) {
    pdl_enter();
    if (!c->done) {
        OpK3Cocg op(c);
        vec_body(c->A.n_rows, op);
    }
    set_cond(c);
}
template <int W, int MODE, int SPLIT>
__global__ void __launch_bounds__(kBlock, spmv_min_blocks(MODE)) k1_cg(SolveCtx* c, const CsrDev A) {
    pdl_enter();
    if (c->done) return;
    stamp_start<S_K1_CG>(c);
    const double2* p = c->p;
        if constexpr (SPLIT == 3) {
        WarpAcc<EpiK1Cg> e(c);
        spmv_any<W, MODE>(A, p, e);
    } else if constexpr (SPLIT == 2) {
        EpiStoreTail<OpRedPq<true, S_K1_CG>> e(c->q, c);
        spmv_any<W, MODE>(A, p, e);
    } else if constexpr (SPLIT == 1) {
        EpiStore e(c->q);
        spmv_any<W, MODE>(A, p, e);
    } else {
        EpiK1Cg e(c);
        spmv_any<W, MODE>(A, p, e);
    }
}
template <bool CONJ, int S>
__global__ void __launch_bounds__(kBlock, ZK_VEC_MINB) rq_kernel(SolveCtx* c) {
    pdl_enter();
    if (c->done) return;
    OpRedPq<CONJ, S> op(c);
    vec_body(c->A.n_rows, op);
}
__global__ void __launch_bounds__(kBlock, ZK_VEC_MINB) k2_cg(SolveCtx* c) {
    pdl_enter();
    if (c->done) return;
    stamp_start<S_K2_CG>(c);
    OpK2Cg op(c);
    vec_body<kSweep>(c->A.n_rows, op);  // ←
}
__global__ void __launch_bounds__(kBlock, ZK_VEC_MINB) k3_cg(SolveCtx* c) {
    pdl_enter();
    if (!c->done) {
        OpK3Cg op(c);
        vec_body(c->A.n_rows, op);
    }
    set_cond(c);
}
template <int W, int MODE>
__global__ void __launch_bounds__(kBlock, spmv_min_blocks(MODE)) k0_tfqmr(SolveCtx* c, const CsrDev A) {  // u1 = v = A y1, σ
    if (c->done) return;
    stamp_start<S_K0_TFQMR>(c);
    const double2* y1 = c->y1;
    EpiT4Tfqmr<S_K0_TFQMR> e(c);
    spmv_any<W, MODE>(A, y1, e);
}
__global__ void __launch_bounds__(kBlock, ZK_VEC_MINB) t1_tfqmr(SolveCtx* c) {
    pdl_enter();
    if (c->done) return;
    stamp_start<S_T1_TFQMR>(c);
    OpT1Tfqmr op(c);
    vec_body(c->A.n_rows, op);  // TFQMR: an even kernel count, fixed directions T1 →, T2 ←, T3 →, T4 ←
}
template <int W, int MODE, int SPLIT>
__global__ void __launch_bounds__(kBlock, ZK_TF_MINB) t2_tfqmr(SolveCtx* c, const CsrDev A) {
    pdl_enter();
    if (c->done) {
        if (c->half != 1 || !A.main_part) return;  // once per SpMV (distributed: 2 partial launches)
        // the first half step ended the loop: only its x += η1·d1, d1 = y1 + c1·d, remains
        double2* __restrict__ x = c->x;
        const double2* __restrict__ d = c->d;
        const double2* __restrict__ y1 = c->y1;
        const double2 eta = c->eta1, coef = c->coef1;
        const int64_t n = c->A.n_rows;
        for (int64_t i = (int64_t)blockIdx.x * kBlock + threadIdx.x; i < n; i += (int64_t)gridDim.x * kBlock) {
            double2 d1 = y1[i];
            cfma(d1, coef, d[i]);
            double2 xn = x[i];
            cfma(xn, eta, d1);
            x[i] = xn;
        }
        return;
    }
    stamp_start<S_T2_TFQMR>(c);
    const double2* y2 = c->y2;
    if constexpr (SPLIT == 2) {
        EpiStoreTail<OpT2bTfqmr> e(c->u2, c);
        spmv_any<W, MODE, kSweep>(A, y2, e);  // ←
    } else if constexpr (SPLIT == 1) {
        EpiStore e(c->u2);
        spmv_any<W, MODE>(A, y2, e);
    } else {
        EpiT2Tfqmr e(c);
        spmv_any<W, MODE>(A, y2, e);
    }
}
__global__ void __launch_bounds__(kBlock, ZK_VEC_MINB) t2b_tfqmr(SolveCtx* c) {
    pdl_enter();
    if (c->done) return;
    OpT2bTfqmr op(c);
    vec_body(c->A.n_rows, op);
}
__global__ void __launch_bounds__(kBlock, ZK_VEC_MINB) t4b_tfqmr(SolveCtx* c) {
    pdl_enter();
    if (c->done) {
        if (c->half && blockIdx.x == 0 && threadIdx.x == 0) c->half = 0;
    } else {
        OpT4bTfqmr op(c);
        vec_body(c->A.n_rows, op);
    }
    set_cond(c);
}
__global__ void __launch_bounds__(kBlock, ZK_VEC_MINB) t3_tfqmr(SolveCtx* c) {
    pdl_enter();
    const bool done = c->done != 0;
    if (done && c->half != 2) return;
    OpT3Tfqmr op(c, done);
    vec_body(c->A.n_rows, op);
}
template <int W, int MODE, int SPLIT>
__global__ void __launch_bounds__(kBlock, ZK_TF_MINB) t4_tfqmr(SolveCtx* c, const CsrDev A) {
    pdl_enter();
    if (c->done) {
        // T2/T3 applied the last x update (split: t4b_tfqmr clears it)
        if (SPLIT != 1 && c->half && blockIdx.x == 0 && threadIdx.x == 0) c->half = 0;
    } else {
        stamp_start<S_T4_TFQMR>(c);
        const double2* y1 = c->y1;
        if constexpr (SPLIT == 2) {
            EpiStoreTail<OpT4bTfqmr> e(c->u1, c);
            spmv_any<W, MODE, kSweep>(A, y1, e);  // ←
        } else if constexpr (SPLIT == 1) {
            EpiStore e(c->u1);
            spmv_any<W, MODE>(A, y1, e);
        } else {
            EpiT4Tfqmr<S_T4_TFQMR> e(c);
            spmv_any<W, MODE>(A, y1, e);
        }
    }
    // split: t4b_tfqmr is the body's last kernel; a distributed SpMV is two launches: count the
    // body once (main_part: the interior launch)
    if (SPLIT != 1 && A.main_part) set_cond(c);
}
// ------------------------------------------------------------------ BiCGStab(ℓ) kernels (NEXT-3)
// One outer cycle (oracle_bicgstab_l): for j = 0..ℓ−1 the BiCG step runs as
//   B1(j)  û_i = r̂_i − β û_i (i ≤ j)
//   S1(j)  û_{j+1} = A û_j ; γ = ⟨r̃, û_{j+1}⟩, ‖û_{j+1}‖²                → α = ρ0/γ
//   B2(j)  r̂_i −= α û_{i+1} (i ≤ j) ; x += α û_0 ; ‖r̂_0‖²                → exit test
//   S2(j)  r̂_{j+1} = A r̂_j ; ρ1 = ⟨r̃, r̂_{j+1}⟩, ‖r̂_{j+1}‖² (j < ℓ−1)    → β = α ρ1/ρ0
// then the minimal-residual part:
//   G      Gram matrix ⟨r̂_a, r̂_b⟩ (a ≤ b ≤ ℓ) in ONE pass over the ℓ+1 vectors → Cholesky, γ, ω
//   U      x += Σ γ_j r̂_{j−1} ; r̂_0 −= Σ γ_j r̂_j ; û_0 −= Σ γ_j û_j ; ‖r̂_0‖², ⟨r̃, r̂_0⟩
//                                                             → hist, tests, next cycle's β
// (writes the WHILE condition).  The vector sets travel as a kernel parameter (constant bank).
struct VecSet {
    double2* r[kMaxEll + 1];
    double2* u[kMaxEll + 1];
};

__global__ void __launch_bounds__(kBlock, ZK_VEC_MINB) bl_b1(SolveCtx* c, VecSet P, int j) {
    pdl_enter();
    if (c->done) return;
    const double2 beta = c->beta;
    const int64_t n = c->A.n_rows;
    constexpr int UE = 4;
    for (int64_t base = (int64_t)blockIdx.x * kBlock * UE + threadIdx.x; base < n;
         base += (int64_t)gridDim.x * kBlock * UE) {
        for (int q = 0; q <= j; q++) {  // û_q = r̂_q − β û_q
            const double2* __restrict__ r = P.r[q];
            double2* __restrict__ u = P.u[q];
            double2 rv[UE], uv[UE];
#pragma unroll
            for (int e = 0; e < UE; e++) {
                const int64_t i = base + e * kBlock;
                if (i < n) {
                    rv[e] = ld_vec(r + i);
                    uv[e] = ld_vec(u + i);
                }
            }
#pragma unroll
            for (int e = 0; e < UE; e++) {
                const int64_t i = base + e * kBlock;
                if (i < n) {
                    double2 o = rv[e];
                    o.x = fma(-beta.x, uv[e].x, fma(beta.y, uv[e].y, o.x));
                    o.y = fma(-beta.x, uv[e].y, fma(-beta.y, uv[e].x, o.y));
                    u[i] = o;
                }
            }
        }
    }
}

__global__ void __launch_bounds__(kBlock, ZK_VEC_MINB) bl_b2(SolveCtx* c, VecSet P, int j) {
    pdl_enter();
    if (c->done) return;
    stamp_start<S_B2_BL>(c);
    const double2 alpha = c->alpha;
    double2* __restrict__ x = c->x;
    const int64_t n = c->A.n_rows;
    constexpr int UE = 2;
    double acc[1] = {0.0};
    for (int64_t base = (int64_t)blockIdx.x * kBlock * UE + threadIdx.x; base < n;
         base += (int64_t)gridDim.x * kBlock * UE) {
        {   // q = 0: r̂_0 −= α û_1 ; x += α û_0 ; ‖r̂_0‖²
            double2 rv[UE], u1[UE], xv[UE], u0[UE];
#pragma unroll
            for (int e = 0; e < UE; e++) {
                const int64_t i = base + e * kBlock;
                if (i < n) {
                    rv[e] = ld_vec(P.r[0] + i);
                    u1[e] = ld_vec(P.u[1] + i);
                    xv[e] = ld_vec(x + i);
                    u0[e] = ld_vec(P.u[0] + i);
                }
            }
#pragma unroll
            for (int e = 0; e < UE; e++) {
                const int64_t i = base + e * kBlock;
                if (i < n) {
                    double2 o = rv[e];
                    o.x = fma(-alpha.x, u1[e].x, fma(alpha.y, u1[e].y, o.x));
                    o.y = fma(-alpha.x, u1[e].y, fma(-alpha.y, u1[e].x, o.y));
                    P.r[0][i] = o;
                    acc[0] += cabs2(o);
                    double2 xn = xv[e];
                    cfma(xn, alpha, u0[e]);
                    x[i] = xn;
                }
            }
        }
        for (int q = 1; q <= j; q++) {  // r̂_q −= α û_{q+1}
            double2* __restrict__ r = P.r[q];
            const double2* __restrict__ u = P.u[q + 1];
            double2 rv[UE], uv[UE];
#pragma unroll
            for (int e = 0; e < UE; e++) {
                const int64_t i = base + e * kBlock;
                if (i < n) {
                    rv[e] = ld_vec(r + i);
                    uv[e] = ld_vec(u + i);
                }
            }
#pragma unroll
            for (int e = 0; e < UE; e++) {
                const int64_t i = base + e * kBlock;
                if (i < n) {
                    double2 o = rv[e];
                    o.x = fma(-alpha.x, uv[e].x, fma(alpha.y, uv[e].y, o.x));
                    o.y = fma(-alpha.x, uv[e].y, fma(-alpha.y, uv[e].x, o.y));
                    r[i] = o;
                }
            }
        }
    }
    reduce_finish<S_B2_BL, 1>(c, acc);
}

template <int S, bool RED>
struct EpiBl {  // out = A v ; {⟨r̃, out⟩, ‖out‖²} when RED
    static constexpr int K = RED ? 3 : 0;
    static constexpr bool kOrdered = !RED;  // store-only (split schedule): as EpiStore (spmv.cuh)
    static constexpr int KA = K > 0 ? K : 1;
    using Pre = double2;
    SolveCtx* c;
    double2* __restrict__ out;
    const double2* __restrict__ rt;
    __device__ EpiBl(SolveCtx* c_, double2* out_) : c(c_), out(out_), rt(c_->rh) {}
    __device__ Pre pre(int64_t i) const {
        if constexpr (RED) return ld_vec(rt + i);
        else return make_double2(0.0, 0.0);
    }
    __device__ void row(int64_t i, double2 y, const Pre& q, double (&acc)[KA]) {
        out[i] = y;
        if constexpr (RED) {
            acc[0] = fma(q.x, y.x, fma(q.y, y.y, acc[0]));
            acc[1] = fma(q.x, y.y, fma(-q.y, y.x, acc[1]));
            acc[2] += cabs2(y);
        }
    }
    __device__ void finish(double (&acc)[KA], int off = 0, int tot = 0) {
        if constexpr (RED) reduce_finish<S, 3>(c, acc, off, tot);
    }
};

template <int W, int MODE, bool RED>
__global__ void __launch_bounds__(kBlock, spmv_min_blocks(MODE)) bl_s1(SolveCtx* c, const CsrDev A, VecSet P, int j) {
    pdl_enter();
    if (c->done) return;
    stamp_start<S_S1_BL>(c);  // RED = false (split): bl_r<S_S1_BL> reduces and closes the timer
    EpiBl<S_S1_BL, RED> e(c, P.u[j + 1]);
    spmv_any<W, MODE>(A, P.u[j], e);
}
template <int W, int MODE, bool RED>
__global__ void __launch_bounds__(kBlock, spmv_min_blocks(MODE)) bl_s2(SolveCtx* c, const CsrDev A, VecSet P, int j,
                                                                    int stamp) {
    pdl_enter();
    if (c->done) return;
    if (stamp) stamp_start<S_S2_BL>(c);
    EpiBl<S_S2_BL, RED> e(c, P.r[j + 1]);
    spmv_any<W, MODE>(A, P.r[j], e);
}

template <int S>
struct OpRedBl {  // {⟨r̃, y⟩, ‖y‖²} of the vector y just produced by S1/S2 (split schedule)
    static constexpr int K = 3;
    struct In { double2 r, y; };
    SolveCtx* c;
    const double2 *__restrict__ rt, *__restrict__ y;
    __device__ OpRedBl(SolveCtx* c_, const double2* y_) : c(c_), rt(c_->rh), y(y_) {}
    __device__ In load(int64_t i) const { return {ld_vec(rt + i), ld_vec(y + i)}; }
    __device__ void apply(int64_t, const In& in, double (&acc)[3]) const {
        acc[0] = fma(in.r.x, in.y.x, fma(in.r.y, in.y.y, acc[0]));
        acc[1] = fma(in.r.x, in.y.y, fma(-in.r.y, in.y.x, acc[1]));
        acc[2] += cabs2(in.y);
    }
    __device__ void finish(double (&acc)[3], int off = 0, int tot = 0) const { reduce_finish<S, 3>(c, acc, off, tot); }
};
template <int S>
__global__ void __launch_bounds__(kBlock, ZK_VEC_MINB) bl_r(SolveCtx* c, const double2* y) {
    pdl_enter();
    if (c->done) return;
    OpRedBl<S> op(c, y);
    vec_body(c->A.n_rows, op);
}

// Gram matrix of r̂_0..ℓ, packed: for a = 0..ℓ: ‖r̂_a‖², then (Re, Im)⟨r̂_a, r̂_b⟩ for b = a+1..ℓ.
template <int L>
__global__ void __launch_bounds__(kBlock, 1) bl_gram(SolveCtx* c, VecSet P) {
    using GP = GramPack<L>;
    constexpr int NV = GP::NV, ND = GP::ND;
    __shared__ double sm[kWarps][ND];
    __shared__ double tot[ND];
    __shared__ bool last;
    pdl_enter();
    if (c->done) return;
    stamp_start<S_G_BL>(c);
    double acc[ND];
#pragma unroll
    for (int k = 0; k < ND; k++) acc[k] = 0.0;
    const int64_t n = c->A.n_rows;
    for (int64_t i = (int64_t)blockIdx.x * kBlock + threadIdx.x; i < n; i += (int64_t)gridDim.x * kBlock) {
        double2 v[NV];
#pragma unroll
        for (int a = 0; a < NV; a++) v[a] = ld_vec(P.r[a] + i);
#pragma unroll
        for (int a = 0; a < NV; a++) {
            acc[GP::diag(a)] += cabs2(v[a]);
#pragma unroll
            for (int b = a + 1; b < NV; b++) {
                double& re = acc[GP::off(a, b)];
                double& im = acc[GP::off(a, b) + 1];
                re = fma(v[a].x, v[b].x, fma(v[a].y, v[b].y, re));
                im = fma(v[a].x, v[b].y, fma(-v[a].y, v[b].x, im));
            }
        }
    }
    warp_sum<ND>(acc);
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    if (lane == 0) {
#pragma unroll
        for (int k = 0; k < ND; k++) sm[warp][k] = acc[k];
    }
    __syncthreads();
    const int G = gridDim.x;
    double* part = c->partials;  // [ND][G]
    for (int k = threadIdx.x; k < ND; k += kBlock) {
        double s = 0.0;
        for (int w = 0; w < kWarps; w++) s += sm[w][k];
        part[k * G + blockIdx.x] = s;
    }
    __threadfence();
    __syncthreads();
    if (threadIdx.x == 0) last = atomicAdd(c->tickets + S_G_BL, 1u) == (unsigned)G - 1;
    __syncthreads();
    if (!last) return;
    __threadfence();
    for (int k = threadIdx.x; k < ND; k += kBlock) {  // fixed order over blocks
        double s = 0.0;
        for (int b = 0; b < G; b++) s += ld_cg(part + k * G + b);
        tot[k] = s;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        c->tickets[S_G_BL] = 0u;
        const unsigned long long st = atomicExch(&c->t0[timer_of(S_G_BL)], ~0ull);
        c->tsum[timer_of(S_G_BL)] += gtimer() - st;
        c->tcnt[timer_of(S_G_BL)] += 1;
        if (c->dist) {  // multi-GPU: the rank's totals go to redg for the allreduce + fin_gram_kernel
            for (int k = 0; k < ND; k++) c->redg[k] = tot[k];
        } else {
            fin_gram_bl<L>(c, tot);
        }
    }
}
template <int L>
__global__ void fin_gram_kernel(SolveCtx* c) {
    if (c->done) return;
    fin_gram_bl<L>(c, c->redg);
}

template <int L>
__global__ void __launch_bounds__(kBlock, 2) bl_u(SolveCtx* c, VecSet P) {
    pdl_enter();
    if (!c->done) {
        stamp_start<S_U_BL>(c);
        double2 g[L + 1];
#pragma unroll
        for (int j = 1; j <= L; j++) g[j] = c->gam[j];
        double2* __restrict__ x = c->x;
        const double2* __restrict__ rt = c->rh;
        const int64_t n = c->A.n_rows;
        double acc[3] = {0.0, 0.0, 0.0};
        for (int64_t i = (int64_t)blockIdx.x * kBlock + threadIdx.x; i < n; i += (int64_t)gridDim.x * kBlock) {
            double2 rv[L + 1], uv[L + 1];
#pragma unroll
            for (int a = 0; a <= L; a++) {
                rv[a] = ld_vec(P.r[a] + i);
                uv[a] = ld_vec(P.u[a] + i);
            }
            double2 xv = ld_vec(x + i);
            const double2 tv = ld_vec(rt + i);
            double2 r0 = rv[0], u0 = uv[0];
#pragma unroll
            for (int j = 1; j <= L; j++) {  // oracle order: j ascending
                cfma(xv, g[j], rv[j - 1]);
                r0.x = fma(-g[j].x, rv[j].x, fma(g[j].y, rv[j].y, r0.x));
                r0.y = fma(-g[j].x, rv[j].y, fma(-g[j].y, rv[j].x, r0.y));
                u0.x = fma(-g[j].x, uv[j].x, fma(g[j].y, uv[j].y, u0.x));
                u0.y = fma(-g[j].x, uv[j].y, fma(-g[j].y, uv[j].x, u0.y));
            }
            x[i] = xv;
            P.r[0][i] = r0;
            P.u[0][i] = u0;
            acc[0] += cabs2(r0);
            acc[1] = fma(tv.x, r0.x, fma(tv.y, r0.y, acc[1]));
            acc[2] = fma(tv.x, r0.y, fma(-tv.y, r0.x, acc[2]));
        }
        reduce_finish<S_U_BL, 3>(c, acc);
    }
    set_cond(c);
}

using BlKernel = void (*)(SolveCtx*, VecSet);
static BlKernel bl_gram_of(int L) {
    switch (L) {
        case 1: return bl_gram<1>;
        case 2: return bl_gram<2>;
        case 3: return bl_gram<3>;
        case 4: return bl_gram<4>;
        case 5: return bl_gram<5>;
        case 6: return bl_gram<6>;
        case 7: return bl_gram<7>;
        default: return bl_gram<8>;
    }
}
using FinKernel = void (*)(SolveCtx*);
static FinKernel fin_gram_of(int L) {
    switch (L) {
        case 1: return fin_gram_kernel<1>;
        case 2: return fin_gram_kernel<2>;
        case 3: return fin_gram_kernel<3>;
        case 4: return fin_gram_kernel<4>;
        case 5: return fin_gram_kernel<5>;
        case 6: return fin_gram_kernel<6>;
        case 7: return fin_gram_kernel<7>;
        default: return fin_gram_kernel<8>;
    }
}
static BlKernel bl_u_of(int L) {
    switch (L) {
        case 1: return bl_u<1>;
        case 2: return bl_u<2>;
        case 3: return bl_u<3>;
        case 4: return bl_u<4>;
        case 5: return bl_u<5>;
        case 6: return bl_u<6>;
        case 7: return bl_u<7>;
        default: return bl_u<8>;
    }
}
static int bl_nd(int L) { return (L + 1) + (L + 1) * L; }

__global__ void k_set_ctx(SolveCtx* c, SolveCtx h) {
    *c = h;
    for (int i = 0; i < kTickets; i++) h.tickets[i] = 0u;  // workspace memory may be recycled
}

// ------------------------------------------------------------------ host side
static int vec_grid(const zk_csr_s* A, const void* k) {
    int cap = A->dev.num_sms * blocks_per_sm(k);
    if (cap > kMaxGrid) cap = kMaxGrid;
    return grid_for(A->n_rows, (int64_t)kBlock * 4, cap);
}

// Jacobi hooks (jacobi.cu)
zk_status jacobi_prepare(zk_csr_s* A, cudaStream_t s);
zk_status cscale(const zk_csr_s* A, const double2* d, const double2* in, double2* out, cudaStream_t s);

// distributed hooks (dist.cu)
zk_status dist_halo(const zk_csr_s* A, double2* xg, cudaStream_t s);           // fill halo slots of xg
zk_status dist_allreduce_ctx(const zk_csr_s* A, double* red, int count, cudaStream_t s);

template <int S>
static zk_status dist_finish(const zk_csr_s* A, SolveCtx* c, int count, cudaStream_t s) {
    ZK_TRY(dist_allreduce_ctx(A, c->red, count, s));
    fin_kernel<S><<<1, 1, 0, s>>>(c);
    ZK_CUDA(cudaGetLastError());
    return ZK_OK;
}

// Split schedule (the SpMV stores its product; its reductions run as the kernel's tail, as a
// warp-reduced epilogue, or — ZK_SPLIT_TAIL=0 / CSR sub-warp mapping — as a separate pass): from
// kSplitRows rows, and always on a distributed matrix, whose SpMVs are split into interior /
// boundary launches around the halo exchange (their fused reductions span both, loop_spmv)
static bool split_reductions(const zk_csr_s* A) {
    if (A->dist) return true;
    if (const char* e = getenv("ZK_SPLIT_RED")) return atoi(e) != 0;
    return A->n_rows >= kSplitRows;
}

// Split schedule with the reduction as the SpMV kernel's tail (EpiStoreTail) instead of a separate
// pass: SELL mapping, one GPU (a distributed SpMV is two launches).  Default; ZK_SPLIT_TAIL=0 keeps
// the separate pass.  Measured (tools/ab_split.py, WHILE graph, µs per iteration, pass → tail):
// Audi3D-4 (C3) BiCGStab 168.0 → 162.2, CG 86.3 → 82.8, TFQMR 173.7 → 165.5; Twingo3D-2 (C3T)
// 133.3 → 128.0, 69.0 → 64.8, 138.0 → 129.7; C4 1707 → 1694, 901 → 908, 1808 → 1797
// (profiles/r02_split_tail.txt).
static bool split_tail(const zk_csr_s* A) {
    if (A->spmv_mode != 3 || !split_reductions(A)) return false;
    // a distributed SpMV is two launches (interior slices, then the boundary after the halo): the
    // fused reductions span them (grid_sum off / total, loop_spmv); ZK_DIST_FUSED=0 keeps the
    // store-only SpMVs and separate reduction passes
    if (A->dist && getenv("ZK_DIST_FUSED") && atoi(getenv("ZK_DIST_FUSED")) == 0) return false;
    if (const char* e = getenv("ZK_SPLIT_TAIL")) return atoi(e) != 0;
    return true;
}
// From 2^20 rows the BiCGStab K1/K3 and CG/COCG K1 SpMVs fuse their dot products again, with
// per-slice warp reductions into shared memory (WarpAcc: no accumulator register across the slice
// loop, the row operand loaded with the slice's last matrix batch) instead of the tail pass — no
// second read of the product vector.  Measured (tools/ab_split.py, µs per iteration, tail →
// warp-reduced): C4 BiCGStab 1749.7 → 1689.5, CG 939.2 → 896.0; C3 BiCGStab 147.9 → 147.9, CG
// 73.1 → 75.2 (profiles/r02_split_wacc.txt), so below 2^20 rows the tail pass stays.
// ZK_SPLIT_TAIL: 0 separate pass, 1 tail, 2 warp-reduced (where the kernel has it), unset = auto.
constexpr int64_t kWarpAccRows = 1 << 20;
static int tail_kind(const zk_csr_s* A) {
    if (!split_tail(A)) return 0;
    if (const char* e = getenv("ZK_SPLIT_TAIL")) return atoi(e) == 2 ? 3 : 2;
    return A->n_rows >= kWarpAccRows ? 3 : 2;
}

bool dist_overlap(const zk_csr_s* A);                                            // dist.cu
void dist_launch_extra(const zk_csr_s* A, int* per_spmv, int* per_allreduce);    // dist.cu
int64_t dist_n_send(const zk_csr_s* A);                                           // dist.cu
void dist_split(const zk_csr_s* A, const CsrDev& a, CsrDev* in, CsrDev* bd);     // dist.cu
zk_status dist_halo_begin(const zk_csr_s* A, double2* xg, cudaStream_t s);       // dist.cu
zk_status dist_halo_end(const zk_csr_s* A, cudaStream_t s);                       // dist.cu

// One store-only loop SpMV y = A·xg.  One GPU: launch(A's view, false).  Distributed: the halo
// exchange of xg runs on the plan's stream while the interior slices (no halo column) compute,
// then the boundary slices (SURVEY.md §8(e) "Halo": pack → send/recv ‖ interior SpMV → boundary
// SpMV); without an interior run (or with ZK_DIST_OVERLAP=0) a blocking exchange first.
// fused: the SpMV kernel's reduction is fused (tail or warp-reduced epilogue): with the overlap its
// two launches share one grid reduction — the interior launch's blocks are partials [0, G1), the
// boundary launch's [G1, G1 + G2), and the boundary launch's last block finishes (grid_sum).
template <class L>
static zk_status loop_spmv(const zk_csr_s* A, const CsrDev& av, double2* xg, cudaStream_t s, L&& launch,
                           const void* fused = nullptr) {
    if (!A->dist) return launch(av, false);
    if (!dist_overlap(A)) {
        ZK_TRY(dist_halo(A, xg, s));
        return launch(av, false);
    }
    CsrDev in, bd;
    dist_split(A, av, &in, &bd);
    if (fused) {
        const int g1 = spmv_cfg_part(A, fused, in).grid;
        const int g2 = bd.sl_cnt > 0 ? spmv_cfg_part(A, fused, bd).grid : 0;
        in.red_off = 0;
        in.red_total = g1 + g2;
        bd.red_off = g1;
        bd.red_total = g1 + g2;
    }
    ZK_TRY(dist_halo_begin(A, xg, s));
    ZK_TRY(launch(in, true));
    ZK_TRY(dist_halo_end(A, s));
    return bd.sl_cnt > 0 ? launch(bd, true) : ZK_OK;
}

// enqueue one iteration of `method`
// loop-kernel launch, with the PDL attribute when `pdl`
template <class... Args>
static zk_status launch_loop(bool pdl, void (*k)(Args...), int grid, int smem, cudaStream_t s, Args... args) {
    cudaLaunchConfig_t cfg;
    memset(&cfg, 0, sizeof cfg);
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(kBlock);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at;
    cfg.numAttrs = pdl ? 1 : 0;
    ZK_CUDA(cudaLaunchKernelEx(&cfg, k, args...));
    return ZK_OK;
}

static zk_status enqueue_iteration(const zk_csr_s* A, SolveCtx* dc, const SolveCtx& hc, int method, cudaStream_t s,
                                   bool pdl = false) {
    const bool dist = A->dist != nullptr;
    if (dist) pdl = false;
    const bool split = split_reductions(A);
    const bool tail = split_tail(A);
    const bool wacc = tail_kind(A) == 3;
    return with_spmv(A, [&](auto wc, auto mc) -> zk_status {
        constexpr int W = decltype(wc)::value, MODE = decltype(mc)::value;
        // a split-schedule SpMV kernel over the slice set `a` (the whole matrix, or one part)
        auto part = [&](auto kf) {
            return [&, kf](const CsrDev& a, bool is_part) -> zk_status {
                const LaunchCfg L = is_part ? spmv_cfg_part(A, (const void*)kf, a) : spmv_cfg(A, (const void*)kf, W, MODE);
                return launch_loop(pdl, kf, L.grid, L.smem, s, dc, a);
            };
        };
        if (method == ZK_BICGSTAB) {
            if (wacc) {
                ZK_TRY(loop_spmv(A, hc.A, hc.p, s, part(k1_bicg<W, MODE, 3>), (const void*)k1_bicg<W, MODE, 3>));
            } else if (tail) {
                ZK_TRY(loop_spmv(A, hc.A, hc.p, s, part(k1_bicg<W, MODE, 2>), (const void*)k1_bicg<W, MODE, 2>));
            } else if (split) {
                ZK_TRY(loop_spmv(A, hc.A, hc.p, s, part(k1_bicg<W, MODE, 1>)));
                ZK_TRY(launch_loop(pdl, r1_bicg, vec_grid(A, (const void*)r1_bicg), 0, s, dc));
            } else {
                auto kf = k1_bicg<W, MODE, 0>;
                const LaunchCfg L = spmv_cfg(A, (const void*)kf, W, MODE);
                ZK_TRY(launch_loop(pdl, kf, L.grid, L.smem, s, dc, hc.A));
            }
            if (dist) ZK_TRY((dist_finish<S_K1_BICG>(A, dc, 3, s)));
            ZK_TRY(launch_loop(pdl, k2_bicg, vec_grid(A, (const void*)k2_bicg), 0, s, dc));
            if (dist) ZK_TRY((dist_finish<S_K2_BICG>(A, dc, 1, s)));
            if (wacc) {
                ZK_TRY(loop_spmv(A, hc.A, hc.s, s, part(k3_bicg<W, MODE, 3>), (const void*)k3_bicg<W, MODE, 3>));
            } else if (tail) {
                ZK_TRY(loop_spmv(A, hc.A, hc.s, s, part(k3_bicg<W, MODE, 2>), (const void*)k3_bicg<W, MODE, 2>));
            } else if (split) {
                ZK_TRY(loop_spmv(A, hc.A, hc.s, s, part(k3_bicg<W, MODE, 1>)));
                ZK_TRY(launch_loop(pdl, r3_bicg, vec_grid(A, (const void*)r3_bicg), 0, s, dc));
            } else {
                auto kf = k3_bicg<W, MODE, 0>;
                const LaunchCfg L = spmv_cfg(A, (const void*)kf, W, MODE);
                ZK_TRY(launch_loop(pdl, kf, L.grid, L.smem, s, dc, hc.A));
            }
            if (dist) ZK_TRY((dist_finish<S_K3_BICG>(A, dc, 3, s)));
            ZK_TRY(launch_loop(pdl, k4_bicg, vec_grid(A, (const void*)k4_bicg), 0, s, dc));
            if (dist) ZK_TRY((dist_finish<S_K4_BICG>(A, dc, 3, s)));
            ZK_TRY(launch_loop(pdl, k5_bicg, vec_grid(A, (const void*)k5_bicg), 0, s, dc));
        } else if (method == kBiCGStabL) {
            VecSet P;
            for (int q = 0; q <= hc.ell; q++) {
                P.r[q] = hc.rl[q];
                P.u[q] = hc.ul[q];
            }
            for (int q = hc.ell + 1; q <= kMaxEll; q++) P.r[q] = P.u[q] = nullptr;
            for (int j = 0; j < hc.ell; j++) {
                ZK_TRY(launch_loop(pdl, bl_b1, vec_grid(A, (const void*)bl_b1), 0, s, dc, P, j));
                if (split) {  // (distributed: always — interior / boundary launches around û_j's halo)
                    auto kf = bl_s1<W, MODE, false>;
                    ZK_TRY(loop_spmv(A, hc.A, P.u[j], s, [&](const CsrDev& a, bool is_part) -> zk_status {
                        const LaunchCfg L = is_part ? spmv_cfg_part(A, (const void*)kf, a) : spmv_cfg(A, (const void*)kf, W, MODE);
                        return launch_loop(pdl, kf, L.grid, L.smem, s, dc, a, P, j);
                    }));
                    auto kr = bl_r<S_S1_BL>;
                    ZK_TRY(launch_loop(pdl, kr, vec_grid(A, (const void*)kr), 0, s, dc, (const double2*)P.u[j + 1]));
                } else {
                    auto kf = bl_s1<W, MODE, true>;
                    const LaunchCfg L = spmv_cfg(A, (const void*)kf, W, MODE);
                    ZK_TRY(launch_loop(pdl, kf, L.grid, L.smem, s, dc, hc.A, P, j));
                }
                if (dist) ZK_TRY((dist_finish<S_S1_BL>(A, dc, 3, s)));
                ZK_TRY(launch_loop(pdl, bl_b2, vec_grid(A, (const void*)bl_b2), 0, s, dc, P, j));
                if (dist) ZK_TRY((dist_finish<S_B2_BL>(A, dc, 1, s)));
                if (j < hc.ell - 1 && !split) {
                    auto kf = bl_s2<W, MODE, true>;
                    const LaunchCfg L = spmv_cfg(A, (const void*)kf, W, MODE);
                    ZK_TRY(launch_loop(pdl, kf, L.grid, L.smem, s, dc, hc.A, P, j, 1));
                } else {
                    auto kf = bl_s2<W, MODE, false>;
                    const int stamp = j < hc.ell - 1 ? 1 : 0;
                    ZK_TRY(loop_spmv(A, hc.A, P.r[j], s, [&](const CsrDev& a, bool is_part) -> zk_status {
                        const LaunchCfg L = is_part ? spmv_cfg_part(A, (const void*)kf, a) : spmv_cfg(A, (const void*)kf, W, MODE);
                        return launch_loop(pdl, kf, L.grid, L.smem, s, dc, a, P, j, stamp);
                    }));
                    if (j < hc.ell - 1) {
                        auto kr = bl_r<S_S2_BL>;
                        ZK_TRY(launch_loop(pdl, kr, vec_grid(A, (const void*)kr), 0, s, dc, (const double2*)P.r[j + 1]));
                        if (dist) ZK_TRY((dist_finish<S_S2_BL>(A, dc, 3, s)));
                    }
                }
            }
            const BlKernel kg = bl_gram_of(hc.ell);
            int gg = A->dev.num_sms * blocks_per_sm((const void*)kg);
            const int gcap = kMaxRed * kMaxGrid / bl_nd(hc.ell);  // partials [ND][grid]
            if (gg > gcap) gg = gcap;
            ZK_TRY(launch_loop(pdl, kg, gg, 0, s, dc, P));
            if (dist) {  // the Gram totals over the ranks, then the (replicated) Cholesky
                ZK_TRY(dist_allreduce_ctx(A, dc->redg, bl_nd(hc.ell), s));
                fin_gram_of(hc.ell)<<<1, 1, 0, s>>>(dc);
                ZK_CUDA(cudaGetLastError());
            }
            const BlKernel ku = bl_u_of(hc.ell);
            ZK_TRY(launch_loop(pdl, ku, vec_grid(A, (const void*)ku), 0, s, dc, P));
            if (dist) ZK_TRY((dist_finish<S_U_BL>(A, dc, 3, s)));
        } else if (method == ZK_TFQMR) {
            ZK_TRY(launch_loop(pdl, t1_tfqmr, vec_grid(A, (const void*)t1_tfqmr), 0, s, dc));
            if (dist) ZK_TRY((dist_finish<S_T1_TFQMR>(A, dc, 1, s)));
            if (tail) {  // (a warp-reduced T2/T4 epilogue carries 2-3 operands: it spills at 80 registers)
                ZK_TRY(loop_spmv(A, hc.A, hc.y2, s, part(t2_tfqmr<W, MODE, 2>), (const void*)t2_tfqmr<W, MODE, 2>));
            } else if (split) {
                ZK_TRY(loop_spmv(A, hc.A, hc.y2, s, part(t2_tfqmr<W, MODE, 1>)));
                ZK_TRY(launch_loop(pdl, t2b_tfqmr, vec_grid(A, (const void*)t2b_tfqmr), 0, s, dc));
            } else {
                auto kf = t2_tfqmr<W, MODE, 0>;
                const LaunchCfg L = spmv_cfg(A, (const void*)kf, W, MODE);
                ZK_TRY(launch_loop(pdl, kf, L.grid, L.smem, s, dc, hc.A));
            }
            if (dist) ZK_TRY((dist_finish<S_T2_TFQMR>(A, dc, 3, s)));
            ZK_TRY(launch_loop(pdl, t3_tfqmr, vec_grid(A, (const void*)t3_tfqmr), 0, s, dc));
            if (tail) {
                ZK_TRY(loop_spmv(A, hc.A, hc.y1, s, part(t4_tfqmr<W, MODE, 2>), (const void*)t4_tfqmr<W, MODE, 2>));
            } else if (split) {
                ZK_TRY(loop_spmv(A, hc.A, hc.y1, s, part(t4_tfqmr<W, MODE, 1>)));
                ZK_TRY(launch_loop(pdl, t4b_tfqmr, vec_grid(A, (const void*)t4b_tfqmr), 0, s, dc));
            } else {
                auto kf = t4_tfqmr<W, MODE, 0>;
                const LaunchCfg L = spmv_cfg(A, (const void*)kf, W, MODE);
                ZK_TRY(launch_loop(pdl, kf, L.grid, L.smem, s, dc, hc.A));
            }
            if (dist) ZK_TRY((dist_finish<S_T4_TFQMR>(A, dc, 2, s)));
        } else if (method == ZK_COCG) {
            if (wacc) {
                ZK_TRY(loop_spmv(A, hc.A, hc.p, s, part(k1_cocg<W, MODE, 3>), (const void*)k1_cocg<W, MODE, 3>));
            } else if (tail) {
                ZK_TRY(loop_spmv(A, hc.A, hc.p, s, part(k1_cocg<W, MODE, 2>), (const void*)k1_cocg<W, MODE, 2>));
            } else if (split) {
                ZK_TRY(loop_spmv(A, hc.A, hc.p, s, part(k1_cocg<W, MODE, 1>)));
                auto kr = rq_kernel<false, S_K1_COCG>;
                ZK_TRY(launch_loop(pdl, kr, vec_grid(A, (const void*)kr), 0, s, dc));
            } else {
                auto kf = k1_cocg<W, MODE, 0>;
                const LaunchCfg L = spmv_cfg(A, (const void*)kf, W, MODE);
                ZK_TRY(launch_loop(pdl, kf, L.grid, L.smem, s, dc, hc.A));
            }
            if (dist) ZK_TRY((dist_finish<S_K1_COCG>(A, dc, 2, s)));
            ZK_TRY(launch_loop(pdl, k2_cocg, vec_grid(A, (const void*)k2_cocg), 0, s, dc));
            if (dist) ZK_TRY((dist_finish<S_K2_COCG>(A, dc, 3, s)));
            ZK_TRY(launch_loop(pdl, k3_cocg, vec_grid(A, (const void*)k3_cocg), 0, s, dc));
        } else {
            if (wacc) {
                ZK_TRY(loop_spmv(A, hc.A, hc.p, s, part(k1_cg<W, MODE, 3>), (const void*)k1_cg<W, MODE, 3>));
            } else if (tail) {
                ZK_TRY(loop_spmv(A, hc.A, hc.p, s, part(k1_cg<W, MODE, 2>), (const void*)k1_cg<W, MODE, 2>));
            } else if (split) {
                ZK_TRY(loop_spmv(A, hc.A, hc.p, s, part(k1_cg<W, MODE, 1>)));
                auto kr = rq_kernel<true, S_K1_CG>;
                ZK_TRY(launch_loop(pdl, kr, vec_grid(A, (const void*)kr), 0, s, dc));
            } else {
                auto kf = k1_cg<W, MODE, 0>;
                const LaunchCfg L = spmv_cfg(A, (const void*)kf, W, MODE);
                ZK_TRY(launch_loop(pdl, kf, L.grid, L.smem, s, dc, hc.A));
            }
            if (dist) ZK_TRY((dist_finish<S_K1_CG>(A, dc, 2, s)));
            ZK_TRY(launch_loop(pdl, k2_cg, vec_grid(A, (const void*)k2_cg), 0, s, dc));
            if (dist) ZK_TRY((dist_finish<S_K2_CG>(A, dc, 1, s)));
            ZK_TRY(launch_loop(pdl, k3_cg, vec_grid(A, (const void*)k3_cg), 0, s, dc));
        }
        return ZK_OK;
    });
}

static void drop_graph(GraphCache& g) {
    if (g.exec) cudaGraphExecDestroy(g.exec);
    if (g.graph) cudaGraphDestroy(g.graph);
    g = GraphCache{};
}

// WHILE-node graph: body = one iteration; condition written by the last kernel of the body.
// Iterations per WHILE-graph body: the conditional node's per-body cost is paid once per
// kWhileUnroll iterations; an exit inside a body leaves at most kWhileUnroll − 1 iterations of
// early-returning kernels.  Measured (tools/ab_unroll.sh, µs per iteration, 1 → 4): Audi3D-4 (C3)
// BiCGStab 148.9 → 147.5, CG 74.2 → 72.2, TFQMR 154.0 → 152.3; Twingo3D-2 116.4 → 114.3, 58.1 →
// 56.2 (profiles/r02_while_unroll_ab.txt).  ZK_WHILE_UNROLL overrides.
constexpr int kWhileUnroll = 4;
static zk_status build_while_graph(zk_csr_s* A, SolveCtx* dc, const SolveCtx& hc, int method, GraphCache& g,
                                   bool pdl) {
    cudaGraph_t graph = nullptr;
    ZK_CUDA(cudaGraphCreate(&graph, 0));
    cudaGraphConditionalHandle h;
    cudaError_t e = cudaGraphConditionalHandleCreate(&h, graph, 1, cudaGraphCondAssignDefault);
    if (e != cudaSuccess) {
        cudaGraphDestroy(graph);
        return cuda_fail(e, "cudaGraphConditionalHandleCreate", __FILE__, __LINE__);
    }
    alignas(cudaGraphNodeParams) unsigned char cp_raw[sizeof(cudaGraphNodeParams)];
    memset(cp_raw, 0, sizeof cp_raw);
    cudaGraphNodeParams& cp = *reinterpret_cast<cudaGraphNodeParams*>(cp_raw);
    cp.type = cudaGraphNodeTypeConditional;
    cp.conditional.handle = h;
    cp.conditional.type = cudaGraphCondTypeWhile;
    cp.conditional.size = 1;
    cudaGraphNode_t node;
    e = cudaGraphAddNode(&node, graph, nullptr, 0, &cp);
    if (e != cudaSuccess) {
        cudaGraphDestroy(graph);
        return cuda_fail(e, "cudaGraphAddNode(conditional)", __FILE__, __LINE__);
    }
    cudaGraph_t body = cp.conditional.phGraph_out[0];
    e = cudaStreamBeginCaptureToGraph(A->cap_stream, body, nullptr, nullptr, 0, cudaStreamCaptureModeRelaxed);
    if (e != cudaSuccess) {
        cudaGraphDestroy(graph);
        return cuda_fail(e, "cudaStreamBeginCaptureToGraph", __FILE__, __LINE__);
    }
    static const int unroll = getenv("ZK_WHILE_UNROLL") ? std::max(1, atoi(getenv("ZK_WHILE_UNROLL"))) : kWhileUnroll;
    zk_status st = ZK_OK;
    for (int u = 0; u < unroll && st == ZK_OK; u++) st = enqueue_iteration(A, dc, hc, method, A->cap_stream, pdl);
    cudaGraph_t captured = nullptr;
    e = cudaStreamEndCapture(A->cap_stream, &captured);
    if (st != ZK_OK || e != cudaSuccess) {
        cudaGraphDestroy(graph);
        return st != ZK_OK ? st : cuda_fail(e, "cudaStreamEndCapture", __FILE__, __LINE__);
    }
    e = cudaGraphInstantiate(&g.exec, graph, 0);
    if (e != cudaSuccess) {
        cudaGraphDestroy(graph);
        g.exec = nullptr;
        return cuda_fail(e, "cudaGraphInstantiate(while)", __FILE__, __LINE__);
    }
    g.graph = graph;
    g.cond = (unsigned long long)h;
    return ZK_OK;
}

constexpr int kChunk = 16;

// plain graph of kChunk iterations (kernels early-exit once done)
static zk_status build_chunk_graph(zk_csr_s* A, SolveCtx* dc, const SolveCtx& hc, int method, GraphCache& g) {
    ZK_CUDA(cudaStreamBeginCapture(A->cap_stream, cudaStreamCaptureModeRelaxed));
    zk_status st = ZK_OK;
    for (int i = 0; i < kChunk && st == ZK_OK; i++) st = enqueue_iteration(A, dc, hc, method, A->cap_stream);
    cudaGraph_t graph = nullptr;
    cudaError_t e = cudaStreamEndCapture(A->cap_stream, &graph);
    if (st != ZK_OK) {
        if (graph) cudaGraphDestroy(graph);
        return st;
    }
    if (e != cudaSuccess) return cuda_fail(e, "cudaStreamEndCapture(chunk)", __FILE__, __LINE__);
    e = cudaGraphInstantiate(&g.exec, graph, 0);
    if (e != cudaSuccess) {
        cudaGraphDestroy(graph);
        return cuda_fail(e, "cudaGraphInstantiate(chunk)", __FILE__, __LINE__);
    }
    g.graph = graph;
    return ZK_OK;
}

struct WsLayout {
    size_t ctx, partials, tickets, hist, vec0, vec_bytes, total;
    int nvec;
};
static size_t up256(size_t v) { return (v + 255) & ~(size_t)255; }
int64_t dist_gather_len(const zk_csr_s* A);  // dist.cu: n_rows + halo slots

static WsLayout ws_layout(const zk_csr_s* A, int method, int32_t maxit, int ell = 0) {
    WsLayout L;
    size_t off = 0;
    L.ctx = off;  // ctx and hist adjacent: the exit readback is one copy
    off += sizeof(SolveCtx);
    L.hist = off;
    off += up256(sizeof(SolveCtx) + sizeof(double) * ((size_t)(maxit > 0 ? maxit : 0) + 1)) - sizeof(SolveCtx);
    L.partials = off;
    off += up256(sizeof(double) * kMaxRed * kMaxGrid);
    L.tickets = off;
    off += up256(sizeof(unsigned int) * kTickets);
    L.vec0 = off;
    const int64_t len = A->dist ? dist_gather_len(A) : A->n_rows;
    L.vec_bytes = up256(sizeof(double2) * (size_t)(len > 0 ? len : 1));
    // BiCGStab: r r̂ p v s t (+ xg gather copy on >1 GPU) ; CG/COCG: r p q (+ xg) ;
    // TFQMR: w y1 y2 u1 u2 v d r̃ (+ xg)
    // BiCGStab(ℓ): r̂_0..ℓ û_0..ℓ r̃
    L.nvec = (method == ZK_BICGSTAB ? 6 : method == ZK_TFQMR ? 8 : method == kBiCGStabL ? 2 * ell + 3 : 3) +
             (A->dist ? 1 : 0);
    off += L.vec_bytes * L.nvec;
    L.total = off;
    return L;
}

}  // namespace zk

using namespace zk;

// method code → (internal method, ℓ); false for an unknown code
static bool decode_method(int32_t code, int* method, int* ell) {
    *ell = 0;
    if (code >= ZK_BICGSTAB && code <= ZK_TFQMR) {
        *method = code;
        return true;
    }
    if (code >= ZK_BICGSTAB_L(1) && code <= ZK_BICGSTAB_L(kMaxEll)) {
        *method = kBiCGStabL;
        *ell = code - ZK_BICGSTAB_L(0);
        return true;
    }
    return false;
}

extern "C" size_t zk_solve_workspace_size(zk_csr A, int32_t code, int32_t maxit) {
    int method, ell;
    if (!A || !decode_method(code, &method, &ell)) return 0;
    if (method == ZK_BICGSTAB_JACOBI) method = ZK_BICGSTAB;
    return ws_layout(A, method, maxit, ell).total;
}

extern "C" zk_status zk_solve(zk_csr A, const zk_z* b, const zk_z* x0, double tol, int32_t maxit, int32_t code,
                              zk_z* x, int32_t* iters, double* resid_hist, zk_solve_info* info, void* workspace,
                              size_t ws_bytes, zk_stream stream) {
    static const bool trace = getenv("ZK_TRACE") != nullptr;  // host-side phase times on stderr
    const auto tr0 = std::chrono::steady_clock::now();
    if (!A || !b || !x || !iters || !resid_hist || !workspace) return fail(ZK_ERR_INVALID_VALUE, "NULL argument");
    int method, ell;
    if (!decode_method(code, &method, &ell)) return fail(ZK_ERR_INVALID_VALUE, "unknown method");
    const bool jacobi = method == ZK_BICGSTAB_JACOBI;
    if (jacobi) {
        ZK_TRY(jacobi_prepare(A, (cudaStream_t)stream));  // A·M⁻¹ built once, cached in the handle
        method = ZK_BICGSTAB;
    }
    if (!(tol > 0.0)) return fail(ZK_ERR_INVALID_VALUE, "tol must be > 0");
    if (maxit < 1) return fail(ZK_ERR_INVALID_VALUE, "maxit must be >= 1");
    if (A->n_cols != A->n_global) return fail(ZK_ERR_DIM, "solve needs a square matrix");
    if ((const void*)b == (const void*)x) return fail(ZK_ERR_ALIAS, "b aliases x");
    if (((uintptr_t)workspace & 255u) != 0) return fail(ZK_ERR_INVALID_VALUE, "workspace must be 256-B aligned");
    const WsLayout L = ws_layout(A, method, maxit, ell);
    if (ws_bytes < L.total) return fail(ZK_ERR_INVALID_VALUE, "workspace too small");
    if (A->n_rows == 0 && !A->dist) return fail(ZK_ERR_ZERO_RHS, "empty system (||b|| = 0)");
    cudaStream_t s = (cudaStream_t)stream;
    char* ws = (char*)workspace;

    SolveCtx* dc = (SolveCtx*)(ws + L.ctx);
    SolveCtx hc;
    memset(&hc, 0, sizeof hc);
    hc.x = (double2*)x;
    hc.b = (const double2*)b;
    hc.partials = (double*)(ws + L.partials);
    hc.tickets = (unsigned int*)(ws + L.tickets);
    hc.hist = (double*)(ws + L.hist);
    double2* vec[2 * kMaxEll + 4];
    for (int i = 0; i < L.nvec; i++) vec[i] = (double2*)(ws + L.vec0 + L.vec_bytes * i);
    if (method == ZK_BICGSTAB) {
        hc.r = vec[0]; hc.rh = vec[1]; hc.p = vec[2]; hc.v = vec[3]; hc.s = vec[4]; hc.t = vec[5];
    } else if (method == ZK_TFQMR) {
        hc.w = vec[0]; hc.y1 = vec[1]; hc.y2 = vec[2]; hc.u1 = vec[3]; hc.u2 = vec[4]; hc.v = vec[5];
        hc.d = vec[6]; hc.rt = vec[7];
        hc.r = hc.w; hc.p = hc.y1; hc.rh = hc.rt;  // the shared init writes r0 into w, y1 and r̃
    } else if (method == kBiCGStabL) {
        for (int q = 0; q <= ell; q++) {
            hc.rl[q] = vec[q];
            hc.ul[q] = vec[ell + 1 + q];
        }
        hc.rh = vec[2 * ell + 2];  // r̃
        hc.r = hc.rl[0];           // the shared init writes r0 into r̂_0, r̃ (and û_1, overwritten later)
        hc.p = hc.ul[1];
        hc.d = hc.ul[0];           // û_0 = 0
        hc.ell = ell;
    } else {
        hc.r = vec[0]; hc.p = vec[1]; hc.q = vec[2];
    }
    double2* xg = A->dist ? vec[L.nvec - 1] : nullptr;  // gather copy of x0 / x with halo slots
    hc.A = csr_dev(A);
    if (jacobi) {  // iterate on A' = A·M⁻¹ (u = M x)
        hc.A.val = A->jac_val;
        hc.A.sl_val = A->jac_sl_val;
    }
    hc.tol = tol;
    hc.maxit = maxit;
    hc.status = ZK_MAXIT;
    hc.true_relres = NAN;
    hc.dist = A->dist ? 1 : 0;
    for (int i = 0; i < 4; i++) hc.t0[i] = ~0ull;

    // ---- loop mode: 1 = WHILE graph (default), 2 = chunked graphs, 3 = direct launches,
    //      5 = the whole loop in one thread-block cluster (default for small systems whose own rows
    //      fit the cluster's shared memory, see cluster_fits).  (A round-1 mode 4, one persistent
    //      cooperative kernel with grid barriers, measured slower on every shape — C1 52 vs 39 µs
    //      per iteration, C3 514 vs 184 — and was removed.)
    int mode = A->dist ? 3 : (cluster_kind(method) >= 0 && A->n_rows <= kClusterDefaultRows ? 5 : 1);
    if (const char* e = getenv("ZK_LOOP_MODE")) {
        int m = atoi(e);
        if (m >= 1 && m <= 5 && m != 4) mode = m;
    }
    if (mode == 5 && (A->dist || !cluster_fits(A, (cudaStream_t)stream, cluster_kind(method), ell)))
        mode = A->dist ? 3 : 1;
    if (A->dist && (mode == 1 || mode == 5)) mode = 3;  // collectives inside WHILE bodies / clusters are not used
    static_assert(kBiCGStabL < (int)(sizeof(((zk_csr_s*)nullptr)->graph) / sizeof(GraphCache)), "graph slot per method");
    // one graph per (method, ℓ, Jacobi) — Jacobi-BiCGStab in its own slot (the ABI's method code), so
    // alternating plain and Jacobi solves on one handle do not rebuild each other's graph; the SpMV
    // kernels take the CSR view (A or A·M⁻¹) as a launch parameter baked into the graph
    GraphCache& gc = A->graph[jacobi ? (int)ZK_BICGSTAB_JACOBI : method];
    const int gkey = ((method * 16 + ell) * 2 + (jacobi ? 1 : 0)) * 4 + tail_kind(A);
    // key: workspace pointer, loop mode, method/ℓ/Jacobi and maxit (ws_layout places the partials,
    // tickets and vectors after hist[maxit+1]; BiCGStab(ℓ) bakes its vector pointers into the graph)
    if (mode <= 2 && (gc.ws != workspace || gc.mode != mode || gc.method != gkey || gc.maxit != maxit || !gc.exec)) {
        drop_graph(gc);
        const bool pdl = !(getenv("ZK_PDL") && atoi(getenv("ZK_PDL")) == 0);
        zk_status st = mode == 1 ? build_while_graph(A, dc, hc, method, gc, pdl) : build_chunk_graph(A, dc, hc, method, gc);
        if (st != ZK_OK && mode == 1 && pdl) {  // PDL edges inside the WHILE body unavailable: retry without
            drop_graph(gc);
            st = build_while_graph(A, dc, hc, method, gc, false);
        }
        if (st != ZK_OK && mode == 1) {  // conditional nodes unavailable: fall back to chunked graphs
            drop_graph(gc);
            mode = 2;
            st = build_chunk_graph(A, dc, hc, method, gc);
        }
        if (st != ZK_OK) {
            drop_graph(gc);
            mode = 3;
        } else {
            gc.ws = workspace;
            gc.mode = mode;
            gc.method = gkey;
            gc.maxit = maxit;
        }
    }
    hc.use_cond = mode == 1 ? 1 : 0;
    hc.cond = mode == 1 ? gc.cond : 0ull;

    for (auto& e : A->ev)
        if (!e) ZK_CUDA(cudaEventCreate(&e));
    cudaEvent_t ev0 = A->ev[0], ev1 = A->ev[1];
    const size_t rb_bytes = sizeof(SolveCtx) + sizeof(double) * ((size_t)maxit + 1);
    if (A->pinned_bytes < rb_bytes) {  // pinned readback staging, grown on demand
        pinned_put(A->pinned, A->pinned_bytes);  // (process-wide free list, api.cu)
        A->pinned = nullptr;
        A->pinned_bytes = 0;
        ZK_CUDA(pinned_get(&A->pinned, rb_bytes, &A->pinned_bytes));
    }
    // mode 5 from x0 = 0: the cluster kernel sets up the context and r0 itself (and TFQMR's K0) —
    // one launch per solve; ZK_CLUSTER_INIT=0 launches k_set_ctx + k_init_zero (+ k0_tfqmr) first
    const bool fused_init = mode == 5 && !x0 && !(getenv("ZK_CLUSTER_INIT") && atoi(getenv("ZK_CLUSTER_INIT")) == 0);
    // zero-copy readback (cluster solve from x0 = 0, no Jacobi exit work after it): the kernel writes
    // the context and the history into the pinned staging itself — no D2H copy after the kernel
    // (C1 fixed cost 63.7 → 55.5 µs, C2 86 → 76); ZK_ZERO_COPY=0 keeps the copy
    bool zero_copy = mode == 5 && fused_init && !jacobi && !(getenv("ZK_ZERO_COPY") && atoi(getenv("ZK_ZERO_COPY")) == 0);
    if (zero_copy) {
        void* dp = nullptr;
        if (cudaHostGetDevicePointer(&dp, A->pinned, 0) == cudaSuccess && dp) {
            hc.out_host = (SolveCtx*)dp;
            hc.hist_host = (double*)((char*)dp + sizeof(SolveCtx));
        } else {
            cudaGetLastError();
            zero_copy = false;
        }
    }
    ZK_CUDA(cudaEventRecord(ev0, s));
    const auto tr1 = std::chrono::steady_clock::now();
    int64_t n_spmv = 0;

    // ---- init: context, r0 = b − A x0 (or b), ‖b‖, hist[0]
    // (mode 5 from x0 = 0: the cluster kernel does both itself — and TFQMR's K0 — one launch per
    // solve, fused_init above)
    if (!fused_init) {
        k_set_ctx<<<1, 1, 0, s>>>(dc, hc);
        ZK_CUDA(cudaGetLastError());
    }
    const int kind = method == ZK_BICGSTAB ? 0 : method == ZK_CG ? 1 : method == ZK_COCG ? 3 : method == ZK_TFQMR ? 4 : 5;
    if (x0) {
        const double2* g0 = (const double2*)x0;
        if (jacobi) {  // u0 = M x0, in the output buffer (x may alias x0)
            ZK_TRY(cscale(A, A->jac_diag, (const double2*)x0, (double2*)x, s));
            g0 = (const double2*)x;
        }
        if (A->dist) {
            ZK_CUDA(cudaMemcpyAsync(xg, x0, sizeof(double2) * A->n_rows, cudaMemcpyDeviceToDevice, s));
            ZK_TRY(dist_halo(A, xg, s));
            g0 = xg;
        }
        ZK_TRY(with_spmv(A, [&](auto wc, auto mc) -> zk_status {
            constexpr int W = decltype(wc)::value, MODE = decltype(mc)::value;
            if (kind == 0) {
                auto k = k_init_x0<W, MODE, S_INIT_BICG>;
                const LaunchCfg L = spmv_cfg(A, (const void*)k, W, MODE);
                k<<<L.grid, kBlock, L.smem, s>>>(dc, g0, 1);
            } else if (kind == 1) {
                auto k = k_init_x0<W, MODE, S_INIT_CG>;
                const LaunchCfg L = spmv_cfg(A, (const void*)k, W, MODE);
                k<<<L.grid, kBlock, L.smem, s>>>(dc, g0, 0);
            } else if (kind == 3) {
                auto k = k_init_x0<W, MODE, S_INIT_COCG>;
                const LaunchCfg L = spmv_cfg(A, (const void*)k, W, MODE);
                k<<<L.grid, kBlock, L.smem, s>>>(dc, g0, 0);
            } else if (kind == 4) {
                auto k = k_init_x0<W, MODE, S_INIT_TFQMR>;
                const LaunchCfg L = spmv_cfg(A, (const void*)k, W, MODE);
                k<<<L.grid, kBlock, L.smem, s>>>(dc, g0, 1);
            } else {
                auto k = k_init_x0<W, MODE, S_INIT_BL>;
                const LaunchCfg L = spmv_cfg(A, (const void*)k, W, MODE);
                k<<<L.grid, kBlock, L.smem, s>>>(dc, g0, 1);
            }
            ZK_CUDA(cudaGetLastError());
            return ZK_OK;
        }));
        n_spmv++;
    } else if (!fused_init) {
        k_init_zero<<<vec_grid(A, (const void*)k_init_zero), kBlock, 0, s>>>(dc, kind);
        ZK_CUDA(cudaGetLastError());
    }
    if (A->dist)
        ZK_TRY(kind == 0   ? dist_finish<S_INIT_BICG>(A, dc, 4, s)
               : kind == 1 ? dist_finish<S_INIT_CG>(A, dc, 4, s)
               : kind == 3 ? dist_finish<S_INIT_COCG>(A, dc, 4, s)
               : kind == 4 ? dist_finish<S_INIT_TFQMR>(A, dc, 4, s)
                           : dist_finish<S_INIT_BL>(A, dc, 4, s));
    if (method == ZK_TFQMR && fused_init) n_spmv++;  // K0 inside the cluster kernel
    if (method == ZK_TFQMR && !fused_init) {  // u1 = v = A y1 and σ = ⟨r̃, v⟩ → α for iteration 1
        if (A->dist) ZK_TRY(dist_halo(A, hc.y1, s));
        ZK_TRY(with_spmv(A, [&](auto wc, auto mc) -> zk_status {
            constexpr int W = decltype(wc)::value, MODE = decltype(mc)::value;
            auto k = k0_tfqmr<W, MODE>;
            const LaunchCfg L = spmv_cfg(A, (const void*)k, W, MODE);
            k<<<L.grid, kBlock, L.smem, s>>>(dc, hc.A);
            ZK_CUDA(cudaGetLastError());
            return ZK_OK;
        }));
        if (A->dist) ZK_TRY(dist_finish<S_K0_TFQMR>(A, dc, 2, s));
        n_spmv++;
    }

    // ---- the loop
    SolveCtx* hdone = nullptr;  // pinned copy of the ctx for the chunked modes
    if (mode == 1) {
        ZK_CUDA(cudaGraphLaunch(gc.exec, s));
    } else if (mode == 5) {
        int csz = 0;
        if (!cluster_launch(A, dc, hc, hc.A, s, &csz, cluster_kind(method), ell, !jacobi, fused_init))  // + true residual
            return fail(ZK_ERR_CUDA, "cluster solver launch failed");
    } else {
        hdone = (SolveCtx*)A->pinned;  // the handle's pinned staging (no per-solve cudaMallocHost)
        int launched = 0;
        const int chunk = mode == 2 ? kChunk : 4;
        for (;;) {
            if (mode == 2) {
                cudaError_t e = cudaGraphLaunch(gc.exec, s);
                if (e != cudaSuccess) return cuda_fail(e, "cudaGraphLaunch", __FILE__, __LINE__);
            } else {
                for (int i = 0; i < chunk; i++) {
                    zk_status st = enqueue_iteration(A, dc, hc, method, s);
                    if (st != ZK_OK) return st;
                }
            }
            launched += chunk;
            cudaError_t e = cudaMemcpyAsync(hdone, dc, sizeof(SolveCtx), cudaMemcpyDeviceToHost, s);
            if (e == cudaSuccess) e = cudaStreamSynchronize(s);
            if (e != cudaSuccess) return cuda_fail(e, "loop poll", __FILE__, __LINE__);
            if (hdone->done || launched > maxit + 1) break;
        }
    }

    // ---- exit: true relative residual ‖b − A x‖/‖b‖ (one more SpMV)
    if (jacobi) ZK_TRY(cscale(A, A->jac_dinv, (const double2*)x, (double2*)x, s));  // x = M⁻¹ u
    const double2* gx = (const double2*)x;
    if (A->dist) {
        ZK_CUDA(cudaMemcpyAsync(xg, x, sizeof(double2) * A->n_rows, cudaMemcpyDeviceToDevice, s));
        ZK_TRY(dist_halo(A, xg, s));
        gx = xg;
    }
    if (!(mode == 5 && !jacobi))  // mode 5 formed it inside the cluster kernel (Jacobi: on the original A here)
        ZK_TRY(with_spmv(A, [&](auto wc, auto mc) -> zk_status {
            constexpr int W = decltype(wc)::value, MODE = decltype(mc)::value;
            { auto kf = k_true<W, MODE>; const LaunchCfg L = spmv_cfg(A, (const void*)kf, W, MODE); kf<<<L.grid, kBlock, L.smem, s>>>(dc, gx, csr_dev(A)); }
            ZK_CUDA(cudaGetLastError());
            return ZK_OK;
        }));
    if (A->dist) ZK_TRY(dist_finish<S_TRUE>(A, dc, 1, s));
    ZK_CUDA(cudaEventRecord(ev1, s));

    SolveCtx out;
    double* hist_pinned = (double*)((char*)A->pinned + sizeof(SolveCtx));
    static_assert(sizeof(SolveCtx) % sizeof(double) == 0, "hist follows the ctx");
    const auto tr2 = std::chrono::steady_clock::now();
    if (!zero_copy) ZK_CUDA(cudaMemcpyAsync(A->pinned, dc, rb_bytes, cudaMemcpyDeviceToHost, s));  // ctx + hist
    cudaError_t e = cudaStreamSynchronize(s);
    const auto tr3 = std::chrono::steady_clock::now();
    if (e != cudaSuccess) return cuda_fail(e, "zk_solve", __FILE__, __LINE__);
    memcpy(&out, A->pinned, sizeof(SolveCtx));
    memcpy(resid_hist, hist_pinned, sizeof(double) * ((size_t)maxit + 1));
    float ms = 0.f;
    cudaEventElapsedTime(&ms, ev0, ev1);

    *iters = out.iters;
    const int passes = out.iters;
    n_spmv += (int64_t)passes * (method == ZK_BICGSTAB || method == ZK_TFQMR ? 2 : method == kBiCGStabL ? 2 * ell : 1) + 1;
    if (info) {
        info->status = out.status == ST_ZERO_RHS ? ZK_CONVERGED : out.status;
        info->iters = out.iters;
        info->true_relres = out.true_relres;
        info->n_spmv = n_spmv;
        info->solve_ms = ms;
        info->loop_mode = mode;
        int per_body = method == ZK_BICGSTAB ? 5 : method == ZK_TFQMR ? 4 : method == kBiCGStabL ? 4 * ell + 2 : 3;
        if (split_reductions(A)) {  // the separate reduction / update passes
            if (method == kBiCGStabL)  // (no tail variant: a warp-reduced S1/S2 measured slower at C4,
                per_body += 2 * ell - 1;  // BiCGStab(8) 16.86 → 17.20 ms per cycle)
            else if (!split_tail(A))
                per_body += method == ZK_BICGSTAB ? 2 : (method == ZK_CG || method == ZK_COCG) ? 1 : 2;
        }
        const int fins = !A->dist ? 0 : method == ZK_BICGSTAB ? 4 : method == ZK_TFQMR ? 3
                       : method == kBiCGStabL ? 3 * ell + 1 : 2;  // dist: 1-thread finish kernels
        const int pre = method == ZK_TFQMR && !fused_init ? (A->dist ? 2 : 1) : 0;               // TFQMR: K0 (+ its finish)
        // mode 5: set_ctx + init (+ TFQMR's K0) + the cluster kernel (+ Jacobi: x = M⁻¹u and k_true)
        info->gpu_launches = mode == 5 ? (fused_init ? 1 : 3) + pre + (jacobi ? 2 : 0)
                                                       : 3 + pre + out.bodies * (per_body + fins) + (A->dist ? 2 : 0);
        if (A->dist) {  // + per SpMV: pack kernel, second (boundary) launch; + per allreduce: LOCAL sum kernel
            int per_spmv = 0, per_red = 0;
            dist_launch_extra(A, &per_spmv, &per_red);
            const int spmv_it = (method == ZK_BICGSTAB || method == ZK_TFQMR) ? 2 : method == kBiCGStabL ? 2 * ell : 1;
            const int red_it = fins;
            const int init_spmv = (x0 ? 1 : 0) + (method == ZK_TFQMR ? 1 : 0) + 1;  // + final true residual
            const int init_red = 2 + (method == ZK_TFQMR ? 1 : 0);
            info->gpu_launches += out.bodies * (spmv_it * per_spmv + red_it * per_red) + init_red * per_red +
                                  init_spmv * (per_spmv > 0 && dist_n_send(A) ? 1 : 0);
        }
        for (int i = 0; i < 4; i++) {
            info->kernel_ms[i] = out.tsum[i] * 1e-6;
            info->kernel_launches[i] = out.tcnt[i];
        }
    }
    if (trace) {
        auto us = [](auto a, auto b) { return std::chrono::duration<double, std::micro>(b - a).count(); };
        fprintf(stderr, "zk_solve: setup %.1f us, enqueue %.1f us, readback+sync %.1f us, rest %.1f us (device %.1f us, mode %d)\n",
                us(tr0, tr1), us(tr1, tr2), us(tr2, tr3), us(tr3, std::chrono::steady_clock::now()), 1e3 * ms, mode);
    }
    if (out.status == ST_ZERO_RHS) return fail(ZK_ERR_ZERO_RHS, "||b|| = 0 (S:361)");
    return ZK_OK;
}
