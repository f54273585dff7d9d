// solve_ctx.cuh — what the solver loops (solve.cu) and the single-cluster solvers (cluster.cu)
// share: the device-resident solve context, the per-method scalar steps (oracle O6/O7 and the NEXT
// rows' steps, line by line, run by one thread: PAPER.md §4, SPEC S:361-392 for the
// tests and breakdowns, DESIGN.md §4 R5-R18 for the readings), the BiCGStab(ℓ) Gram/Cholesky step
// (R18), and the cluster solver's host entry points.  See solve.cu's header for the schedules.
#pragma once
#include <cuda_runtime.h>

#include <cooperative_groups.h>

#include "spmv.cuh"
#include "zk_host.h"

namespace zk {

enum { ST_ZERO_RHS = 7 };  // internal outcome → ZK_ERR_ZERO_RHS at the ABI
constexpr int kTickets = 64;  // workspace ticket slots (256 B)
constexpr int kMaxEll = 8;    // BiCGStab(ℓ): ℓ ≤ 8
constexpr int kBiCGStabL = 5; // internal method id of ZK_BICGSTAB_L(ℓ)

struct SolveCtx {
    // vectors (device)
    double2* x;
    const double2* b;
    double2 *r, *rh, *p, *v, *s, *t, *q;
    double2 *w, *y1, *y2, *u1, *u2, *d, *rt;  // TFQMR (r/p/rh alias w/y1/rt for the shared init)
    double2 *rl[kMaxEll + 1], *ul[kMaxEll + 1];      // BiCGStab(ℓ) r̂_0..ℓ, û_0..ℓ (r/rh alias r̂_0/r̃)
    double* hist;
    double* partials;       // [kMaxRed][kMaxGrid]
    unsigned int* tickets;  // [kTickets], one per reduction stage (self-resetting; cleared at solve start)
    CsrDev A;
    // scalars
    double2 rho, alpha, omega, beta;
    double nb, nrh, rnorm, gamma, alpha_cg, beta_cg;
    double2 eta, eta1, coef1, coef2;  // TFQMR η (η1: first half step's) and the d coefficients (θ²/α)·η
    double theta, tau;      // TFQMR θ, τ
    double2 gam[kMaxEll + 1];  // BiCGStab(ℓ) minimal-residual coefficients γ_1..ℓ
    int ell;
    double tol;
    int maxit;
    int j;       // iteration being executed (1-based)
    int done;    // loop finished (any outcome)
    int half;    // BiCGStab half-step exit pending (K4 applies x += αp); TFQMR exit inside an
                 // iteration: 1 → T2 applies x += η1·d1 only, 2 → T3 applies its d, x updates only
    int status;  // ZK_CONVERGED ... / ST_ZERO_RHS
    int iters;
    double true_relres;
    unsigned long long cond;  // cudaGraphConditionalHandle of the WHILE node
    int use_cond;
    int dist;                 // multi-GPU: last blocks publish red[] for an NCCL allreduce
    double red[kMaxRed];
    double redg[96];          // multi-GPU BiCGStab(ℓ): the Gram totals (≤ 81 doubles) for the allreduce
    int bodies;               // loop bodies executed (counts launches for zk_solve_info)
    // zero-copy readback of a cluster solve (zk_solve, loop mode 5 from x0 = 0): CTA 0 writes the
    // final context and hist[0..iters] straight into the handle's pinned staging (device-mapped)
    SolveCtx* out_host;
    double* hist_host;
    // in-loop kernel timers (device global timer): per class, min block start of the running
    // launch, summed durations and launch counts (zk_solve_info.kernel_ms)
    unsigned long long t0[4];
    unsigned long long tsum[4];
    int tcnt[4];
};

__device__ __forceinline__ unsigned long long gtimer() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}

// Programmatic dependent launch: the loop kernels are launched with the PDL attribute so the
// next kernel's blocks are scheduled while the previous one drains; each waits for the previous
// grid's completion (and memory) before touching the context.  No-ops without the attribute.
__device__ __forceinline__ void pdl_enter() {
    asm volatile("griddepcontrol.wait;" ::: "memory");
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}

// Opposite sweeps: a streaming kernel of a solver loop that walks its rows last to
// first starts on the rows its predecessor (a first-to-last sweep) touched last — the lines still
// in L2 (126 MB against 128 MB per vector at C4; a same-direction sweep finds the oldest lines of
// the previous sweep evicted first).  Fixed per kernel: BiCGStab K2 and K4, CG/COCG K2 and
// TFQMR T2/T4 run backwards, the rest forwards (an odd kernel count per iteration leaves one
// same-direction boundary: BiCGStab K5 → K1, CG K3 → K1).  -DZK_SWEEP=0 makes every sweep forward.
#ifndef ZK_SWEEP
#define ZK_SWEEP 1
#endif
constexpr bool kSweep = ZK_SWEEP != 0;

__device__ __forceinline__ void set_cond(SolveCtx* c) {
    if (blockIdx.x == 0 && threadIdx.x == 0) {
        c->bodies += 1;
        if (c->use_cond) cudaGraphSetConditional((cudaGraphConditionalHandle)c->cond, c->done ? 0u : 1u);
    }
}

// ------------------------------------------------------------------ scalar steps (one thread)
// Each follows oracle O6/O7 line by line (same tests, same order, same complex division).
__device__ inline void fin_init_bicg(SolveCtx* c, const double* tot) {  // tot = {‖b‖², ‖r0‖²}
    c->iters = 0;
    c->nb = sqrt(tot[0]);
    if (c->nb == 0.0) { c->status = ST_ZERO_RHS; c->done = 1; return; }
    c->rnorm = sqrt(tot[1]);
    c->hist[0] = c->rnorm / c->nb;
    if (!isfinite(c->hist[0])) { c->status = ZK_NONFINITE; c->done = 1; return; }
    if (c->hist[0] <= c->tol) { c->status = ZK_CONVERGED; c->done = 1; return; }
    c->nrh = c->rnorm;                           // r̂ = r0
    c->rho = make_double2(tot[1], 0.0);          // ρ1 = ⟨r̂, r0⟩ = ‖r0‖²
    c->alpha = c->omega = make_double2(1.0, 0.0);
    if (cabs_(c->rho) <= 1e-30 * c->nrh * c->rnorm) { c->status = ZK_BREAKDOWN_RHO; c->done = 1; return; }
    c->j = 1;
}
__device__ inline void fin_k1_bicg(SolveCtx* c, const double* tot) {  // {Re σ, Im σ, ‖v‖²}
    const double2 sigma = make_double2(tot[0], tot[1]);
    const double vnorm = sqrt(tot[2]);
    if (!cfinite(sigma)) { c->status = ZK_NONFINITE; c->done = 1; return; }
    if (cabs_(sigma) <= 1e-30 * c->nrh * vnorm) { c->status = ZK_BREAKDOWN_SIGMA; c->done = 1; return; }
    c->alpha = cdiv(c->rho, sigma);
}
__device__ inline void fin_k2_bicg(SolveCtx* c, const double* tot) {  // {‖s‖²}
    const double snorm = sqrt(tot[0]);
    if (!isfinite(snorm)) { c->status = ZK_NONFINITE; c->done = 1; return; }
    if (snorm / c->nb <= c->tol) {               // half-step exit (L6): K4 applies x += αp
        c->hist[c->j] = snorm / c->nb;
        c->iters = c->j;
        c->status = ZK_CONVERGED;
        c->half = 1;
        c->done = 1;
    }
}
__device__ inline void fin_k3_bicg(SolveCtx* c, const double* tot) {  // {Re⟨t,s⟩, Im⟨t,s⟩, τ}
    const double tau = tot[2];
    if (!isfinite(tau)) { c->status = ZK_NONFINITE; c->done = 1; return; }
    if (tau == 0.0) { c->status = ZK_BREAKDOWN_OMEGA; c->done = 1; return; }
    c->omega = make_double2(tot[0] / tau, tot[1] / tau);
}
__device__ inline void fin_k4_bicg(SolveCtx* c, const double* tot) {  // {‖r‖², Re ρ', Im ρ'}
    const int j = c->j;
    c->rnorm = sqrt(tot[0]);
    c->hist[j] = c->rnorm / c->nb;
    c->iters = j;
    if (!isfinite(c->hist[j]) || !cfinite(c->omega)) { c->status = ZK_NONFINITE; c->done = 1; return; }
    if (c->hist[j] <= c->tol) { c->status = ZK_CONVERGED; c->done = 1; return; }
    if (cabs_(c->omega) <= 1e-30) { c->status = ZK_BREAKDOWN_OMEGA; c->done = 1; return; }
    if (j >= c->maxit) { c->status = ZK_MAXIT; c->done = 1; return; }
    // start of iteration j+1 of O6: ρ = ⟨r̂, r⟩, breakdown test, β = (ρ/ρ_prev)(α/ω)
    const double2 rho = make_double2(tot[1], tot[2]);
    if (!cfinite(rho)) { c->status = ZK_NONFINITE; c->done = 1; return; }
    if (cabs_(rho) <= 1e-30 * c->nrh * c->rnorm) { c->status = ZK_BREAKDOWN_RHO; c->done = 1; return; }
    c->beta = cmul(cdiv(rho, c->rho), cdiv(c->alpha, c->omega));
    c->rho = rho;
    c->j = j + 1;
}
__device__ inline void fin_init_cg(SolveCtx* c, const double* tot) {  // {‖b‖², ‖r0‖²}
    c->iters = 0;
    c->nb = sqrt(tot[0]);
    if (c->nb == 0.0) { c->status = ST_ZERO_RHS; c->done = 1; return; }
    c->gamma = tot[1];
    c->hist[0] = sqrt(c->gamma) / c->nb;
    if (!isfinite(c->hist[0])) { c->status = ZK_NONFINITE; c->done = 1; return; }
    if (c->hist[0] <= c->tol) { c->status = ZK_CONVERGED; c->done = 1; return; }
    c->j = 1;
}
__device__ inline void fin_k1_cg(SolveCtx* c, const double* tot) {  // {Re δ, Im δ}
    const double2 delta = make_double2(tot[0], tot[1]);
    if (!cfinite(delta)) { c->status = ZK_NONFINITE; c->done = 1; return; }
    if (delta.x <= 0.0) { c->status = ZK_NOT_HPD; c->done = 1; return; }
    c->alpha_cg = c->gamma / delta.x;
}
__device__ inline void fin_k2_cg(SolveCtx* c, const double* tot) {  // {γ'}
    const int j = c->j;
    const double g = tot[0];
    c->hist[j] = sqrt(g) / c->nb;
    c->iters = j;
    if (!isfinite(c->hist[j])) { c->status = ZK_NONFINITE; c->done = 1; return; }
    if (c->hist[j] <= c->tol) { c->status = ZK_CONVERGED; c->done = 1; return; }
    if (j >= c->maxit) { c->status = ZK_MAXIT; c->done = 1; return; }
    c->beta_cg = g / c->gamma;
    c->gamma = g;
    c->j = j + 1;
}
// NEXT-4 COCG (van der Vorst & Melissen): CG with the unconjugated form for complex symmetric A
__device__ inline void fin_init_cocg(SolveCtx* c, const double* tot) {  // {‖b‖², ‖r0‖², Re r0ᵀr0, Im r0ᵀr0}
    c->iters = 0;
    c->nb = sqrt(tot[0]);
    if (c->nb == 0.0) { c->status = ST_ZERO_RHS; c->done = 1; return; }
    c->rho = make_double2(tot[2], tot[3]);
    c->hist[0] = sqrt(tot[1]) / c->nb;
    if (!isfinite(c->hist[0])) { c->status = ZK_NONFINITE; c->done = 1; return; }
    if (c->hist[0] <= c->tol) { c->status = ZK_CONVERGED; c->done = 1; return; }
    c->j = 1;
}
__device__ inline void fin_k1_cocg(SolveCtx* c, const double* tot) {  // {Re μ, Im μ}, μ = pᵀq
    const double2 mu = make_double2(tot[0], tot[1]);
    if (!cfinite(mu)) { c->status = ZK_NONFINITE; c->done = 1; return; }
    if (mu.x == 0.0 && mu.y == 0.0) { c->status = ZK_BREAKDOWN_SIGMA; c->done = 1; return; }
    c->alpha = cdiv(c->rho, mu);
}
__device__ inline void fin_k2_cocg(SolveCtx* c, const double* tot) {  // {‖r‖², Re ρ', Im ρ'}, ρ' = rᵀr
    const int j = c->j;
    const double rn2 = tot[0];
    c->hist[j] = sqrt(rn2) / c->nb;
    c->iters = j;
    if (!isfinite(c->hist[j])) { c->status = ZK_NONFINITE; c->done = 1; return; }
    if (c->hist[j] <= c->tol) { c->status = ZK_CONVERGED; c->done = 1; return; }
    if (j >= c->maxit) { c->status = ZK_MAXIT; c->done = 1; return; }
    const double2 rho = make_double2(tot[1], tot[2]);
    if (!cfinite(rho)) { c->status = ZK_NONFINITE; c->done = 1; return; }
    if (cabs_(rho) <= 1e-30 * rn2) { c->status = ZK_BREAKDOWN_RHO; c->done = 1; return; }
    c->beta = cdiv(rho, c->rho);
    c->rho = rho;
    c->j = j + 1;
}
// NEXT-2 TFQMR — the scalar steps of oracle_tfqmr in its order (θ, c, τ, η, bound; ρ', β; σ, α)
__device__ inline void fin_init_tfqmr(SolveCtx* c, const double* tot) {  // {‖b‖², ‖r0‖², ·, ·}
    c->iters = 0;
    c->nb = sqrt(tot[0]);
    if (c->nb == 0.0) { c->status = ST_ZERO_RHS; c->done = 1; return; }
    c->tau = sqrt(tot[1]);
    c->hist[0] = c->tau / c->nb;
    if (!isfinite(c->hist[0])) { c->status = ZK_NONFINITE; c->done = 1; return; }
    if (c->hist[0] <= c->tol) { c->status = ZK_CONVERGED; c->done = 1; return; }
    c->nrh = c->tau;                     // ‖r̃‖, r̃ = r0
    c->rho = make_double2(tot[1], 0.0);  // ρ = ⟨r̃, r0⟩ = ‖r0‖²
    c->theta = 0.0;
    c->eta = make_double2(0.0, 0.0);
    c->j = 1;
}
__device__ inline void fin_sigma_tfqmr(SolveCtx* c, const double* tot) {  // {Re σ, Im σ}, σ = ⟨r̃, v⟩
    const double2 sigma = make_double2(tot[0], tot[1]);
    if (!cfinite(sigma)) { c->status = ZK_NONFINITE; c->done = 1; return; }
    if (sigma.x == 0.0 && sigma.y == 0.0) { c->status = ZK_BREAKDOWN_SIGMA; c->done = 1; return; }
    c->alpha = cdiv(c->rho, sigma);
    c->coef1 = cmul(cdiv(make_double2(c->theta * c->theta, 0.0), c->alpha), c->eta);  // for half step 1
}
// one half step's scalars from ‖w‖²; returns false when the loop ends (x += η·d still pending)
__device__ inline bool half_tfqmr(SolveCtx* c, double ww, int m, bool second) {
    c->theta = sqrt(ww) / c->tau;
    const double cc = 1.0 / sqrt(1.0 + c->theta * c->theta);
    c->tau = c->tau * c->theta * cc;
    c->eta = make_double2(cc * cc * c->alpha.x, cc * cc * c->alpha.y);
    const double bound = c->tau * sqrt((double)m + 1.0) / c->nb;
    if (!isfinite(bound)) { c->status = ZK_NONFINITE; c->iters = c->j; c->done = 1; return false; }
    if (second || bound <= c->tol) c->hist[c->j] = bound;
    if (bound <= c->tol) { c->status = ZK_CONVERGED; c->iters = c->j; c->done = 1; return false; }
    return true;
}
// Any exit inside an iteration leaves the d, x updates of its half steps to the next kernel (the
// oracle applies them before testing): c->half = 1 (T2 does x += η1·d1) or 2 (T3 does its updates).
__device__ inline void fin_t1_tfqmr(SolveCtx* c, const double* tot) {  // {‖w‖²}
    const bool go = half_tfqmr(c, tot[0], 2 * c->j - 1, false);
    c->eta1 = c->eta;
    if (!go) { c->half = 1; return; }
    c->coef2 = cmul(cdiv(make_double2(c->theta * c->theta, 0.0), c->alpha), c->eta);  // for half step 2
}
__device__ inline void fin_t2_steps(SolveCtx* c, const double* tot) {
    const int j = c->j;
    if (!half_tfqmr(c, tot[0], 2 * j, true)) return;
    c->iters = j;
    const double2 rho = make_double2(tot[1], tot[2]);
    if (!cfinite(rho)) { c->status = ZK_NONFINITE; c->done = 1; return; }
    if (cabs_(rho) <= 1e-30 * c->nrh * sqrt(tot[0])) { c->status = ZK_BREAKDOWN_RHO; c->done = 1; return; }
    c->beta = cdiv(rho, c->rho);
    c->rho = rho;
    if (j >= c->maxit) { c->status = ZK_MAXIT; c->done = 1; return; }
    c->j = j + 1;
}
__device__ inline void fin_t2_tfqmr(SolveCtx* c, const double* tot) {  // {‖w‖², Re ρ', Im ρ'}
    fin_t2_steps(c, tot);
    if (c->done) c->half = 2;
}
// NEXT-3 BiCGStab(ℓ) — the scalar steps of oracle_bicgstab_l in its order; c->rho is ρ0
__device__ inline bool bl_rho(SolveCtx* c, double2 rho1, double rn) {  // ρ1 = ⟨r̃, r̂_j⟩, rn = ‖r̂_j‖
    if (!cfinite(rho1)) { c->status = ZK_NONFINITE; c->done = 1; return false; }
    if (cabs_(rho1) <= 1e-30 * c->nrh * rn) { c->status = ZK_BREAKDOWN_RHO; c->done = 1; return false; }
    c->beta = cdiv(cmul(c->alpha, rho1), c->rho);  // β = α ρ1 / ρ0
    c->rho = rho1;
    return true;
}
__device__ inline void bl_cycle_start(SolveCtx* c) {  // iters = k (an exit inside the cycle counts it); ρ0 = −ω ρ0
    c->iters = c->j;
    c->rho = cmul(make_double2(-c->omega.x, -c->omega.y), c->rho);
}
__device__ inline void fin_init_bl(SolveCtx* c, const double* tot) {  // {‖b‖², ‖r0‖², ·, ·}
    c->iters = 0;
    c->nb = sqrt(tot[0]);
    if (c->nb == 0.0) { c->status = ST_ZERO_RHS; c->done = 1; return; }
    c->rnorm = sqrt(tot[1]);
    c->hist[0] = c->rnorm / c->nb;
    if (!isfinite(c->hist[0])) { c->status = ZK_NONFINITE; c->done = 1; return; }
    if (c->hist[0] <= c->tol) { c->status = ZK_CONVERGED; c->done = 1; return; }
    c->nrh = c->rnorm;  // r̃ = r0
    c->rho = make_double2(1.0, 0.0);
    c->alpha = make_double2(0.0, 0.0);
    c->omega = make_double2(1.0, 0.0);
    c->j = 1;
    bl_cycle_start(c);
    bl_rho(c, make_double2(tot[1], 0.0), c->rnorm);  // ρ1 = ⟨r̃, r0⟩ = ‖r0‖²
}
__device__ inline void fin_s1_bl(SolveCtx* c, const double* tot) {  // {Re γ, Im γ, ‖û_{j+1}‖²}
    const double2 g = make_double2(tot[0], tot[1]);
    if (!cfinite(g)) { c->status = ZK_NONFINITE; c->done = 1; return; }
    if (cabs_(g) <= 1e-30 * c->nrh * sqrt(tot[2])) { c->status = ZK_BREAKDOWN_SIGMA; c->done = 1; return; }
    c->alpha = cdiv(c->rho, g);
}
__device__ inline void fin_b2_bl(SolveCtx* c, const double* tot) {  // {‖r̂_0‖²} after x += α û_0
    const double rn = sqrt(tot[0]);
    if (!isfinite(rn)) { c->status = ZK_NONFINITE; c->done = 1; return; }
    if (rn / c->nb <= c->tol) {
        c->hist[c->j] = rn / c->nb;
        c->status = ZK_CONVERGED;
        c->done = 1;
    }
}
__device__ inline void fin_s2_bl(SolveCtx* c, const double* tot) {  // {Re ρ1, Im ρ1, ‖r̂_{j+1}‖²}
    bl_rho(c, make_double2(tot[0], tot[1]), sqrt(tot[2]));
}
__device__ inline void fin_u_bl(SolveCtx* c, const double* tot) {  // {‖r̂_0‖², Re ρ1, Im ρ1}
    const int j = c->j;
    c->rnorm = sqrt(tot[0]);
    c->hist[j] = c->rnorm / c->nb;
    c->iters = j;
    if (!isfinite(c->hist[j]) || !cfinite(c->omega)) { c->status = ZK_NONFINITE; c->done = 1; return; }
    if (c->hist[j] <= c->tol) { c->status = ZK_CONVERGED; c->done = 1; return; }
    if (cabs_(c->omega) <= 1e-30) { c->status = ZK_BREAKDOWN_OMEGA; c->done = 1; return; }
    if (j >= c->maxit) { c->status = ZK_MAXIT; c->done = 1; return; }
    c->j = j + 1;
    bl_cycle_start(c);
    bl_rho(c, make_double2(tot[1], tot[2]), c->rnorm);
}
__device__ inline void fin_true(SolveCtx* c, const double* tot) {  // {‖b − Ax‖²}
    c->true_relres = c->nb > 0.0 ? sqrt(tot[0]) / c->nb : NAN;
}


template <int L>
struct GramPack {
    static constexpr int NV = L + 1;
    static constexpr int ND = NV + NV * (NV - 1);  // doubles
    __host__ __device__ static constexpr int diag(int a) { return a + a * (2 * NV - a - 1); }  // entry (a, a)
    __host__ __device__ static constexpr int off(int a, int b) { return diag(a) + 1 + 2 * (b - a - 1); }  // a < b
};

// the minimal-residual system from the packed Gram totals: M γ = v with M_ik = ⟨r̂_{i+1}, r̂_{k+1}⟩,
// v_i = ⟨r̂_{i+1}, r̂_0⟩, by Cholesky M = L·Lᴴ (the oracle's algorithm, written independently)
template <int L>
__device__ inline void fin_gram_bl(SolveCtx* c, const double* g) {
    using GP = GramPack<L>;
    auto G = [&](int a, int b) -> double2 {  // ⟨r̂_a, r̂_b⟩
        if (a == b) return make_double2(g[GP::diag(a)], 0.0);
        if (a < b) return make_double2(g[GP::off(a, b)], g[GP::off(a, b) + 1]);
        return make_double2(g[GP::off(b, a)], -g[GP::off(b, a) + 1]);
    };
    double2 Lm[L][L];
    for (int jj = 0; jj < L; jj++) {
        double d = G(jj + 1, jj + 1).x;
        for (int q = 0; q < jj; q++) d -= Lm[jj][q].x * Lm[jj][q].x + Lm[jj][q].y * Lm[jj][q].y;
        if (!(d > 0.0) || !isfinite(d)) {
            c->status = ZK_BREAKDOWN_OMEGA;  // singular ℓ×ℓ minimal-residual system
            c->done = 1;
            return;
        }
        const double l = sqrt(d);
        Lm[jj][jj] = make_double2(l, 0.0);
        for (int i = jj + 1; i < L; i++) {
            double2 s = G(i + 1, jj + 1);
            for (int q = 0; q < jj; q++) s = csub(s, cmul(Lm[i][q], make_double2(Lm[jj][q].x, -Lm[jj][q].y)));
            Lm[i][jj] = make_double2(s.x / l, s.y / l);
        }
    }
    double2 y[L];
    for (int i = 0; i < L; i++) {  // L y = v
        double2 s = G(i + 1, 0);
        for (int q = 0; q < i; q++) s = csub(s, cmul(Lm[i][q], y[q]));
        y[i] = make_double2(s.x / Lm[i][i].x, s.y / Lm[i][i].x);
    }
    for (int i = L - 1; i >= 0; i--) {  // Lᴴ γ = y
        double2 s = y[i];
        for (int q = i + 1; q < L; q++) s = csub(s, cmul(make_double2(Lm[q][i].x, -Lm[q][i].y), c->gam[q + 1]));
        c->gam[i + 1] = make_double2(s.x / Lm[i][i].x, s.y / Lm[i][i].x);
    }
    c->omega = c->gam[L];
}


// ---- the single-cluster solvers (loop mode 5, cluster.cu)
#ifndef ZK_CLUSTER_DEFAULT_ROWS
#define ZK_CLUSTER_DEFAULT_ROWS 16384
#endif
constexpr int64_t kClusterDefaultRows = ZK_CLUSTER_DEFAULT_ROWS;  // default up to this size
// cluster solver kind of a method: 0 BiCGStab (and Jacobi-BiCGStab), 1 TFQMR, 2 CG, 3 COCG,
// 4 BiCGStab(ℓ); −1 none
int cluster_kind(int method);
// can the cluster solver hold this system (own rows + the block's columns in shared memory)?
bool cluster_fits(zk_csr_s* A, cudaStream_t s, int kind, int ell);
// launch the whole solve loop on one cluster (A or A·M⁻¹ in av); false when unavailable
bool cluster_launch(zk_csr_s* A, SolveCtx* dc, const SolveCtx& hc, const CsrDev& av, cudaStream_t s, int* out_cs,
                    int kind, int ell, bool do_true, bool init);
}  // namespace zk
