/*
 * zk_oracle.c — TEST INFRASTRUCTURE ONLY.  The plain, slow, obviously correct CPU
 * oracle for the hot path of arXiv 2112.11880 ("Alinea" complex-double Krylov).
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
 * --impl reference legs may load this.  It shares no code, header, table or
 * helper with the CUDA library (paper_2112_11880_b200/csrc); neither includes
 * or links the other.
 *
 * Every routine is the plain definition (SpMV, dot, norm, axpy, scal) or the
 * textbook algorithm step by step (BiCGStab, CG), in IEEE binary64, complex
 * numbers as interleaved (re, im) pairs, complex products written out as
 * (a+bi)(c+di) = (ac − bd) + (ad + bc)i.  Compile with -ffp-contract=off
 * (no FMA contraction) and without -ffast-math.
 *
 * Citations: P:L = /root/reference/PAPER.md line L; S:L = SPEC.md line L;
 * SURVEY.md §8(c) O1–O7 and ledger L1–L21 give the readings; DESIGN.md lists them.
 *
 * Pins: tests/test_oracle_*.py (dense brute force, closed-form eigenvectors,
 * integer exactness, closed-form sums, A = cI, DST-I direct solves, gauge and
 * phase invariance, true-vs-recurrence residual).  Parity unpinned: nothing
 * here reproduces PAPER.md T9/T10 iteration counts (other matrices and an
 * unnamed preconditioner).
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

/* summation orders */
enum { ORD_SEQ = 0, ORD_REV = 1, ORD_BLOCK256 = 2, ORD_NEUMAIER = 3 };

/* solver outcomes */
enum {
    ST_CONVERGED = 0, ST_MAXIT = 1, ST_BREAKDOWN_RHO = 2, ST_BREAKDOWN_SIGMA = 3,
    ST_BREAKDOWN_OMEGA = 4, ST_NOT_HPD = 5, ST_NONFINITE = 6, ST_ZERO_RHS = 7
};

#define RE(v, i) ((v)[2 * (i)])
#define IM(v, i) ((v)[2 * (i) + 1])

/* Timing-only OpenMP build (liboracle_omp.so, bench.py's all-core cpu_baseline row, SURVEY.md
 * §8(d) "CPU oracle timing"): ROWWISE marks loops whose iterations are independent (one output
 * row / element each, computed exactly as in the serial loop), so splitting them over threads
 * changes no bit of any result.  Sums over i (dot, norm) stay sequential.  The default build has
 * no -fopenmp and ROWWISE expands to nothing. */
#ifdef _OPENMP
#define ROWWISE _Pragma("omp parallel for schedule(static)")
#else
#define ROWWISE
#endif

/* ------------------------------------------------------------------------ */
/* summation helper: adds term[i] for i in [0,n) in the requested order     */
/* ------------------------------------------------------------------------ */
typedef double (*term_fn)(const void* ctx, int64_t i);

static double ordered_sum(int64_t n, term_fn f, const void* ctx, int order) {
    double s = 0.0;
    if (order == ORD_REV) {
        for (int64_t i = n - 1; i >= 0; i--) s += f(ctx, i);
    } else if (order == ORD_BLOCK256) {
        /* partial per block of 256 in ascending order, then partials in ascending order
           (the "two distinct tasks" reduction of P:199-200) */
        for (int64_t b0 = 0; b0 < n; b0 += 256) {
            double part = 0.0;
            int64_t e = b0 + 256 < n ? b0 + 256 : n;
            for (int64_t i = b0; i < e; i++) part += f(ctx, i);
            s += part;
        }
    } else if (order == ORD_NEUMAIER) {
        double c = 0.0;
        for (int64_t i = 0; i < n; i++) {
            double t = f(ctx, i);
            double u = s + t;
            if (fabs(s) >= fabs(t)) c += (s - u) + t;
            else c += (t - u) + s;
            s = u;
        }
        s += c;
    } else {
        for (int64_t i = 0; i < n; i++) s += f(ctx, i);
    }
    return s;
}

typedef struct { const double* x; const double* y; } pair_ctx;

/* Re(conj(x_i) y_i) = xr·yr + xi·yi ;  Im(conj(x_i) y_i) = xr·yi − xi·yr   (O2) */
static double dot_re_term(const void* c, int64_t i) {
    const pair_ctx* p = (const pair_ctx*)c;
    return RE(p->x, i) * RE(p->y, i) + IM(p->x, i) * IM(p->y, i);
}
static double dot_im_term(const void* c, int64_t i) {
    const pair_ctx* p = (const pair_ctx*)c;
    return RE(p->x, i) * IM(p->y, i) - IM(p->x, i) * RE(p->y, i);
}
static double sq_term(const void* c, int64_t i) {
    const pair_ctx* p = (const pair_ctx*)c;
    return RE(p->x, i) * RE(p->x, i) + IM(p->x, i) * IM(p->x, i);
}

/* O2 zdotc: Σ conj(x_i)·y_i, conjugating the FIRST argument (L1; BLAS zdotc).
   PAPER.md P:199-200 (ZDOT, "two distinct tasks"). */
void oracle_zdotc(int64_t n, const double* x, const double* y, int order, double* out) {
    pair_ctx c = {x, y};
    out[0] = ordered_sum(n, dot_re_term, &c, order);
    out[1] = ordered_sum(n, dot_im_term, &c, order);
}

/* Σ re² + im² (no scaling, L3) */
double oracle_sumsq(int64_t n, const double* x, int order) {
    pair_ctx c = {x, x};
    return ordered_sum(n, sq_term, &c, order);
}

/* O3 dznrm2: sqrt(Σ re² + im²).  PAPER.md P:257 (ZNORM, T7). */
double oracle_dznrm2(int64_t n, const double* x, int order) {
    return sqrt(oracle_sumsq(n, x, order));
}

/* O4 zaxpy: y_i ← α·x_i + y_i.  PAPER.md P:143-150 (listing "d_y[idx] = alpha * d_x[idx] + d_y[idx]"). */
void oracle_zaxpy(int64_t n, double ar, double ai, const double* x, double* y) {
    for (int64_t i = 0; i < n; i++) {
        double pr = ar * RE(x, i) - ai * IM(x, i);
        double pi = ar * IM(x, i) + ai * RE(x, i);
        RE(y, i) = pr + RE(y, i);
        IM(y, i) = pi + IM(y, i);
    }
}

/* O5 zscal: x_i ← α·x_i.  PAPER.md P:116-122 (listing "d_x[idx] = alpha * d_x[idx]"). */
void oracle_zscal(int64_t n, double ar, double ai, double* x) {
    for (int64_t i = 0; i < n; i++) {
        double xr = RE(x, i), xi = IM(x, i);
        RE(x, i) = ar * xr - ai * xi;
        IM(x, i) = ar * xi + ai * xr;
    }
}

/* O1 zcsrmv: y_i ← α·Σ_{p ∈ row i} values[p]·x[col[p]] + β·y_i, row entries in stored order
   (order = ORD_REV accumulates each row back to front; used only for the BiCGStab envelope, L11).
   β = 0 ⇒ y is not read.  PAPER.md P:279-281 (SpMV CSR, T8). */
void oracle_zcsrmv(int64_t n_rows, const int64_t* row_ptr, const int32_t* col, const double* val,
                   double ar, double ai, const double* x, double br, double bi, double* y,
                   int order) {
    ROWWISE
    for (int64_t i = 0; i < n_rows; i++) {
        double sr = 0.0, si = 0.0;
        if (order == ORD_REV) {
            for (int64_t p = row_ptr[i + 1] - 1; p >= row_ptr[i]; p--) {
                double a = RE(val, p), b = IM(val, p);
                double c = RE(x, col[p]), d = IM(x, col[p]);
                sr += a * c - b * d;
                si += a * d + b * c;
            }
        } else {
            for (int64_t p = row_ptr[i]; p < row_ptr[i + 1]; p++) {
                double a = RE(val, p), b = IM(val, p);
                double c = RE(x, col[p]), d = IM(x, col[p]);
                sr += a * c - b * d;
                si += a * d + b * c;
            }
        }
        double yr = ar * sr - ai * si;
        double yi = ar * si + ai * sr;
        if (br != 0.0 || bi != 0.0) {
            double qr = br * RE(y, i) - bi * IM(y, i);
            double qi = br * IM(y, i) + bi * RE(y, i);
            yr += qr;
            yi += qi;
        }
        RE(y, i) = yr;
        IM(y, i) = yi;
    }
}

/* ------------------------------------------------------------------------ */
/* complex scalar helpers (written out; no Annex-G handling)                 */
/* ------------------------------------------------------------------------ */
typedef struct { double re, im; } cplx;
static cplx make_cplx_real(double a) { cplx r = {a, 0.0}; return r; }
static cplx cmul(cplx a, cplx b) { cplx r = {a.re * b.re - a.im * b.im, a.re * b.im + a.im * b.re}; return r; }
static cplx cdiv(cplx a, cplx b) {
    double den = b.re * b.re + b.im * b.im;
    cplx r = {(a.re * b.re + a.im * b.im) / den, (a.im * b.re - a.re * b.im) / den};
    return r;
}
static double cabs_(cplx a) { return sqrt(a.re * a.re + a.im * a.im); }
static int cfinite(cplx a) { return isfinite(a.re) && isfinite(a.im); }

typedef struct {
    int64_t n;
    const int64_t* row_ptr;
    const int32_t* col;
    const double* val;
    int order;
} csr_t;

static void spmv(const csr_t* A, const double* x, double* y) {
    oracle_zcsrmv(A->n, A->row_ptr, A->col, A->val, 1.0, 0.0, x, 0.0, 0.0, y,
                  A->order == ORD_REV ? ORD_REV : ORD_SEQ);
}
static cplx dotc(const csr_t* A, const double* x, const double* y) {
    double o[2];
    oracle_zdotc(A->n, x, y, A->order, o);
    cplx r = {o[0], o[1]};
    return r;
}
static double nrm(const csr_t* A, const double* x) { return oracle_dznrm2(A->n, x, A->order); }

/* true_relres = ‖b − A x‖/nb */
static double true_relres(const csr_t* A, const double* b, const double* x, double nb, double* tmp) {
    spmv(A, x, tmp);
    for (int64_t i = 0; i < 2 * A->n; i++) tmp[i] = b[i] - tmp[i];
    return nrm(A, tmp) / nb;
}

/*
 * O6 BiCGStab (van der Vorst 1992, Barrett et al. "Templates" form, Hermitian inner product).
 * PAPER.md §4 P:308-310 (P-Bi-CGSTAB; residual tolerance, zero initial guess, maxit);
 * unpreconditioned per L8; half-step exit per L6; breakdown floors per L20.
 * x0 may be NULL (zero initial guess).  hist has room for maxit+1 entries.
 * Returns the status; *iters = completed loop passes (half-step exit counts as one, L7).
 */
int oracle_bicgstab(int64_t n, const int64_t* row_ptr, const int32_t* col, const double* val,
                    const double* b, const double* x0, double tol, int32_t maxit, int order,
                    double* x, int32_t* iters, double* hist, double* out_true_relres) {
    csr_t A = {n, row_ptr, col, val, order};
    size_t bytes = (size_t)(2 * n) * sizeof(double);
    double *r = malloc(bytes), *rh = malloc(bytes), *p = malloc(bytes), *v = malloc(bytes),
           *s = malloc(bytes), *t = malloc(bytes);
    int status = ST_MAXIT;
    *iters = 0;
    *out_true_relres = NAN;

    /* r = b − A x0 (r = b if x0 = 0) */
    if (x0) {
        memcpy(x, x0, bytes);
        spmv(&A, x, r);
        for (int64_t i = 0; i < 2 * n; i++) r[i] = b[i] - r[i];
    } else {
        memset(x, 0, bytes);
        memcpy(r, b, bytes);
    }
    double nb = nrm(&A, b);
    if (nb == 0.0) { status = ST_ZERO_RHS; goto done; }
    double rnorm = nrm(&A, r);
    hist[0] = rnorm / nb;
    if (!isfinite(hist[0])) { status = ST_NONFINITE; goto done; }
    if (hist[0] <= tol) { status = ST_CONVERGED; goto done_true; }

    memcpy(rh, r, bytes);                      /* r̂ = r0 (L6) */
    double nrh = rnorm;
    cplx rho_prev = {1, 0}, alpha = {1, 0}, omega = {1, 0};
    memset(p, 0, bytes);
    memset(v, 0, bytes);

    for (int32_t j = 1; j <= maxit; j++) {
        cplx rho = dotc(&A, rh, r);                            /* ρ = ⟨r̂, r⟩ */
        if (!cfinite(rho)) { status = ST_NONFINITE; break; }
        if (cabs_(rho) <= 1e-30 * nrh * rnorm) { status = ST_BREAKDOWN_RHO; break; }
        if (j == 1) {
            memcpy(p, r, bytes);                               /* p = r */
        } else {
            cplx beta = cmul(cdiv(rho, rho_prev), cdiv(alpha, omega));  /* β = (ρ/ρ_prev)(α/ω) */
            ROWWISE
            for (int64_t i = 0; i < n; i++) {                  /* p = r + β(p − ω v) */
                cplx pv = {RE(p, i), IM(p, i)}, vv = {RE(v, i), IM(v, i)};
                cplx wv = cmul(omega, vv);
                cplx d = {pv.re - wv.re, pv.im - wv.im};
                cplx bd = cmul(beta, d);
                RE(p, i) = RE(r, i) + bd.re;
                IM(p, i) = IM(r, i) + bd.im;
            }
        }
        spmv(&A, p, v);                                        /* v = A p */
        cplx sigma = dotc(&A, rh, v);                          /* σ = ⟨r̂, v⟩ */
        double vnorm = nrm(&A, v);
        if (!cfinite(sigma)) { status = ST_NONFINITE; break; }
        if (cabs_(sigma) <= 1e-30 * nrh * vnorm) { status = ST_BREAKDOWN_SIGMA; break; }
        alpha = cdiv(rho, sigma);                              /* α = ρ/σ */
        ROWWISE
        for (int64_t i = 0; i < n; i++) {                      /* s = r − α v */
            cplx vv = {RE(v, i), IM(v, i)};
            cplx av = cmul(alpha, vv);
            RE(s, i) = RE(r, i) - av.re;
            IM(s, i) = IM(r, i) - av.im;
        }
        double snorm = nrm(&A, s);
        if (!isfinite(snorm)) { status = ST_NONFINITE; break; }
        if (snorm / nb <= tol) {                               /* half-step exit (L6) */
            for (int64_t i = 0; i < n; i++) {
                cplx pv = {RE(p, i), IM(p, i)};
                cplx ap = cmul(alpha, pv);
                RE(x, i) += ap.re;
                IM(x, i) += ap.im;
            }
            hist[j] = snorm / nb;
            *iters = j;
            status = ST_CONVERGED;
            goto done_true;
        }
        spmv(&A, s, t);                                        /* t = A s */
        double tau = oracle_sumsq(n, t, order);                /* τ = ⟨t, t⟩ */
        if (!isfinite(tau)) { status = ST_NONFINITE; break; }
        if (tau == 0.0) { status = ST_BREAKDOWN_OMEGA; break; }
        cplx ts = dotc(&A, t, s);                              /* ω = ⟨t, s⟩/τ */
        omega.re = ts.re / tau;
        omega.im = ts.im / tau;
        ROWWISE
        for (int64_t i = 0; i < n; i++) {                      /* x += αp + ωs ; r = s − ωt */
            cplx pv = {RE(p, i), IM(p, i)}, sv = {RE(s, i), IM(s, i)}, tv = {RE(t, i), IM(t, i)};
            cplx ap = cmul(alpha, pv), ws = cmul(omega, sv), wt = cmul(omega, tv);
            RE(x, i) += ap.re + ws.re;
            IM(x, i) += ap.im + ws.im;
            RE(r, i) = sv.re - wt.re;
            IM(r, i) = sv.im - wt.im;
        }
        rnorm = nrm(&A, r);
        hist[j] = rnorm / nb;
        *iters = j;
        if (!isfinite(hist[j]) || !cfinite(omega)) { status = ST_NONFINITE; break; }
        if (hist[j] <= tol) { status = ST_CONVERGED; break; }
        if (cabs_(omega) <= 1e-30) { status = ST_BREAKDOWN_OMEGA; break; }
        rho_prev = rho;
    }
done_true:
    *out_true_relres = true_relres(&A, b, x, nb, t);
done:
    free(r); free(rh); free(p); free(v); free(s); free(t);
    return status;
}

/*
 * O7 CG (Hestenes–Stiefel, Hermitian inner product; A Hermitian positive definite).
 * Not in the paper (north-star addition, SPEC S:410 lists it as a non-goal of the CPU program);
 * run on the gauge-twisted η = 0 variant (L9).  NOT_HPD if Re⟨p, Ap⟩ ≤ 0.
 */
int oracle_cg(int64_t n, const int64_t* row_ptr, const int32_t* col, const double* val,
              const double* b, const double* x0, double tol, int32_t maxit, int order, double* x,
              int32_t* iters, double* hist, double* out_true_relres) {
    csr_t A = {n, row_ptr, col, val, order};
    size_t bytes = (size_t)(2 * n) * sizeof(double);
    double *r = malloc(bytes), *p = malloc(bytes), *q = malloc(bytes);
    int status = ST_MAXIT;
    *iters = 0;
    *out_true_relres = NAN;

    if (x0) {                                                  /* r = b − A x0 */
        memcpy(x, x0, bytes);
        spmv(&A, x, r);
        for (int64_t i = 0; i < 2 * n; i++) r[i] = b[i] - r[i];
    } else {
        memset(x, 0, bytes);
        memcpy(r, b, bytes);
    }
    double nb = nrm(&A, b);
    if (nb == 0.0) { status = ST_ZERO_RHS; goto done; }
    memcpy(p, r, bytes);                                       /* p = r */
    double gamma = oracle_sumsq(n, r, order);                  /* γ = ⟨r, r⟩ */
    hist[0] = sqrt(gamma) / nb;
    if (!isfinite(hist[0])) { status = ST_NONFINITE; goto done; }
    if (hist[0] <= tol) { status = ST_CONVERGED; goto done_true; }

    for (int32_t j = 1; j <= maxit; j++) {
        spmv(&A, p, q);                                        /* q = A p */
        cplx delta = dotc(&A, p, q);                           /* δ = ⟨p, q⟩ */
        if (!cfinite(delta)) { status = ST_NONFINITE; break; }
        if (delta.re <= 0.0) { status = ST_NOT_HPD; break; }
        double alpha = gamma / delta.re;                       /* α = γ / Re δ */
        for (int64_t i = 0; i < 2 * n; i++) {                  /* x += α p ; r −= α q */
            x[i] += alpha * p[i];
            r[i] -= alpha * q[i];
        }
        double gamma_new = oracle_sumsq(n, r, order);          /* γ' = ⟨r, r⟩ */
        hist[j] = sqrt(gamma_new) / nb;
        *iters = j;
        if (!isfinite(hist[j])) { status = ST_NONFINITE; break; }
        if (hist[j] <= tol) { status = ST_CONVERGED; break; }
        double beta = gamma_new / gamma;                       /* p = r + (γ'/γ) p */
        for (int64_t i = 0; i < 2 * n; i++) p[i] = r[i] + beta * p[i];
        gamma = gamma_new;
    }
done_true:
    *out_true_relres = true_relres(&A, b, x, nb, q);
done:
    free(r); free(p); free(q);
    return status;
}

/*
 * NEXT-1: Jacobi-preconditioned BiCGStab, the paper's "P-Bi-CGSTAB" (§4; the
 * preconditioner is unnamed there, SPEC S:296-322 reads it as Jacobi).  The Templates
 * preconditioned BiCGSTAB step by step with M = diag(A) (complex reciprocal of the stored
 * diagonal): p̂ = M⁻¹p, v = A p̂, ŝ = M⁻¹s, t = A ŝ, x += α p̂ + ω ŝ.  Residuals, tests and
 * breakdown floors are those of O6 (unpreconditioned r, so tol is comparable).
 * A row without a stored nonzero diagonal makes M singular: returns ST_BREAKDOWN_RHO with
 * iters = 0 and hist[0] unset (the GPU reports ZK_ERR_DIM at setup instead).
 */
static int jacobi_inverse(const csr_t* A, double* dinv) {
    for (int64_t i = 0; i < A->n; i++) {
        cplx d = {0, 0};
        int found = 0;
        for (int64_t p = A->row_ptr[i]; p < A->row_ptr[i + 1]; p++)
            if (A->col[p] == i) { d.re = RE(A->val, p); d.im = IM(A->val, p); found = 1; }
        if (!found || (d.re == 0.0 && d.im == 0.0)) return 0;
        cplx one = {1, 0};
        cplx q = cdiv(one, d);                                  /* 1/d written out (R7) */
        RE(dinv, i) = q.re;
        IM(dinv, i) = q.im;
    }
    return 1;
}

static void apply_jacobi(int64_t n, const double* dinv, const double* in, double* out) {
    for (int64_t i = 0; i < n; i++) {
        cplx d = {RE(dinv, i), IM(dinv, i)}, v = {RE(in, i), IM(in, i)};
        cplx r = cmul(d, v);
        RE(out, i) = r.re;
        IM(out, i) = r.im;
    }
}

int oracle_bicgstab_jacobi(int64_t n, const int64_t* row_ptr, const int32_t* col, const double* val,
                           const double* b, const double* x0, double tol, int32_t maxit, int order,
                           double* x, int32_t* iters, double* hist, double* out_true_relres) {
    csr_t A = {n, row_ptr, col, val, order};
    size_t bytes = (size_t)(2 * n) * sizeof(double);
    double *r = malloc(bytes), *rh = malloc(bytes), *p = malloc(bytes), *v = malloc(bytes),
           *s = malloc(bytes), *t = malloc(bytes), *ph = malloc(bytes), *sh = malloc(bytes),
           *dinv = malloc(bytes);
    int status = ST_MAXIT;
    *iters = 0;
    *out_true_relres = NAN;
    if (!jacobi_inverse(&A, dinv)) { status = ST_BREAKDOWN_RHO; goto done; }

    if (x0) {                                                  /* r = b − A x0 */
        memcpy(x, x0, bytes);
        spmv(&A, x, r);
        for (int64_t i = 0; i < 2 * n; i++) r[i] = b[i] - r[i];
    } else {
        memset(x, 0, bytes);
        memcpy(r, b, bytes);
    }
    double nb = nrm(&A, b);
    if (nb == 0.0) { status = ST_ZERO_RHS; goto done; }
    double rnorm = nrm(&A, r);
    hist[0] = rnorm / nb;
    if (!isfinite(hist[0])) { status = ST_NONFINITE; goto done; }
    if (hist[0] <= tol) { status = ST_CONVERGED; goto done_true; }

    memcpy(rh, r, bytes);                                      /* r̂ = r0 */
    double nrh = rnorm;
    cplx rho_prev = {1, 0}, alpha = {1, 0}, omega = {1, 0};
    memset(p, 0, bytes);
    memset(v, 0, bytes);

    for (int32_t j = 1; j <= maxit; j++) {
        cplx rho = dotc(&A, rh, r);                            /* ρ = ⟨r̂, r⟩ */
        if (!cfinite(rho)) { status = ST_NONFINITE; break; }
        if (cabs_(rho) <= 1e-30 * nrh * rnorm) { status = ST_BREAKDOWN_RHO; break; }
        if (j == 1) {
            memcpy(p, r, bytes);
        } else {
            cplx beta = cmul(cdiv(rho, rho_prev), cdiv(alpha, omega));
            for (int64_t i = 0; i < n; i++) {                  /* p = r + β(p − ω v) */
                cplx pv = {RE(p, i), IM(p, i)}, vv = {RE(v, i), IM(v, i)};
                cplx wv = cmul(omega, vv);
                cplx d = {pv.re - wv.re, pv.im - wv.im};
                cplx bd = cmul(beta, d);
                RE(p, i) = RE(r, i) + bd.re;
                IM(p, i) = IM(r, i) + bd.im;
            }
        }
        apply_jacobi(n, dinv, p, ph);                          /* p̂ = M⁻¹ p */
        spmv(&A, ph, v);                                       /* v = A p̂ */
        cplx sigma = dotc(&A, rh, v);
        double vnorm = nrm(&A, v);
        if (!cfinite(sigma)) { status = ST_NONFINITE; break; }
        if (cabs_(sigma) <= 1e-30 * nrh * vnorm) { status = ST_BREAKDOWN_SIGMA; break; }
        alpha = cdiv(rho, sigma);
        for (int64_t i = 0; i < n; i++) {                      /* s = r − α v */
            cplx vv = {RE(v, i), IM(v, i)};
            cplx av = cmul(alpha, vv);
            RE(s, i) = RE(r, i) - av.re;
            IM(s, i) = IM(r, i) - av.im;
        }
        double snorm = nrm(&A, s);
        if (!isfinite(snorm)) { status = ST_NONFINITE; break; }
        if (snorm / nb <= tol) {                               /* half-step exit: x += α p̂ */
            for (int64_t i = 0; i < n; i++) {
                cplx pv = {RE(ph, i), IM(ph, i)};
                cplx ap = cmul(alpha, pv);
                RE(x, i) += ap.re;
                IM(x, i) += ap.im;
            }
            hist[j] = snorm / nb;
            *iters = j;
            status = ST_CONVERGED;
            goto done_true;
        }
        apply_jacobi(n, dinv, s, sh);                          /* ŝ = M⁻¹ s */
        spmv(&A, sh, t);                                       /* t = A ŝ */
        double tau = oracle_sumsq(n, t, order);
        if (!isfinite(tau)) { status = ST_NONFINITE; break; }
        if (tau == 0.0) { status = ST_BREAKDOWN_OMEGA; break; }
        cplx ts = dotc(&A, t, s);                              /* ω = ⟨t, s⟩/τ */
        omega.re = ts.re / tau;
        omega.im = ts.im / tau;
        for (int64_t i = 0; i < n; i++) {                      /* x += α p̂ + ω ŝ ; r = s − ω t */
            cplx pv = {RE(ph, i), IM(ph, i)}, sv = {RE(sh, i), IM(sh, i)}, tv = {RE(t, i), IM(t, i)};
            cplx ap = cmul(alpha, pv), ws = cmul(omega, sv), wt = cmul(omega, tv);
            RE(x, i) += ap.re + ws.re;
            IM(x, i) += ap.im + ws.im;
            RE(r, i) = RE(s, i) - wt.re;
            IM(r, i) = IM(s, i) - wt.im;
        }
        rnorm = nrm(&A, r);
        hist[j] = rnorm / nb;
        *iters = j;
        if (!isfinite(hist[j]) || !cfinite(omega)) { status = ST_NONFINITE; break; }
        if (hist[j] <= tol) { status = ST_CONVERGED; break; }
        if (cabs_(omega) <= 1e-30) { status = ST_BREAKDOWN_OMEGA; break; }
        rho_prev = rho;
    }
done_true:
    *out_true_relres = true_relres(&A, b, x, nb, t);
done:
    free(r); free(rh); free(p); free(v); free(s); free(t); free(ph); free(sh); free(dinv);
    return status;
}

/* NEXT-4: ZASSIGN — "assign of a vector" (§3, T2), read as a fill x_i ← α
   (T2's bytes per element imply a write-only pass). */
void oracle_zassign(int64_t n, double ar, double ai, double* x) {
    for (int64_t i = 0; i < n; i++) {
        RE(x, i) = ar;
        IM(x, i) = ai;
    }
}

/* NEXT-4: ZAXMY — element-wise product y_i ← x_i · y_i ("EWProduct", T5;
   the listing's unused α is ignored, L17). */
void oracle_zaxmy(int64_t n, const double* x, double* y) {
    for (int64_t i = 0; i < n; i++) {
        double a = RE(x, i), b = IM(x, i), c = RE(y, i), d = IM(y, i);
        RE(y, i) = a * c - b * d;
        IM(y, i) = a * d + b * c;
    }
}

/* unconjugated bilinear form Σ x_i·y_i (COCG) */
static cplx dotu(const csr_t* A, const double* x, const double* y) {
    /* Re Σ x y = Σ (xr·yr − xi·yi), Im = Σ (xr·yi + xi·yr), in the requested order via the
       conjugated routine: Σ x y = Σ conj(conj(x)) y → conjugate x into a scratch copy. */
    size_t bytes = (size_t)(2 * A->n) * sizeof(double);
    double* xc = malloc(bytes);
    for (int64_t i = 0; i < A->n; i++) { RE(xc, i) = RE(x, i); IM(xc, i) = -IM(x, i); }
    cplx r = dotc(A, xc, y);
    free(xc);
    return r;
}

/*
 * NEXT-4: COCG (van der Vorst & Melissen 1990) — CG with the unconjugated bilinear form for
 * complex SYMMETRIC A (Aᵀ = A, the Helmholtz matrices with absorption, η > 0), where Hermitian
 * CG does not apply (L9).  Step by step:
 *   r = b − A x0; p = r; ρ = rᵀr; hist[0] = ‖r‖/‖b‖
 *   loop: q = A p; μ = pᵀq (μ = 0 → BREAKDOWN_SIGMA); α = ρ/μ; x += α p; r −= α q;
 *         hist[j] = ‖r‖/‖b‖ (tests as O7); ρ' = rᵀr (|ρ'| ≤ 1e-30‖r‖² → BREAKDOWN_RHO);
 *         p = r + (ρ'/ρ) p; ρ = ρ'.
 */
int oracle_cocg(int64_t n, const int64_t* row_ptr, const int32_t* col, const double* val, const double* b,
                const double* x0, double tol, int32_t maxit, int order, double* x, int32_t* iters,
                double* hist, double* out_true_relres) {
    csr_t A = {n, row_ptr, col, val, order};
    size_t bytes = (size_t)(2 * n) * sizeof(double);
    double *r = malloc(bytes), *p = malloc(bytes), *q = malloc(bytes);
    int status = ST_MAXIT;
    *iters = 0;
    *out_true_relres = NAN;
    if (x0) {
        memcpy(x, x0, bytes);
        spmv(&A, x, r);
        for (int64_t i = 0; i < 2 * n; i++) r[i] = b[i] - r[i];
    } else {
        memset(x, 0, bytes);
        memcpy(r, b, bytes);
    }
    double nb = nrm(&A, b);
    if (nb == 0.0) { status = ST_ZERO_RHS; goto done; }
    memcpy(p, r, bytes);
    cplx rho = dotu(&A, r, r);
    hist[0] = nrm(&A, r) / nb;
    if (!isfinite(hist[0])) { status = ST_NONFINITE; goto done; }
    if (hist[0] <= tol) { status = ST_CONVERGED; goto done_true; }
    for (int32_t j = 1; j <= maxit; j++) {
        spmv(&A, p, q);                                        /* q = A p */
        cplx mu = dotu(&A, p, q);                              /* μ = pᵀ q */
        if (!cfinite(mu)) { status = ST_NONFINITE; break; }
        if (mu.re == 0.0 && mu.im == 0.0) { status = ST_BREAKDOWN_SIGMA; break; }
        cplx alpha = cdiv(rho, mu);                            /* α = ρ/μ */
        for (int64_t i = 0; i < n; i++) {                      /* x += α p ; r −= α q */
            cplx pv = {RE(p, i), IM(p, i)}, qv = {RE(q, i), IM(q, i)};
            cplx ap = cmul(alpha, pv), aq = cmul(alpha, qv);
            RE(x, i) += ap.re;
            IM(x, i) += ap.im;
            RE(r, i) -= aq.re;
            IM(r, i) -= aq.im;
        }
        double rn2 = oracle_sumsq(n, r, order);
        hist[j] = sqrt(rn2) / nb;
        *iters = j;
        if (!isfinite(hist[j])) { status = ST_NONFINITE; break; }
        if (hist[j] <= tol) { status = ST_CONVERGED; break; }
        cplx rho_new = dotu(&A, r, r);                         /* ρ' = rᵀ r */
        if (!cfinite(rho_new)) { status = ST_NONFINITE; break; }
        if (cabs_(rho_new) <= 1e-30 * rn2) { status = ST_BREAKDOWN_RHO; break; }
        cplx beta = cdiv(rho_new, rho);                        /* p = r + (ρ'/ρ) p */
        for (int64_t i = 0; i < n; i++) {
            cplx pv = {RE(p, i), IM(p, i)};
            cplx bp = cmul(beta, pv);
            RE(p, i) = RE(r, i) + bp.re;
            IM(p, i) = IM(r, i) + bp.im;
        }
        rho = rho_new;
    }
done_true:
    *out_true_relres = true_relres(&A, b, x, nb, q);
done:
    free(r); free(p); free(q);
    return status;
}

/*
 * NEXT-2: TFQMR (Freund 1993), the paper's "P-TFQMR" without preconditioner (§4 P:308,
 * Tables 9/10), in Kelley's two-half-step form ("Iterative Methods for Linear and
 * Nonlinear Equations", Alg. tfqmr), complex arithmetic with the Hermitian product, r̃ = r0:
 *   w = y1 = r0; u1 = v = A y1; d = 0; τ = ‖r0‖; θ = η = 0; ρ = ⟨r̃, r0⟩
 *   outer iteration k = 1, 2, ...:
 *     σ = ⟨r̃, v⟩ (0 → BREAKDOWN_SIGMA); α = ρ/σ; y2 = y1 − α v; u2 = A y2
 *     half steps j = 1, 2 (m = 2k − 2 + j):
 *        w = w − α u_j; d = y_j + (θ² η / α) d; θ = ‖w‖/τ; c = (1 + θ²)^(-1/2); τ = τ θ c;
 *        η = c² α; x = x + η d;  converged if τ √(m+1) / ‖b‖ ≤ tol (the quasi-residual bound, an
 *        upper bound on ‖r_m‖/‖b‖) → iters = k (a first-half-step exit counts as one)
 *     ρ' = ⟨r̃, w⟩ (|ρ'| ≤ 1e-30‖r̃‖‖w‖ → BREAKDOWN_RHO); β = ρ'/ρ; ρ = ρ'
 *     y1 = w + β y2; u1 = A y1; v = u1 + β (u2 + β v)
 *   hist[k] = τ √(2k+1)/‖b‖ after the second half step (hist[0] = 1 for x0 = 0... = ‖r0‖/‖b‖),
 *   or the first half step's bound on a half-step exit.  θ, c, τ are real; α, β, ρ, σ, η complex.
 */
int oracle_tfqmr(int64_t n, const int64_t* row_ptr, const int32_t* col, const double* val, const double* b,
                 const double* x0, double tol, int32_t maxit, int order, double* x, int32_t* iters,
                 double* hist, double* out_true_relres) {
    csr_t A = {n, row_ptr, col, val, order};
    size_t bytes = (size_t)(2 * n) * sizeof(double);
    double *r = malloc(bytes), *w = malloc(bytes), *y1 = malloc(bytes), *y2 = malloc(bytes), *u1 = malloc(bytes),
           *u2 = malloc(bytes), *v = malloc(bytes), *d = malloc(bytes), *rt = malloc(bytes);
    int status = ST_MAXIT;
    *iters = 0;
    *out_true_relres = NAN;
    if (x0) {
        memcpy(x, x0, bytes);
        spmv(&A, x, r);
        for (int64_t i = 0; i < 2 * n; i++) r[i] = b[i] - r[i];
    } else {
        memset(x, 0, bytes);
        memcpy(r, b, bytes);
    }
    double nb = nrm(&A, b);
    if (nb == 0.0) { status = ST_ZERO_RHS; goto done; }
    double tau = nrm(&A, r);
    hist[0] = tau / nb;
    if (!isfinite(hist[0])) { status = ST_NONFINITE; goto done; }
    if (hist[0] <= tol) { status = ST_CONVERGED; goto done_true; }
    memcpy(w, r, bytes);
    memcpy(y1, r, bytes);
    memcpy(rt, r, bytes);
    spmv(&A, y1, u1);                                          /* u1 = v = A y1 */
    memcpy(v, u1, bytes);
    memset(d, 0, bytes);
    double theta = 0.0, nrt = tau;
    cplx eta = {0, 0};
    cplx rho = dotc(&A, rt, r);
    for (int32_t k = 1; k <= maxit; k++) {
        cplx sigma = dotc(&A, rt, v);                          /* σ = ⟨r̃, v⟩ */
        if (!cfinite(sigma)) { status = ST_NONFINITE; break; }
        if (sigma.re == 0.0 && sigma.im == 0.0) { status = ST_BREAKDOWN_SIGMA; break; }
        cplx alpha = cdiv(rho, sigma);                         /* α = ρ/σ */
        for (int64_t i = 0; i < n; i++) {                      /* y2 = y1 − α v */
            cplx vv = {RE(v, i), IM(v, i)};
            cplx av = cmul(alpha, vv);
            RE(y2, i) = RE(y1, i) - av.re;
            IM(y2, i) = IM(y1, i) - av.im;
        }
        spmv(&A, y2, u2);                                      /* u2 = A y2 */
        int conv = 0;
        for (int j = 1; j <= 2 && !conv; j++) {
            const int m = 2 * k - 2 + j;
            const double* yj = j == 1 ? y1 : y2;
            const double* uj = j == 1 ? u1 : u2;
            cplx coef = cdiv(make_cplx_real(theta * theta), alpha);   /* θ² η / α */
            coef = cmul(coef, eta);
            for (int64_t i = 0; i < n; i++) {                  /* w −= α u_j ; d = y_j + coef d */
                cplx uv = {RE(uj, i), IM(uj, i)}, dv = {RE(d, i), IM(d, i)};
                cplx au = cmul(alpha, uv), cd = cmul(coef, dv);
                RE(w, i) -= au.re;
                IM(w, i) -= au.im;
                RE(d, i) = RE(yj, i) + cd.re;
                IM(d, i) = IM(yj, i) + cd.im;
            }
            theta = nrm(&A, w) / tau;                          /* θ = ‖w‖/τ */
            double c = 1.0 / sqrt(1.0 + theta * theta);
            tau = tau * theta * c;
            eta.re = c * c * alpha.re;                          /* η = c² α */
            eta.im = c * c * alpha.im;
            for (int64_t i = 0; i < n; i++) {                  /* x += η d */
                cplx dv = {RE(d, i), IM(d, i)};
                cplx ed = cmul(eta, dv);
                RE(x, i) += ed.re;
                IM(x, i) += ed.im;
            }
            double bound = tau * sqrt((double)m + 1.0) / nb;
            if (!isfinite(bound)) { status = ST_NONFINITE; conv = 2; break; }
            if (j == 2 || bound <= tol) hist[k] = bound;
            if (bound <= tol) conv = 1;
        }
        *iters = k;
        if (conv == 2) break;
        if (conv == 1) { status = ST_CONVERGED; break; }
        cplx rho_new = dotc(&A, rt, w);                        /* ρ' = ⟨r̃, w⟩ */
        if (!cfinite(rho_new)) { status = ST_NONFINITE; break; }
        if (cabs_(rho_new) <= 1e-30 * nrt * nrm(&A, w)) { status = ST_BREAKDOWN_RHO; break; }
        cplx beta = cdiv(rho_new, rho);
        rho = rho_new;
        for (int64_t i = 0; i < n; i++) {                      /* y1 = w + β y2 */
            cplx yv = {RE(y2, i), IM(y2, i)};
            cplx by = cmul(beta, yv);
            RE(y1, i) = RE(w, i) + by.re;
            IM(y1, i) = IM(w, i) + by.im;
        }
        spmv(&A, y1, u1);                                      /* u1 = A y1 */
        for (int64_t i = 0; i < n; i++) {                      /* v = u1 + β (u2 + β v) */
            cplx vv = {RE(v, i), IM(v, i)}, u2v = {RE(u2, i), IM(u2, i)};
            cplx bv = cmul(beta, vv);
            cplx t = {u2v.re + bv.re, u2v.im + bv.im};
            cplx bt = cmul(beta, t);
            RE(v, i) = RE(u1, i) + bt.re;
            IM(v, i) = IM(u1, i) + bt.im;
        }
    }
done_true:
    *out_true_relres = true_relres(&A, b, x, nb, u2);
done:
    free(r); free(w); free(y1); free(y2); free(u1); free(u2); free(v); free(d); free(rt);
    return status;
}

/*
 * NEXT-3: BiCGStab(ℓ) (Sleijpen & Fokkema 1993), the paper's "P-BiCGSTAB parametered (l)" /
 * "P-BiCGSTAB(8)" without preconditioner (§4, T9/T10 headers),
 * complex arithmetic with the Hermitian product ⟨x, y⟩ = Σ conj(x_i) y_i, r̃ = r0.
 * One outer cycle k (2ℓ SpMVs; hist/iters count cycles, SURVEY.md §8 A2 / T9-T10 "#iter"):
 *   ρ0 = −ω ρ0
 *   BiCG part, j = 0..ℓ−1:
 *     ρ1 = ⟨r̃, r̂_j⟩ (|ρ1| ≤ 1e-30‖r̃‖‖r̂_j‖ → BREAKDOWN_RHO); β = α ρ1 / ρ0; ρ0 = ρ1
 *     û_i = r̂_i − β û_i (i = 0..j);  û_{j+1} = A û_j
 *     γ = ⟨r̃, û_{j+1}⟩ (|γ| ≤ 1e-30‖r̃‖‖û_{j+1}‖ → BREAKDOWN_SIGMA); α = ρ0 / γ
 *     r̂_i = r̂_i − α û_{i+1} (i = 0..j);  x̂ = x̂ + α û_0
 *     ‖r̂_0‖/‖b‖ ≤ tol → CONVERGED inside the cycle (BiCGStab's half-step test, L6)
 *     r̂_{j+1} = A r̂_j
 *   MR part ("coefficients solve the l×l least-squares system of inner products"):
 *     G_ij = ⟨r̂_i, r̂_j⟩ (i, j = 0..ℓ); solve G[1..ℓ,1..ℓ] γ = G[1..ℓ,0] by Cholesky (a non-positive
 *     or non-finite pivot → BREAKDOWN_OMEGA); ω = γ_ℓ
 *     x̂ = x̂ + Σ_j γ_j r̂_{j−1};  r̂_0 = r̂_0 − Σ_j γ_j r̂_j;  û_0 = û_0 − Σ_j γ_j û_j   (j = 1..ℓ)
 *   hist[k] = ‖r̂_0‖/‖b‖; converged if ≤ tol; |ω| ≤ 1e-30 → BREAKDOWN_OMEGA.
 * Start: x̂ = x0, r̂_0 = b − A x0, û_0 = 0, ρ0 = 1, α = 0, ω = 1.  *iters = the cycle in which the
 * loop ended (an exit inside a cycle, convergence or breakdown, counts that cycle).  With ℓ = 1 this is BiCGStab
 * (O6) up to rounding (pinned in tests/test_oracle_solvers.py).  ℓ ∈ [1, 8].
 */
int oracle_bicgstab_l(int64_t n, const int64_t* row_ptr, const int32_t* col, const double* val, const double* b,
                      const double* x0, double tol, int32_t maxit, int order, int ell, double* x, int32_t* iters,
                      double* hist, double* out_true_relres) {
    csr_t A = {n, row_ptr, col, val, order};
    if (ell < 1 || ell > 8) return -1;
    size_t bytes = (size_t)(2 * n) * sizeof(double);
    double* rr[9];
    double* uu[9];
    for (int i = 0; i <= ell; i++) {
        rr[i] = malloc(bytes);
        uu[i] = calloc((size_t)(2 * n), sizeof(double));
    }
    double* rt = malloc(bytes);
    int status = ST_MAXIT;
    *iters = 0;
    *out_true_relres = NAN;
    double* r = rr[0];
    if (x0) {
        memcpy(x, x0, bytes);
        spmv(&A, x, r);
        for (int64_t i = 0; i < 2 * n; i++) r[i] = b[i] - r[i];
    } else {
        memset(x, 0, bytes);
        memcpy(r, b, bytes);
    }
    double nb = nrm(&A, b);
    if (nb == 0.0) { status = ST_ZERO_RHS; goto done; }
    double rnorm = nrm(&A, r);
    hist[0] = rnorm / nb;
    if (!isfinite(hist[0])) { status = ST_NONFINITE; goto done; }
    if (hist[0] <= tol) { status = ST_CONVERGED; goto done_true; }
    memcpy(rt, r, bytes);
    double nrt = rnorm;
    cplx rho0 = {1, 0}, alpha = {0, 0}, omega = {1, 0};
    for (int32_t k = 1; k <= maxit; k++) {
        *iters = k;                                                 /* an exit inside a cycle counts it */
        cplx mw = {-omega.re, -omega.im};
        rho0 = cmul(mw, rho0);                                      /* ρ0 = −ω ρ0 */
        for (int j = 0; j < ell; j++) {
            cplx rho1 = dotc(&A, rt, rr[j]);                        /* ρ1 = ⟨r̃, r̂_j⟩ */
            if (!cfinite(rho1)) { status = ST_NONFINITE; goto done_true; }
            if (cabs_(rho1) <= 1e-30 * nrt * nrm(&A, rr[j])) { status = ST_BREAKDOWN_RHO; goto done_true; }
            cplx beta = cdiv(cmul(alpha, rho1), rho0);              /* β = α ρ1 / ρ0 */
            rho0 = rho1;
            for (int i = 0; i <= j; i++)                            /* û_i = r̂_i − β û_i */
                for (int64_t e = 0; e < n; e++) {
                    cplx uv = {RE(uu[i], e), IM(uu[i], e)};
                    cplx bu = cmul(beta, uv);
                    RE(uu[i], e) = RE(rr[i], e) - bu.re;
                    IM(uu[i], e) = IM(rr[i], e) - bu.im;
                }
            spmv(&A, uu[j], uu[j + 1]);                             /* û_{j+1} = A û_j */
            cplx gam = dotc(&A, rt, uu[j + 1]);                     /* γ = ⟨r̃, û_{j+1}⟩ */
            if (!cfinite(gam)) { status = ST_NONFINITE; goto done_true; }
            if (cabs_(gam) <= 1e-30 * nrt * nrm(&A, uu[j + 1])) { status = ST_BREAKDOWN_SIGMA; goto done_true; }
            alpha = cdiv(rho0, gam);                                /* α = ρ0 / γ */
            for (int i = 0; i <= j; i++)                            /* r̂_i = r̂_i − α û_{i+1} */
                for (int64_t e = 0; e < n; e++) {
                    cplx uv = {RE(uu[i + 1], e), IM(uu[i + 1], e)};
                    cplx au = cmul(alpha, uv);
                    RE(rr[i], e) -= au.re;
                    IM(rr[i], e) -= au.im;
                }
            for (int64_t e = 0; e < n; e++) {                       /* x̂ = x̂ + α û_0 */
                cplx uv = {RE(uu[0], e), IM(uu[0], e)};
                cplx au = cmul(alpha, uv);
                RE(x, e) += au.re;
                IM(x, e) += au.im;
            }
            double rn = nrm(&A, rr[0]);
            if (!isfinite(rn)) { status = ST_NONFINITE; goto done_true; }
            if (rn / nb <= tol) {                                   /* exit inside the cycle */
                hist[k] = rn / nb;
                status = ST_CONVERGED;
                goto done_true;
            }
            spmv(&A, rr[j], rr[j + 1]);                             /* r̂_{j+1} = A r̂_j */
        }
        /* MR part: G_ij = ⟨r̂_i, r̂_j⟩ ; M γ = g with M = G[1..ℓ,1..ℓ], g_i = G[i][0] */
        cplx G[9][9];
        for (int i = 0; i <= ell; i++)
            for (int j = i; j <= ell; j++) {
                G[i][j] = dotc(&A, rr[i], rr[j]);
                cplx c = {G[i][j].re, -G[i][j].im};
                G[j][i] = c;
            }
        /* Cholesky M = L Lᴴ (L lower, real positive diagonal), written out */
        cplx L[8][8];
        int bad = 0;
        for (int j = 0; j < ell && !bad; j++) {
            double dsum = G[j + 1][j + 1].re;
            for (int q = 0; q < j; q++) dsum -= L[j][q].re * L[j][q].re + L[j][q].im * L[j][q].im;
            if (!(dsum > 0.0) || !isfinite(dsum)) { bad = 1; break; }
            double ljj = sqrt(dsum);
            L[j][j] = make_cplx_real(ljj);
            for (int i = j + 1; i < ell; i++) {
                cplx s = G[i + 1][j + 1];
                for (int q = 0; q < j; q++) {                       /* s −= L_iq conj(L_jq) */
                    cplx cj = {L[j][q].re, -L[j][q].im};
                    cplx t = cmul(L[i][q], cj);
                    s.re -= t.re;
                    s.im -= t.im;
                }
                L[i][j].re = s.re / ljj;
                L[i][j].im = s.im / ljj;
            }
        }
        if (bad) { status = ST_BREAKDOWN_OMEGA; goto done_true; }
        cplx y[8], gm[9];
        for (int i = 0; i < ell; i++) {                             /* L y = g */
            cplx s = G[i + 1][0];
            for (int q = 0; q < i; q++) {
                cplx t = cmul(L[i][q], y[q]);
                s.re -= t.re;
                s.im -= t.im;
            }
            y[i].re = s.re / L[i][i].re;
            y[i].im = s.im / L[i][i].re;
        }
        for (int i = ell - 1; i >= 0; i--) {                        /* Lᴴ γ = y */
            cplx s = y[i];
            for (int q = i + 1; q < ell; q++) {                     /* s −= conj(L_qi) γ_q */
                cplx cq = {L[q][i].re, -L[q][i].im};
                cplx t = cmul(cq, gm[q + 1]);
                s.re -= t.re;
                s.im -= t.im;
            }
            gm[i + 1].re = s.re / L[i][i].re;
            gm[i + 1].im = s.im / L[i][i].re;
        }
        omega = gm[ell];                                            /* ω = γ_ℓ */
        for (int64_t e = 0; e < n; e++) {
            double xr = RE(x, e), xi = IM(x, e), r0r = RE(rr[0], e), r0i = IM(rr[0], e);
            double u0r = RE(uu[0], e), u0i = IM(uu[0], e);
            for (int j = 1; j <= ell; j++) {
                cplx rp = {RE(rr[j - 1], e), IM(rr[j - 1], e)}, rj = {RE(rr[j], e), IM(rr[j], e)};
                cplx uj = {RE(uu[j], e), IM(uu[j], e)};
                cplx a = cmul(gm[j], rp), c = cmul(gm[j], rj), d = cmul(gm[j], uj);
                xr += a.re; xi += a.im;                             /* x̂ += γ_j r̂_{j−1} */
                r0r -= c.re; r0i -= c.im;                           /* r̂_0 −= γ_j r̂_j   */
                u0r -= d.re; u0i -= d.im;                           /* û_0 −= γ_j û_j   */
            }
            RE(x, e) = xr; IM(x, e) = xi;
            RE(rr[0], e) = r0r; IM(rr[0], e) = r0i;
            RE(uu[0], e) = u0r; IM(uu[0], e) = u0i;
        }
        rnorm = nrm(&A, rr[0]);
        hist[k] = rnorm / nb;
        if (!isfinite(hist[k]) || !cfinite(omega)) { status = ST_NONFINITE; break; }
        if (hist[k] <= tol) { status = ST_CONVERGED; break; }
        if (cabs_(omega) <= 1e-30) { status = ST_BREAKDOWN_OMEGA; break; }
    }
done_true:
    *out_true_relres = true_relres(&A, b, x, nb, uu[1]);
done:
    for (int i = 0; i <= ell; i++) { free(rr[i]); free(uu[i]); }
    free(rt);
    return status;
}
