/*
 * helmholtz_gen.c — seeded synthetic input generator (shared by the CUDA path's
 * tests/bench and by the CPU oracle's tests).  It holds NONE of the solver's
 * arithmetic (no SpMV, no dot, no Krylov step): it only writes the CSR arrays
 * of the discretised operator, following SURVEY.md Appendix A.
 *
 * What it builds (the input recipe of DESIGN.md §"Inputs"):
 *   Q1 (trilinear) hexahedral finite elements on a node box Nx×Ny×Nz with
 *   spacing h, for the Helmholtz operator of PAPER.md §1 (P:23,
 *   "-∇²u - k²u = g", k = 2π/λ) with the absorbing term of the north star:
 *         A = K − (1 + iη)·k²·M.
 *   On a uniform grid K and M are Kronecker sums/products of the 1-D P1
 *   matrices  K1 = (1/h)·tridiag(−1,2,−1),  M1 = (h/6)·tridiag(1,4,1):
 *         K = Kz⊗My⊗Mx + Mz⊗Ky⊗Mx + Mz⊗My⊗Kx,   M = Mz⊗My⊗Mx,
 *   so the entry for node offset (dx,dy,dz) ∈ {−1,0,1}³ is
 *         k(dz)m(dy)m(dx) + m(dz)k(dy)m(dx) + m(dz)m(dy)k(dx)
 *       − (1+iη)k²·m(dx)m(dy)m(dz),
 *   with k(0)=2/h, k(±1)=−1/h, m(0)=2h/3, m(±1)=h/6.
 *   Dirichlet nodes ("Dirichlet boundary conditions along a part
 *   of Γ") are eliminated symmetrically: their columns are dropped from free
 *   rows and, when `shell` is set, they stay in the numbering as identity rows
 *   with value d = Re(interior diagonal) = 8h/3.  `pad`
 *   further identity rows are appended so n matches PAPER.md Table 1.
 *   Numbering is x fastest: id = ix + Nx·(iy + Ny·iz).
 *   Structural zeros are kept (face-neighbour stiffness is exactly 0; L21).
 *
 *   Optional gauge twist: entry (i,j) is multiplied by
 *   e^{i(φ_i − φ_j)}; φ is passed in (drawn by the Python wrapper from a
 *   seeded numpy generator).  With η = 0 this gives a Hermitian positive
 *   definite matrix with fully complex off-diagonals.
 *
 * Rows [row_begin,row_end) can be generated on their own (one rank's slab).
 */
#include <stdint.h>
#include <math.h>
#include <string.h>

typedef struct {
    int64_t nx, ny, nz;   /* node box */
    int64_t shell;        /* 1: boundary nodes are identity rows; 0: box = free nodes only */
    int64_t pad;          /* identity rows appended after the box */
    double h, k, eta;
} gen_box;

static int64_t box_nodes(const gen_box* g) { return g->nx * g->ny * g->nz; }

int64_t gen_n_rows(const gen_box* g) { return box_nodes(g) + g->pad; }

static int axis_free(int64_t i, int64_t n, int64_t shell) {
    return shell ? (i >= 1 && i <= n - 2) : (i >= 0 && i <= n - 1);
}

/* number of free neighbours (incl. self) of free coordinate i along one axis */
static int64_t axis_count(int64_t i, int64_t n, int64_t shell) {
    int64_t c = 1;
    if (axis_free(i - 1, n, shell)) c++;
    if (axis_free(i + 1, n, shell)) c++;
    return c;
}

static int row_is_free(const gen_box* g, int64_t row, int64_t* ix, int64_t* iy, int64_t* iz) {
    if (row >= box_nodes(g)) return 0;
    *ix = row % g->nx;
    *iy = (row / g->nx) % g->ny;
    *iz = row / (g->nx * g->ny);
    return axis_free(*ix, g->nx, g->shell) && axis_free(*iy, g->ny, g->shell) &&
           axis_free(*iz, g->nz, g->shell);
}

int64_t gen_row_nnz(const gen_box* g, int64_t row) {
    int64_t ix, iy, iz;
    if (!row_is_free(g, row, &ix, &iy, &iz)) return 1;
    return axis_count(ix, g->nx, g->shell) * axis_count(iy, g->ny, g->shell) *
           axis_count(iz, g->nz, g->shell);
}

/* row_ptr[0..m] for rows [r0,r1), local (row_ptr[0] = 0); returns nnz */
int64_t gen_row_ptr(const gen_box* g, int64_t r0, int64_t r1, int64_t* row_ptr) {
    int64_t m = r1 - r0;
    row_ptr[0] = 0;
    for (int64_t i = 0; i < m; i++) row_ptr[i + 1] = row_ptr[i] + gen_row_nnz(g, r0 + i);
    return row_ptr[m];
}

/* stencil value for offset (dx,dy,dz) */
static void stencil(const gen_box* g, int dx, int dy, int dz, double* re, double* im,
                    double* kstiff) {
    const double h = g->h;
    double k1[3] = {-1.0 / h, 2.0 / h, -1.0 / h};
    double m1[3] = {h / 6.0, 2.0 * h / 3.0, h / 6.0};
    double K = k1[dz + 1] * m1[dy + 1] * m1[dx + 1] + m1[dz + 1] * k1[dy + 1] * m1[dx + 1] +
               m1[dz + 1] * m1[dy + 1] * k1[dx + 1];
    double M = m1[dx + 1] * m1[dy + 1] * m1[dz + 1];
    double k2 = g->k * g->k;
    *re = K - k2 * M;
    *im = -g->eta * k2 * M;
    *kstiff = K;
}

/* Fill rows [r0,r1).  row_ptr must come from gen_row_ptr over the same range.
 * val is interleaved (re,im).  phase: NULL or n_rows gauge angles. */
void gen_fill(const gen_box* g, int64_t r0, int64_t r1, const int64_t* row_ptr, int32_t* col,
              double* val, const double* phase) {
    double st_re[27], st_im[27], st_k[27];
    for (int dz = -1; dz <= 1; dz++)
        for (int dy = -1; dy <= 1; dy++)
            for (int dx = -1; dx <= 1; dx++) {
                int s = (dz + 1) * 9 + (dy + 1) * 3 + (dx + 1);
                stencil(g, dx, dy, dz, &st_re[s], &st_im[s], &st_k[s]);
            }
    const double d_ident = st_k[13]; /* 8h/3: real stiffness diagonal (identity rows, L15) */
#pragma omp parallel for schedule(static)
    for (int64_t r = r0; r < r1; r++) {
        int64_t p = row_ptr[r - r0];
        int64_t ix, iy, iz;
        if (!row_is_free(g, r, &ix, &iy, &iz)) {
            col[p] = (int32_t)r;
            val[2 * p] = d_ident;
            val[2 * p + 1] = 0.0;
            continue;
        }
        for (int dz = -1; dz <= 1; dz++) {
            if (!axis_free(iz + dz, g->nz, g->shell)) continue;
            for (int dy = -1; dy <= 1; dy++) {
                if (!axis_free(iy + dy, g->ny, g->shell)) continue;
                for (int dx = -1; dx <= 1; dx++) {
                    if (!axis_free(ix + dx, g->nx, g->shell)) continue;
                    int64_t c = (ix + dx) + g->nx * ((iy + dy) + g->ny * (iz + dz));
                    int s = (dz + 1) * 9 + (dy + 1) * 3 + (dx + 1);
                    double re = st_re[s], im = st_im[s];
                    if (phase) {
                        double t = phase[r] - phase[c];
                        double cr = cos(t), ci = sin(t);
                        double nr = re * cr - im * ci;
                        double ni = re * ci + im * cr;
                        re = nr;
                        im = ni;
                    }
                    col[p] = (int32_t)c;
                    val[2 * p] = re;
                    val[2 * p + 1] = im;
                    p++;
                }
            }
        }
    }
}

/* 1 where the row is a free (PDE) row, 0 for identity rows */
void gen_free_mask(const gen_box* g, int64_t r0, int64_t r1, uint8_t* mask) {
#pragma omp parallel for schedule(static)
    for (int64_t r = r0; r < r1; r++) {
        int64_t ix, iy, iz;
        mask[r - r0] = (uint8_t)row_is_free(g, r, &ix, &iy, &iz);
    }
}
