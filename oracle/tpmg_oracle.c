/*
 * tpmg_oracle.c -- CPU ORACLE.  TEST INFRASTRUCTURE ONLY.
 *
 * Plain, slow, obviously-correct fp64 implementation of what the paper's
 * hot path computes (Mueller, Scheichl, Vainikko, "Petascale elliptic solvers
 * for anisotropic PDEs on GPU clusters", arXiv:1402.3545).  Line citations
 * "P:n" refer to /root/reference/PAPER.md, "S:n" to SPEC.md.
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
 * --impl reference legs may load this library.  It shares no code, header,
 * table or constant generator with the CUDA product path
 * (paper_1402_3545_b200/); the two meet only through the seeded inputs of
 * inputs/ and through the tests that compare them.
 *
 * Conventions
 *   - Fields are stored z-contiguous (the CPU-friendly ordering of P:59):
 *       ZC(i,j,k) = (j*nx + i)*nz + k,  0 <= i < nx, 0 <= j < ny, 0 <= k < nz.
 *     The paper's 1-based horizontal indices (i,j) in [1,nx]x[1,ny]
 *     map to i-1, j-1 here.
 *   - Level index l: l = L is the finest, l = 1 the coarsest.
 *   - Built with -ffp-contract=off: every multiply and add is rounded
 *     separately, in the order written.
 *   - Reductions are deterministic: each horizontal row j is summed serially
 *     in (i,k) order, then the row sums are added serially in j order.
 *
 * Readings of the paper where it is silent or garbled are listed in
 * DESIGN.md section "Readings"; each is cited at the point of use as [Rn].
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

#define OR_OK 0
#define OR_E_PARAM 1
#define OR_E_SHAPE 2
#define OR_E_SINGULAR 4
#define OR_E_BREAKDOWN 5
#define OR_E_OOM 9

/* ------------------------------------------------------------------------ */
/* Operator of one multigrid level, in the notation of eqn:LocalMatrixStencil
 * (P:250-256):
 *     A_{T,T'} = alpha_{T,T'} diag(d)
 *     A_T      = |T| diag(a) - alpha_T diag(d) + |T| tridiag(-(b+c), b, c)
 * For the flat box of P:140-150 every column has the same scalars:
 *     |T| = 1,  a_k = d_k = 1,
 *     alpha_{T,T'} = -omega^2/h_l^2           ("A_{(i,j),(i',j')} = -omega^2/h^2 I")
 *     alpha_T      = sum over the 4 faces of alpha_{T,T'} = -4 omega^2/h_l^2
 *                    (including boundary faces: ghost value 0 Dirichlet [R1]);
 *                    with boundary = 1 (face Dirichlet [R25]) a boundary face counts
 *                    twice (the face is h_l/2 from the cell centre), so a column with
 *                    nb boundary faces has alpha_T = (4 + nb) alpha_{T,T'}
 *     b_k = -omega^2 lambda^2/h_z^2 for k > 0, b_0 = 0          (Neumann)
 *     c_k = -omega^2 lambda^2/h_z^2 for k < nz-1, c_{nz-1} = 0
 * so that the interior diagonal is 1 + 4 omega^2/h^2 + 2 omega^2 lambda^2/h_z^2
 * and the vertical off-diagonals are -omega^2 lambda^2/h_z^2, exactly P:150.
 * tridiag(-(b+c), b, c): b multiplies u_{k-1}, c multiplies u_{k+1}. */
typedef struct {
    long nx, ny;      /* horizontal cells of this level (whole domain) */
    int nz;           /* vertical levels (never coarsened) */
    double area;      /* |T| */
    double alpha_TT;  /* alpha_{T,T'} */
    double alpha_T;   /* alpha_T of an interior column */
    int boundary;     /* 0: ghost-zero Dirichlet [R1]; 1: face Dirichlet [R25] */
    double *a, *b, *c, *d; /* vertical profiles, length nz */
    /* per-column horizontal fields of this level ("|T|, alpha_{T,T'} and alpha_T are
     * different for each horizontal grid cell T (and depend on the multigrid level)"), or NULL
     * for the flat box (the scalars above):
     *   fa[j*nx + i]      = |T| of column (i,j)
     *   fx[j*(nx+1) + i]  = alpha_{T,T'} of the x-face between columns (i-1,j) and (i,j),
     *                       i = 0..nx (faces 0 and nx lie on the boundary)
     *   fy[j*nx + i]      = alpha_{T,T'} of the y-face between columns (i,j-1) and (i,j),
     *                       j = 0..ny (faces 0 and ny lie on the boundary) */
    double *fa, *fx, *fy;
} or_op;

/* alpha_T of column (i,j) ("alpha_T ... different for each horizontal grid cell").
 * [R1]: every column has 4 alpha_{T,T'}.  [R25] (face Dirichlet, the cell-centred
 * finite-volume boundary of P:131 and P:139): the flux through a boundary face is
 * omega^2 (0 - u_T)/(h/2), i.e. 2 alpha_{T,T'} per boundary face. */
static inline double or_alpha_T(const or_op *op, long i, long j)
{
    if (op->fa) {   /* per-column fields: alpha_T = sum over the 4 faces of alpha_{T,T'} [R1];
                     * [R25] counts a boundary face twice */
        const long nx = op->nx, ny = op->ny;
        double w = op->fx[j * (nx + 1) + i], e = op->fx[j * (nx + 1) + i + 1];
        double s = op->fy[j * nx + i], n = op->fy[(j + 1) * nx + i];
        double aT = w + e + s + n;
        if (op->boundary) {
            if (i == 0) aT += w;
            if (i == nx - 1) aT += e;
            if (j == 0) aT += s;
            if (j == ny - 1) aT += n;
        }
        return aT;
    }
    if (!op->boundary) return op->alpha_T;
    int nb = (i == 0) + (i == op->nx - 1) + (j == 0) + (j == op->ny - 1);
    return op->alpha_T + (double)nb * op->alpha_TT;
}

static inline size_t ZC(const or_op *op, long i, long j, long k)
{
    return ((size_t)j * (size_t)op->nx + (size_t)i) * (size_t)op->nz + (size_t)k;
}

/* Problem parameters (defaults P:415-418 and [R3]). */
typedef struct {
    long nx, ny;      /* global horizontal cells of the finest level */
    int nz;
    double nu_cfl;    /* nu_CFL, omega = nu h / 2 (eqn:OmegaNumerical) */
    double H;         /* depth ratio; h_z = H / nz */
    double lambda;
    int L;            /* multigrid levels */
    int pre, post;    /* smoothing steps (1 and 1) */
    int coarse_sweeps;/* smoother iterations on the coarsest level (2) */
    double rho;       /* rho_relax = 2/3 */
    int boundary;     /* horizontal Dirichlet reading: 0 = ghost zero [R1], 1 = face [R25] */
    /* vertical profiles a, b, c, d of eqn:LocalMatrixStencil, length nz, in the
     * units of A (b, c include omega^2 lambda^2 / h_z^2, d multiplies alpha_{T,T'});
     * NULL: the flat-box values [R2].  Requirements (a symmetric, diagonally dominant
     * column block): b_0 = 0, c_{nz-1} = 0, b_{k+1} = c_k, a >= 0, b <= 0, c <= 0, d > 0. */
    const double *prof_a, *prof_b, *prof_c, *prof_d;
    /* per-column horizontal fields of the FINEST level, or NULL for the flat box:
     * field_area[ny][nx] = |T| > 0, field_ax[ny][nx+1] and field_ay[ny+1][nx] = alpha_{T,T'}
     * <= 0 of the x- and y-faces (layout of or_op.fa/fx/fy, global indices).  Coarser
     * levels follow reading [R26] (or_op_init). */
    const double *field_area, *field_ax, *field_ay;
} or_params;

/* Per-column fields of level l from the finest level's (reading [R26]): with
 * s = L - l and F = 2^s fine columns per coarse column and direction,
 *   |T|_l(I,J)        = (1/F^2) sum of |T|_L over the F x F fine columns of (I,J)
 *                       (the mean: |T| is normalised, the flat box has |T| = 1 on every level),
 *   alpha_l(x-face I) = 8^-s  sum of alpha_L over the F fine x-faces on that face
 *   alpha_l(y-face J) = 8^-s  sum of alpha_L over the F fine y-faces on that face.
 * One level down, a face has 2 fine faces: the mean coefficient (1/2), times the
 * normalised-area ratio of the rediscretisation (1/4) [R4]; so constant fields |T| = 1,
 * alpha = -omega^2/h^2 give exactly the flat box's alpha_{T,T'} = -omega^2/h_l^2. */
static int or_fields_init(const or_params *p, int l, or_op *op)
{
    const long F = 1L << (p->L - l), nxf = p->nx, nx = p->nx / F, ny = p->ny / F;
    if (!p->field_ax || !p->field_ay) return OR_E_PARAM;
    for (long q = 0; q < nxf * p->ny; ++q)
        if (!(p->field_area[q] > 0) || !isfinite(p->field_area[q])) return OR_E_PARAM;
    for (long q = 0; q < (nxf + 1) * p->ny; ++q)
        if (!(p->field_ax[q] <= 0) || !isfinite(p->field_ax[q])) return OR_E_PARAM;
    for (long q = 0; q < nxf * (p->ny + 1); ++q)
        if (!(p->field_ay[q] <= 0) || !isfinite(p->field_ay[q])) return OR_E_PARAM;
    double scale = 1.0;
    for (int s = 0; s < p->L - l; ++s) scale /= 8.0;
    op->fa = (double *)malloc(sizeof(double) * (size_t)(nx * ny));
    op->fx = (double *)malloc(sizeof(double) * (size_t)((nx + 1) * ny));
    op->fy = (double *)malloc(sizeof(double) * (size_t)(nx * (ny + 1)));
    if (!op->fa || !op->fx || !op->fy) return OR_E_OOM;
    for (long J = 0; J < ny; ++J)
        for (long I = 0; I < nx; ++I) {
            double sum = 0.0;
            for (long b = 0; b < F; ++b)
                for (long a = 0; a < F; ++a) sum += p->field_area[(J * F + b) * nxf + I * F + a];
            op->fa[J * nx + I] = sum / (double)(F * F);
        }
    for (long J = 0; J < ny; ++J)
        for (long I = 0; I <= nx; ++I) {
            double sum = 0.0;
            for (long b = 0; b < F; ++b) sum += p->field_ax[(J * F + b) * (nxf + 1) + I * F];
            op->fx[J * (nx + 1) + I] = sum * scale;
        }
    for (long J = 0; J <= ny; ++J)
        for (long I = 0; I < nx; ++I) {
            double sum = 0.0;
            for (long a = 0; a < F; ++a) sum += p->field_ay[(J * F) * nxf + I * F + a];
            op->fy[J * nx + I] = sum * scale;
        }
    return OR_OK;
}

/* Build the operator of level l (1 <= l <= L) by rediscretisation [R4]:
 * the horizontal mesh width on level l is h_l = h * 2^(L-l) (horizontal-only
 * semicoarsening); omega, lambda and h_z are the same on every level. */
int or_op_init(const or_params *p, int l, or_op *op)
{
    memset(op, 0, sizeof(*op));   /* or_op_free is safe after any early return */
    if (p->nx <= 0 || p->ny <= 0 || p->nz <= 0 || p->L <= 0 || l < 1 || l > p->L)
        return OR_E_PARAM;
    if (!(p->nu_cfl > 0) || !(p->H > 0) || !(p->lambda > 0)) return OR_E_PARAM;
    if (p->boundary != 0 && p->boundary != 1) return OR_E_PARAM;
    long f = 1L << (p->L - l);
    if (p->nx % f || p->ny % f) return OR_E_SHAPE;
    double h = 1.0 / (double)p->nx;              /* unit square, equidistant */
    double hz = p->H / (double)p->nz;            /* h_z = H / n_z */
    double omega = 0.5 * p->nu_cfl * h;          /* eqn:OmegaNumerical */
    double hl = h * (double)f;
    double omega2 = omega * omega;
    double vert = omega2 * (p->lambda * p->lambda) / (hz * hz); /* omega^2 lambda^2 / h_z^2 */
    op->nx = p->nx / f;
    op->ny = p->ny / f;
    op->nz = p->nz;
    op->area = 1.0;
    op->alpha_TT = -omega2 / (hl * hl);
    op->alpha_T = 4.0 * op->alpha_TT;
    op->boundary = p->boundary;
    op->a = (double *)malloc(sizeof(double) * p->nz);
    op->b = (double *)malloc(sizeof(double) * p->nz);
    op->c = (double *)malloc(sizeof(double) * p->nz);
    op->d = (double *)malloc(sizeof(double) * p->nz);
    op->fa = op->fx = op->fy = NULL;
    if (!op->a || !op->b || !op->c || !op->d) return OR_E_OOM;
    if (p->field_area) {
        int st = or_fields_init(p, l, op);
        if (st != OR_OK) return st;
    }
    if (p->prof_a) {   /* general vertical profiles ("derived from the vertical
                        * stiffness- and mass-matrices"; the same on every level) */
        if (!p->prof_b || !p->prof_c || !p->prof_d) return OR_E_PARAM;
        for (int k = 0; k < p->nz; ++k) {
            if (!(p->prof_a[k] >= 0) || !(p->prof_b[k] <= 0) || !(p->prof_c[k] <= 0) || !(p->prof_d[k] > 0))
                return OR_E_PARAM;
            if (k + 1 < p->nz && p->prof_b[k + 1] != p->prof_c[k]) return OR_E_PARAM;
        }
        if (p->prof_b[0] != 0.0 || p->prof_c[p->nz - 1] != 0.0) return OR_E_PARAM;
        for (int k = 0; k < p->nz; ++k) {
            op->a[k] = p->prof_a[k];
            op->b[k] = p->prof_b[k];
            op->c[k] = p->prof_c[k];
            op->d[k] = p->prof_d[k];
        }
        return OR_OK;
    }
    for (int k = 0; k < p->nz; ++k) {
        op->a[k] = 1.0;
        op->d[k] = 1.0;
        op->b[k] = (k > 0) ? -vert : 0.0;
        op->c[k] = (k < p->nz - 1) ? -vert : 0.0;
    }
    return OR_OK;
}

void or_op_free(or_op *op)
{
    free(op->a); free(op->b); free(op->c); free(op->d);
    free(op->fa); free(op->fx); free(op->fy);
    op->a = op->b = op->c = op->d = NULL;
    op->fa = op->fx = op->fy = NULL;
}

/* ------------------------------------------------------------------------ */
/* y = A x for one column T = (i,j), eqn:TridiagonalPDE:
 *   (A x)^(T) = A_T x^(T) + sum_{T' in N(T)} A_{T,T'} x^(T'),
 * with x^(T') = 0 for T' outside the horizontal domain [R1]. */
void or_apply_col(const or_op *op, const double *x, long i, long j, double *ycol)
{
    const int nz = op->nz;
    const int has_w = i > 0, has_e = i < op->nx - 1, has_s = j > 0, has_n = j < op->ny - 1;
    const double area = op->fa ? op->fa[j * op->nx + i] : op->area;
    for (int k = 0; k < nz; ++k) {
        double xk = x[ZC(op, i, j, k)];
        /* A_T x^(T) */
        double y = area * op->a[k] * xk - or_alpha_T(op, i, j) * op->d[k] * xk
                 + area * (-(op->b[k] + op->c[k])) * xk;
        if (k > 0) y += area * op->b[k] * x[ZC(op, i, j, k - 1)];
        if (k < nz - 1) y += area * op->c[k] * x[ZC(op, i, j, k + 1)];
        /* sum_{T'} A_{T,T'} x^(T') */
        if (op->fa) {   /* per-face alpha_{T,T'} */
            const long nx = op->nx;
            double nb = 0.0;
            if (has_w) nb += op->fx[j * (nx + 1) + i] * x[ZC(op, i - 1, j, k)];
            if (has_e) nb += op->fx[j * (nx + 1) + i + 1] * x[ZC(op, i + 1, j, k)];
            if (has_s) nb += op->fy[j * nx + i] * x[ZC(op, i, j - 1, k)];
            if (has_n) nb += op->fy[(j + 1) * nx + i] * x[ZC(op, i, j + 1, k)];
            y += op->d[k] * nb;
        } else {
            double nb = 0.0;
            if (has_w) nb += x[ZC(op, i - 1, j, k)];
            if (has_e) nb += x[ZC(op, i + 1, j, k)];
            if (has_s) nb += x[ZC(op, i, j - 1, k)];
            if (has_n) nb += x[ZC(op, i, j + 1, k)];
            y += op->alpha_TT * op->d[k] * nb;
        }
        ycol[k] = y;
    }
}

/* y = A x (Kernel "SpMV", eqn:SpMVPrec). */
void or_apply(const or_op *op, const double *x, double *y)
{
#pragma omp parallel for schedule(static)
    for (long j = 0; j < op->ny; ++j)
        for (long i = 0; i < op->nx; ++i)
            or_apply_col(op, x, i, j, y + ZC(op, i, j, 0));
}

/* r = f - A u (Kernel "Residual", alg:VCycle P:197) for one column. */
void or_residual_col(const or_op *op, const double *u, const double *f, long i, long j,
                     double *rcol)
{
    or_apply_col(op, u, i, j, rcol);
    for (int k = 0; k < op->nz; ++k) rcol[k] = f[ZC(op, i, j, k)] - rcol[k];
}

void or_residual(const or_op *op, const double *u, const double *f, double *r)
{
#pragma omp parallel for schedule(static)
    for (long j = 0; j < op->ny; ++j)
        for (long i = 0; i < op->nx; ++i)
            or_residual_col(op, u, f, i, j, r + ZC(op, i, j, 0));
}

/* ------------------------------------------------------------------------ */
/* Thomas algorithm (textbook form):
 *   s: sub-diagonal (s[0] unused), dg: diagonal, t: super-diagonal (t[n-1]
 *   unused), g: right-hand side.  Solves the n x n tridiagonal system.
 *   t'_0 = t_0/dg_0, g'_0 = g_0/dg_0;
 *   m_k = dg_k - s_k t'_{k-1}, t'_k = t_k/m_k, g'_k = (g_k - s_k g'_{k-1})/m_k;
 *   x_{n-1} = g'_{n-1}, x_k = g'_k - t'_k x_{k+1}.
 * work: 2n doubles.  Returns OR_E_SINGULAR on a zero pivot. */
int or_thomas(int n, const double *s, const double *dg, const double *t, const double *g,
              double *x, double *work)
{
    double *tp = work, *gp = work + n;
    if (n <= 0) return OR_OK;
    if (dg[0] == 0.0) return OR_E_SINGULAR;
    tp[0] = (n > 1) ? t[0] / dg[0] : 0.0;
    gp[0] = g[0] / dg[0];
    for (int k = 1; k < n; ++k) {
        double m = dg[k] - s[k] * tp[k - 1];
        if (m == 0.0) return OR_E_SINGULAR;
        tp[k] = (k < n - 1) ? t[k] / m : 0.0;
        gp[k] = (g[k] - s[k] * gp[k - 1]) / m;
    }
    x[n - 1] = gp[n - 1];
    for (int k = n - 2; k >= 0; --k) x[k] = gp[k] - tp[k] * x[k + 1];
    return OR_OK;
}

/* The three diagonals of the column block A_T = M_T (M keeps only the
 * first term of eqn:TridiagonalPDE). */
static void or_block_diagonals(const or_op *op, long i, long j, double *s, double *dg, double *t)
{
    const double alpha_T = or_alpha_T(op, i, j);
    const double area = op->fa ? op->fa[j * op->nx + i] : op->area;
    for (int k = 0; k < op->nz; ++k) {
        s[k] = area * op->b[k];
        t[k] = area * op->c[k];
        dg[k] = area * op->a[k] - alpha_T * op->d[k]
              + area * (-(op->b[k] + op->c[k]));
    }
}

/* z = M^{-1} r for column (i,j) (vertical line relaxation). */
int or_precondition_col(const or_op *op, const double *rcol, long i, long j, double *zcol)
{
    const int nz = op->nz;
    double buf[5 * nz]; /* column workspace (no global temporaries) */
    double *s = buf, *dg = buf + nz, *t = buf + 2 * nz, *work = buf + 3 * nz;
    or_block_diagonals(op, i, j, s, dg, t);
    return or_thomas(nz, s, dg, t, rcol, zcol, work);
}

/* z = M^{-1} r on the whole field (Kernel "Preconditioner", eqn:SpMVPrec). */
int or_precondition(const or_op *op, const double *r, double *z)
{
    int status = OR_OK;
#pragma omp parallel for schedule(static)
    for (long j = 0; j < op->ny; ++j)
        for (long i = 0; i < op->nx; ++i) {
            int st = or_precondition_col(op, r + ZC(op, i, j, 0), i, j, z + ZC(op, i, j, 0));
            if (st != OR_OK) {
#pragma omp critical
                status = st;
            }
        }
    return status;
}

/* Block-Jacobi smoother, eqn:MultigridSmoother, one column:
 *   u_out = u + rho M^{-1} (f - A u);  all columns read the OLD u (Jacobi). */
int or_smooth_col(const or_op *op, const double *u, const double *f, double rho, long i,
                  long j, double *ucol_out)
{
    const int nz = op->nz;
    double r[nz], z[nz];
    or_residual_col(op, u, f, i, j, r);
    int st = or_precondition_col(op, r, i, j, z);
    for (int k = 0; k < nz; ++k) ucol_out[k] = u[ZC(op, i, j, k)] + rho * z[k];
    return st;
}

/* Out-of-place smoother over the whole field: u_out = u + rho M^{-1}(f - A u). */
int or_smooth(const or_op *op, const double *u, const double *f, double rho, double *u_out)
{
    int status = OR_OK;
#pragma omp parallel for schedule(static)
    for (long j = 0; j < op->ny; ++j)
        for (long i = 0; i < op->nx; ++i) {
            int st = or_smooth_col(op, u, f, rho, i, j, u_out + ZC(op, i, j, 0));
            if (st != OR_OK) {
#pragma omp critical
                status = st;
            }
        }
    return status;
}

/* ------------------------------------------------------------------------ */
/* Restriction R_{l,l+1}: "simple cell-average" in the horizontal direction
 * only [R6].  Coarse cell (I,J) has the fine children
 * (2I+a, 2J+b), a,b in {0,1} (0-based), at the same k:
 *   f_c(I,J,k) = 1/4 * sum_{a,b} r_f(2I+a, 2J+b, k). */
void or_restrict(const or_op *fine, const or_op *coarse, const double *rf, double *fc)
{
#pragma omp parallel for schedule(static)
    for (long J = 0; J < coarse->ny; ++J)
        for (long I = 0; I < coarse->nx; ++I)
            for (int k = 0; k < coarse->nz; ++k) {
                double s = rf[ZC(fine, 2 * I, 2 * J, k)] + rf[ZC(fine, 2 * I + 1, 2 * J, k)]
                         + rf[ZC(fine, 2 * I, 2 * J + 1, k)] + rf[ZC(fine, 2 * I + 1, 2 * J + 1, k)];
                fc[ZC(coarse, I, J, k)] = 0.25 * s;
            }
}

/* Coarse value with the ghosts of the boundary reading: zero outside the domain
 * [R7]; with face Dirichlet [R25] the ghost is the linear continuation through the
 * boundary value 0 on the face, u_c(-1) = -u_c(0) (per direction, so a corner ghost
 * is +u_c of the corner cell). */
static inline double or_coarse_at(const or_op *c, const double *uc, long I, long J, int k)
{
    if (!c->boundary) {
        if (I < 0 || I >= c->nx || J < 0 || J >= c->ny) return 0.0;
        return uc[ZC(c, I, J, k)];
    }
    double sign = 1.0;
    if (I < 0) { I = 0; sign = -sign; }
    if (I >= c->nx) { I = c->nx - 1; sign = -sign; }
    if (J < 0) { J = 0; sign = -sign; }
    if (J >= c->ny) { J = c->ny - 1; sign = -sign; }
    return sign * uc[ZC(c, I, J, k)];
}

/* Prolongation P_{l,l-1} and add: u_f += P u_c (Kernel "Prolongate", P:201,
 * P:276).  "(piecewise) linear interpolation ... in the horizontal direction
 * only" read as cell-centred bilinear interpolation [R7]: the fine
 * cell (i,j) (0-based) has parent (I,J) = (i/2, j/2); its nearer coarse
 * neighbour in x is I+sx with sx = -1 for even i, +1 for odd i (likewise sy);
 *   u_f(i,j,k) += (9 u_c(I,J) + 3 u_c(I+sx,J) + 3 u_c(I,J+sy) + u_c(I+sx,J+sy)) / 16
 * with u_c outside the domain from or_coarse_at (zero [R7] or reflected [R25]). */
void or_prolong_add(const or_op *coarse, const or_op *fine, const double *uc, double *uf)
{
#pragma omp parallel for schedule(static)
    for (long j = 0; j < fine->ny; ++j)
        for (long i = 0; i < fine->nx; ++i) {
            long I = i / 2, J = j / 2;
            long sx = (i % 2 == 0) ? -1 : 1, sy = (j % 2 == 0) ? -1 : 1;
            for (int k = 0; k < fine->nz; ++k) {
                double v = 9.0 * or_coarse_at(coarse, uc, I, J, k)
                         + 3.0 * or_coarse_at(coarse, uc, I + sx, J, k)
                         + 3.0 * or_coarse_at(coarse, uc, I, J + sy, k)
                         + 1.0 * or_coarse_at(coarse, uc, I + sx, J + sy, k);
                uf[ZC(fine, i, j, k)] += v / 16.0;
            }
        }
}

/* ------------------------------------------------------------------------ */
/* Deterministic inner product <x, y> over one level's cells. */
double or_dot(const or_op *op, const double *x, const double *y)
{
    double *rows = (double *)malloc(sizeof(double) * (size_t)op->ny);
    if (!rows) return NAN;
    const size_t rowlen = (size_t)op->nx * (size_t)op->nz;
#pragma omp parallel for schedule(static)
    for (long j = 0; j < op->ny; ++j) {
        double s = 0.0;
        const double *xr = x + (size_t)j * rowlen, *yr = y + (size_t)j * rowlen;
        for (size_t q = 0; q < rowlen; ++q) s += xr[q] * yr[q];
        rows[j] = s;
    }
    double s = 0.0;
    for (long j = 0; j < op->ny; ++j) s += rows[j];
    free(rows);
    return s;
}

/* ------------------------------------------------------------------------ */
/* Multigrid hierarchy: u^(l), f^(l), r^(l) for l = 1..L. */
typedef struct {
    or_params p;
    or_op op[33];          /* op[l], l = 1..L */
    double *u[33], *f[33], *r[33], *tmp[33];
} or_mg;

void or_mg_free(or_mg *mg)
{
    for (int l = 1; l <= mg->p.L; ++l) {
        if (l < mg->p.L) { free(mg->u[l]); free(mg->f[l]); }
        free(mg->r[l]); free(mg->tmp[l]);
        or_op_free(&mg->op[l]);
    }
}

int or_mg_init(const or_params *p, or_mg *mg)
{
    memset(mg, 0, sizeof(*mg));
    if (p->L < 1 || p->L > 32) return OR_E_PARAM;
    mg->p = *p;
    for (int l = 1; l <= p->L; ++l) {
        int st = or_op_init(p, l, &mg->op[l]);
        if (st != OR_OK) return st;
        size_t n = (size_t)mg->op[l].nx * (size_t)mg->op[l].ny * (size_t)mg->op[l].nz;
        if (l < p->L) {
            mg->u[l] = (double *)calloc(n, sizeof(double));
            mg->f[l] = (double *)calloc(n, sizeof(double));
            if (!mg->u[l] || !mg->f[l]) return OR_E_OOM;
        }
        mg->r[l] = (double *)calloc(n, sizeof(double));
        mg->tmp[l] = (double *)calloc(n, sizeof(double));
        if (!mg->r[l] || !mg->tmp[l]) return OR_E_OOM;
    }
    return OR_OK;
}

static size_t or_size(const or_op *op)
{
    return (size_t)op->nx * (size_t)op->ny * (size_t)op->nz;
}

/* Kernel-call trace of the V-cycle (test instrumentation only, no arithmetic): when
 * or_trace_counts is set, counts[OR_NK * l + kind] is incremented once per kernel of
 * alg:VCycle that runs on level l, with the kernel names of
 * tab:TimingBreakdownMultigrid. */
enum { OR_K_SMOOTH = 0, OR_K_RESSMOOTH = 1, OR_K_RESIDUAL = 2, OR_K_PROLONGATE = 3, OR_NK = 4 };
static int *or_trace_counts = NULL;
static inline void or_trace(int l, int kind)
{
    if (or_trace_counts) or_trace_counts[OR_NK * l + kind] += 1;
}

/* In-place smoother on level l: u^(l) <- u + rho M^{-1}(f - A u). */
static int or_mg_smooth(or_mg *mg, int l)
{
    or_trace(l, OR_K_SMOOTH);
    int st = or_smooth(&mg->op[l], mg->u[l], mg->f[l], mg->p.rho, mg->tmp[l]);
    memcpy(mg->u[l], mg->tmp[l], sizeof(double) * or_size(&mg->op[l]));
    return st;
}

/* Kernel "RestrictSmooth": f^(l) = R r^(l+1); u^(l) = rho M^{-1} f^(l),
 * i.e. one smoother step from the zero initial guess of P:278. */
static int or_mg_restrict_smooth(or_mg *mg, int l)
{
    or_trace(l, OR_K_RESSMOOTH);
    or_restrict(&mg->op[l + 1], &mg->op[l], mg->r[l + 1], mg->f[l]);
    int st = or_precondition(&mg->op[l], mg->f[l], mg->u[l]);
    size_t n = or_size(&mg->op[l]);
    for (size_t q = 0; q < n; ++q) mg->u[l][q] = mg->p.rho * mg->u[l][q];
    return st;
}

/* Subroutine VCycle of alg:VCycle with pre/post smoothing counts
 * and the coarse "A^{-1}" replaced by coarse_sweeps smoother
 * iterations, the first of which is the fused RestrictSmooth [R5]. */
static int or_vcycle_rec(or_mg *mg, int l)
{
    int st = OR_OK;
    const int L = mg->p.L;
    if (l == 1 && L > 1) {
        /* Restrict residual and solve on coarsest level */
        st |= or_mg_restrict_smooth(mg, 1);
        for (int s = 1; s < mg->p.coarse_sweeps; ++s) st |= or_mg_smooth(mg, 1);
        return st;
    }
    if (l == 1 && L == 1) {
        /* single-level hierarchy: the coarse solve is coarse_sweeps smoother
         * iterations on the given u */
        for (int s = 0; s < mg->p.coarse_sweeps; ++s) st |= or_mg_smooth(mg, 1);
        return st;
    }
    if (l == L) {
        /* Smooth on finest level */
        for (int s = 0; s < mg->p.pre; ++s) st |= or_mg_smooth(mg, l);
    } else {
        /* restrict residual and smooth once (RestrictSmooth) */
        st |= or_mg_restrict_smooth(mg, l);
        for (int s = 1; s < mg->p.pre; ++s) st |= or_mg_smooth(mg, l);
    }
    /* Calculate residual */
    or_trace(l, OR_K_RESIDUAL);
    or_residual(&mg->op[l], mg->u[l], mg->f[l], mg->r[l]);
    /* Recursive call */
    st |= or_vcycle_rec(mg, l - 1);
    /* Add prolongated coarse grid correction */
    or_trace(l, OR_K_PROLONGATE);
    or_prolong_add(&mg->op[l - 1], &mg->op[l], mg->u[l - 1], mg->u[l]);
    /* Postsmoothing */
    for (int s = 0; s < mg->p.post; ++s) st |= or_mg_smooth(mg, l);
    return st;
}

/* One V-cycle on the finest level, u and f caller-owned (z-contiguous). */
int or_vcycle(const or_params *p, double *u, const double *f)
{
    or_mg mg;
    int st = or_mg_init(p, &mg);
    if (st != OR_OK) { or_mg_free(&mg); return st; }
    mg.u[p->L] = u;
    mg.f[p->L] = (double *)f;
    st = or_vcycle_rec(&mg, p->L);
    or_mg_free(&mg);
    return st;
}

/* One V-cycle (as or_vcycle) with the kernel-call trace: counts has OR_NK * (L + 1)
 * entries, zeroed here; counts[OR_NK * l + kind] = calls of `kind` on level l. */
int or_api_vcycle_trace(const or_params *p, double *u, const double *f, int *counts)
{
    if (p->L < 1 || p->L > 32) return OR_E_PARAM;
    memset(counts, 0, sizeof(int) * (size_t)(OR_NK * (p->L + 1)));
    or_trace_counts = counts;
    int st = or_vcycle(p, u, f);
    or_trace_counts = NULL;
    return st;
}

/* Multigrid solve: u_0 = 0 [R9]; repeat V-cycles until
 * ||f - A u||_2 / ||r_0||_2 < eps (eqn:epsilonTolerance) [R10], at most
 * max_iter cycles.  history[it] = ||r_it|| (it = 0..iterations), if non-NULL
 * with history_cap entries. */
int or_solve_mg(const or_params *p, const double *f, double *u, double eps, int max_iter,
                int *iterations, int *converged, double *history, int history_cap)
{
    or_mg mg;
    int st = or_mg_init(p, &mg);
    if (st != OR_OK) { or_mg_free(&mg); return st; }
    const int L = p->L;
    const or_op *op = &mg.op[L];
    size_t n = or_size(op);
    memset(u, 0, sizeof(double) * n);
    mg.u[L] = u;
    mg.f[L] = (double *)f;
    or_residual(op, u, f, mg.r[L]);
    double r0 = sqrt(or_dot(op, mg.r[L], mg.r[L]));
    if (history && history_cap > 0) history[0] = r0;
    *iterations = 0;
    *converged = (r0 == 0.0);
    for (int it = 1; !*converged && it <= max_iter; ++it) {
        st |= or_vcycle_rec(&mg, L);
        or_residual(op, u, f, mg.r[L]);
        double rn = sqrt(or_dot(op, mg.r[L], mg.r[L]));
        if (history && it < history_cap) history[it] = rn;
        *iterations = it;
        if (rn / r0 < eps) *converged = 1;
        if (!(rn == rn)) break; /* NaN */
    }
    or_mg_free(&mg);
    return st;
}

/* Preconditioned CG, textbook form [R10]:
 *   u = 0, r = f, z = M^{-1} r, p = z, zeta = <r,z>
 *   loop: q = A p; alpha = zeta/<p,q>; u += alpha p; r -= alpha q;
 *         if ||r||/||r_0|| < eps stop;   (iterations = number of A p products)
 *         z = M^{-1} r; zeta' = <r,z>; p = z + (zeta'/zeta) p; zeta = zeta'.
 * Breakdown (<p,q> <= 0 or zeta <= 0) returns OR_E_BREAKDOWN. */
int or_solve_cg(const or_params *p, const double *f, double *u, double eps, int max_iter,
                int *iterations, int *converged, double *history, int history_cap)
{
    or_op op;
    int st = or_op_init(p, p->L, &op);
    if (st != OR_OK) { or_op_free(&op); return st; }
    size_t n = or_size(&op);
    double *r = (double *)malloc(sizeof(double) * n);
    double *z = (double *)malloc(sizeof(double) * n);
    double *pp = (double *)malloc(sizeof(double) * n);
    double *q = (double *)malloc(sizeof(double) * n);
    if (!r || !z || !pp || !q) { st = OR_E_OOM; goto done; }
    memset(u, 0, sizeof(double) * n);
    memcpy(r, f, sizeof(double) * n);
    double r0 = sqrt(or_dot(&op, r, r));
    if (history && history_cap > 0) history[0] = r0;
    *iterations = 0;
    *converged = (r0 == 0.0);
    if (*converged) goto done;
    st = or_precondition(&op, r, z);
    if (st != OR_OK) goto done;
    memcpy(pp, z, sizeof(double) * n);
    double zeta = or_dot(&op, r, z);
    for (int it = 1; it <= max_iter; ++it) {
        if (!(zeta > 0)) { st = OR_E_BREAKDOWN; break; }
        or_apply(&op, pp, q);
        double sigma = or_dot(&op, pp, q);
        if (!(sigma > 0)) { st = OR_E_BREAKDOWN; break; }
        double alpha = zeta / sigma;
        for (size_t m = 0; m < n; ++m) u[m] = u[m] + alpha * pp[m];
        for (size_t m = 0; m < n; ++m) r[m] = r[m] - alpha * q[m];
        double rn = sqrt(or_dot(&op, r, r));
        if (history && it < history_cap) history[it] = rn;
        *iterations = it;
        if (rn / r0 < eps) { *converged = 1; break; }
        st = or_precondition(&op, r, z);
        if (st != OR_OK) break;
        double zeta_new = or_dot(&op, r, z);
        double beta = zeta_new / zeta;
        for (size_t m = 0; m < n; ++m) pp[m] = z[m] + beta * pp[m];
        zeta = zeta_new;
    }
done:
    free(r); free(z); free(pp); free(q);
    or_op_free(&op);
    return st;
}

/* ------------------------------------------------------------------------ */
/* Thin entry points for the ctypes wrapper (oracle/oracle.py): each builds
 * the level operator from the parameters, runs one operation, frees it. */
#define OR_WITH_OP(p, l, body)                       \
    do {                                             \
        or_op op_;                                   \
        int st_ = or_op_init((p), (l), &op_);        \
        if (st_ == OR_OK) { body; }                  \
        or_op_free(&op_);                            \
        return st_;                                  \
    } while (0)

int or_api_apply(const or_params *p, int l, const double *x, double *y)
{ OR_WITH_OP(p, l, or_apply(&op_, x, y)); }

int or_api_residual(const or_params *p, int l, const double *u, const double *f, double *r)
{ OR_WITH_OP(p, l, or_residual(&op_, u, f, r)); }

int or_api_precondition(const or_params *p, int l, const double *r, double *z)
{ OR_WITH_OP(p, l, st_ = or_precondition(&op_, r, z)); }

int or_api_smooth(const or_params *p, int l, const double *u, const double *f, double *u_out)
{ OR_WITH_OP(p, l, st_ = or_smooth(&op_, u, f, p->rho, u_out)); }

int or_api_dot(const or_params *p, int l, const double *x, const double *y, double *out)
{ OR_WITH_OP(p, l, *out = or_dot(&op_, x, y)); }

/* Column samplers for full-size parity checks: compute the listed columns
 * (ii[m], jj[m]) of A x, of M^{-1} r, or of the smoother, m = 0..ncols-1,
 * into out[m*nz .. m*nz+nz-1]. */
int or_api_apply_cols(const or_params *p, int l, const double *x, int ncols, const long *ii,
                      const long *jj, double *out)
{ OR_WITH_OP(p, l, for (int m = 0; m < ncols; ++m) or_apply_col(&op_, x, ii[m], jj[m], out + (size_t)m * op_.nz)); }

int or_api_residual_cols(const or_params *p, int l, const double *u, const double *f, int ncols,
                         const long *ii, const long *jj, double *out)
{ OR_WITH_OP(p, l, for (int m = 0; m < ncols; ++m) or_residual_col(&op_, u, f, ii[m], jj[m], out + (size_t)m * op_.nz)); }

int or_api_precondition_cols(const or_params *p, int l, const double *r, int ncols,
                             const long *ii, const long *jj, double *out)
{ OR_WITH_OP(p, l, for (int m = 0; m < ncols; ++m) { int s_ = or_precondition_col(&op_, r + ZC(&op_, ii[m], jj[m], 0), ii[m], jj[m], out + (size_t)m * op_.nz); if (s_) st_ = s_; }); }

int or_api_smooth_cols(const or_params *p, int l, const double *u, const double *f, int ncols,
                       const long *ii, const long *jj, double *out)
{ OR_WITH_OP(p, l, for (int m = 0; m < ncols; ++m) { int s_ = or_smooth_col(&op_, u, f, p->rho, ii[m], jj[m], out + (size_t)m * op_.nz); if (s_) st_ = s_; }); }

int or_api_restrict(const or_params *p, int fine_level, const double *rf, double *fc)
{
    or_op fine, coarse;
    if (fine_level < 2) return OR_E_PARAM;
    int st = or_op_init(p, fine_level, &fine);
    if (st == OR_OK) st = or_op_init(p, fine_level - 1, &coarse);
    if (st == OR_OK) or_restrict(&fine, &coarse, rf, fc);
    or_op_free(&fine); or_op_free(&coarse);
    return st;
}

int or_api_prolong_add(const or_params *p, int coarse_level, const double *uc, double *uf)
{
    or_op fine, coarse;
    if (coarse_level < 1 || coarse_level >= p->L) return OR_E_PARAM;
    int st = or_op_init(p, coarse_level, &coarse);
    if (st == OR_OK) st = or_op_init(p, coarse_level + 1, &fine);
    if (st == OR_OK) or_prolong_add(&coarse, &fine, uc, uf);
    or_op_free(&fine); or_op_free(&coarse);
    return st;
}

int or_api_thomas(int n, const double *s, const double *dg, const double *t, const double *g,
                  double *x)
{
    double *work = (double *)malloc(sizeof(double) * 2 * (size_t)(n > 0 ? n : 1));
    if (!work) return OR_E_OOM;
    int st = or_thomas(n, s, dg, t, g, x, work);
    free(work);
    return st;
}

/* Per-column fields of level l (reading [R26]); area[ny_l*nx_l], ax[ny_l*(nx_l+1)],
 * ay[(ny_l+1)*nx_l].  OR_E_PARAM when the parameters carry no fields. */
int or_api_level_fields(const or_params *p, int l, double *area, double *ax, double *ay)
{
    or_op op;
    int st = or_op_init(p, l, &op);
    if (st == OR_OK && !op.fa) st = OR_E_PARAM;
    if (st == OR_OK) {
        memcpy(area, op.fa, sizeof(double) * (size_t)(op.nx * op.ny));
        memcpy(ax, op.fx, sizeof(double) * (size_t)((op.nx + 1) * op.ny));
        memcpy(ay, op.fy, sizeof(double) * (size_t)(op.nx * (op.ny + 1)));
    }
    or_op_free(&op);
    return st;
}

/* Level shape and coefficients as the oracle sees them (for reporting). */
int or_api_level_info(const or_params *p, int l, long *nx, long *ny, double *alpha_TT,
                      double *vert)
{
    or_op op;
    int st = or_op_init(p, l, &op);
    if (st == OR_OK) {
        *nx = op.nx; *ny = op.ny; *alpha_TT = op.alpha_TT; *vert = -op.b[op.nz > 1 ? 1 : 0];
    }
    or_op_free(&op);
    return st;
}

void or_api_set_threads(int n)
{
#ifdef _OPENMP
    if (n > 0) omp_set_num_threads(n);
#else
    (void)n;
#endif
}

int or_api_num_threads(void)
{
#ifdef _OPENMP
    return omp_get_max_threads();
#else
    return 1;
#endif
}
