/*
 * tpmg.h -- C ABI of libtpmg.so: B200-native (sm_100a, fp64) tensor-product
 * multigrid and line-preconditioned CG for the sign-positive anisotropic
 * Helmholtz equation of Mueller, Scheichl & Vainikko, "Petascale elliptic
 * solvers for anisotropic PDEs on GPU clusters" (arXiv:1402.3545).
 *
 * Citations "P:n" are lines of the paper's text; equation and
 * algorithm names are the paper's LaTeX labels.  DESIGN.md section 3 lists
 * every reading of the paper the library makes ([R1]..[R26]).
 *
 * ----------------------------------------------------------------------------
 * Problem (flat-box instance of eqn:ModelEquation):
 *   -omega^2 (Laplace_2D u + lambda^2 d^2u/dz^2) + u = f  on [0,1]^2 x [0,H],
 *   homogeneous Dirichlet horizontally (zero ghost cells [R1]),
 *   homogeneous Neumann at top and bottom,
 *   omega = nu_CFL h / 2 (eqn:OmegaNumerical), h = 1/nx, h_z = H/nz.
 * Cell-centred finite volumes give, per vertical column T = (i,j)
 * (eqn:TridiagonalPDE, eqn:LocalMatrixStencil):
 *   (A u)^(T) = A_T u^(T) + sum_{T' in N(T)} A_{T,T'} u^(T'),
 *   A_{T,T'} = -omega^2/h^2 I,
 *   A_T = tridiag(-omega^2 lambda^2/h_z^2,
 *                 1 + 4 omega^2/h^2 + omega^2 lambda^2/h_z^2 [(k>0)+(k<nz-1)],
 *                 -omega^2 lambda^2/h_z^2).
 * Coarse levels rediscretise with h_l = 2^(L-l) h (horizontal-only
 * semicoarsening; [R4]).
 *
 * ----------------------------------------------------------------------------
 * Data layout (every vector argument):
 *   DEVICE pointer, IEEE fp64, the calling rank's owned cells of one level in
 *   the paper's x-contiguous order Lambda (eqn:MemoryMapSingleGPU),
 *   0-based:   idx(i, j, k) = (j * nz + k) * nx_l + i,
 *   0 <= i < nx_l, 0 <= j < ny_l (local rows), 0 <= k < nz.
 *   A torch tensor of shape [ny_l, nz, nx_l] is such a vector.  There is no
 *   padding and no halo in caller memory: halos live in library-owned slabs.
 *   Pointers must be 16-byte aligned (cudaMalloc / torch allocations are).
 *   Level l = L is the finest, l = 1 the coarsest; tpmg_local_box
 *   returns the shape of every level.
 *
 * Domain decomposition: nranks y-strips of ny/nranks rows each;
 * columns are never split.  Calls marked COLLECTIVE must be made by
 * every rank with matching arguments; the others are rank-local.
 *
 * Ownership: the caller owns every vector and the tpmg_result.history array;
 * the library owns the context, halo slabs, multigrid and CG work vectors
 * and the NCCL communicator.  No caller pointer is retained after a call
 * returns.
 *
 * Streams: every call enqueues on the context stream (the one given to
 * tpmg_create, or tpmg_set_stream).  Single-operator calls return without
 * synchronising unless they return a host-side scalar.  The solvers and
 * tpmg_vcycle synchronise before returning (the convergence test reads the
 * residual norm on the host).
 *
 * Errors: every call returns a tpmg_status; on failure tpmg_last_error(ctx)
 * describes it.  Argument errors are detected before any work is enqueued.
 * CUDA and NCCL failures (TPMG_E_CUDA, TPMG_E_NCCL) leave the context usable
 * only for tpmg_destroy.
 */
#ifndef TPMG_H
#define TPMG_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define TPMG_VERSION_MAJOR 0
#define TPMG_VERSION_MINOR 1

typedef enum {
    TPMG_OK = 0,
    TPMG_E_PARAM = 1,     /* non-positive nu, H, lambda; rho not in (0,2); bad counts or boundary; NULL pointer */
    TPMG_E_SHAPE = 2,     /* nx or ny not divisible by 2^(L-1); ny not divisible by nranks*2^(L-1);
                             nz too large for the on-chip Thomas buffer; x == y where forbidden */
    TPMG_E_RANGE = 3,     /* level not in [1, L] */
    TPMG_E_SINGULAR = 4,  /* zero Thomas pivot (cannot happen for valid parameters: the column
                             blocks are strictly diagonally dominant by 1 + 4 omega^2/h^2) */
    TPMG_E_BREAKDOWN = 5, /* CG: <p, A p> <= 0 or <r, M^-1 r> <= 0, or a NaN residual */
    TPMG_E_TOPOLOGY = 6,  /* rank / nranks / communicator mismatch */
    TPMG_E_CUDA = 7,
    TPMG_E_NCCL = 8,
    TPMG_E_OOM = 9
} tpmg_status;

typedef enum { TPMG_SOLVER_CG = 0, TPMG_SOLVER_MG = 1 } tpmg_solver;

/* Reading of the horizontal homogeneous Dirichlet condition on the
 * cell-centred grid:
 *   TPMG_BC_GHOST_ZERO [R1] (default): the value 0 sits in the ghost cell, every
 *       column has alpha_T = 4 alpha_{T,T'}; coarse ghosts of the prolongation are 0 [R7];
 *   TPMG_BC_FACE [R25]: the value 0 sits on the boundary face (half a cell away), a
 *       column with nb boundary faces has alpha_T = (4 + nb) alpha_{T,T'}, its line
 *       block M_T changes accordingly, and the prolongation's coarse ghost is the
 *       linear continuation through 0 (-u_c across an edge, +u_c across a corner).
 *       The boundary is then at the same place on every level, which keeps MG
 *       robust for large nu_CFL (sec:Robustness). */
typedef enum { TPMG_BC_GHOST_ZERO = 0, TPMG_BC_FACE = 1 } tpmg_boundary;

/* Problem and solver parameters.  A zero field selects its default. */
typedef struct {
    int64_t nx, ny;        /* GLOBAL horizontal cells of the finest level (required, > 0) */
    int32_t nz;            /* vertical levels; default 128 */
    double nu_cfl;         /* CFL number; default 8.4 (eqn:OmegaNumerical) */
    double H;              /* depth ratio, h_z = H/nz; default 0.01 [R3] */
    double lambda;         /* vertical coefficient; default 1 [R3] */
    int32_t levels;        /* multigrid levels L; default 5 */
    int32_t pre, post;     /* smoothing steps per level; default 1, 1 */
    int32_t coarse_sweeps; /* smoother iterations on the coarsest level; default 2 */
    double rho;            /* block-Jacobi relaxation rho_relax; default 2/3 */
    int32_t boundary;      /* tpmg_boundary; default TPMG_BC_GHOST_ZERO [R1] */
} tpmg_params;

/* Solve report.  history (optional, caller-owned HOST array of history_cap
 * doubles) receives ||r_it||_2 for it = 0..iterations (global norms). */
typedef struct {
    int32_t iterations;    /* V-cycles (MG) or A-applications (CG) performed */
    int32_t converged;     /* 1 if ||r||/||r_0|| < eps (eqn:epsilonTolerance) */
    double r0_norm;        /* ||r_0||_2 = ||f||_2 (u_0 = 0, [R9]) */
    double rel_residual;   /* final ||r||/||r_0|| (MG: true residual; CG: recurrence residual [R10]) */
    double seconds;        /* device time of the solve (CUDA events on the context stream) */
    double *history;
    int32_t history_cap;
} tpmg_result;

/* Counters for benchmarking. */
typedef struct {
    int64_t kernel_launches;   /* kernels launched by the library since creation / reset */
    int64_t halo_exchanges;    /* halo exchange calls (nranks > 1) */
    int64_t allreduces;        /* NCCL all-reduce calls (nranks > 1) */
    int64_t graph_launches;    /* CUDA graph launches: always 0 (the solvers enqueue their kernels
                                  directly, run-ahead on device flags) */
    int64_t p2p_halo;          /* 1: halos by device-initiated NVLink stores (decided collectively at
                                  create: every rank's neighbours reachable peer-to-peer on one host);
                                  0: NCCL send/recv (or one rank) */
    int64_t p2p_allreduce;     /* 1: global sums by the device-initiated NVLink allreduce (P2P mode,
                                  <= 8 ranks); 0: ncclAllReduce (TPMG_ALLREDUCE=nccl, or one rank) */
} tpmg_stats;

typedef struct tpmg_ctx tpmg_ctx;

/* Library version as MAJOR*1000 + MINOR. */
int32_t tpmg_version(void);

/* Fill *p with the defaults (nx = ny = 0). */
void tpmg_params_default(tpmg_params *p);

/* Rank 0: generate a 128-byte NCCL unique id into id128 (caller-owned, 128
 * bytes); the caller broadcasts it to every rank (e.g. torch.distributed). */
tpmg_status tpmg_nccl_id(void *id128);

/* Domain decomposition without a GPU (host-only, pure): validates params for
 * nranks y-strips exactly as tpmg_create does (TPMG_E_PARAM / TPMG_E_SHAPE /
 * TPMG_E_TOPOLOGY) and returns rank `rank`'s first global row y0 and row count
 * ny on level `level` (1..L; TPMG_E_RANGE otherwise).  Strips are contiguous and
 * equal: ny_l = ny / (nranks 2^(L-l)), y0 = rank ny_l (columns never
 * split P:306). */
tpmg_status tpmg_partition(const tpmg_params *params, int32_t rank, int32_t nranks, int32_t level,
                           int64_t *y0, int64_t *ny);

/* Create a context on CUDA device `device` for rank `rank` of `nranks`.
 * id128: the NCCL unique id (ignored when nranks == 1, may be NULL).
 * cuda_stream: a cudaStream_t on `device`, or NULL for the legacy default
 * stream.  Validates the parameters (TPMG_E_PARAM / TPMG_E_SHAPE), builds
 * the per-level coefficient tables (a1 of SURVEY 8a), allocates the
 * multigrid hierarchy and CG work vectors, and (nranks > 1) joins the NCCL
 * communicator: COLLECTIVE.  *out receives the context. */
tpmg_status tpmg_create(const tpmg_params *params, int32_t rank, int32_t nranks,
                        const void *id128, int32_t device, void *cuda_stream,
                        tpmg_ctx **out);

/* Release everything the context owns.  Accepts NULL. COLLECTIVE if nranks > 1. */
tpmg_status tpmg_destroy(tpmg_ctx *ctx);

/* Replace the context stream (a cudaStream_t on the context's device).  Work already
 * enqueued on the old stream is ordered before everything enqueued on the new one (an event
 * recorded on the old stream, waited for by the new): the two never race on the library's
 * scratch, reduction slots or halo slabs. */
tpmg_status tpmg_set_stream(tpmg_ctx *ctx, void *cuda_stream);

/* Shape of level `level` on this rank: first owned global row y0, local
 * nx, ny, and nz.  Any output pointer may be NULL. */
tpmg_status tpmg_local_box(const tpmg_ctx *ctx, int32_t level, int64_t *y0, int64_t *nx,
                           int64_t *ny, int32_t *nz);

/* y = A x on level `level` (Kernel SpMV, eqn:SpMVPrec P:168-171; matrix-free
 * stencil eqn:LocalMatrixStencil).  x != y.  COLLECTIVE (halo of x). */
tpmg_status tpmg_apply(tpmg_ctx *ctx, int32_t level, const double *x, double *y);

/* r = f - A u (Kernel Residual, alg:VCycle P:197).  r may be NULL
 * (norm only); r must not alias u.  If norm2 (HOST pointer) is non-NULL it
 * receives the global sum of r^2 and the call synchronises.  COLLECTIVE. */
tpmg_status tpmg_residual(tpmg_ctx *ctx, int32_t level, const double *u, const double *f,
                          double *r, double *norm2);

/* z = M^{-1} r: vertical line relaxation, one Thomas solve per column with
 * M = blockdiag(A_T) (eqn:SpMVPrec).  r != z.  Rank-local. */
tpmg_status tpmg_precondition(tpmg_ctx *ctx, int32_t level, const double *r, double *z);

/* `sweeps` block-Jacobi smoother steps in place on u:
 * u <- u + rho_relax M^{-1} (f - A u)  (eqn:MultigridSmoother P:215-218,
 * Kernel Smooth P:273); every column reads the old u (Jacobi).  COLLECTIVE. */
tpmg_status tpmg_smooth(tpmg_ctx *ctx, int32_t level, double *u, const double *f,
                        int32_t sweeps);

/* f_coarse = R r_fine: cell average over the 2x2 horizontal children
 * (P:219-226).  fine_level in [2, L].  Rank-local. */
tpmg_status tpmg_restrict(tpmg_ctx *ctx, int32_t fine_level, const double *r_fine,
                          double *f_coarse);

/* u_fine += P u_coarse: cell-centred bilinear interpolation, weights
 * (9,3,3,1)/16, zero coarse ghosts at the physical boundary [R7]
 * (Kernel Prolongate P:276).  coarse_level in [1, L-1].  COLLECTIVE (halo
 * of u_coarse). */
tpmg_status tpmg_prolong_add(tpmg_ctx *ctx, int32_t coarse_level, const double *u_coarse,
                             double *u_fine);

/* One V-cycle (alg:VCycle P:181-208) on the finest level, in place on u:
 * 1 pre- / 1 post-smooth (params), RestrictSmooth on the coarse levels, the
 * coarsest problem solved by coarse_sweeps smoother iterations [R5].
 * COLLECTIVE. Synchronises. */
tpmg_status tpmg_vcycle(tpmg_ctx *ctx, double *u, const double *f);

/* Solve A u = f from u_0 = 0 to ||r||_2/||r_0||_2 < eps (eqn:epsilonTolerance,
 * P:177-180) with at most max_iter iterations.  Not converging is not an
 * error (result->converged = 0).  u and f must not alias.  COLLECTIVE.
 * tpmg_solve_mg: repeated V-cycles, true residual after each.
 * tpmg_solve_cg: preconditioned CG with vertical line relaxation
 *   (P:160-173), two fused kernels per iteration. */
tpmg_status tpmg_solve_mg(tpmg_ctx *ctx, const double *f, double *u, double eps,
                          int32_t max_iter, tpmg_result *result);
tpmg_status tpmg_solve_cg(tpmg_ctx *ctx, const double *f, double *u, double eps,
                          int32_t max_iter, tpmg_result *result);

/* The same solves with HOST buffers (Lambda layout of the rank's fine-level
 * cells): copies f in, solves on the device, copies u out (the paper's
 * "total solution time" path, P:427 minus the transposition).  Pageable or
 * pinned memory; pinned is faster.  COLLECTIVE. */
tpmg_status tpmg_solve_host(tpmg_ctx *ctx, tpmg_solver solver, const double *f_host,
                            double *u_host, double eps, int32_t max_iter,
                            tpmg_result *result);

/* Both solvers on one host right-hand side -- the benchmark's step (an MG solve and a PCG
 * solve of the same f, BASELINE.json): f is copied in ONCE, the MG solve runs into a device
 * buffer, its solution's device->host copy runs on a separate copy stream while the PCG solve
 * computes, then the PCG solution is copied out.  Host buffers as tpmg_solve_host (pinned for
 * the overlap; pageable still works, without it); results for each solver (either may be
 * NULL).  max_iter_mg / max_iter_cg as tpmg_solve_mg / tpmg_solve_cg.  COLLECTIVE; returns
 * after both copies have completed. */
tpmg_status tpmg_solve_host_pair(tpmg_ctx *ctx, const double *f_host, double *u_mg_host, double *u_cg_host,
                                 double eps, int32_t max_iter_mg, int32_t max_iter_cg, tpmg_result *res_mg,
                                 tpmg_result *res_cg);

/* Layout conversion (the fields are z-contiguous on the host, "transposing the fields
 * from a z-contiguous data format on the host to the x-contiguous format ... on the GPU").
 * z-contiguous: idx = (j*nx + i)*nz + k (columns contiguous, the CPU ordering of P:59);
 * Lambda: idx = (j*nz + k)*nx + i (eqn:MemoryMapSingleGPU).  Over the rank's local
 * box of `level`; src and dst are DEVICE pointers of that many doubles, must not alias.
 * Pure data movement (bit-exact).  Errors: TPMG_E_PARAM (direction, NULL, aliasing),
 * TPMG_E_RANGE (level).  Asynchronous on the context stream. */
typedef enum { TPMG_ZC_TO_LAMBDA = 0, TPMG_LAMBDA_TO_ZC = 1 } tpmg_layout_direction;
tpmg_status tpmg_transpose(tpmg_ctx *ctx, int32_t level, int32_t direction, const double *src, double *dst);

/* tpmg_solve_host with HOST buffers in the z-contiguous layout: the paper's "total solution
 * time" path (tab:SingleGPUTiming's t_MemCpy+transpose): copy f in, transpose to
 * Lambda on the device, solve, transpose u back, copy out.  Same arguments and errors as
 * tpmg_solve_host.  COLLECTIVE. */
tpmg_status tpmg_solve_host_zc(tpmg_ctx *ctx, tpmg_solver solver, const double *f_host,
                               double *u_host, double eps, int32_t max_iter,
                               tpmg_result *result);

/* General vertical profiles a, b, c, d of eqn:LocalMatrixStencil ("derived
 * from the vertical stiffness- and mass-matrices", the same for every column and level),
 * e.g. a stretched vertical grid or height-dependent lambda / density:
 *   A_T      = diag(a) - alpha_T diag(d) + tridiag(-(b+c), b, c),
 *   A_{T,T'} = alpha_{T,T'} diag(d),   alpha_{T,T'} = -omega^2 / h_l^2 on level l,
 * in the units of A (b, c include omega^2 lambda^2 / h_z^2; the flat box [R2] is a = d = 1,
 * b_k = -gamma [k > 0], c_k = -gamma [k < nz-1]).  Host arrays of nz doubles, copied.
 * Requirements (symmetric, diagonally dominant column blocks): b[0] = 0, c[nz-1] = 0,
 * b[k+1] = c[k], a >= 0, b <= 0, c <= 0, d > 0, else TPMG_E_PARAM.  All NULL: back to the
 * flat box.  Synchronises the context stream and rebuilds the per-level Thomas tables;
 * applies to every later call.  COLLECTIVE in the sense that all ranks must pass the same
 * profiles.  The fused prolongation and the k-split CG preconditioner options are flat-box
 * only (the library falls back to the general kernels). */
tpmg_status tpmg_set_profiles(tpmg_ctx *ctx, const double *a, const double *b, const double *c,
                              const double *d);

/* Per-column horizontal fields of eqn:LocalMatrixStencil: "the coefficients
 * alpha_{T,T'} and alpha_T are different for each horizontal grid cell T (and depend on the
 * multigrid level)", with |T| the (normalised) cell size:
 *   A_T      = |T| diag(a) - alpha_T diag(d) + |T| tridiag(-(b+c), b, c),
 *   A_{T,T'} = alpha_{T,T'} diag(d),   alpha_T = sum of the column's 4 face alpha_{T,T'} [R1]
 *   (the face-Dirichlet reading [R25] counts a boundary face twice).
 * HOST arrays over the GLOBAL finest level (every rank passes the same arrays; each takes its
 * strip), row-major, copied:
 *   area[ny][nx]    |T| > 0 of column (i, j);
 *   ax[ny][nx+1]    alpha_{T,T'} <= 0 of the x-face between columns (i-1, j) and (i, j);
 *                   faces 0 and nx are boundary faces (they enter alpha_T only);
 *   ay[ny+1][nx]    alpha_{T,T'} <= 0 of the y-face between columns (i, j-1) and (i, j).
 * The flat box is area = 1, ax = ay = -omega^2/h^2.  Coarse levels follow reading [R26]
 * (DESIGN.md): |T| averages the 2x2 children, a coarse face alpha is 1/8 of the sum of the
 * two fine faces on it (flat fields reproduce the rediscretisation [R4] exactly).  Works
 * with the vertical profiles of tpmg_set_profiles (either order).  All NULL: back to
 * the uniform coefficients.  Errors: TPMG_E_PARAM (missing array, |T| <= 0, alpha > 0, non-
 * finite values, cp.async loader), TPMG_E_SHAPE (nz too large for the on-chip per-column
 * Thomas buffers).  Synchronises the context stream.  With fields every line kernel runs the
 * one-thread-per-column form, which computes each column's Thomas pivots on the fly
 * (the k-split and fused-prolongation options fall back). */
tpmg_status tpmg_set_fields(tpmg_ctx *ctx, const double *area, const double *ax, const double *ay);

/* Halo-exchange primitives of the multi-rank path (y-strips with halo width 1),
 * exposed so that the exchange kernels can be checked on a single GPU.  The solvers call the
 * same kernels on the neighbours' IPC-mapped slabs (P2P mode).
 * tpmg_halo_push: one launch of the push kernel -- dst_lo <- row 0 of src, dst_hi <- row
 *   ny_l - 1 of src (each row a plane of nz * nx_l doubles of `level`, Lambda order); either
 *   destination may be NULL (a physical boundary).  Device pointers, caller-owned; src must
 *   not overlap a destination.  Rank-local, asynchronous on the context stream.
 * tpmg_cg_halo: the CG direction kernel's local update of the p halo (the halo of
 *   p = z + beta p_old without sending p): out = fma(beta, p, z) element by element on each
 *   non-NULL triple of fine-level planes (nz * nx_L doubles).  Rank-local; synchronises. */
tpmg_status tpmg_halo_push(tpmg_ctx *ctx, int32_t level, const double *src, double *dst_lo, double *dst_hi);
tpmg_status tpmg_cg_halo(tpmg_ctx *ctx, double beta, double *out_lo, const double *z_lo, const double *p_lo,
                         double *out_hi, const double *z_hi, const double *p_hi);

/* Counters (kernel launches etc.); tpmg_stats_reset zeroes them. */
tpmg_status tpmg_get_stats(const tpmg_ctx *ctx, tpmg_stats *out);
tpmg_status tpmg_stats_reset(tpmg_ctx *ctx);

/* Kernel classes for tpmg_profile_read. */
typedef enum {
    TPMG_K_APPLY = 0,             /* y = A x */
    TPMG_K_RESIDUAL = 1,          /* r = f - A u (+ norm) */
    TPMG_K_PRECONDITION = 2,      /* z = s M^-1 r (also the zero-guess coarse smooth) */
    TPMG_K_SMOOTH = 3,            /* fused stencil + Thomas + relaxation */
    TPMG_K_CG_DIRECTION = 4,      /* p = z + beta p, <p, A p> */
    TPMG_K_CG_PRECONDITION = 5,   /* r -= alpha A p, u += alpha p, z = M^-1 r, norms */
    TPMG_K_RESIDUAL_RESTRICT = 6, /* f_c = R (f - A u) */
    TPMG_K_RESTRICT = 7,          /* f_c = R r */
    TPMG_K_PROLONG_ADD = 8,       /* u_f += P u_c */
    TPMG_K_DOT = 9,               /* global inner product */
    TPMG_K_SMOOTH_PROLONG = 10,   /* post-smooth of u + P u_c, prolongation fused */
    TPMG_K_COUNT = 11
} tpmg_kernel;

/* Per-kernel-class device timing with CUDA events on the context stream.
 * tpmg_profile(ctx, 1) clears the totals and brackets every later launch with
 * a pair of events; tpmg_profile(ctx, 0) stops recording.  tpmg_profile_read
 * synchronises the stream and returns, for one class, the number of launches,
 * their summed device time (ms) and the summed number of grid cells they
 * processed (fine cells for the transfer kernels). */
tpmg_status tpmg_profile(tpmg_ctx *ctx, int32_t enable);
/* Like tpmg_profile for the classes in mask (bit k = tpmg_kernel k) only; 0 stops.
 * Each bracketed launch costs a timing-event pair on the stream (a few microseconds
 * of serialisation), so a benchmark can time one class live and leave the others
 * unbracketed. */
tpmg_status tpmg_profile_mask(tpmg_ctx *ctx, uint32_t mask);
tpmg_status tpmg_profile_read(tpmg_ctx *ctx, int32_t kernel, int64_t *launches, double *ms,
                              double *cells);

/* Message for the last failing call on ctx ("" if none); never NULL.
 * With ctx == NULL: the last error of a failed tpmg_create on this thread. */
const char *tpmg_last_error(const tpmg_ctx *ctx);

#ifdef __cplusplus
}
#endif

#endif /* TPMG_H */
