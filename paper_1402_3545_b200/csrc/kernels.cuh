// kernels.cuh -- launch interface of the sm_100a kernels of libtpmg.
//
// Every vector is fp64 in the paper's Lambda layout:
//   idx(i, j, k) = (j * nz + k) * nx + i   (0-based, local rows j).
// A "halo'd" field is read at the 4 horizontal neighbours; rows j = -1 and
// j = ny come from the slabs lo / hi (one nz x nx plane each) or are zero
// when the slab pointer is null (physical boundary, zero ghosts [R1]).
#pragma once
#include <cstdint>
#include <cuda.h>
#include <cuda_runtime.h>
#include <utility>

namespace tpmg {

// A field read with its horizontal neighbours.
struct HaloField {
    const double* base;  // owned rows
    const double* lo;    // row j = -1 (nullptr: zero)
    const double* hi;    // row j = ny (nullptr: zero)
};

// Per-level operator constants.
struct LevelConst {
    int64_t nx, ny;     // local horizontal cells
    int32_t nz;
    double c;           // omega^2 / h_l^2        (minus alpha_{T,T'})
    double gamma;       // omega^2 lambda^2 / h_z^2 (minus the vertical off-diagonal)
    const double* tab;  // device: per column class [diag, invm, gim, afw, P, Q][nz] (Thomas factors of M_T)
    int32_t bc;         // tpmg_boundary: 0 ghost-zero [R1] (class 0 only), 1 face Dirichlet [R25]
    int32_t bnd_lo, bnd_hi;   // local row 0 / ny-1 lies on the physical boundary
    int32_t gen;        // 1: general vertical profiles (stencil couplings from prof, not gamma / c);
                        // 2: per-column horizontal fields (fld) with the profiles a, b, c, d
    const double* prof; // device, gen 1: [b_k][c_k][c_l d_k]; gen 2: [a_k-b_k-c_k][b_k][c_k][d_k];
                        // nz each
    const double* fld;  // device, gen 2: [|T|][alpha_T][alpha_W][alpha_E][alpha_S][alpha_N], each
                        // [ny][nx] over the local columns ("different for each horizontal
                        // grid cell T (and depend on the multigrid level)")
};

// Column classes of the face-Dirichlet reading: nb = number of boundary faces (0..4).
constexpr int kBoundaryClasses = 5;
constexpr int kTabArrays = 6;   // doubles per class: kTabArrays * nz

// Does the tile of columns [i0, i0+tx) x [j0, j0+ty) contain a column whose line
// block differs from the interior one (face Dirichlet only)?
__host__ __device__ inline bool tile_on_boundary(const LevelConst& L, int64_t i0, int64_t j0, int tx, int ty)
{
    return L.bc && (i0 == 0 || i0 + tx >= L.nx || (L.bnd_lo && j0 == 0) || (L.bnd_hi && j0 + ty >= L.ny));
}

// Class (boundary-face count) of column (i, j); 0 for out-of-range columns.
__host__ __device__ inline int column_class(const LevelConst& L, int64_t i, int64_t j)
{
    if (i < 0 || i >= L.nx || j < 0 || j >= L.ny) return 0;
    return (i == 0) + (i == L.nx - 1) + (L.bnd_lo && j == 0) + (L.bnd_hi && j == L.ny - 1);
}

// Deterministic reduction slot: per-block partials, a ticket counter and the
// result (nvals doubles).  The last block to finish sums the partials in
// block order, so the result is independent of scheduling.
struct ReduceSlot {
    double* partials;   // >= gridDim.x * nvals
    unsigned* ticket;   // zero on entry, reset to zero by the last block
    double* result;     // nvals doubles (device)
    int accumulate;     // 1: result += sum (second launch of an interior/boundary pair)
};

// Tile-row subsets for overlapping a halo exchange with interior work:
// PART_ALL every tile row; PART_INTERIOR rows 1 .. nty-2 (they read no halo row);
// PART_BOUNDARY rows 0 and nty-1.
enum TilePart : int { PART_ALL = 0, PART_INTERIOR = 1, PART_BOUNDARY = 2 };
__host__ __device__ inline int part_rows(int part, int nty)
{
    return part == PART_ALL ? nty : part == PART_INTERIOR ? (nty > 2 ? nty - 2 : 0) : (nty < 2 ? nty : 2);
}
__host__ __device__ inline int part_row(int part, int nty, int idx)
{
    return part == PART_ALL ? idx : part == PART_INTERIOR ? idx + 1 : (idx == 0 ? 0 : nty - 1);
}

// Tile-row order of a launch that pushes its boundary rows to the neighbours (fused halo
// push): the strip-boundary tile rows come first, so their remote stores drain while the
// rest of the grid is computed.
__host__ __device__ inline int push_row(int r, int nrows, bool lo, bool hi)
{
    if (nrows < 2 || !hi) return r;          // row 0 is first anyway
    if (lo) return r == 0 ? 0 : (r == 1 ? nrows - 1 : r - 1);
    return r == 0 ? nrows - 1 : r - 1;
}

// Scalar ratio read on the device: value = num_idx < 0 ? 0 : s[num]/s[den].
struct DevRatio {
    const double* s;
    int num, den;
};

enum LineMode : int {
    MODE_APPLY = 0,   // out0 = A x                                   (halo: x)
    MODE_RESID = 1,   // out0 = f - A u (optional), sum r^2           (halo: u; plain: f)
    MODE_PREC = 2,    // out0 = scale * M^-1 r                        (plain: r)
    MODE_SMOOTH = 3,  // out0 = u + rho M^-1 (f - A u), sum r^2       (halo: u; plain: f)
    MODE_CGDIR = 4,   // p = z + beta p_old; out0 = p; sum <p, A p>   (halo: z, p_old)
    MODE_CGPREC = 5,  // r -= alpha A p; u += alpha p; z = M^-1 r;
                      // sums ||r||^2, <r, z>                         (halo: p; plain: r, u)
    MODE_RESTRICT = 6,// out0 (coarse) = R (f - A u): fine residual restricted (halo: u; plain: f)
    MODE_SMOOTH_PROLONG = 7, // out0 = smooth(u + P u_c), sum r^2  (halo: u, coarse u_c; plain: f;
                             // k-split kernel only)
    // CG preconditioner with the u update paired over two iterations (the level-1 BLAS
    // fused into the two kernels): odd iterations leave u alone, even ones add both steps;
    // r, z, the sums and hence the iteration are bit-identical to MODE_CGPREC's
    MODE_CGPREC_D = 8,  // r -= alpha A p; z = M^-1 r; sums (no u)          (halo: p; plain: r)
    MODE_CGPREC_P = 9,  // as MODE_CGPREC with u += alpha2 p_prev + alpha p  (halo: p; plain: r, u, p_prev)
};
__host__ __device__ constexpr bool is_cgprec(int mode)
{
    return mode == MODE_CGPREC || mode == MODE_CGPREC_D || mode == MODE_CGPREC_P;
}

// TMA descriptors of one halo'd field: the whole (TY+2)-row box, a one-row box,
// and the halo slabs (rows j = -1 / j = ny) when present.
struct TmaHalo {
    CUtensorMap main, row, lo, hi;
    CUtensorMap m1;   // k-split in-place layout: the box minus one row (a strip-boundary tile loads
                      // its in-domain rows with it and the slab row separately)
    int has_lo, has_hi, has_m1;
};
struct TmaMaps {
    TmaHalo h[2];
    CUtensorMap q[4];   // plain inputs; q[NP] = the pivot field of the precomputed-pivot form
    CUtensorMap o[3];   // TMA stores of the CG preconditioner (LineArgs::tst): r, u (TY-row boxes), z (one row)
};

// Tile geometry of the line kernels: TX = 32 columns along x per tile row,
// TY rows per tile (4, or fewer when nz needs a larger Thomas buffer), KB
// levels per pipeline stage.
constexpr int kTileX = 32;
constexpr int kStageK = 8;
constexpr int kSegK = 32;   // k-split kernel: levels per column segment

// P2P halo exchange: dst_lo <- src_first (my row 0 into the lower neighbour's slab),
// dst_hi <- src_last (my row ny-1 into the upper neighbour's); n doubles each, remote
// stores over NVLink.  Carried by k_halo_push and by producer kernels (LineArgs::push,
// k_prolong_add) that store their strip-boundary output rows into the neighbours' slabs
// themselves (fused push; src_* unused).  The epoch flags are published by the stream
// after the kernel (write-value with its memory fence), not by the kernel.
struct HaloPush {
    const double* src_first;
    const double* src_last;
    double* dst_lo;
    double* dst_hi;
    int64_t n;
    // k_halo_push only (device-side publish, TPMG_DEV_PUBLISH): the last CTA to finish its
    // remote stores (ticket counter `done`, reset by it) stores `epoch` into the neighbours'
    // flag words with st.release.sys -- instead of two stream write-values after the kernel
    unsigned* flag_lo;
    unsigned* flag_hi;
    unsigned* done;
    unsigned epoch;
};
// In-kernel halo wait (P2P overlap in ONE launch): flag[0] / flag[1] are my pool's epoch
// flags "data from the lower / upper neighbour".  When set, the line kernels walk their
// tile rows with the strip-boundary rows deferred (boundary_deferred_row) and the loader
// waits (ld.acquire.sys) until flag >= epoch before it loads a tile row that reads that halo
// slab, so interior rows run while the neighbours' rows are still on the way.  nullptr: no
// wait.
struct HaloWait {
    const unsigned* flag[2];
    unsigned epoch;
};
// Tile-row order with the two strip-boundary rows deferred by d rows (nrows >= 3):
// 1, ..., d, 0, nrows-1, d+1, ..., nrows-2.  A few µs of interior work cover the NVLink
// push; deferring them to the very end (d = nrows-2) made them the kernel's tail (r2s:
// +15% for the fine-level restriction).
__host__ __device__ inline int boundary_deferred_row(int r, int nrows, int d)
{
    if (nrows < 3) return r;
    d = d < nrows - 2 ? d : nrows - 2;
    return r < d ? r + 1 : (r == d ? 0 : (r == d + 1 ? nrows - 1 : r - 1));
}
constexpr int kHaloDefer = 8;   // tile rows of interior work before the boundary rows

struct LineArgs {
    LevelConst L;
    double rho;        // smoother relaxation (MODE_SMOOTH)
    double scale;      // MODE_PREC output scale (1 or rho for the zero-guess smooth)
    HaloField h0, h1;  // halo'd inputs
    const double* q0;  // plain inputs
    const double* q1;
    const double* q2;  // MODE_CGPREC_P: p of the previous iteration
    double* out0;
    double* out1;
    double* out2;
    DevRatio ratio;    // beta (CGDIR) or alpha (CGPREC)
    DevRatio ratio2;   // MODE_CGPREC_P: alpha of the previous iteration
    ReduceSlot red;    // result may be nullptr: no reduction
    int use_tma;       // 1: loads by TMA (tma must be filled), 0: cp.async
    const int* skip;   // device flag: the kernel returns at once when *skip != 0 (solver run-ahead)
    int part;          // TilePart: which tile rows this launch covers
    HaloPush push;     // fused halo push of the output (dst == nullptr: none)
    HaloWait hw;       // in-kernel wait for the halo'd input's slabs (P2P overlap)
    int band_w;        // k_line: tile columns per band on wide grids (0: row by row)
    int cgdir_ctas;    // k_line<CGDIR> CTAs per SM (0: automatic)
    int tst;           // k_line<CGPREC>: outputs staged in shared memory and written by TMA stores (tma.o)
    int l2hint;        // k_line TMA loads: bit 0 = halo'd fields evict_last in L2, bit 1 = plain fields evict_first
    int dbg;           // debug experiments: bit 0 = k-split in-place boxes row by row (TPMG_DBG_PERROW)
    const double* im;  // per-column fields: 1/m_k of every column's line block (Lambda layout, this
                       // level), precomputed once per operator (launch_pivots); the Thomas modes then
                       // stream it with the data instead of running the pivot recurrence
    TmaMaps tma;
};

struct Launcher {
    cudaStream_t stream;
    int num_sms;
    int64_t* launch_counter;
    int reserve_sms;   // SMs left free (for NCCL kernels running concurrently)
    bool pdl = false;  // programmatic dependent launch: overlap a kernel's launch and
                       // prologue with the previous kernel's tail (griddepcontrol)
    bool tmem = true;  // one-thread-per-column Thomas kernels keep g' in Tensor Memory (nz <= 128)
    int tm_stages = 3; // their TMA ring depth (3; 4, 5 for CGPREC A/B)
    bool carveout_fit = false;   // line kernels: the smallest shared-memory carveout for their resident CTAs (TPMG_CARVEOUT=fit)
    int tm_ctas = 1;   // CTAs per SM of those kernels (TMEM holds 2; 1 and 2 measured equal: r2c, r2f, r2k, r2p; 1 keeps every CG variant on the same grid, so the reductions -- and the iteration -- are identical)
};

// Shared-memory carveout (percent of the 228 KB maximum) that holds `ctas` CTAs of `smem`
// dynamic bytes each (+ the 1 KB per-CTA reserve); the rest of the SM's 256 KB is L1.
inline int carveout_pct(size_t smem, int64_t ctas)
{
    const size_t need = (size_t)ctas * (smem + 1024);
    const size_t maxs = (size_t)228 * 1024;
    int pct = (int)((need * 100 + maxs - 1) / maxs);
    return pct < 1 ? 1 : pct > 100 ? 100 : pct;
}

// Launch with the PDL attribute when ln.pdl.  Every kernel launched this way executes
// griddepcontrol.wait (dev::pdl_wait) in every CTA before touching global data, so it
// still observes all writes of the kernels before it.
template <typename... KArgs, typename... Args>
cudaError_t launch_kernel(const Launcher& ln, void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem,
                          Args&&... args)
{
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = ln.stream;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at;
    cfg.numAttrs = ln.pdl ? 1 : 0;
    cudaError_t e = cudaLaunchKernelEx(&cfg, kern, std::forward<Args>(args)...);
    if (e == cudaSuccess && ln.launch_counter) ++*ln.launch_counter;
    return e;
}

// Tile rows of the line kernel that will run for (mode, nz, nx) (TY of the chosen kernel).
int line_launch_rows(int mode, int nz, int nx, int use_tma, int ksplit_cfg);

cudaError_t launch_line(const Launcher& ln, int mode, const LineArgs& a);
// Tile rows TY the launcher uses for `mode` at this nz (the TMA boxes depend on it).
int line_tile_rows(int mode, int nz, int gen = 0, bool tm = false, int64_t nx = 0);   // gen: vertical profiles / fields; tm: TMEM form
bool line_gen_fits(int nz, int gen = 1);   // the line kernels' on-chip buffers fit nz (gen 1: profiles, 2: fields)
// Largest nz the on-chip Thomas buffer supports.
int line_max_nz();

// k-split line kernel (kernels_ksplit.cu) for MODE_SMOOTH / MODE_PREC.
// Per-level tables passed in the kernel parameter space: diag, 1/m, b = gamma/m,
// a = gamma/m_{k-1}, forward propagator P, backward propagator Q.
constexpr int kKsplitMaxNZ = 128;
struct KTables {
    double t[6][kKsplitMaxNZ];
};
struct KsplitBoxes {
    int ty;      // tile rows
    int kb;      // levels per chunk (f box depth)
    int hx;      // halo'd row width (u box x extent)
    int depth;   // u box depth (kb + 2)
    int xo;      // u box starts at column i0 - xo
    int hxc;     // coarse box row width (SMOOTH_PROLONG)
    int xoc;     // coarse box starts at column i0/2 - xoc
};
bool ksplit_supported(int mode, int nz, int nx);
// The launchers that have an in-kernel halo wait (LineArgs::hw) instantiation
bool ksplit_halo_wait(int mode, int cfg, int gen);
bool line_halo_wait(int mode, int nz, int gen, bool use_tma, bool tmem);
KsplitBoxes ksplit_boxes(int mode, int cfg);
cudaError_t launch_line_ksplit(const Launcher& ln, int mode, int cfg, const LineArgs& a, const KTables& T);

// z-contiguous (zc[j][i][k]) <-> Lambda (lam[j][k][i]) layout of an nx x ny x nz field
cudaError_t launch_transpose(const Launcher& ln, bool to_lambda, const double* src, double* dst, int64_t nx,
                             int64_t ny, int nz);
// f_c = 1/4 sum of the 2x2 fine children of r (plain restriction)
cudaError_t launch_restrict(const Launcher& ln, const LevelConst& fine, const LevelConst& coarse,
                            const double* r, double* fc);
// u_f += P u_c (bilinear; coarse ghosts per the boundary reading); push: fused halo push
// of the updated fine boundary rows (optional)
cudaError_t launch_prolong_add(const Launcher& ln, const LevelConst& coarse,
                               const LevelConst& fine, HaloField uc, double* uf, const int* skip = nullptr,
                               int part = PART_ALL, const HaloPush* push = nullptr, const HaloWait* hw = nullptr);
// Per-column fields: the Thomas pivots of every column's block M_T:
// m_0 = dg_0, m_k = dg_k - s_k t_{k-1} / m_{k-1}; im[(j nz + k) nx + i] = 1 / m_k.  They depend
// on the coefficients only, so they are computed once per operator (tpmg_set_fields).
cudaError_t launch_pivots(const Launcher& ln, const LevelConst& L, double* im);
// dst = src (n doubles) unless *skip
cudaError_t launch_copy(const Launcher& ln, double* dst, const double* src, int64_t n, const int* skip);

cudaError_t launch_halo_push(const Launcher& ln, const HaloPush& hp);

// Device-initiated allreduce over NVLink (P2P mode, up to kMaxP2PRanks ranks): every rank's
// halo pool holds slots[2][kMaxP2PRanks][4] doubles and flags[kMaxP2PRanks] (uint32), mapped
// into every other rank by CUDA IPC.  One single-warp kernel per allreduce of n <= 4 doubles:
// store my values into slot [E&1][me] of every rank, fence, publish epoch E in every rank's
// flags[me], wait until all flags[r] of my pool reached E, then sum slots [E&1][0..N-1] in rank
// order -- the same sum, bit for bit, on every rank.  A wait longer than ~20 s (a rank that
// died) writes NaN instead of hanging.
constexpr int kMaxP2PRanks = 8;
struct P2PReduce {
    double* slots[kMaxP2PRanks];     // rank r's slot array (r == me: my own pool)
    unsigned* flags[kMaxP2PRanks];   // rank r's flag array
    int me, nranks;
};
cudaError_t launch_allreduce_p2p(const Launcher& ln, double* d, int n, const P2PReduce& P, unsigned epoch);

// CG multi-GPU: p halo slabs updated locally, out = fma(beta, p, z) on each non-null slab.
cudaError_t launch_cg_halo(const Launcher& ln, double* out_lo, const double* z_lo, const double* p_lo, double* out_hi,
                           const double* z_hi, const double* p_hi, int64_t n, DevRatio beta, const int* skip);

// Solver run-ahead: convergence / breakdown flags computed on the device.
// Flag codes: 0 continue, 1 converged, 2 breakdown, 3 NaN, 4 iteration limit.
// CG iteration m (m >= 1): scal[3m] = sigma, scal[3m+1] = ||r||^2, scal[3m+2] = zeta; m = 0 is the
// setup (scal[1] = ||r_0||^2, scal[2] = zeta_0).  flags[m] = flags[m-1] if set, else the test.
cudaError_t launch_cg_check(const Launcher& ln, const double* scal, int m, double eps, int* flags, int* hflags);
// MG cycle n: norm2 = ||f - A u_n||^2, r0_2 = ||r_0||^2.
cudaError_t launch_mg_check(const Launcher& ln, const double* norm2, const double* r0_2, int n, double eps,
                            int max_iter, int* flags, int* hflags);
// result = sum x*y over n elements (deterministic)
cudaError_t launch_dot(const Launcher& ln, const double* x, const double* y, int64_t n,
                       ReduceSlot red);

}  // namespace tpmg
