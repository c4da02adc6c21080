// kernels.cu -- sm_100a kernels of libtpmg (fp64, memory-bound; no tensor cores:
// nothing on this path is a dense contraction).
//
// The central kernel, k_line, is the paper's "one thread per vertical column,
// loop over k" design rebuilt for B200:
//   * a CTA owns a TX x TY tile of columns (TX = 32 = one warp along the
//     x-contiguous rows of the Lambda layout) and streams the
//     tile's k-planes, with a 1-cell horizontal halo, through an NS-stage
//     cp.async ring in shared memory, KB levels per stage;
//   * the 7-point stencil (eqn:LocalMatrixStencil) reads the neighbours from
//     shared memory, the vertical neighbours from registers (k-lag by one);
//   * the Thomas forward sweep keeps the modified right-hand
//     side g'_k of every column on chip (shared memory, 8*nz bytes/column), the
//     backward sweep writes the result once: each vector crosses HBM once;
//   * the CTA is persistent over tiles, and the next tile's loads are issued
//     before the current tile's backward sweep.
// Modes fuse the paper's kernels: Smooth in ONE out-of-place pass,
// the preconditioner, and the two CG kernels (re-fused, see
// DESIGN.md).  The Thomas factors of the column block are per-level tables
// (every column has the same A_T in the flat box), so there is no per-cell
// division.
#include "kernels.cuh"
#include "device_util.cuh"

#include <algorithm>
#include <cstdlib>
#include <type_traits>

namespace tpmg {
namespace {
using namespace dev;

constexpr int TX = kTileX;  // columns per tile row (one warp, 256 B per row segment)
constexpr int KB = kStageK; // vertical levels per pipeline stage
constexpr int kNS = 3;  // pipeline stages
constexpr int kNsCgdir = 3;   // the CG direction kernel (8-row tiles, one CTA per SM): 2 stages = 3 (r2ba), 4 stages 20% slower (r2ay)
// the CG preconditioner with per-column fields keeps 4 tile rows (4 warps per SM) with 2 stages
template <int MODE, int GEN>
__host__ __device__ constexpr int stages() { return (GEN == 2 && is_cgprec(MODE)) ? 2 : (MODE == MODE_CGDIR ? kNsCgdir : kNS); }

// 1/x for the per-column pivots: the approximate reciprocal (MUFU) refined by two Newton
// steps (error ~2^-92 before rounding, i.e. correctly rounded up to an ulp) -- 5 instructions
// instead of the IEEE division's subroutine, which made the fields kernels instruction-bound.
__device__ __forceinline__ double rcp_nr(double x)
{
    double r;
    asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x));
    double e = fma(-x, r, 1.0);
    r = fma(r, e, r);
    e = fma(-x, r, 1.0);
    return fma(r, e, r);
}

// CG preconditioner tile rows in the TMEM form: 4 (one 4-warp CTA per SM, default) or 8
// (TPMG_CGPREC_TY=8: one 8-warp CTA, g' of warps 4..7 in TMEM columns 256..511).
static int cgprec_rows()
{
    const char* e = std::getenv("TPMG_CGPREC_TY");   // (read per call, like TPMG_CGDIR_TY)
    return (e && std::atoi(e) == 8) ? 8 : 4;
}

template <int MODE>
struct Traits;
template <> struct Traits<MODE_APPLY>  { static constexpr int NH = 1, NP = 0, THOMAS = 0, NR = 0; };
template <> struct Traits<MODE_RESID>  { static constexpr int NH = 1, NP = 1, THOMAS = 0, NR = 1; };
template <> struct Traits<MODE_PREC>   { static constexpr int NH = 0, NP = 1, THOMAS = 1, NR = 0; };
template <> struct Traits<MODE_SMOOTH> { static constexpr int NH = 1, NP = 1, THOMAS = 1, NR = 1; };
template <> struct Traits<MODE_CGDIR>  { static constexpr int NH = 2, NP = 0, THOMAS = 0, NR = 1; };
template <> struct Traits<MODE_CGPREC> { static constexpr int NH = 1, NP = 2, THOMAS = 1, NR = 2; };
template <> struct Traits<MODE_RESTRICT> { static constexpr int NH = 1, NP = 1, THOMAS = 0, NR = 0; };
template <> struct Traits<MODE_CGPREC_D> { static constexpr int NH = 1, NP = 1, THOMAS = 1, NR = 2; };
template <> struct Traits<MODE_CGPREC_P> { static constexpr int NH = 1, NP = 3, THOMAS = 1, NR = 2; };

template <int NH, int NP, int TY>
struct Geom {
    // halo rows span i0-2 .. i0+TX+1: TMA needs a 16-byte aligned (even) start column
    static constexpr int HX = TX + 4, HY = TY + 2, NT = TX * TY;
    static constexpr int HALO_ROW = KB * HX;          // one (row, all kk) block
    static constexpr int PLAIN_BASE = NH * HY * KB * HX;
    static constexpr int STAGE = PLAIN_BASE + NP * TY * KB * TX;  // doubles per stage
};

// Issue the cp.async copies of one stage (levels k0..k0+KB-1 of the tile).
// One warp per (field, row, level) segment; out-of-domain cells are zero-filled.
template <int NH, int NP, int TY>
__device__ __forceinline__ void load_stage(double* st, const LineArgs& a, int64_t i0, int64_t j0, int k0)
{
    using G = Geom<NH, NP, TY>;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    constexpr int NW = G::NT / 32;
    constexpr int NSEG_H = NH * G::HY * KB;
    constexpr int NSEG = NSEG_H + NP * TY * KB;
    const int64_t nx = a.L.nx, ny = a.L.ny;
    const int nz = a.L.nz;
    const int64_t plane = nx * (int64_t)nz;
    for (int seg = warp; seg < NSEG; seg += NW) {
        if (seg < NSEG_H) {
            const int f = seg / (G::HY * KB);
            const int rem = seg - f * (G::HY * KB);
            const int r = rem / KB, kk = rem - (rem / KB) * KB;
            const HaloField& H = (f == 0) ? a.h0 : a.h1;
            const int64_t j = j0 - 1 + r;
            const int k = k0 + kk;
            const double* row = (j < 0) ? H.lo : (j >= ny ? H.hi : H.base + j * plane);
            const bool rowok = (row != nullptr) && (k < nz);
            double* dst = st + ((f * G::HY + r) * KB + kk) * G::HX;
#pragma unroll
            for (int x = lane; x < G::HX; x += 32) {
                const int64_t i = i0 - 2 + x;
                const bool ok = rowok && i >= 0 && i < nx;
                cp_async8(dst + x, ok ? row + (int64_t)k * nx + i : H.base, ok);
            }
        } else {
            const int s2 = seg - NSEG_H;
            const int f = s2 / (TY * KB);
            const int rem = s2 - f * (TY * KB);
            const int r = rem / KB, kk = rem - (rem / KB) * KB;
            const double* Q = (f == 0) ? a.q0 : (f == 1 ? a.q1 : a.q2);
            const int64_t j = j0 + r;
            const int k = k0 + kk;
            const bool rowok = (j < ny) && (k < nz);
            double* dst = st + G::PLAIN_BASE + ((f * TY + r) * KB + kk) * TX;
            const int64_t i = i0 + lane;
            const bool ok = rowok && i < nx;
            cp_async8(dst + lane, ok ? Q + j * plane + (int64_t)k * nx + i : Q, ok);
        }
    }
}

// Issue the TMA copies of one stage (thread 0 only).  Box layout in shared
// memory is identical to load_stage's: halo field f, row r, level kk, x.
template <int NH, int NP, int TY>
__device__ __forceinline__ void tma_stage(double* st, const LineArgs& a, int64_t i0, int64_t j0, int k0,
                                          uint64_t* bar, uint64_t pol_h = 0, uint64_t pol_q = 0)
{
    // a.l2hint: the main boxes carry an L2 policy (pol_h for the halo'd fields, pol_q for the plain ones)
    auto load_h = [&](double* dst, const CUtensorMap* m, int x, int y, int z) {
        if (a.l2hint & 1) tma_load_3d_hint(dst, m, x, y, z, bar, pol_h);
        else tma_load_3d(dst, m, x, y, z, bar);
    };
    using G = Geom<NH, NP, TY>;
    mbar_expect_tx(bar, (uint32_t)(G::STAGE * sizeof(double)));
    const int64_t ny = a.L.ny;
    const int x0 = (int)i0 - 2;
#pragma unroll
    for (int f = 0; f < NH; ++f) {
        const TmaHalo& M = a.tma.h[f];
        double* dst = st + f * G::HY * G::HALO_ROW;
        const bool lo = M.has_lo && j0 == 0, hi = M.has_hi && j0 + TY >= ny;
        if (!lo && !hi) {
            load_h(dst, &M.main, x0, k0, (int)j0 - 1);
        } else if (M.has_m1 && lo != hi && (lo || j0 + TY == ny)) {   // (a ragged last row: row by row)
            // strip-boundary tile: the in-domain rows as one box, the slab row by itself (a
            // row-by-row tile is several times slower and its CTA sets the kernel time)
            if (lo) {
                tma_load_3d(dst, &M.lo, x0, k0, 0, bar);
                tma_load_3d(dst + G::HALO_ROW, &M.m1, x0, k0, (int)j0, bar);
            } else {
                tma_load_3d(dst, &M.m1, x0, k0, (int)j0 - 1, bar);
                tma_load_3d(dst + (G::HY - 1) * G::HALO_ROW, &M.hi, x0, k0, 0, bar);
            }
        } else {
            for (int r = 0; r < G::HY; ++r) {
                const int64_t j = j0 - 1 + r;
                const CUtensorMap* m = &M.row;
                int jj = (int)j;
                if (j < 0 && M.has_lo) { m = &M.lo; jj = 0; }
                else if (j == ny && M.has_hi) { m = &M.hi; jj = 0; }
                tma_load_3d(dst + r * G::HALO_ROW, m, x0, k0, jj, bar);
            }
        }
    }
#pragma unroll
    for (int f = 0; f < NP; ++f) {
        if (a.l2hint & 2) tma_load_3d_hint(st + G::PLAIN_BASE + f * TY * KB * TX, &a.tma.q[f], (int)i0, k0, (int)j0, bar, pol_q);
        else tma_load_3d(st + G::PLAIN_BASE + f * TY * KB * TX, &a.tma.q[f], (int)i0, k0, (int)j0, bar);
    }
}

// The line kernel.  LOADER = 0: cp.async (all threads); 1: TMA (thread 0) with an
// mbarrier per stage.  The CTA walks its tiles (tile = blockIdx.x + t*gridDim.x)
// as one global sequence of KB-level chunks, so the loads of the next tile's
// first chunks overlap the current tile's backward sweep.
// GEN: 0 flat box, 1 general vertical profiles, 2 per-column horizontal fields (|T|, alpha_T
// and the 4 face alpha_{T,T'} of every column; profiles a, b, c, d as well).  With
// fields the Thomas factors differ from column to column: the forward sweep computes the
// pivots of its own column through the leading principal minors, p_k = diag_k p_{k-1} -
// s_k t_{k-1} p_{k-2}, m_k = p_k / p_{k-1} (a linear recurrence: one FMA per level on the
// dependency chain, the division 1/m_k = p_{k-1}/p_k off it), renormalised at every KB-th level
// to (p_{k-1}, p_{k-2}) = (m_{k-1}, 1), and checkpoints m_{k-1} there next to g'_k in shared
// memory ((nz + nz/KB) * 8 bytes per column).  The backward sweep recomputes each chunk's
// pivots from its checkpoint with the same arithmetic instead of keeping all nz on chip.
// TM: the Thomas intermediates g'_k live in Tensor Memory instead of shared memory (flat box,
// 4 warps = the 4 TMEM lane quarters, nz <= 128): the 8*nz bytes per column of shared memory
// that held one CTA per SM leave room for two, i.e. twice the warps to hide the recurrences'
// latency; TMEM itself (256 columns = 128 levels per CTA) holds exactly two CTAs.
constexpr uint32_t kTmemCols = 256;
// HW: the in-kernel halo wait of the P2P overlap (LineArgs::hw), a separate instantiation
// GEN 3: per-column fields with the pivots precomputed (LineArgs::im): like GEN 2, but 1/m_k
// arrives as one more plain field through the TMA ring and the Thomas sweeps run no pivot
// recurrence; g'_k and 1/m_k both live in TMEM (4 columns per level, the whole TMEM of the SM).
// TST: the CG preconditioner's outputs r, u (forward sweep) and z (backward sweep) are staged
// in shared memory and written by TMA stores (LineArgs::tst, tma.o) instead of one STG per cell
// and output with its 64-bit address arithmetic: r, u in groups of KB levels (3 buffers: the
// group being written, the one whose last level is finalised one chunk later, the one in
// flight), z per warp in KB-level rows (2 buffers).
template <int MODE, int TY, int LOADER, int GEN, int TMS = 0, bool HW = false, bool TST = false>
__global__ void __launch_bounds__(TX* TY) k_line(const __grid_constant__ LineArgs a)
{
    static_assert(!TST || (MODE == MODE_CGPREC && TMS > 0 && GEN == 0 && LOADER == 1 && !HW), "TMA stores: TMEM CGPREC");
    using T = Traits<MODE>;
    constexpr bool TM = TMS > 0;   // TMS: pipeline stages of the TMEM form (the freed shared memory deepens it)
    static_assert(!TM || ((TY == 4 || (TY == 8 && GEN == 0)) && T::THOMAS),
                  "TMEM g' buffer: 4 warps (the 4 TMEM lane quarters) or 8 (two column halves), Thomas modes");
    static_assert(GEN != 3 || (TM && T::THOMAS), "precomputed pivots: TMEM form of the Thomas modes");
    constexpr int NH = T::NH, NR = T::NR;
    constexpr int NP = T::NP + (GEN == 3 ? 1 : 0);   // + the pivot field
    constexpr uint32_t NCOL = (GEN == 3 || TY == 8) ? 512u : kTmemCols;
    using G = Geom<NH, NP, TY>;
    constexpr int NT = G::NT;
    constexpr int NS = TM ? TMS : stages<MODE, GEN>();

    extern __shared__ __align__(128) double smem_raw[];
    __shared__ __align__(8) uint64_t full_bar[NS];
    // TMA destinations must be 128-byte aligned: align the dynamic window explicitly
    double* smem = reinterpret_cast<double*>(
        reinterpret_cast<char*>(smem_raw) + ((128u - (smem_u32(smem_raw) & 127u)) & 127u));
    const int nz = a.L.nz;
    const int64_t nx = a.L.nx, ny = a.L.ny;
    const int tabn = (3 * nz + 15) & ~15;    // keep the stages 128-byte aligned
    const int ptn = (GEN >= 2) ? ((4 * nz + 15) & ~15) : tabn;   // GEN 3 uses GEN 2's profile table
    double* tab = smem;                      // diag[nz], invm[nz], gim[nz]
    double* ptab = smem + tabn;              // GEN 1: b_k, c_k, c_l d_k; GEN 2: a_k-b_k-c_k, b_k, c_k, d_k
    double* stage = ptab + (GEN ? ptn : 0);  // NS stages
    double* gbuf = stage + NS * G::STAGE;    // g'[nz][NT] (Thomas modes)
    const int nck = (nz + KB - 1) / KB;
    double* cbuf = gbuf + (TM ? 0 : nz * NT);           // GEN 2: m_{c KB - 1}[nck][NT], the pivot checkpoints
    // MODE_RESTRICT: x-pair sums [2][TY][KB+1][TX/2] (a chunk completes up to KB+1 levels)
    constexpr int RS = KB + 1;
    double* rbuf = gbuf + (T::THOMAS ? ((TM ? 0 : nz) + (GEN == 2 ? nck : 0)) * NT : 0);
    double* scratch = rbuf + (MODE == MODE_RESTRICT ? 2 * TY * RS * (TX / 2) : 0);  // reduction scratch
    // TST staging (128-byte aligned TMA sources): sfw[3][2][KB][TY][TX] (r, u), sbw[2][TY][KB][TX] (z)
    // (pointer arithmetic only, so that the compiler keeps the shared state space: STS, not ST)
    double* sfw = scratch + 64 + ((128u - (smem_u32(scratch + 64) & 127u)) & 127u) / 8u;
    double* sbw = sfw + 3 * 2 * KB * G::NT;

    const int tid = threadIdx.x, tx = tid & 31, ty = tid >> 5;
    for (int q = tid; q < 3 * nz; q += NT) tab[q] = a.L.tab[q];   // interior class (0)
    if constexpr (GEN != 0)
        for (int q = tid; q < (GEN >= 2 ? 4 : 3) * nz; q += NT) ptab[q] = a.L.prof[q];
    const double* diag_s = tab;
    const double* invm_s = tab + nz;
    const double* gim_s = tab + 2 * nz;
    const double c0 = a.L.c, gamma = a.L.gamma;
    if constexpr (LOADER == 1) {
        if (tid == 0) {
            for (int s = 0; s < NS; ++s) mbar_init(&full_bar[s], 1);
            asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
        }
    }

    // prologue above (tables, barriers) overlaps the previous kernel's tail under PDL
    pdl_wait();
    pdl_trigger();
    if (a.skip && *a.skip) return;   // solver run-ahead: this iteration is not needed

    auto put = [](double* q, double v) { *q = v; };   // (st.global.cs measured no different, r2o)
    constexpr bool CGP = is_cgprec(MODE);
    double ratio = 0.0, ratio2 = 0.0;
    if constexpr (MODE == MODE_CGDIR || CGP)
        if (a.ratio.num >= 0) ratio = a.ratio.s[a.ratio.num] / a.ratio.s[a.ratio.den];
    if constexpr (MODE == MODE_CGPREC_P)
        if (a.ratio2.num >= 0) ratio2 = a.ratio2.s[a.ratio2.num] / a.ratio2.s[a.ratio2.den];

    double acc[NR > 0 ? NR : 1];
#pragma unroll
    for (int r = 0; r < (NR > 0 ? NR : 1); ++r) acc[r] = 0.0;
    const bool want_red = (NR > 0) && (a.red.result != nullptr);

    // 32-bit bookkeeping (tiles < 2^31); the producer and consumer walk the same chunk
    // sequence with incremental cursors (no per-chunk integer division).
    const int ntx = (int)((nx + TX - 1) / TX), nty = (int)((ny + TY - 1) / TY);
    const int ntiles = ntx * part_rows(a.part, nty);
    const int nch = (nz + KB - 1) / KB;
    const int my_tiles = ((int)blockIdx.x < ntiles) ? (ntiles - (int)blockIdx.x + (int)gridDim.x - 1) / (int)gridDim.x : 0;
    const int total = my_tiles * nch;
    __shared__ uint32_t tmem_slot;
    if constexpr (TM) {
        if (ty == 0) tmem_alloc<NCOL>(&tmem_slot);
        tmem_fence_before();
    }
    __syncthreads();
    uint32_t tbase = 0;   // TM: this warp's lane quarter, column 0
    if constexpr (TM) {
        tmem_fence_after();
        // warp ty: lane quarter ty % 4; with 8 warps the second four use columns 256..511
        tbase = tmem_slot + ((uint32_t)((ty & 3) * 32) << 16) + (uint32_t)(ty >> 2) * kTmemCols;
    }

    // producer cursor: next chunk to load
    int p_count = 0, p_ch = 0, p_slot = 0, p_tile = blockIdx.x;
    const bool plo = a.push.dst_lo != nullptr, phi = a.push.dst_hi != nullptr;
    const int nrows = part_rows(a.part, nty);
    // Wide grids (a.band_w > 0 tile columns per band, ntx > band_w): the tiles are walked band by
    // band, so the CTAs working at any moment cover a band_w-tile-wide strip several tile rows
    // deep -- vertically adjacent tiles (which share halo rows) are in flight together and the
    // halo rows are re-read from L2, as on a 1024-wide grid (round 1: 2.1x the algorithmic
    // reads at nx = 4096 without it).
    const int bw = (a.band_w > 0 && ntx > a.band_w) ? a.band_w : ntx;
    auto col_of = [&](int t) {
        const int b = t / (bw * nrows), rt = t - b * bw * nrows, w = min(bw, ntx - b * bw);
        return b * bw + rt % w;
    };
    auto raw_row = [&](int t) {
        const int b = t / (bw * nrows), rt = t - b * bw * nrows, w = min(bw, ntx - b * bw);
        return rt / w;
    };
    auto row_of = [&](int t) {
        if constexpr (HW) return boundary_deferred_row(raw_row(t), nrows, kHaloDefer);   // in-kernel halo wait
        return part_row(a.part, nty, push_row(raw_row(t), nrows, plo, phi));
    };
    int p_i0 = col_of(p_tile) * TX, p_j0 = row_of(p_tile) * TY;
    uint64_t pol_h = 0, pol_q = 0;
    if constexpr (LOADER == 1)
        if (tid == 0 && a.l2hint) {
            pol_h = l2_policy_evict_last();
            pol_q = l2_policy_evict_first();
        }
    auto issue = [&]() {
        if (p_count < total) {
            double* st = stage + p_slot * G::STAGE;
            if constexpr (HW)   // the first load of a tile row that reads a halo slab waits for its epoch
                if (p_ch == 0 && (LOADER == 0 || tid == 0)) halo_tile_wait(a.hw, (int)p_j0, TY, (int)ny);
            if constexpr (LOADER == 0) {
                load_stage<NH, NP, TY>(st, a, p_i0, p_j0, p_ch * KB);
            } else {
                if (tid == 0) {
                    asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
                    tma_stage<NH, NP, TY>(st, a, p_i0, p_j0, p_ch * KB, &full_bar[p_slot], pol_h, pol_q);
                }
            }
            ++p_count;
            if (++p_slot == NS) p_slot = 0;
            if (++p_ch == nch) {
                p_ch = 0;
                p_tile += gridDim.x;
                p_i0 = col_of(p_tile) * TX;
                p_j0 = row_of(p_tile) * TY;
            }
        }
        if constexpr (LOADER == 0) cp_async_commit();
    };
    // consumer cursor
    int c_slot = 0;
    uint32_t c_phase = 0;
    auto wait = [&]() {
        if constexpr (LOADER == 0) {
            cp_async_wait<NS - 1>();
            __syncthreads();
        } else {
            mbar_wait(&full_bar[c_slot], c_phase);
        }
    };
    auto advance = [&]() {
        if (++c_slot == NS) {
            c_slot = 0;
            c_phase ^= 1u;
        }
    };

#pragma unroll
    for (int s = 0; s < NS - 1; ++s) issue();

    int gi = 0;
    // One tile.  BND: the tile holds columns of other classes (face Dirichlet [R25]); each
    // thread then reads its column's Thomas factors from the global class tables.
    auto tile_body = [&](auto bnd_t, int tl) {
        constexpr bool BND = decltype(bnd_t)::value;
        const int tile = (int)blockIdx.x + tl * (int)gridDim.x;
        const int64_t i0 = (int64_t)col_of(tile) * TX, j0 = (int64_t)row_of(tile) * TY;
        const int64_t i = i0 + tx, j = j0 + ty;
        const bool valid = (i < nx) && (j < ny);
        const int64_t colbase = j * nx * (int64_t)nz + i;  // + k*nx
        const double* ctab = BND ? a.L.tab + (size_t)column_class(a.L, i, j) * kTabArrays * nz : nullptr;
        const double* diag = BND ? ctab : diag_s;
        const double* invm = BND ? ctab + nz : invm_s;
        const double* gim = BND ? ctab + 2 * nz : gim_s;
        // GEN 2: this column's |T|, alpha_T and face alpha_{T,T'} (W, E, S, N), fields SoA
        // [6][ny][nx] (a phantom column of a ragged tile gets |T| = 1 and no couplings)
        double fT = 1.0, faT = 0.0, fw = 0.0, fe = 0.0, fs = 0.0, fn = 0.0;
        double pm1 = 1.0, pm2 = 0.0, tkm1 = 0.0;   // GEN 2 pivot state: p_{k-1}, p_{k-2}, t_{k-1}
        // GEN 2: one step of the minor recurrence at level k, returns 1/m_k (S:267's pivot)
        auto pivot_step = [&](int k, double& p1, double& p2, double& t1) {
            const double sk = fT * ptab[nz + k];
            const double tk = fT * ptab[2 * nz + k];
            const double dgk = fma(fT, ptab[k], -faT * ptab[3 * nz + k]);
            const double p = fma(dgk, p1, -(sk * t1) * p2);
            const double im = p1 * rcp_nr(p);
            p2 = p1;
            p1 = p;
            t1 = tk;
            return im;
        };
        if constexpr (GEN >= 2) {
            if (valid) {
                const int64_t ncol = nx * ny, cc = j * nx + i;
                const double* F = a.L.fld + cc;
                fT = __ldg(F);
                faT = __ldg(F + ncol);
                fw = __ldg(F + 2 * ncol);
                fe = __ldg(F + 3 * ncol);
                fs = __ldg(F + 4 * ncol);
                fn = __ldg(F + 5 * ncol);
            }
        }

        // rolling state for the k-lag: values at level km = k-1 and km-1
        double um1 = 0.0, u0 = 0.0, S0 = 0.0, qa = 0.0, qb = 0.0, qc = 0.0, qd = 0.0, gprev = 0.0;   // qc: 1/m_k (GEN 3), qd: p_prev
        double* rbuf_cur = rbuf;   // MODE_RESTRICT: buffer of the current chunk
        // forward-pass outputs of level km live at ofw0/ofw1 (advanced by nx per level)
        double* ofw0 = (MODE == MODE_APPLY || MODE == MODE_RESID || MODE == MODE_CGDIR || CGP) && a.out0
                           ? a.out0 + colbase : nullptr;
        double* ofw1 = (MODE == MODE_CGPREC || MODE == MODE_CGPREC_P) ? a.out1 + colbase : nullptr;

        // Complete level km (its upper neighbour up1 has arrived): stencil, the mode's
        // pointwise work and one Thomas forward-elimination step.
        auto finalize = [&](double up1, double dgk, double imk, double* gslot, int rslot, int km, double* sbo) {
            // (M_T u)_k and the coefficient of the horizontal neighbour sum: -gamma and c in
            // the flat box; b_k, c_k and c_l d_k with general profiles (GEN, shared memory)
            double Mu, c, sk = -gamma, tk = 0.0;
            if constexpr (GEN >= 2) {
                // A_T = |T| (diag(a) + tridiag(-(b+c), b, c)) - alpha_T diag(d)
                sk = fT * ptab[nz + km];
                tk = fT * ptab[2 * nz + km];
                dgk = fma(fT, ptab[km], -faT * ptab[3 * nz + km]);
                Mu = fma(sk, um1, fma(tk, up1, dgk * u0));
                c = -ptab[3 * nz + km];   // A u = M_T u + d_k sum_T' alpha_TT' u_T'
            } else if constexpr (GEN == 1) {
                sk = ptab[km];
                Mu = fma(sk, um1, fma(ptab[nz + km], up1, dgk * u0));
                c = ptab[2 * nz + km];
            } else {
                Mu = fma(-gamma, um1 + up1, dgk * u0);
                c = c0;
            }
            double g = 0.0;
            if constexpr (MODE == MODE_APPLY) {
                if (valid) *ofw0 = fma(-c, S0, Mu);                 // (A u)_k = (M_T u)_k - c sum(nbrs)
            } else if constexpr (MODE == MODE_RESID) {
                const double r = fma(c, S0, qa) - Mu;               // f - A u
                if (valid) {
                    if (ofw0) *ofw0 = r;
                    acc[0] = fma(r, r, acc[0]);
                }
            } else if constexpr (MODE == MODE_PREC) {
                g = a.scale * qa;
            } else if constexpr (MODE == MODE_SMOOTH) {
                const double r = fma(c, S0, qa) - Mu;               // f - A u
                g = fma(a.rho, r, Mu);   // = rho f + (M - rho A) u   (one-pass smoother)
                if (valid) acc[0] = fma(r, r, acc[0]);
            } else if constexpr (MODE == MODE_CGDIR) {
                const double Ap = fma(-c, S0, Mu);
                if (valid) {
                    put(ofw0, u0);
                    acc[0] = fma(u0, Ap, acc[0]);
                }
            } else if constexpr (MODE == MODE_RESTRICT) {
                // r = f - A u, summed over the x-pair (2I, 2I+1) of fine columns
                const double r = fma(c, S0, qa) - Mu;
                const double rs = r + __shfl_xor_sync(0xffffffffu, r, 1);
                if ((tx & 1) == 0) rbuf_cur[(ty * RS + rslot) * (TX / 2) + (tx >> 1)] = rs;
            } else if constexpr (TST) {   // (MODE_CGPREC) r, u staged for the group's TMA stores
                const double Ap = fma(-c, S0, Mu);
                const double rn = fma(-ratio, Ap, qa);
                sbo[0] = rn;
                sbo[KB * NT] = fma(ratio, u0, qb);
                if (valid) acc[0] = fma(rn, rn, acc[0]);
                g = rn;
            } else if constexpr (CGP) {
                const double Ap = fma(-c, S0, Mu);
                const double rn = fma(-ratio, Ap, qa);
                if (valid) {
                    put(ofw0, rn);
                    if constexpr (MODE == MODE_CGPREC) put(ofw1, fma(ratio, u0, qb));
                    if constexpr (MODE == MODE_CGPREC_P) put(ofw1, fma(ratio, u0, fma(ratio2, qd, qb)));
                    acc[0] = fma(rn, rn, acc[0]);
                }
                g = rn;
            }
            if constexpr ((MODE == MODE_APPLY || MODE == MODE_RESID || MODE == MODE_CGDIR || CGP) && !TST) {
                if constexpr (MODE == MODE_RESID) {   // the only mode whose out0 may be absent
                    if (ofw0) ofw0 += nx;
                } else {
                    ofw0 += nx;
                }
                if constexpr (MODE == MODE_CGPREC || MODE == MODE_CGPREC_P) ofw1 += nx;
            }
            if constexpr (T::THOMAS) {
                if constexpr (GEN == 2) {
                    // this column's pivot: m_k = diag_k - s_k t'_{k-1}, t'_k = t_k / m_k
                    imk = pivot_step(km, pm1, pm2, tkm1);
                } else if constexpr (GEN == 3) {
                    imk = qc;   // this column's 1/m_k, precomputed (launch_pivots)
                }
                const double y = fma(-sk, gprev, g);     // y = L^-1 g   (M = L D L^T; sub-diagonal s_k)
                const double gp = y * imk;               // g'_k = (g_k - s_k g'_{k-1}) / m_k
                if constexpr (GEN == 3)
                    tmem_st_f64x2(tbase + 4u * (uint32_t)km, gp, imk);   // the backward sweep needs both
                else if constexpr (TM)
                    tmem_st_f64(tbase + 2u * (uint32_t)km, gp);
                else
                    *gslot = gp;
                if constexpr (CGP)
                    if (valid) acc[1] = fma(gp, y, acc[1]);   // <g, M^-1 g> = sum y_k^2 / m_k
                gprev = gp;
            }
        };

        // One KB-level chunk.  FULL: an interior chunk (ch >= 1, k0 + KB <= nz) needs no
        // bounds checks.  All offsets are compile-time constants from per-chunk bases.
        auto do_chunk = [&](auto full_t, int ch, const double* st) {
            constexpr bool FULL = decltype(full_t)::value;
            const int k0 = ch * KB;
            double ecv[KB], Sv[KB], pav[KB], pbv[KB], pcv[KB], pdv[KB];
            const double* hp = st + (ty + 1) * G::HALO_ROW + tx + 2;           // own column
            const double* pp = st + G::PLAIN_BASE + ty * (KB * TX) + tx;       // plain field 0
#pragma unroll
            for (int kk = 0; kk < KB; ++kk) {
                ecv[kk] = 0.0; Sv[kk] = 0.0; pav[kk] = 0.0; pbv[kk] = 0.0; pcv[kk] = 0.0; pdv[kk] = 0.0;
                if constexpr (NH >= 1) {
                    const double* h = hp + kk * G::HX;
                    ecv[kk] = h[0];
                    // neighbour sum; GEN 2: weighted by the face alpha_{T,T'}
                    auto nsum = [&](const double* q) {
                        if constexpr (GEN >= 2)
                            return fma(fw, q[-1], fe * q[1]) + fma(fs, q[-G::HALO_ROW], fn * q[G::HALO_ROW]);
                        else
                            return (q[-1] + q[1]) + (q[-G::HALO_ROW] + q[G::HALO_ROW]);
                    };
                    Sv[kk] = nsum(h);
                    if constexpr (MODE == MODE_CGDIR) {
                        const double* p = h + G::HY * G::HALO_ROW;  // field 1 = p_old
                        ecv[kk] = fma(ratio, p[0], ecv[kk]);
                        Sv[kk] = fma(ratio, nsum(p), Sv[kk]);
                    }
                }
                if constexpr (T::NP >= 1) pav[kk] = pp[kk * TX];
                if constexpr (T::NP >= 2) pbv[kk] = pp[TY * KB * TX + kk * TX];
                if constexpr (T::NP >= 3) pdv[kk] = pp[2 * TY * KB * TX + kk * TX];   // MODE_CGPREC_P: p_prev
                if constexpr (GEN == 3) pcv[kk] = pp[T::NP * TY * KB * TX + kk * TX];   // the pivot field
            }
            if constexpr (TST) {
                fence_proxy_async_smem();           // my staged r, u before the barrier
                if (tid == 0) bulk_wait_read<0>();  // the group stored one chunk ago has left its buffer
            }
            __syncthreads();   // slot gi % NS is free for chunk gi + NS
            if constexpr (TST)
                if (tid == 0 && ch >= 2) {   // group ch-2 is complete (its last level was finalised in chunk ch-1)
                    const double* src = sfw + ((gi + 1) % 3) * (2 * KB * NT);
                    tma_store_3d(&a.tma.o[0], (int)i0, (ch - 2) * KB, (int)j0, src);
                    tma_store_3d(&a.tma.o[1], (int)i0, (ch - 2) * KB, (int)j0, src + KB * NT);
                    bulk_commit();
                }
            if constexpr (MODE == MODE_RESTRICT) rbuf_cur = rbuf + (gi & 1) * (TY * RS * (TX / 2));
            const double* dg = diag + (k0 - 1);      // level km = k0 - 1 + kk
            const double* im = invm + (k0 - 1);
            double* gb = gbuf + (k0 - 1) * NT + tid;
            // TST staging: level k0-1 closes the previous group (buffer (gi+2)%3, slot KB-1), the
            // chunk's other levels open group gi (buffer gi%3); box layout [row][level][x]
            double* sbp = sfw + ((gi + 2) % 3) * (2 * KB * NT) + ty * (KB * TX) + tx + (KB - 1) * TX;
            double* sbc = sfw + (gi % 3) * (2 * KB * NT) + ty * (KB * TX) + tx - TX;
#pragma unroll
            for (int kk = 0; kk < KB; ++kk) {
                const int k = k0 + kk;
                if (FULL || k < nz) {
                    if (FULL || k > 0) finalize(ecv[kk], dg[kk], im[kk], gb + kk * NT, kk, k - 1, kk == 0 ? sbp : sbc + kk * TX);
                    if constexpr (GEN == 2 && T::THOMAS)
                        if (kk == 0 && ch > 0) {   // renormalise and checkpoint m_{k0-1}
                            const double m = pm1 * rcp_nr(pm2);
                            pm1 = m;
                            pm2 = 1.0;
                            cbuf[ch * NT + tid] = m;
                        }
                    um1 = u0; u0 = ecv[kk]; S0 = Sv[kk]; qa = pav[kk]; qb = pbv[kk]; qc = pcv[kk]; qd = pdv[kk];
                }
            }
        };

        for (int ch = 0; ch < nch; ++ch, ++gi) {
            issue();
            wait();
            const double* st = stage + c_slot * G::STAGE;
            advance();
            if (ch >= 1 && (ch + 1) * KB <= nz)
                do_chunk(std::true_type{}, ch, st);
            else
                do_chunk(std::false_type{}, ch, st);
            if (ch == nch - 1)
                finalize(0.0, diag[nz - 1], invm[nz - 1], gbuf + (nz - 1) * NT + tid, nz - ch * KB, nz - 1,
                         sfw + (gi % 3) * (2 * KB * NT) + ty * (KB * TX) + tx + (KB - 1) * TX);
            if constexpr (MODE == MODE_RESTRICT) {
                // f_c(I, J, k) = 1/4 (x-pair sum of row 2J + x-pair sum of row 2J+1);
                // this chunk completed levels ch*KB-1 .. ch*KB+KB-2 (and nz-1 if last), slot
                // s holding level ch*KB-1+s
                __syncthreads();
                const int slot_base = ch * KB - 1;
                const int lo = (ch == 0) ? 0 : ch * KB - 1;
                const int hi = (ch == nch - 1) ? nz - 1 : ch * KB + KB - 2;
                const int64_t nxc = nx >> 1, nyc = ny >> 1;
                const int nlev = hi - lo + 1;
                for (int it = tid; it < (TY / 2) * RS * (TX / 2); it += NT) {
                    const int l = it % (TX / 2);
                    const int sl = (it / (TX / 2)) % RS;
                    const int jp = it / ((TX / 2) * RS);
                    const int km = lo + sl;
                    if (sl < nlev) {
                        const int slot = km - slot_base;
                        const int64_t I = (i0 >> 1) + l, J = (j0 >> 1) + jp;
                        if (I < nxc && J < nyc)
                            a.out0[(J * nz + km) * nxc + I] =
                                0.25 * (rbuf_cur[((2 * jp) * RS + slot) * (TX / 2) + l] +
                                        rbuf_cur[((2 * jp + 1) * RS + slot) * (TX / 2) + l]);
                    }
                }
            }
        }
        if constexpr (TST) {   // the tile's last two groups (gi is one past the last chunk)
            fence_proxy_async_smem();
            __syncthreads();
            if (tid == 0) {
                const double* s1 = sfw + ((gi + 1) % 3) * (2 * KB * NT);   // group nch-2
                const double* s2 = sfw + ((gi + 2) % 3) * (2 * KB * NT);   // group nch-1
                tma_store_3d(&a.tma.o[0], (int)i0, (nch - 2) * KB, (int)j0, s1);
                tma_store_3d(&a.tma.o[1], (int)i0, (nch - 2) * KB, (int)j0, s1 + KB * NT);
                bulk_commit();
                tma_store_3d(&a.tma.o[0], (int)i0, (nch - 1) * KB, (int)j0, s2);
                tma_store_3d(&a.tma.o[1], (int)i0, (nch - 1) * KB, (int)j0, s2 + KB * NT);
                bulk_commit();
            }
        }

        if constexpr (T::THOMAS && GEN == 3) {
            // backward substitution x_k = g'_k - (t_k / m_k) x_{k+1}, 8 levels per TMEM load of
            // (g'_k, 1/m_k) pairs
            double* op = (CGP ? a.out2 : a.out0) + colbase + (int64_t)(nz - 1) * nx;
            double x = 0.0;
            int k = nz - 1;
            tmem_wait_st();   // the forward sweep's stores have landed
            for (; k >= KB - 1; k -= KB) {
                double v[2 * KB];   // v[2q] = g'_{k0+q}, v[2q+1] = 1/m_{k0+q}, k0 = k-KB+1
                tmem_ld_f64x16(tbase + 4u * (uint32_t)(k - (KB - 1)), v);
#pragma unroll
                for (int q = KB - 1; q >= 0; --q) {
                    const int kq = k - (KB - 1) + q;
                    const double tp = fT * ptab[2 * nz + kq] * v[2 * q + 1];   // t'_k = t_k / m_k
                    x = fma(-tp, x, v[2 * q]);
                    if (valid) put(op, x);
                    op -= nx;
                }
            }
            for (; k >= 0; --k) {
                double v2[2];
                {
                    uint32_t lo0, hi0, lo1, hi1;
                    asm volatile(
                        "tcgen05.ld.sync.aligned.32x32b.x4.b32 {%0, %1, %2, %3}, [%4];\n"
                        "tcgen05.wait::ld.sync.aligned;\n"
                        : "=r"(lo0), "=r"(hi0), "=r"(lo1), "=r"(hi1)
                        : "r"(tbase + 4u * (uint32_t)k)
                        : "memory");
                    v2[0] = __hiloint2double((int)hi0, (int)lo0);
                    v2[1] = __hiloint2double((int)hi1, (int)lo1);
                }
                x = fma(-(fT * ptab[2 * nz + k] * v2[1]), x, v2[0]);
                if (valid) put(op, x);
                op -= nx;
            }
        }
        if constexpr (T::THOMAS && GEN == 2) {
            // backward substitution per KB-level chunk: the chunk's t'_k recomputed from its
            // checkpoint with the forward sweep's arithmetic, then x_k = g'_k - t'_k x_{k+1}
            // (software-pipelining the next chunk's recompute into this loop measured slower:
            // 1869 vs 1770 us for the fine-level smoother, more registers, same stalls)
            double* obase = (CGP ? a.out2 : a.out0) + colbase;
            double x = 0.0;
            if constexpr (TM) tmem_wait_st();   // the forward sweep's g' stores have landed
            for (int c = nck - 1; c >= 0; --c) {
                const int kb0 = c * KB;
                double p1 = c ? cbuf[c * NT + tid] : 1.0, p2 = c ? 1.0 : 0.0;
                double t1 = c ? fT * ptab[2 * nz + kb0 - 1] : 0.0;
                double tq[KB], gv[KB];
                if constexpr (TM) {   // g' of this chunk from Tensor Memory (warp-uniform loads)
                    if (kb0 + KB <= nz) {
                        tmem_ld_f64x8(tbase + 2u * (uint32_t)kb0, gv);
                    } else {
#pragma unroll
                        for (int q = 0; q < KB; ++q)
                            if (kb0 + q < nz) gv[q] = tmem_ld_f64(tbase + 2u * (uint32_t)(kb0 + q));
                    }
                }
#pragma unroll
                for (int q = 0; q < KB; ++q) {
                    const int k = kb0 + q;
                    if (k < nz) {
                        const double tk = fT * ptab[2 * nz + k];
                        tq[q] = -(tk * pivot_step(k, p1, p2, t1));   // -t'_k = -t_k / m_k
                        if constexpr (!TM) gv[q] = gbuf[k * NT + tid];
                    }
                }
#pragma unroll
                for (int q = KB - 1; q >= 0; --q) {
                    const int k = kb0 + q;
                    if (k < nz) {
                        x = fma(tq[q], x, gv[q]);
                        if (valid) obase[(int64_t)k * nx] = x;
                    }
                }
            }
        }
        if constexpr (T::THOMAS && GEN < 2) {
            // backward substitution x_k = g'_k - t'_k x_{k+1}, KB levels per step with
            // the shared-memory loads issued ahead of the dependent FMA chain
            double* op = (CGP ? a.out2 : a.out0) + colbase + (int64_t)(nz - 1) * nx;
            double x = 0.0;
            int k = nz - 1;
            // TM: the chunk's g' comes from Tensor Memory, 8 levels per load (a software-pipelined
            // form with the next chunk's load in flight measured the same, r2k, at 237 registers)
            if constexpr (TM) tmem_wait_st();   // the forward sweep's g' stores have landed
            int bg = 0;   // TST: this warp's z staging buffer
            for (; k >= KB - 1; k -= KB) {
                const double* gq = gbuf + (k - (KB - 1)) * NT + tid;   // levels k-KB+1 .. k
                const double* mq = gim + (k - (KB - 1));
                double gv[KB], gm[KB];
                if constexpr (TM) {
                    static_assert(KB == 8, "16 TMEM columns = 8 levels per chunk");
                    double g8[KB];
                    tmem_ld_f64x8(tbase + 2u * (uint32_t)(k - (KB - 1)), g8);
#pragma unroll
                    for (int q = 0; q < KB; ++q) gv[q] = g8[KB - 1 - q];
                }
#pragma unroll
                for (int q = 0; q < KB; ++q) {
                    if constexpr (!TM) gv[q] = gq[(KB - 1 - q) * NT];
                    gm[q] = mq[KB - 1 - q];
                }
                if constexpr (TST) {
                    double* zb = sbw + (bg * TY + ty) * (KB * TX);
                    if (tx == 0) bulk_wait_read<1>();   // this buffer's store (two groups ago) has read it
                    __syncwarp();
#pragma unroll
                    for (int q = 0; q < KB; ++q) {
                        x = fma(gm[q], x, gv[q]);
                        zb[(KB - 1 - q) * TX + tx] = x;   // box [level][x] of row j
                    }
                    fence_proxy_async_smem();
                    __syncwarp();
                    if (tx == 0) {
                        tma_store_3d(&a.tma.o[2], (int)i0, k - (KB - 1), (int)j, zb);
                        bulk_commit();
                    }
                    bg ^= 1;
                } else {
#pragma unroll
                    for (int q = 0; q < KB; ++q) {
                        x = fma(gm[q], x, gv[q]);
                        if (valid) put(op, x);
                        op -= nx;
                    }
                }
            }
            for (; k >= 0; --k) {
                x = fma(gim[k], x, TM ? tmem_ld_f64(tbase + 2u * (uint32_t)k) : gbuf[k * NT + tid]);
                if (valid) *op = x;
                op -= nx;
            }
        }
        if constexpr (T::THOMAS) {
            // fused halo push: a strip-boundary row also goes to the neighbour's slab (read
            // back from L1/L2, outside the recurrence loop)
            if (valid && ((j == 0 && a.push.dst_lo) || (j == ny - 1 && a.push.dst_hi))) {
                const double* src = (CGP ? a.out2 : a.out0) + colbase;
                double* dst = (j == 0 ? a.push.dst_lo : a.push.dst_hi) + i;
                double* dst2 = (j == 0 && j == ny - 1) ? a.push.dst_hi : nullptr;   // a one-row strip
                // batches of 16 independent loads: the copy is latency-, not bandwidth-bound
                int kk = 0;
                for (; kk + 16 <= nz; kk += 16) {
                    double v[16];
#pragma unroll
                    for (int q = 0; q < 16; ++q) v[q] = src[(int64_t)(kk + q) * nx];
#pragma unroll
                    for (int q = 0; q < 16; ++q) {
                        dst[(int64_t)(kk + q) * nx] = v[q];
                        if (dst2) dst2[(int64_t)(kk + q) * nx + i] = v[q];
                    }
                }
                for (; kk < nz; ++kk) {
                    dst[(int64_t)kk * nx] = src[(int64_t)kk * nx];
                    if (dst2) dst2[(int64_t)kk * nx + i] = src[(int64_t)kk * nx];
                }
            }
        }
    };
    for (int tl = 0; tl < my_tiles; ++tl) {
        const int tile = (int)blockIdx.x + tl * (int)gridDim.x;
        if (GEN < 2 && tile_on_boundary(a.L, (int64_t)col_of(tile) * TX, (int64_t)row_of(tile) * TY, TX, TY))
            tile_body(std::true_type{}, tl);
        else
            tile_body(std::false_type{}, tl);
    }
    if constexpr (LOADER == 0) cp_async_wait<0>();
    if constexpr (TST)
        if (tx == 0) bulk_wait<0>();   // my TMA stores are complete before the CTA (and its staging) ends
    if constexpr (TM) {   // every warp is done with its lanes; the allocating warp frees them
        tmem_fence_before();
        __syncthreads();
        if (ty == 0) {
            tmem_fence_after();
            tmem_dealloc<NCOL>(tmem_slot);
        }
    }
    if (want_red) grid_reduce<NR>(a.red, acc, scratch);
}

template <int MODE, int TY>
size_t line_smem_bytes(int nz, int gen = 0, int tms = 0, bool tst = false)
{
    using T = Traits<MODE>;
    using G = Geom<T::NH, T::NP, TY>;
    using G3 = Geom<T::NH, T::NP + 1, TY>;   // GEN 3: + the pivot field
    if (gen == 3)
        return (size_t)(((3 * nz + 15) & ~15) + ((4 * nz + 15) & ~15) + (size_t)tms * G3::STAGE + 64 + 16) * sizeof(double);
    const bool tm = tms > 0;
    size_t d = ((3 * nz + 15) & ~15) + (gen >= 2 ? ((4 * nz + 15) & ~15) : gen ? ((3 * nz + 15) & ~15) : 0) +
               (size_t)(tm ? tms : gen == 2 ? stages<MODE, 2>() : gen ? stages<MODE, 1>() : stages<MODE, 0>()) * G::STAGE + (T::THOMAS ? (size_t)((tm ? 0 : nz) + (gen == 2 ? (nz + KB - 1) / KB : 0)) * G::NT : 0) + 64 + 16 +
               (MODE == MODE_RESTRICT ? 2 * TY * (KB + 1) * (TX / 2) : 0) +
               (tst ? 16 + (3 * 2 + 2) * KB * TY * TX : 0);   // TST staging + its 128-byte alignment
    return d * sizeof(double);
}

constexpr size_t kMaxSmem = 227 * 1024 - 1024;  // leave room for static smem (barriers, flags)

template <int MODE, int TY, int LOADER, int GEN, int TMS = 0, bool HW = false, bool TST = false>
cudaError_t launch_line_l(const Launcher& ln, const LineArgs& a)
{
    constexpr bool TM = TMS > 0;
    const size_t smem = line_smem_bytes<MODE, TY>(a.L.nz, GEN, TMS, TST);
    auto kern = k_line<MODE, TY, LOADER, GEN, TMS, HW, TST>;
    static size_t limit = 0;   // per instantiation
    if (!limit) {
        limit = dyn_smem_limit(kern);
        cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)limit);
        if (e != cudaSuccess) return e;
        // the largest shared-memory carveout, so that the occupancy query below (and the first
        // launch) sees every CTA that fits, not the default carveout's count
        e = cudaFuncSetAttribute(kern, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
        if (e != cudaSuccess) return e;
    }
    if (smem > limit) return cudaErrorInvalidConfiguration;
    int per_sm = 0;
    static int carve = 100;   // per instantiation: the carveout last set
    if (ln.carveout_fit && carve != 100) {   // query the occupancy at the largest carveout
        cudaError_t e2 = cudaFuncSetAttribute(kern, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
        if (e2 != cudaSuccess) return e2;
        carve = 100;
    }
    cudaError_t e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, TX * TY, smem);
    if (e != cudaSuccess) return e;
    per_sm = std::max(per_sm, 1);
    if (TM) per_sm = std::min<int>(per_sm, std::min<int>(ln.tm_ctas, 512 / kTmemCols));   // resident CTAs must all get their TMEM
    if (GEN == 3 || (TM && TY == 8)) per_sm = 1;   // 512 TMEM columns per CTA
    const int64_t ntiles = ((a.L.nx + TX - 1) / TX) * part_rows(a.part, (int)((a.L.ny + TY - 1) / TY));
    // CG direction (two halo'd fields) with 4-row tiles: on wide grids two CTAs per SM
    // re-read the halo rows from HBM (2.1x the algorithmic reads at 4096 x 1024 x 128, ncu),
    // so one CTA per SM there (the 8-row default fits one CTA per SM anyway).
    if (MODE == MODE_CGDIR && a.L.nx > 32 * TX && a.cgdir_ctas == 0) per_sm = 1;
    if (MODE == MODE_CGDIR && a.cgdir_ctas > 0) per_sm = std::min(per_sm, a.cgdir_ctas);
    const int64_t grid = std::min<int64_t>(ntiles, (int64_t)std::max(1, ln.num_sms - ln.reserve_sms) * per_sm);
    if (grid <= 0) return cudaSuccess;
    if (ln.carveout_fit) {   // the smallest carveout that holds the resident CTAs: the rest stays L1
        const int pct = carveout_pct(smem, std::min<int64_t>(per_sm, grid));
        if (pct != carve) {
            e = cudaFuncSetAttribute(kern, cudaFuncAttributePreferredSharedMemoryCarveout, pct);
            if (e != cudaSuccess) return e;
            carve = pct;
        }
    }
    return launch_kernel(ln, kern, dim3((unsigned)grid), dim3(TX * TY), smem, a);
}

template <int MODE, int TY>
cudaError_t launch_line_t(const Launcher& ln, const LineArgs& a)
{
    if constexpr (MODE == MODE_CGPREC && TY == 8) {   // 8 warps, g' in both TMEM column halves
        if (!a.hw.flag[0] && !a.hw.flag[1] && !a.L.gen && ln.tmem && a.use_tma && a.L.nz <= (int)(kTmemCols / 2))
            return launch_line_l<MODE, 8, 1, 0, 3>(ln, a);
        return cudaErrorNotSupported;
    } else {
    if (a.hw.flag[0] || a.hw.flag[1]) {   // P2P overlap with the in-kernel halo wait (line_halo_wait())
        if constexpr (TY == 4 && (MODE == MODE_CGDIR || MODE == MODE_RESTRICT))
            if (!a.L.gen && a.use_tma) return launch_line_l<MODE, 4, 1, 0, 0, true>(ln, a);
        if constexpr (TY == 8 && MODE == MODE_CGDIR)
            if (!a.L.gen && a.use_tma) return launch_line_l<MODE, 8, 1, 0, 0, true>(ln, a);
        if constexpr (TY == 4 && MODE == MODE_SMOOTH)
            if (!a.L.gen && a.use_tma && ln.tmem && a.L.nz <= (int)(kTmemCols / 2))
                return launch_line_l<MODE, 4, 1, 0, 3, true>(ln, a);
        return cudaErrorNotSupported;
    }
    if (a.L.gen) {   // general vertical profiles / per-column fields: TMA loader only
        if (!a.use_tma) return cudaErrorNotSupported;
        if constexpr (Traits<MODE>::THOMAS && TY == 4)   // precomputed pivots streamed with the data
            if (a.L.gen >= 2 && a.im && ln.tmem && a.L.nz <= (int)(kTmemCols / 2))
                return launch_line_l<MODE, 4, 1, 3, 3>(ln, a);
        if constexpr (Traits<MODE>::THOMAS && TY == 4)   // g' in Tensor Memory, 2 CTAs per SM
            if (ln.tmem && a.L.nz <= (int)(kTmemCols / 2)) {
                if (a.L.gen >= 2) return launch_line_l<MODE, 4, 1, 2, (is_cgprec(MODE) ? 2 : 3)>(ln, a);
                return launch_line_l<MODE, 4, 1, 1, 3>(ln, a);
            }
        return a.L.gen >= 2 ? launch_line_l<MODE, TY, 1, 2>(ln, a) : launch_line_l<MODE, TY, 1, 1>(ln, a);
    }
    if constexpr (Traits<MODE>::THOMAS && TY == 4)   // g' in Tensor Memory (flat box, TMA loader)
        if (ln.tmem && a.use_tma && a.L.nz <= (int)(kTmemCols / 2)) {
            // TMA ring depth (stages of 8 levels): the shared memory freed from g' would hold 7,
            // but 7 measured 16% slower than 3 for CGPREC (r2e: 1.29 vs 1.11 ms); TPMG_TM_STAGES
            // selects 3 (default), 4 or 5 for the CG preconditioner
            if constexpr (MODE == MODE_CGPREC) {
                if (a.tst) return launch_line_l<MODE, 4, 1, 0, 3, false, true>(ln, a);
                if (ln.tm_stages == 2) return launch_line_l<MODE, 4, 1, 0, 2>(ln, a);
                if (ln.tm_stages == 4) return launch_line_l<MODE, 4, 1, 0, 4>(ln, a);
                if (ln.tm_stages == 5) return launch_line_l<MODE, 4, 1, 0, 5>(ln, a);
            }
            return launch_line_l<MODE, 4, 1, 0, 3>(ln, a);
        }
    return a.use_tma ? launch_line_l<MODE, TY, 1, 0>(ln, a) : launch_line_l<MODE, TY, 0, 0>(ln, a);
    }
}

template <int MODE>
cudaError_t launch_line_ty(const Launcher& ln, const LineArgs& a)
{
    if (ln.tmem && a.use_tma && a.L.nz <= (int)(kTmemCols / 2)) {
        if constexpr (MODE == MODE_CGPREC)
            if (cgprec_rows() == 8 && !a.L.gen) return launch_line_t<MODE, 8>(ln, a);
        return launch_line_t<MODE, 4>(ln, a);
    }
    if (line_smem_bytes<MODE, 4>(a.L.nz, a.L.gen) <= kMaxSmem) return launch_line_t<MODE, 4>(ln, a);
    if (line_smem_bytes<MODE, 2>(a.L.nz, a.L.gen) <= kMaxSmem) return launch_line_t<MODE, 2>(ln, a);
    return launch_line_t<MODE, 1>(ln, a);
}

// ------------------------------------------------------------------ simple streaming kernels

__global__ void k_restrict(const LevelConst F, const LevelConst Cc, const double* __restrict__ r,
                           double* __restrict__ fc)
{
    pdl_wait();
    pdl_trigger();
    const int64_t I = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    const int k = blockIdx.y;
    const int64_t J = blockIdx.z;
    if (I >= Cc.nx) return;
    const int64_t nx = F.nx;
    const double* r0 = r + ((2 * J) * F.nz + k) * nx;
    const double* r1 = r + ((2 * J + 1) * F.nz + k) * nx;
    const double s = (__ldg(r0 + 2 * I) + __ldg(r0 + 2 * I + 1)) + (__ldg(r1 + 2 * I) + __ldg(r1 + 2 * I + 1));
    fc[(J * Cc.nz + k) * Cc.nx + I] = 0.25 * s;
}

// u_f += P u_c: a thread owns coarse column (I, J) of a 32 x 4 block and walks lpt
// levels, updating the 2 x 2 fine children with 16-byte loads/stores (fine level:
// 402 us = 6.0 TB/s at 1024^2 x 128, was 531 us before the loads were batched).  The 3 x 3 coarse
// neighbourhood is read through L1 (neighbouring threads share it); no integer
// division in the loop.
// The work of k_prolong_add; threads outside the grid return early (no barrier here).
template <bool PUSH, int PB>
__device__ __forceinline__ void prolong_body(const LevelConst& Cc, const LevelConst& F, const HaloField& uc,
                                             double* __restrict__ uf, int lpt, int part, const HaloPush& push,
                                             const HaloWait& hw)
{
    const int64_t nxc = Cc.nx, nyc = Cc.ny;
    const int nz = Cc.nz;
    const int64_t I = blockIdx.x * 32 + threadIdx.x;
    // PART_INTERIOR: coarse rows 1 .. nyc-2 (no halo row read); PART_BOUNDARY: rows 0, nyc-1.
    // In-kernel halo wait (hw): the block rows with coarse rows 0 / nyc-1 are deferred by a
    // few block rows, and their threads wait for the halo epoch before they read the slabs.
    const bool hwait = hw.flag[0] || hw.flag[1];
    const int by = hwait ? boundary_deferred_row((int)blockIdx.y, (int)gridDim.y, kHaloDefer) : (int)blockIdx.y;
    int64_t J = by * 4 + threadIdx.y;
    if (part == PART_INTERIOR) J += 1;
    else if (part == PART_BOUNDARY) J = (J == 0) ? 0 : ((J == 1 && nyc > 1) ? nyc - 1 : nyc);
    if (part == PART_INTERIOR && J >= nyc - 1) return;
    const int kbeg = blockIdx.z * lpt, kend = min(nz, kbeg + lpt);   // levels of this thread
    if (I >= nxc || J >= nyc) return;
    if (hwait) {
        if (J == 0 && hw.flag[0]) halo_flag_wait(hw.flag[0], hw.epoch);
        if (J == nyc - 1 && hw.flag[1]) halo_flag_wait(hw.flag[1], hw.epoch);
    }
    // coarse rows J-1, J, J+1 and columns I-1, I, I+1.  Ghosts outside the physical domain
    // are a factor times an in-domain value: 0 (zero coarse ghosts [R7]) or -1 (face
    // Dirichlet [R25]: the linear continuation through 0; a corner gets (-1)(-1) = +1), so
    // every load is unconditional and in bounds.
    const int64_t cplane = nxc * nz;
    const bool face = Cc.bc != 0;
    const double ghost = face ? -1.0 : 0.0;
    const double* rows[3];
    double fr[3];
#pragma unroll
    for (int d = 0; d < 3; ++d) {
        const int64_t JJ = J - 1 + d;
        const double* r = (JJ < 0) ? uc.lo : (JJ >= nyc ? uc.hi : uc.base + JJ * cplane);
        rows[d] = r ? r : uc.base + J * cplane;
        fr[d] = r ? 1.0 : ghost;
    }
    const int64_t iw = I > 0 ? I - 1 : I, ie = I < nxc - 1 ? I + 1 : I;
    const double fw = I > 0 ? 1.0 : ghost, fe = I < nxc - 1 ? 1.0 : ghost;
    const int64_t fplane = F.nx * (int64_t)F.nz;
    double* f0 = uf + (2 * J) * fplane + 2 * I;     // fine row 2J, level 0
    double* f1 = f0 + fplane;                        // fine row 2J+1
    // PB levels per step: all loads of the step are issued before its stores (the fine
    // read-modify-write would otherwise serialise on memory latency level by level)
    for (int k0 = kbeg; k0 < kend; k0 += PB) {
        double2 fv[PB][2];
        double cc[PB][3][3];
#pragma unroll
        for (int q = 0; q < PB; ++q) {
            const int k = min(k0 + q, kend - 1);
            fv[q][0] = *reinterpret_cast<const double2*>(f0 + (int64_t)k * F.nx);
            fv[q][1] = *reinterpret_cast<const double2*>(f1 + (int64_t)k * F.nx);
#pragma unroll
            for (int d = 0; d < 3; ++d) {
                const double* r = rows[d] + (int64_t)k * nxc;
                // plain loads, not ld.global.nc: with the in-kernel halo wait the slab rows are
                // written (by the neighbour) while this kernel runs
                cc[q][d][0] = r[iw];
                cc[q][d][1] = r[I];
                cc[q][d][2] = r[ie];
            }
        }
#pragma unroll
        for (int q = 0; q < PB; ++q) {
            if (k0 + q >= kend) break;
            double c[3][3];
#pragma unroll
            for (int d = 0; d < 3; ++d) {
                c[d][0] = fr[d] * (fw * cc[q][d][0]);
                c[d][1] = fr[d] * cc[q][d][1];
                c[d][2] = fr[d] * (fe * cc[q][d][2]);
            }
#pragma unroll
            for (int b = 0; b < 2; ++b) {          // fine row 2J + b: sy = -1 (b = 0), +1 (b = 1)
                const int sy = b ? 2 : 0;
                // fine columns 2I (sx = -1) and 2I+1 (sx = +1)
                const double v0 = 9.0 * c[1][1] + 3.0 * c[1][0] + 3.0 * c[sy][1] + 1.0 * c[sy][0];
                const double v1 = 9.0 * c[1][1] + 3.0 * c[1][2] + 3.0 * c[sy][1] + 1.0 * c[sy][2];
                double2 w = fv[q][b];
                w.x = w.x + v0 / 16.0;
                w.y = w.y + v1 / 16.0;
                *reinterpret_cast<double2*>((b ? f1 : f0) + (int64_t)(k0 + q) * F.nx) = w;
                if constexpr (PUSH) {   // fused halo push of the fine strip-boundary rows
                    const int64_t jf = 2 * J + b, off = (int64_t)(k0 + q) * F.nx + 2 * I;
                    if (jf == 0 && push.dst_lo) *reinterpret_cast<double2*>(push.dst_lo + off) = w;
                    if (jf == F.ny - 1 && push.dst_hi) *reinterpret_cast<double2*>(push.dst_hi + off) = w;
                }
            }
        }
    }

}

template <bool PUSH, int PB = 2>   // PB: levels per load batch (4 measured slower, r2ac)
__global__ void __launch_bounds__(128) k_prolong_add(const LevelConst Cc, const LevelConst F, const HaloField uc,
                                                     double* __restrict__ uf, int lpt, const int* skip, int part,
                                                     const HaloPush push, const HaloWait hw)
{
    pdl_wait();
    pdl_trigger();
    if (skip && *skip) return;
    prolong_body<PUSH, PB>(Cc, F, uc, uf, lpt, part, push, hw);
}


// One thread per column (i, j): the Thomas pivots of its block M_T = |T| (diag(a) + tridiag(-(b+c),
// b, c)) - alpha_T diag(d) (eqn:LocalMatrixStencil, the fields layout of LevelConst::fld and the
// profile table [a-b-c][b][c][d]): m_0 = dg_0, m_k = dg_k - s_k t_{k-1} / m_{k-1}, stored as 1/m_k.
__global__ void __launch_bounds__(128) k_pivots(const LevelConst L, double* __restrict__ im)
{
    const int64_t nx = L.nx, ny = L.ny;
    const int nz = L.nz;
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x, j = blockIdx.y;
    if (i >= nx || j >= ny) return;
    const int64_t ncol = nx * ny, cc = j * nx + i;
    const double fT = L.fld[cc], faT = L.fld[ncol + cc];
    const double* pr = L.prof;   // [a-b-c][b][c][d], nz each
    double m = 0.0, tprev = 0.0;
    for (int k = 0; k < nz; ++k) {
        const double sk = fT * pr[nz + k], tk = fT * pr[2 * nz + k];
        const double dg = fma(fT, pr[k], -faT * pr[3 * nz + k]);
        m = (k == 0) ? dg : dg - sk * tprev / m;
        im[(j * nz + k) * nx + i] = 1.0 / m;
        tprev = tk;
    }
}

__global__ void __launch_bounds__(256) k_dot(const double* __restrict__ x, const double* __restrict__ y,
                                             int64_t n, ReduceSlot red)
{
    pdl_wait();
    pdl_trigger();
    __shared__ double scratch[64];
    double acc[1] = {0.0};
    for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < n; q += (int64_t)gridDim.x * blockDim.x)
        acc[0] += x[q] * y[q];
    grid_reduce<1>(red, acc, scratch);
}

__global__ void __launch_bounds__(256) k_copy(double* __restrict__ dst, const double* __restrict__ src, int64_t n,
                                              const int* skip)
{
    pdl_wait();
    pdl_trigger();
    if (skip && *skip) return;
    for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < n; q += (int64_t)gridDim.x * blockDim.x)
        dst[q] = src[q];
}

__global__ void __launch_bounds__(256) k_cg_halo(double* out_lo, const double* z_lo, const double* p_lo, double* out_hi,
                                                 const double* z_hi, const double* p_hi, int64_t n, DevRatio r,
                                                 const int* skip)
{
    pdl_wait();
    pdl_trigger();
    if (skip && *skip) return;
    const double beta = (r.num >= 0) ? r.s[r.num] / r.s[r.den] : 0.0;
    for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < n; q += (int64_t)gridDim.x * blockDim.x) {
        if (out_lo) out_lo[q] = fma(beta, p_lo[q], z_lo[q]);   // same arithmetic as k_line<CGDIR>
        if (out_hi) out_hi[q] = fma(beta, p_hi[q], z_hi[q]);
    }
}

template <typename V>
__global__ void __launch_bounds__(256) k_halo_push(const HaloPush hp, int64_t n)
{
    const V* sf = reinterpret_cast<const V*>(hp.src_first);
    const V* sl = reinterpret_cast<const V*>(hp.src_last);
    V* dl = reinterpret_cast<V*>(hp.dst_lo);
    V* dh = reinterpret_cast<V*>(hp.dst_hi);
    for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < n; q += (int64_t)gridDim.x * blockDim.x) {
        if (dl) dl[q] = sf[q];
        if (dh) dh[q] = sl[q];
    }
    if (hp.done) {   // device-side publish: the last CTA releases the epoch to both neighbours
        __threadfence_system();   // my CTA's remote stores before its ticket
        __syncthreads();
        if (threadIdx.x == 0) {
            const unsigned t = atomicAdd(hp.done, 1u);
            if (t == gridDim.x - 1) {
                *hp.done = 0u;          // every CTA has taken its ticket: reset for the next push
                __threadfence_system(); // (cumulative) every CTA's stores before the flags
                if (hp.flag_lo) asm volatile("st.release.sys.global.u32 [%0], %1;\n" ::"l"(hp.flag_lo), "r"(hp.epoch) : "memory");
                if (hp.flag_hi) asm volatile("st.release.sys.global.u32 [%0], %1;\n" ::"l"(hp.flag_hi), "r"(hp.epoch) : "memory");
            }
        }
    }
}

__global__ void __launch_bounds__(32) k_allreduce_p2p(double* d, int n, const P2PReduce P, unsigned E)
{
    pdl_wait();
    pdl_trigger();
    const int t = threadIdx.x;
    const int b = (int)(E & 1u);
    if (t < n) {
        const double v = d[t];
        for (int r = 0; r < P.nranks; ++r) P.slots[r][(b * kMaxP2PRanks + P.me) * 4 + t] = v;   // NVLink stores
    }
    __threadfence_system();   // my values are visible everywhere before my flag is
    __syncwarp();
    if (t < P.nranks) asm volatile("st.release.sys.global.u32 [%0], %1;\n" ::"l"(P.flags[t] + P.me), "r"(E) : "memory");
    bool timed_out = false;
    if (t < P.nranks) {
        const unsigned* f = P.flags[P.me] + t;
        uint64_t t0, now;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
        for (;;) {
            unsigned v;
            asm volatile("ld.acquire.sys.global.u32 %0, [%1];\n" : "=r"(v) : "l"(f) : "memory");
            if ((int)(v - E) >= 0) break;
            asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(now));
            if (now - t0 > 20000000000ull) { timed_out = true; break; }
            __nanosleep(64);
        }
    }
    timed_out = __any_sync(0xffffffffu, timed_out);
    __syncwarp();
    __threadfence_system();
    if (t < n) {
        double s = 0.0;
        const volatile double* mine = P.slots[P.me] + b * kMaxP2PRanks * 4 + t;
        for (int r = 0; r < P.nranks; ++r) s += mine[r * 4];   // rank order: identical on every rank
        d[t] = timed_out ? __longlong_as_double(0x7ff8000000000000ll) : s;
    }
}

// Convergence test of PCG iteration m on the device: ||r_m|| / ||r_0|| < eps
// (eqn:epsilonTolerance), breakdown when <p, A p> <= 0 or <r, M^-1 r> <= 0.
// The host reads the flag from pinned memory after an event behind the check kernel:
// a system-scope store instead of a 4-byte copy in the stream (no copy-engine bubble).
__device__ __forceinline__ void publish_flag(int* hflags, int m, int code)
{
    if (!hflags) return;
    *reinterpret_cast<volatile int*>(hflags + m) = code;
    __threadfence_system();
}

__global__ void k_cg_check(const double* scal, int m, double eps, int* flags, int* hflags)
{
    pdl_wait();
    pdl_trigger();
    const int prev = (m >= 1) ? flags[m - 1] : 0;
    int code = prev;
    if (!prev) {
        const double rr0 = scal[1], rr = scal[3 * m + 1], zeta = scal[3 * m + 2];
        if (m >= 1 && !(scal[3 * m] > 0.0)) code = 2;
        else if (rr != rr) code = 3;
        else if (rr0 == 0.0 || sqrt(rr) / sqrt(rr0) < eps) code = 1;
        else if (!(zeta > 0.0)) code = 2;
    }
    flags[m] = code;
    publish_flag(hflags, m, code);
}

// Convergence test of MG cycle n: ||f - A u_n|| / ||r_0|| < eps, or the cycle limit.
__global__ void k_mg_check(const double* norm2, const double* r0_2, int n, double eps, int max_iter, int* flags,
                           int* hflags)
{
    pdl_wait();
    pdl_trigger();
    const int prev = (n >= 1) ? flags[n - 1] : 0;
    int code = prev;
    if (!prev) {
        const double rn2 = *norm2;
        if (rn2 != rn2) code = 3;
        else if (sqrt(rn2) / sqrt(*r0_2) < eps) code = 1;
        else if (n >= max_iter) code = 4;
    }
    flags[n] = code;
    publish_flag(hflags, n, code);
}

}  // namespace

cudaError_t launch_copy(const Launcher& ln, double* dst, const double* src, int64_t n, const int* skip)
{
    if (n <= 0) return cudaSuccess;
    const int64_t grid = std::min<int64_t>((n + 255) / 256, (int64_t)ln.num_sms * 8);
    return launch_kernel(ln, k_copy, dim3((unsigned)grid), dim3(256), 0, dst, src, n, skip);
}

cudaError_t launch_cg_halo(const Launcher& ln, double* out_lo, const double* z_lo, const double* p_lo, double* out_hi,
                           const double* z_hi, const double* p_hi, int64_t n, DevRatio beta, const int* skip)
{
    if (!out_lo && !out_hi) return cudaSuccess;
    const int64_t grid = std::min<int64_t>((n + 255) / 256, (int64_t)ln.num_sms * 4);
    return launch_kernel(ln, k_cg_halo, dim3((unsigned)grid), dim3(256), 0, out_lo, z_lo, p_lo, out_hi, z_hi, p_hi, n, beta, skip);
}

cudaError_t launch_halo_push(const Launcher& ln, const HaloPush& hp)
{
    if (!hp.dst_lo && !hp.dst_hi) return cudaSuccess;
    const bool vec = (hp.n % 2 == 0) && ((uintptr_t)hp.src_first % 16 == 0) && ((uintptr_t)hp.src_last % 16 == 0);
    const int64_t m = vec ? hp.n / 2 : hp.n;
    const unsigned grid = (unsigned)std::max<int64_t>(std::min<int64_t>((m + 255) / 256, 64), 1);
    if (vec) k_halo_push<double2><<<grid, 256, 0, ln.stream>>>(hp, m);
    else k_halo_push<double><<<grid, 256, 0, ln.stream>>>(hp, m);
    if (ln.launch_counter) ++*ln.launch_counter;
    return cudaGetLastError();
}

cudaError_t launch_allreduce_p2p(const Launcher& ln, double* d, int n, const P2PReduce& P, unsigned epoch)
{
    if (n < 1 || n > 4 || P.nranks > kMaxP2PRanks) return cudaErrorInvalidValue;
    return launch_kernel(ln, k_allreduce_p2p, dim3(1), dim3(32), 0, d, n, P, epoch);
}

cudaError_t launch_cg_check(const Launcher& ln, const double* scal, int m, double eps, int* flags, int* hflags)
{
    return launch_kernel(ln, k_cg_check, dim3(1), dim3(1), 0, scal, m, eps, flags, hflags);
}

cudaError_t launch_mg_check(const Launcher& ln, const double* norm2, const double* r0_2, int n, double eps,
                            int max_iter, int* flags, int* hflags)
{
    return launch_kernel(ln, k_mg_check, dim3(1), dim3(1), 0, norm2, r0_2, n, eps, max_iter, flags, hflags);
}

bool line_halo_wait(int mode, int nz, int gen, bool use_tma, bool tmem)
{
    if (gen || !use_tma) return false;
    if (mode == MODE_CGDIR || mode == MODE_RESTRICT) return true;
    return mode == MODE_SMOOTH && tmem && nz <= (int)(kTmemCols / 2);
}

int line_launch_rows(int mode, int nz, int nx, int use_tma, int ksplit_cfg)
{
    if (use_tma && ksplit_cfg >= 0 && ksplit_supported(mode, nz, nx)) return ksplit_boxes(mode, ksplit_cfg).ty;
    return line_tile_rows(mode, nz, 0, false, nx);
}

bool line_gen_fits(int nz, int gen) { return line_smem_bytes<MODE_CGPREC, 1>(nz, gen) <= kMaxSmem; }

// CG direction tile rows: 8 (one 8-warp CTA per SM: the warps of two 4-row CTAs, one halo
// box for both -- (TY+2)/TY = 1.25 instead of 1.5 halo rows per row, and no second CTA
// re-reading the halo rows on wide grids).  r2ak, TB/s under the power cap, 8 vs 4 rows:
// nx = 1024 5.84 vs 5.46; 2048 5.78 vs 4.31; 4096 5.63 vs 4.21.  TPMG_CGDIR_TY=4: 4 rows.
static int cgdir_rows(int64_t)
{
    const char* e = std::getenv("TPMG_CGDIR_TY");   // (read per call: the tests switch it per context)
    return (e && std::atoi(e) == 4) ? 4 : 8;
}

int line_tile_rows(int mode, int nz, int gen, bool tm, int64_t nx)
{
    if (mode == MODE_CGDIR) return cgdir_rows(nx);
    if (tm && nz <= (int)(kTmemCols / 2) && mode == MODE_CGPREC && !gen) return cgprec_rows();
    // the Tensor Memory form of the Thomas modes always runs 4 tile rows (the lane quarters)
    if (tm && nz <= (int)(kTmemCols / 2) && (mode == MODE_PREC || mode == MODE_SMOOTH || is_cgprec(mode))) return 4;
    switch (mode) {
    case MODE_PREC: return line_smem_bytes<MODE_PREC, 4>(nz, gen) <= kMaxSmem ? 4 : line_smem_bytes<MODE_PREC, 2>(nz, gen) <= kMaxSmem ? 2 : 1;
    case MODE_SMOOTH: return line_smem_bytes<MODE_SMOOTH, 4>(nz, gen) <= kMaxSmem ? 4 : line_smem_bytes<MODE_SMOOTH, 2>(nz, gen) <= kMaxSmem ? 2 : 1;
    case MODE_CGPREC: return line_smem_bytes<MODE_CGPREC, 4>(nz, gen) <= kMaxSmem ? 4 : line_smem_bytes<MODE_CGPREC, 2>(nz, gen) <= kMaxSmem ? 2 : 1;
    case MODE_CGPREC_D: return line_smem_bytes<MODE_CGPREC_D, 4>(nz, gen) <= kMaxSmem ? 4 : line_smem_bytes<MODE_CGPREC_D, 2>(nz, gen) <= kMaxSmem ? 2 : 1;
    case MODE_CGPREC_P: return line_smem_bytes<MODE_CGPREC_P, 4>(nz, gen) <= kMaxSmem ? 4 : line_smem_bytes<MODE_CGPREC_P, 2>(nz, gen) <= kMaxSmem ? 2 : 1;
    default: return 4;
    }
}

int line_max_nz()
{
    // Thomas modes at TY = 1 are the binding case
    int nz = 8;
    while (line_smem_bytes<MODE_CGPREC, 1>(nz + 8) <= kMaxSmem) nz += 8;
    return nz;
}

cudaError_t launch_line(const Launcher& ln, int mode, const LineArgs& a)
{
    switch (mode) {
    case MODE_APPLY: return launch_line_t<MODE_APPLY, 4>(ln, a);
    case MODE_RESID: return launch_line_t<MODE_RESID, 4>(ln, a);
    case MODE_PREC: return launch_line_ty<MODE_PREC>(ln, a);
    case MODE_SMOOTH: return launch_line_ty<MODE_SMOOTH>(ln, a);
    case MODE_CGDIR: return cgdir_rows(a.L.nx) == 8 ? launch_line_t<MODE_CGDIR, 8>(ln, a) : launch_line_t<MODE_CGDIR, 4>(ln, a);
    case MODE_CGPREC: return launch_line_ty<MODE_CGPREC>(ln, a);
    case MODE_CGPREC_D: return launch_line_ty<MODE_CGPREC_D>(ln, a);
    case MODE_CGPREC_P: return launch_line_ty<MODE_CGPREC_P>(ln, a);
    case MODE_RESTRICT: return launch_line_t<MODE_RESTRICT, 4>(ln, a);
    default: return cudaErrorInvalidValue;
    }
}

// z-contiguous <-> Lambda layout ("transposing the fields from a z-contiguous data
// format on the host to the x-contiguous format ... on the GPU", after Harris's tiled
// transpose): for every row j the nx x nz block zc[j][i][k] is transposed to lam[j][k][i].
// A 32 x 32 tile through shared memory (one padding column: no bank conflicts), both global
// sides coalesced.  TO_LAMBDA: src zc, dst Lambda; else the reverse.
template <bool TO_LAMBDA>
__global__ void __launch_bounds__(256) k_transpose(const double* __restrict__ src, double* __restrict__ dst,
                                                   int64_t nx, int nz)
{
    __shared__ double tile[32][33];
    pdl_wait();
    pdl_trigger();
    const int64_t i0 = (int64_t)blockIdx.x * 32, j = blockIdx.z;
    const int k0 = blockIdx.y * 32;
    const int tx = threadIdx.x, ty = threadIdx.y;
    const int64_t slab = j * nx * (int64_t)nz;
    if (TO_LAMBDA) {
        // read: k fastest (zc), tile[i][k]
        for (int r = ty; r < 32; r += 8) {
            const int64_t i = i0 + r;
            const int k = k0 + tx;
            if (i < nx && k < nz) tile[r][tx] = src[slab + i * nz + k];
        }
        __syncthreads();
        for (int r = ty; r < 32; r += 8) {
            const int k = k0 + r;
            const int64_t i = i0 + tx;
            if (i < nx && k < nz) dst[slab + (int64_t)k * nx + i] = tile[tx][r];
        }
    } else {
        // read: i fastest (Lambda), tile[k][i]
        for (int r = ty; r < 32; r += 8) {
            const int k = k0 + r;
            const int64_t i = i0 + tx;
            if (i < nx && k < nz) tile[r][tx] = src[slab + (int64_t)k * nx + i];
        }
        __syncthreads();
        for (int r = ty; r < 32; r += 8) {
            const int64_t i = i0 + r;
            const int k = k0 + tx;
            if (i < nx && k < nz) dst[slab + i * nz + k] = tile[tx][r];
        }
    }
}

cudaError_t launch_transpose(const Launcher& ln, bool to_lambda, const double* src, double* dst, int64_t nx,
                             int64_t ny, int nz)
{
    if (nx <= 0 || ny <= 0 || nz <= 0) return cudaSuccess;
    const dim3 grid((unsigned)((nx + 31) / 32), (unsigned)((nz + 31) / 32), (unsigned)ny), block(32, 8);
    return to_lambda ? launch_kernel(ln, k_transpose<true>, grid, block, 0, src, dst, nx, nz)
                     : launch_kernel(ln, k_transpose<false>, grid, block, 0, src, dst, nx, nz);
}

cudaError_t launch_restrict(const Launcher& ln, const LevelConst& fine, const LevelConst& coarse,
                            const double* r, double* fc)
{
    dim3 block(64), grid((unsigned)((coarse.nx + 63) / 64), (unsigned)coarse.nz, (unsigned)coarse.ny);
    if (coarse.ny <= 0 || coarse.nx <= 0) return cudaSuccess;
    return launch_kernel(ln, k_restrict, dim3(grid), dim3(block), 0, fine, coarse, r, fc);
}

cudaError_t launch_prolong_add(const Launcher& ln, const LevelConst& coarse, const LevelConst& fine,
                               HaloField uc, double* uf, const int* skip, int part, const HaloPush* push,
                               const HaloWait* hw)
{
    if (coarse.nx <= 0 || coarse.ny <= 0) return cudaSuccess;
    // levels per thread: enough threads to fill the GPU on the coarse levels
    const int64_t cols = coarse.nx * coarse.ny;
    // (measured at 1024^2 x 128: 16384 threads' worth per SM, >= 4 levels per thread)
    const int64_t want = (int64_t)ln.num_sms * 16384;
    int lpt = coarse.nz;
    while (lpt > 4 && cols * ((coarse.nz + lpt - 1) / lpt) < want) lpt = (lpt + 1) / 2;
    dim3 grid((unsigned)((coarse.nx + 31) / 32), (unsigned)((coarse.ny + 3) / 4), (unsigned)((coarse.nz + lpt - 1) / lpt)),
        block(32, 4);
    if (part == PART_INTERIOR) grid.y = (unsigned)((std::max<int64_t>(coarse.ny - 2, 0) + 3) / 4);
    if (part == PART_BOUNDARY) grid.y = 1;
    if (grid.y == 0) return cudaSuccess;
    const HaloPush hp = push ? *push : HaloPush{};
    const HaloWait w = hw ? *hw : HaloWait{};
    if (hp.dst_lo || hp.dst_hi)
        return launch_kernel(ln, k_prolong_add<true>, dim3(grid), dim3(block), 0, coarse, fine, uc, uf, lpt, skip, part, hp, w);
    return launch_kernel(ln, k_prolong_add<false>, dim3(grid), dim3(block), 0, coarse, fine, uc, uf, lpt, skip, part, hp, w);
}

cudaError_t launch_pivots(const Launcher& ln, const LevelConst& L, double* im)
{
    if (L.nx <= 0 || L.ny <= 0 || L.gen < 2 || !L.fld || !L.prof) return cudaErrorInvalidValue;
    return launch_kernel(ln, k_pivots, dim3((unsigned)((L.nx + 127) / 128), (unsigned)L.ny), dim3(128), 0, L, im);
}

cudaError_t launch_dot(const Launcher& ln, const double* x, const double* y, int64_t n, ReduceSlot red)
{
    int64_t grid = std::min<int64_t>((n + 255) / 256, (int64_t)ln.num_sms * 4);
    grid = std::max<int64_t>(grid, 1);
    return launch_kernel(ln, k_dot, dim3((unsigned)grid), dim3(256), 0, x, y, n, red);
}

}  // namespace tpmg
