// kernels_ksplit.cu -- the k-split line kernel (smoother, preconditioner,
// residual->restriction, and prolongation fused with the post-smooth).
//
// The one-thread-per-column kernel (kernels.cu) keeps a column's Thomas
// intermediates g'_k in shared memory (8*nz bytes per column), which at nz = 128
// limits an SM to 128 columns = one warp per SMSP, and the k-recurrence then
// runs latency-bound.  Here each column is split into NSEG segments of SL = 32
// levels handled by NSEG threads (the paper's outlook, "assign several threads
// to work on each vertical column ... substructuring"):
//
//  forward   y = L^-1 g  (M_T = L D L^T, y_k = g_k + a_k y_{k-1}, a_k = gamma/m_{k-1})
//            each thread: local recurrence from 0, yhat (32 values, in REGISTERS);
//            true y_k = yhat_k + P_k Y_s, P_k = prod_{j=k_s..k} a_j (level tables),
//            Y_s = y_{k_s - 1} chained through the segments' last values;
//  scale     g'_k = y_k / m_k;
//  backward  x_k = g'_k + b_k x_{k+1} (b_k = gamma/m_k): local xhat from 0, then
//            x_k = xhat_k + Q_k X_s, Q_k = prod_{j=k..k_e} b_j, X_s = x_{k_e + 1}
//            chained through the segments' first values.
//
// This is exact algebra on the same recurrences (only the rounding order
// differs), so the result matches a sequential Thomas solve to rounding.  With no
// g' buffer in shared memory a CTA holds TY * NSEG warps.
//
// Shared memory per stage and segment (TMA, 128-byte aligned blocks):
//   u box   (TY+2 rows) x (KB+2 levels) x HX columns (see KGeom): the
//           vertical neighbours of the chunk's first and last level come with the
//           box, so chunks are independent; each row block is 128-byte aligned so a
//           tile on a strip boundary loads its halo row from the neighbour's slab
//           with one TMA per row;
//   f box   TY rows x KB levels x 32 columns;
//   c box   (SMOOTH_PROLONG) the coarse u_c rows j0/2-1 .. j0/2+TY/2, columns
//           i0/2-8 .. i0/2+23, KB+2 levels: the post-smooth's input u + P u_c is
//           formed in shared memory (bilinear (9,3,3,1)/16, zero coarse ghosts).
#include "kernels.cuh"
#include "device_util.cuh"

#include <algorithm>
#include <type_traits>

namespace tpmg {
namespace {
using namespace dev;

constexpr int TX = kTileX;
constexpr int SL = kSegK;      // levels per segment
constexpr int HXC = 32;        // coarse box row width: coarse columns i0/2-8 .. i0/2+23
constexpr int XOC = 8;         // coarse box column of i0/2

__host__ __device__ constexpr int r16(int n) { return (n + 15) & ~15; }

// Two u-box layouts.  Smoother: rows of HX = 36 columns (i0-2 .. i0+33) loaded as
// one box; at a strip boundary the halo row comes from the neighbour's slab into a
// separate 128-byte aligned slot (SROW) and the stencil reads it through a row
// pointer.  Restriction and fused prolongation ("in place"): rows of 40 columns
// (i0-4 .. i0+35) so every row block is 128-byte aligned and a slab row is loaded in
// place (one TMA per row); this layout needs no slab slots (restriction: 3 stages fit)
// and lets the fused prolongation form u + P u_c on the whole box, slab rows included.
template <int MODE, int TY, int KB>
struct KGeom {
    static constexpr bool HALO = (MODE == MODE_SMOOTH || MODE == MODE_RESTRICT || MODE == MODE_SMOOTH_PROLONG ||
                                  MODE == MODE_CGPREC);
    static constexpr bool PROL = (MODE == MODE_SMOOTH_PROLONG);
    static constexpr bool INPLACE = PROL || MODE == MODE_RESTRICT;  // aligned rows, slab rows in place
    static constexpr int HX = INPLACE ? TX + 8 : TX + 4;        // u box row width
    static constexpr int XO = INPLACE ? 4 : 2;                  // box column of i0
    static constexpr int D = KB + 2;                            // box depth (levels k0-1 .. k0+KB)
    static constexpr int UROW = D * HX;                         // one u row block
    static constexpr int UBOX = HALO ? r16((TY + 2) * UROW) : 0;
    static constexpr int SROW = (HALO && !INPLACE) ? r16(UROW) : 0;  // one slab row slot
    static constexpr int FBOX = TY * KB * TX;
    static constexpr int FBOX2 = (MODE == MODE_CGPREC) ? FBOX : 0;   // CG: u next to r
    static constexpr int CROWS = TY / 2 + 2;
    static constexpr int CROW = D * HXC;
    static constexpr int CBOX = PROL ? CROWS * CROW : 0;
    static constexpr int SEGST = UBOX + 2 * SROW + FBOX + FBOX2 + CBOX;  // doubles per segment per stage
    static_assert(!INPLACE || ((UROW * 8) % 128 == 0 && (CROW * 8) % 128 == 0), "TMA row alignment");
    // exchange buffer: Thomas segment chaining [2][TY][NSEG][32], or (MODE_RESTRICT)
    // x-pair residual sums [2 (chunk parity)][TY][NSEG][KB][16]
    template <int NSEG>
    static constexpr int bnd() { return MODE == MODE_RESTRICT ? 2 * TY * NSEG * KB * 16 : 2 * TY * NSEG * 32; }
};

// Rows r0 .. r0+nrows-1 (local row index of the box's first row = jb) of a halo'd
// field into dst: one box TMA when no row comes from a slab, else one TMA per row.
__device__ __forceinline__ void tma_rows(double* dst, const TmaHalo& M, int rows, int rowst, int x, int k, int jb,
                                         int nyl, uint64_t* bar, bool force_rows = false)
{
    const bool lo = M.has_lo && jb < 0, hi = M.has_hi && jb + rows - 1 >= nyl;
    if (!force_rows && !lo && !hi) {
        tma_load_3d(dst, &M.main, x, k, jb, bar);
        return;
    }
    // a strip-boundary tile: the in-domain rows as one box, the slab row by itself (row-by-row
    // loads measured 4.5x slower per tile, and the kernel waits for its slowest CTA: r2r)
    if (!force_rows && M.has_m1 && lo != hi && (lo || jb + rows - 1 == nyl)) {   // (ragged last row: row by row)
        if (lo) {
            tma_load_3d(dst, &M.lo, x, k, 0, bar);
            tma_load_3d(dst + rowst, &M.m1, x, k, jb + 1, bar);
        } else {
            tma_load_3d(dst, &M.m1, x, k, jb, bar);
            tma_load_3d(dst + (rows - 1) * rowst, &M.hi, x, k, 0, bar);
        }
        return;
    }
    for (int r = 0; r < rows; ++r) {
        const int j = jb + r;
        if (j == -1 && M.has_lo) tma_load_3d(dst + r * rowst, &M.lo, x, k, 0, bar);
        else if (j == nyl && M.has_hi) tma_load_3d(dst + r * rowst, &M.hi, x, k, 0, bar);
        else tma_load_3d(dst + r * rowst, &M.row, x, k, j, bar);   // out of range: zero fill
    }
}

// Issue the TMA copies of step (tile origin i0, j0; chunk cc of every segment).
template <int MODE, int TY, int KB, int NSEG>
__device__ __forceinline__ void tma_step(double* st, const LineArgs& a, int i0, int j0, int cc, uint64_t* bar)
{
    using G = KGeom<MODE, TY, KB>;
    const int ny = (int)a.L.ny;
    uint32_t bytes = NSEG * ((G::HALO ? (TY + 2) * G::UROW : 0) + G::FBOX + G::FBOX2 + G::CBOX) * 8;
    bool lo = false, hi = false;
    if constexpr (G::HALO && !G::INPLACE) {
        lo = a.tma.h[0].has_lo && j0 == 0;
        hi = a.tma.h[0].has_hi && j0 + TY >= ny;
        bytes += NSEG * ((lo ? 1 : 0) + (hi ? 1 : 0)) * G::UROW * 8;
    }
    mbar_expect_tx(bar, bytes);
#pragma unroll
    for (int s = 0; s < NSEG; ++s) {
        double* seg = st + s * G::SEGST;
        const int k0 = s * SL + cc * KB;
        if constexpr (G::INPLACE) {
            tma_rows(seg, a.tma.h[0], TY + 2, G::UROW, i0 - G::XO, k0 - 1, j0 - 1, ny, bar, a.dbg & 1);
            if constexpr (G::PROL)
                tma_rows(seg + G::UBOX + G::FBOX, a.tma.h[1], G::CROWS, G::CROW, i0 / 2 - XOC, k0 - 1, j0 / 2 - 1,
                         ny / 2, bar);
        } else if constexpr (G::HALO) {
            tma_load_3d(seg, &a.tma.h[0].main, i0 - G::XO, k0 - 1, j0 - 1, bar);
            if (lo) tma_load_3d(seg + G::UBOX, &a.tma.h[0].lo, i0 - G::XO, k0 - 1, 0, bar);
            if (hi) tma_load_3d(seg + G::UBOX + G::SROW, &a.tma.h[0].hi, i0 - G::XO, k0 - 1, 0, bar);
        }
        tma_load_3d(seg + G::UBOX + 2 * G::SROW, &a.tma.q[0], i0, k0, j0, bar);
        if constexpr (G::FBOX2 > 0) tma_load_3d(seg + G::UBOX + 2 * G::SROW + G::FBOX, &a.tma.q[1], i0, k0, j0, bar);
    }
}

// HW: the in-kernel halo wait of the P2P overlap (LineArgs::hw), a separate instantiation
// so that the single-GPU kernels carry none of its code
template <int MODE, int TY, int NSEG, int KB, int NS2, bool PUSH, bool GEN, bool HW = false>
__global__ void __launch_bounds__(32 * TY * NSEG, 1) k_linek(const __grid_constant__ LineArgs a,
                                                             const __grid_constant__ KTables T)
{
    using G = KGeom<MODE, TY, KB>;
    constexpr int NT = 32 * TY * NSEG;
    constexpr int NCC = SL / KB;           // chunks per segment
    constexpr int STG = NSEG * G::SEGST;
    constexpr bool CGP = (MODE == MODE_CGPREC);
    constexpr bool NORM = (MODE == MODE_SMOOTH || MODE == MODE_SMOOTH_PROLONG || CGP);
    constexpr bool THOMAS = (MODE != MODE_RESTRICT);
    constexpr int NR = CGP ? 2 : 1;   // CG: ||r||^2 and zeta = <r, M^-1 r>

    extern __shared__ __align__(128) double smem_raw[];
    __shared__ __align__(8) uint64_t full_bar[NS2];
    double* smem = reinterpret_cast<double*>(reinterpret_cast<char*>(smem_raw) +
                                             ((128u - (smem_u32(smem_raw) & 127u)) & 127u));
    const int nz = a.L.nz;
    const int64_t nx = a.L.nx, ny = a.L.ny;
    double* stage = smem;                               // NS2 stages (128-byte aligned)
    double* tab = stage + NS2 * STG;                    // diag, invm, gim, afw, Pfw, Qbw (nz each)
    double* bnd = tab + r16(6 * nz);
    double* scratch = bnd + G::template bnd<NSEG>();

    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int s = warp % NSEG, ty = warp / NSEG;
    // per-level tables, staged in shared memory (warp-uniform broadcast reads)
    for (int q = tid; q < 6 * nz; q += NT) tab[q] = T.t[q / nz][q % nz];   // interior class (0)
    const double c0 = a.L.c, gamma = a.L.gamma, rho = a.rho, scale = a.scale;
    if (tid == 0) {
        for (int q = 0; q < NS2; ++q) mbar_init(&full_bar[q], 1);
        asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    }
    // prologue above (tables, barriers) overlaps the previous kernel's tail under PDL
    pdl_wait();
    pdl_trigger();
    if (a.skip && *a.skip) return;   // solver run-ahead: this iteration is not needed
    double acc[NR];
#pragma unroll
    for (int q = 0; q < NR; ++q) acc[q] = 0.0;
    // CG: alpha = zeta_{m-1} / sigma_m from the device scalars (written by earlier kernels)
    double alpha = 0.0;
    if constexpr (CGP)
        if (a.ratio.num >= 0) alpha = a.ratio.s[a.ratio.num] / a.ratio.s[a.ratio.den];

    const int ntx = (int)((nx + TX - 1) / TX), nty = (int)((ny + TY - 1) / TY);
    const int nrows = part_rows(a.part, nty);
    const int ntiles = ntx * nrows;
    const bool plo = PUSH && a.push.dst_lo != nullptr, phi = PUSH && a.push.dst_hi != nullptr;
    auto row_of = [&](int t) {
        if constexpr (HW) return boundary_deferred_row(t / ntx, nrows, kHaloDefer);   // in-kernel halo wait
        return part_row(a.part, nty, PUSH ? push_row(t / ntx, nrows, plo, phi) : t / ntx);
    };
    const int my_tiles = ((int)blockIdx.x < ntiles) ? (ntiles - (int)blockIdx.x + (int)gridDim.x - 1) / (int)gridDim.x : 0;
    const int total = my_tiles * NCC;
    __syncthreads();

    // producer (thread 0) and consumer cursors over the CTA's (tile, chunk) steps
    int p_count = 0, p_cc = 0, p_slot = 0, p_tile = blockIdx.x;
    auto issue = [&]() {
        if (tid == 0 && p_count < total) {
            if constexpr (HW)
                if (p_cc == 0) halo_tile_wait(a.hw, row_of(p_tile) * TY, TY, (int)ny);   // a strip-boundary tile row
                                                                                          // waits for the halo epoch
            asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
            tma_step<MODE, TY, KB, NSEG>(stage + p_slot * STG, a, (p_tile % ntx) * TX, row_of(p_tile) * TY, p_cc,
                                         &full_bar[p_slot]);
        }
        ++p_count;
        if (++p_slot == NS2) p_slot = 0;
        if (++p_cc == NCC) {
            p_cc = 0;
            p_tile += gridDim.x;
        }
    };
    int c_slot = 0;
    uint32_t c_phase = 0;

#pragma unroll
    for (int q = 0; q < NS2 - 1; ++q) issue();
    int rstep = 0;   // MODE_RESTRICT: chunk counter (exchange-buffer parity)

    // One tile.  BND: the tile holds columns of other classes (face Dirichlet [R25]); each
    // thread then reads its column's tables from the global class tables.
    auto tile_body = [&](auto bnd_t, int tl) {
        constexpr bool BND = decltype(bnd_t)::value;
        const int tile = (int)blockIdx.x + tl * (int)gridDim.x;
        const int i0 = (tile % ntx) * TX, j0 = row_of(tile) * TY;
        const int64_t i = i0 + lane, j = j0 + ty;
        const bool valid = (i < nx) && (j < ny);
        const double* ct = BND ? a.L.tab + (size_t)column_class(a.L, i, j) * kTabArrays * nz : tab;
        const double* diag = ct;
        const double* invm = ct + nz;
        const double* gim = ct + 2 * nz;
        const double* afw = ct + 3 * nz;
        const double* Pfw = ct + 4 * nz;
        const double* Qbw = ct + 5 * nz;
        // halo rows of this warp's row j kept in the slab slots (layout without in-place rows)
        const bool s_slab = G::SROW && a.tma.h[0].has_lo && j0 == 0 && ty == 0;
        const bool n_slab = G::SROW && a.tma.h[0].has_hi && (j0 + ty + 1 == ny);

        double yv[THOMAS ? SL : 1];
        double yprev = 0.0;
#pragma unroll
        for (int cc = 0; cc < NCC; ++cc) {
            issue();
            mbar_wait(&full_bar[c_slot], c_phase);
            double* seg = stage + c_slot * STG + s * G::SEGST;
            if (++c_slot == NS2) { c_slot = 0; c_phase ^= 1u; }
            if constexpr (G::PROL) {
                // u <- u + P u_c on the u box of this segment (the TY warps of the segment
                // share it; named barrier s+1).  Only in-domain fine cells change: the zero
                // ghosts stay zero; halo rows from a neighbour's slab get the correction too.
                const double* cb = seg + G::UBOX + 2 * G::SROW + G::FBOX;
                const int tseg = ty * 32 + lane;   // thread index within the segment's warps
                const bool slo = a.tma.h[0].has_lo, shi = a.tma.h[0].has_hi;
                for (int e = tseg; e < (TY + 2) * G::D * (TX + 2); e += TY * 32) {
                    const int x = G::XO - 1 + e % (TX + 2);       // box columns read by the stencil
                    const int rd = e / (TX + 2);
                    const int d = rd % G::D, r = rd / G::D;
                    const int ig = i0 - G::XO + x, jg = j0 - 1 + r;
                    const bool in = ig >= 0 && ig < nx &&
                                    ((jg >= 0 && jg < ny) || (jg == -1 && slo) || (jg == ny && shi));
                    if (in) {
                        const int cx = (ig >> 1) - (i0 >> 1) + XOC, cy = (jg >> 1) - (j0 >> 1) + 1;
                        const int sx = (ig & 1) ? 1 : -1, sy = (jg & 1) ? HXC * G::D : -HXC * G::D;
                        const double* cp = cb + (cy * G::D + d) * HXC + cx;
                        const double v = 9.0 * cp[0] + 3.0 * cp[sx] + 3.0 * cp[sy] + 1.0 * cp[sy + sx];
                        double* up = seg + (r * G::D + d) * G::HX + x;
                        *up = *up + v / 16.0;
                    }
                }
                asm volatile("bar.sync %0, %1;\n" ::"r"(s + 1), "r"(TY * 32) : "memory");
            }
            const double* fb = seg + G::UBOX + 2 * G::SROW + ty * (KB * TX) + lane;
            double gv[KB], rv[KB];
            if constexpr (G::HALO) {
                constexpr int HX = G::HX;
                const double* rc = seg + (ty + 1) * G::UROW + lane + G::XO;                    // own row
                const double* rs = s_slab ? seg + G::UBOX + lane + G::XO : rc - G::UROW;         // south row
                const double* rn = n_slab ? seg + G::UBOX + G::SROW + lane + G::XO : rc + G::UROW;  // north row
                double ud = rc[0], uc = rc[HX];
#pragma unroll
                for (int kk = 0; kk < KB; ++kk) {
                    const int dd = kk + 1;                 // box level of k = k0 + kk
                    const int k = s * SL + cc * KB + kk;
                    const double uu = rc[(dd + 1) * HX];
                    const double S = (rc[dd * HX - 1] + rc[dd * HX + 1]) + (rs[dd * HX] + rn[dd * HX]);
                    double Mu, c = c0;                                          // (M_T u)_k
                    if constexpr (GEN) {   // general vertical profiles: b_k, c_k, c_l d_k
                        Mu = fma(__ldg(a.L.prof + k), ud, fma(__ldg(a.L.prof + nz + k), uu, diag[k] * uc));
                        c = __ldg(a.L.prof + 2 * nz + k);
                    } else {
                        Mu = fma(-gamma, ud + uu, diag[k] * uc);
                    }
                    if constexpr (CGP) {
                        // (Fused) Tridiag: r -= alpha A p, u += alpha p, then z = M^-1 r
                        // (the box field is p, fb is r, fb + FBOX is u)
                        const double Ap = fma(-c, S, Mu);
                        const double rnew = fma(-alpha, Ap, fb[kk * TX]);
                        const double unew = fma(alpha, uc, fb[G::FBOX + kk * TX]);
                        if (valid) {
                            const int64_t o = (j * nz + k) * nx + i;
                            a.out0[o] = rnew;
                            a.out1[o] = unew;
                        }
                        gv[kk] = rnew;
                        rv[kk] = rnew;
                    } else {
                        const double r = fma(c, S, fb[kk * TX]) - Mu;           // f - A u
                        gv[kk] = fma(rho, r, Mu);        // g = (M - rho A) u + rho f  (one-pass smoother)
                        rv[kk] = r;
                    }
                    ud = uc;
                    uc = uu;
                }
            } else {
#pragma unroll
                for (int kk = 0; kk < KB; ++kk) { gv[kk] = scale * fb[kk * TX]; rv[kk] = 0.0; }
            }
            if constexpr (MODE == MODE_RESTRICT) {
                // f_c(I, J, k) = 1/4 (sum over the 2 x 2 fine children of f - A u):
                // x-pairs by shuffle, y-pairs (rows ty, ty+1 = two warps) through shared memory
                double* rb = bnd + (rstep++ & 1) * (TY * NSEG * KB * 16);
#pragma unroll
                for (int kk = 0; kk < KB; ++kk) {
                    const double rsum = rv[kk] + __shfl_xor_sync(0xffffffffu, rv[kk], 1);
                    if ((lane & 1) == 0) rb[((ty * NSEG + s) * KB + kk) * 16 + (lane >> 1)] = rsum;
                }
                __syncthreads();   // every warp is done with this slot; the x-pair sums are visible
                if ((ty & 1) == 0) {
                    const int64_t nxc = nx >> 1, nyc = ny >> 1;
                    const int64_t J = (j0 + ty) >> 1;
                    const int l = lane & 15;
                    const int64_t I = (i0 >> 1) + l;
#pragma unroll
                    for (int kk = lane >> 4; kk < KB; kk += 2) {
                        const int k = s * SL + cc * KB + kk;
                        const double v = 0.25 * (rb[((ty * NSEG + s) * KB + kk) * 16 + l] +
                                                 rb[(((ty + 1) * NSEG + s) * KB + kk) * 16 + l]);
                        if (I < nxc && J < nyc) a.out0[(J * nz + k) * nxc + I] = v;
                    }
                }
                continue;
            } else {
                // local forward recurrence yhat_k = g_k + a_k yhat_{k-1} (yhat = 0 before the segment)
#pragma unroll
                for (int kk = 0; kk < KB; ++kk) {
                    const int k = s * SL + cc * KB + kk;
                    yprev = (cc == 0 && kk == 0) ? gv[kk] : fma(afw[k], yprev, gv[kk]);
                    yv[cc * KB + kk] = yprev;
                    if constexpr (NORM)
                        if (valid) acc[0] = fma(rv[kk], rv[kk], acc[0]);   // phantom columns of ragged tiles excluded
                }
                __syncthreads();   // every warp is done with this slot
            }
        }
        if constexpr (THOMAS) {
            // chain the segments: Y_s = y_{k_s - 1} (true), from the segments' last yhat
            double* bF = bnd + (ty * NSEG) * 32 + lane;               // [ty][seg][lane]
            double* bB = bnd + TY * NSEG * 32 + (ty * NSEG) * 32 + lane;
            bF[s * 32] = yv[SL - 1];
            __syncthreads();
            double Y = 0.0;
#pragma unroll
            for (int q = 0; q < NSEG - 1; ++q)
                if (q < s) Y = fma(Pfw[(q + 1) * SL - 1], Y, bF[q * 32]);
            // g'_k = (yhat_k + P_k Y) / m_k, then the local backward recurrence
            const int kb = s * SL;
#pragma unroll
            for (int q = 0; q < SL; ++q) {
                const double yt = fma(Pfw[kb + q], Y, yv[q]);   // y = L^-1 g
                yv[q] = yt * invm[kb + q];                        // g' = D^-1 y
                if constexpr (CGP)
                    if (valid) acc[1] = fma(yv[q], yt, acc[1]);   // zeta = sum y_k g'_k [R22]
            }
            double xh = 0.0;
#pragma unroll
            for (int q = SL - 1; q >= 0; --q) {
                xh = fma(gim[kb + q], xh, yv[q]);
                yv[q] = xh;
            }
            bB[s * 32] = yv[0];
            __syncthreads();
            double X = 0.0;                                           // x_{k_e + 1} (true)
#pragma unroll
            for (int q = NSEG - 1; q >= 1; --q)
                if (q > s) X = fma(Qbw[q * SL], X, bB[q * 32]);
            double* op = (CGP ? a.out2 : a.out0) + (j * nz + kb) * nx + i;
#pragma unroll
            for (int q = 0; q < SL; ++q) {
                const double x = fma(Qbw[kb + q], X, yv[q]);
                if (valid) {
                    *op = x;
                    // fused halo push (PUSH instantiation only): a strip-boundary row also
                    // goes to the neighbour's slab over NVLink
                    if constexpr (PUSH) push_out(a.push, j, ny, (int64_t)(kb + q) * nx + i, x);
                }
                op += nx;
            }
            // bnd is reused by the next tile only after its forward chunks (>= 1 __syncthreads)
        }
    };
    for (int tl = 0; tl < my_tiles; ++tl) {
        const int tile = (int)blockIdx.x + tl * (int)gridDim.x;
        if (tile_on_boundary(a.L, (int64_t)(tile % ntx) * TX, (int64_t)row_of(tile) * TY, TX, TY))
            tile_body(std::true_type{}, tl);
        else
            tile_body(std::false_type{}, tl);
    }
    if (NORM && a.red.result != nullptr) grid_reduce<NR>(a.red, acc, scratch);
}

template <int MODE, int TY, int NSEG, int KB, int NS2>
size_t ksmem(int nz)
{
    using G = KGeom<MODE, TY, KB>;
    return (size_t)(NS2 * NSEG * G::SEGST + r16(6 * nz) + G::template bnd<NSEG>() + 64 + 16) * sizeof(double);
}

template <int MODE, int TY, int NSEG, int KB, int NS2, bool PUSH, bool GEN = false, bool HW = false>
cudaError_t launch_k_push(const Launcher& ln, const LineArgs& a, const KTables& T)
{
    auto kern = k_linek<MODE, TY, NSEG, KB, NS2, PUSH, GEN, HW>;
    const size_t smem = ksmem<MODE, TY, NSEG, KB, NS2>(a.L.nz);
    static size_t limit = 0;
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
    cudaError_t e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, 32 * TY * NSEG, smem);
    if (e != cudaSuccess) return e;
    per_sm = std::max(per_sm, 1);
    const int64_t ntiles = ((a.L.nx + TX - 1) / TX) * part_rows(a.part, (int)((a.L.ny + TY - 1) / TY));
    const int64_t grid = std::min<int64_t>(ntiles, (int64_t)std::max(1, ln.num_sms - ln.reserve_sms) * per_sm);
    if (grid <= 0) return cudaSuccess;
    return launch_kernel(ln, kern, dim3((unsigned)grid), dim3(32 * TY * NSEG), smem, a, T);
}

// The fused halo push (multi-GPU, P2P) has its own instantiation, so single-GPU launches
// carry none of its code.  Only the smoother and the preconditioner push.
template <int MODE, int TY, int NSEG, int KB, int NS2, bool HWOK = false>
cudaError_t launch_k(const Launcher& ln, const LineArgs& a, const KTables& T)
{
    if (a.hw.flag[0] || a.hw.flag[1]) {   // P2P overlap with the in-kernel halo wait
        if constexpr (HWOK && (MODE == MODE_SMOOTH || MODE == MODE_RESTRICT))
            if (!a.L.gen && !a.push.dst_lo && !a.push.dst_hi)
                return launch_k_push<MODE, TY, NSEG, KB, NS2, false, false, true>(ln, a, T);
        return cudaErrorNotSupported;   // the host checks ksplit_halo_wait() first
    }
    if constexpr (MODE == MODE_SMOOTH || MODE == MODE_RESTRICT) {
        if (a.L.gen) {   // general vertical profiles: the stencil's couplings per level
            if constexpr (MODE == MODE_SMOOTH)
                if (a.push.dst_lo || a.push.dst_hi) return launch_k_push<MODE, TY, NSEG, KB, NS2, true, true>(ln, a, T);
            return launch_k_push<MODE, TY, NSEG, KB, NS2, false, true>(ln, a, T);
        }
    } else if constexpr (MODE != MODE_PREC) {
        if (a.L.gen) return cudaErrorNotSupported;   // fused prolongation / k-split CG: flat box only
    }
    if constexpr (MODE == MODE_SMOOTH || MODE == MODE_PREC)
        if (a.push.dst_lo || a.push.dst_hi) return launch_k_push<MODE, TY, NSEG, KB, NS2, true>(ln, a, T);
    return launch_k_push<MODE, TY, NSEG, KB, NS2, false>(ln, a, T);
}

template <int MODE, int TY, int KB, int NS2, bool HWOK = false>
cudaError_t launch_k_nseg(const Launcher& ln, const LineArgs& a, const KTables& T)
{
    switch (a.L.nz / SL) {
    case 1: return launch_k<MODE, TY, 1, KB, NS2, HWOK>(ln, a, T);
    case 2: return launch_k<MODE, TY, 2, KB, NS2, HWOK>(ln, a, T);
    case 4: return launch_k<MODE, TY, 4, KB, NS2, HWOK>(ln, a, T);
    default: return cudaErrorInvalidValue;
    }
}

// configurations (rows TY, levels per chunk KB): 0 = 2 x 8; 1 = 4 x 4 (default); 2 = 2 x 4
struct Cfg { int ty, kb; };
constexpr Cfg kCfg[3] = {{2, 8}, {4, 4}, {2, 4}};

}  // namespace

bool ksplit_halo_wait(int mode, int cfg, int gen)
{
    return (mode == MODE_SMOOTH || mode == MODE_RESTRICT) && cfg == 1 && gen == 0;
}

bool ksplit_supported(int mode, int nz, int nx)
{
    // TMA row strides must be multiples of 16 bytes: even nx (and even coarse nx for the
    // fused prolongation)
    return (mode == MODE_SMOOTH || mode == MODE_PREC || mode == MODE_RESTRICT || mode == MODE_SMOOTH_PROLONG ||
            mode == MODE_CGPREC) &&
           nz % SL == 0 && nz <= kKsplitMaxNZ && (nz / SL == 1 || nz / SL == 2 || nz / SL == 4) && nx % 2 == 0 &&
           (mode != MODE_SMOOTH_PROLONG || nx % 4 == 0);
}

KsplitBoxes ksplit_boxes(int mode, int cfg)
{
    const Cfg c = kCfg[cfg < 0 || cfg > 2 ? 0 : cfg];
    const bool inplace = (mode == MODE_SMOOTH_PROLONG || mode == MODE_RESTRICT);
    return KsplitBoxes{c.ty, c.kb, inplace ? TX + 8 : TX + 4, c.kb + 2, inplace ? 4 : 2, HXC, XOC};
}

cudaError_t launch_line_ksplit(const Launcher& ln, int mode, int cfg, const LineArgs& a, const KTables& T)
{
    if (mode == MODE_SMOOTH) {
        if (cfg == 1) return launch_k_nseg<MODE_SMOOTH, 4, 4, 3, true>(ln, a, T);
        if (cfg == 2) return launch_k_nseg<MODE_SMOOTH, 2, 4, 3>(ln, a, T);
        return launch_k_nseg<MODE_SMOOTH, 2, 8, 2>(ln, a, T);
    }
    if (mode == MODE_SMOOTH_PROLONG) {
        if (cfg == 1) return launch_k_nseg<MODE_SMOOTH_PROLONG, 4, 4, 2>(ln, a, T);
        if (cfg == 2) return launch_k_nseg<MODE_SMOOTH_PROLONG, 2, 4, 3>(ln, a, T);
        return launch_k_nseg<MODE_SMOOTH_PROLONG, 2, 8, 2>(ln, a, T);
    }
    if (mode == MODE_PREC) {   // no u box: deeper pipelines are cheap
        if (cfg == 1) return launch_k_nseg<MODE_PREC, 4, 4, 6>(ln, a, T);
        if (cfg == 2) return launch_k_nseg<MODE_PREC, 2, 4, 6>(ln, a, T);
        return launch_k_nseg<MODE_PREC, 2, 8, 4>(ln, a, T);
    }
    if (mode == MODE_CGPREC) {     // p box + r and u boxes: two stages fit at 4 x 4
        if (cfg == 1) return launch_k_nseg<MODE_CGPREC, 4, 4, 2>(ln, a, T);
        if (cfg == 2) return launch_k_nseg<MODE_CGPREC, 2, 4, 3>(ln, a, T);
        return launch_k_nseg<MODE_CGPREC, 2, 8, 2>(ln, a, T);
    }
    if (mode == MODE_RESTRICT) {   // no Thomas: the exchange buffer replaces the chaining buffer
        if (cfg == 1) return launch_k_nseg<MODE_RESTRICT, 4, 4, 3, true>(ln, a, T);
        if (cfg == 2) return launch_k_nseg<MODE_RESTRICT, 2, 4, 3>(ln, a, T);
        return launch_k_nseg<MODE_RESTRICT, 2, 8, 2>(ln, a, T);
    }
    return cudaErrorInvalidValue;
}

}  // namespace tpmg
