// api.cpp -- the C ABI of libtpmg.so (include/tpmg.h): context, per-level
// operator tables, multigrid hierarchy, PCG, halo exchange and reductions.
//
// Host orchestration only: every arithmetic step of the hot path runs in the
// sm_100a kernels of kernels.cu.  Multi-GPU plumbing is NCCL over NVLink:
// halo slabs with ncclSend/ncclRecv (y-strip decomposition) and
// ncclAllReduce for the solver's global sums.
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>
#include <nccl.h>

#include <unistd.h>

#include <algorithm>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <string>
#include <tuple>
#include <vector>

#include "../../include/tpmg.h"
#include "kernels.cuh"

using namespace tpmg;

namespace {

thread_local std::string g_create_error;

struct LevelData {
    LevelConst lc{};
    double* d_tab = nullptr;
    double* u[2] = {nullptr, nullptr};  // MG iterate ping-pong (fine level: u[0] = caller's u)
    int cur = 0;
    double* f = nullptr;                // MG right-hand side (coarse levels)
    KTables ktab{};                     // k-split tables (kernel parameter space)
    double* d_prof = nullptr;           // general vertical profiles: [b_k][c_k][c_l d_k] (device)
    double* d_fprof = nullptr;          // with per-column fields: [a_k-b_k-c_k][b_k][c_k][d_k] (device)
    double* d_fld = nullptr;            // per-column fields, LevelConst::fld layout (device)
    double* d_im = nullptr;             // per-column fields: 1/m_k of every column's block (Lambda layout)
    bool im_ok = false;                 // d_im is current
    double* slab_lo = nullptr;          // halo rows j = -1 / j = ny for this level (nranks > 1)
    double* slab_hi = nullptr;
    size_t n() const { return (size_t)lc.nx * (size_t)lc.ny * (size_t)lc.nz; }
    size_t plane() const { return (size_t)lc.nx * (size_t)lc.nz; }
};

}  // namespace

struct tpmg_ctx {
    tpmg_params p{};
    int rank = 0, nranks = 1, device = 0;
    cudaStream_t stream = nullptr;
    int num_sms = 148;
    int L = 0;
    int64_t ny_loc = 0, y0 = 0;
    std::vector<LevelData> lv;  // index 1..L
    std::vector<double> prof_abcd;   // the vertical profiles a, b, c, d in use (4 nz; set by build_tables)
    bool fields = false;             // per-column horizontal fields set (tpmg_set_fields)
    bool gen_profiles = false;       // general vertical profiles set (tpmg_set_profiles)
    // reductions
    double* d_partials = nullptr;
    unsigned* d_ticket = nullptr;
    double* d_scal = nullptr;   // CG per-iteration scalars / norms
    int scal_cap = 0;
    double* h_pinned = nullptr; // pinned host scalars
    // solver run-ahead: device flags per iteration, their pinned host copies, events
    int* d_flags = nullptr;
    int* h_flags = nullptr;
    int* dh_flags = nullptr;            // device view of h_flags (mapped pinned memory)
    int flags_cap = 0;
    const int* skip = nullptr;  // predicate put into every launch while set
    cudaEvent_t ev_it[8] = {};
    // work vectors (lazily allocated)
    bool mg_ready = false, cg_ready = false;
    double* scratch = nullptr;   // fine-size scratch (single-op ping-pong)
    double *cg_r = nullptr, *cg_z = nullptr, *cg_p[2] = {nullptr, nullptr};
    double *cg_zlo = nullptr, *cg_zhi = nullptr, *cg_plo[2] = {nullptr, nullptr}, *cg_phi[2] = {nullptr, nullptr};
    double *host_f = nullptr, *host_u = nullptr;  // device buffers for tpmg_solve_host
    double* host_u2 = nullptr;                     // ... the second solution of tpmg_solve_host_pair
    cudaStream_t copy_stream = nullptr;            // tpmg_solve_host_pair's overlapped device->host copy
    cudaEvent_t ev_copy = nullptr;
    ncclComm_t comm = nullptr;
    // halo channels (nranks > 1): 1..L = levels, L+1 = CG z.  Each has double-buffered slabs
    // in one pool allocation; in P2P mode the neighbours write into them over NVLink.
    struct Chan {
        size_t plane = 0;
        int64_t nyl = 0;
        double* lo[2] = {nullptr, nullptr};
        double* hi[2] = {nullptr, nullptr};
        double** cur_lo = nullptr;      // where consumers look for the current slabs
        double** cur_hi = nullptr;
        int epoch = 0;
        size_t off_lo[2] = {0, 0}, off_hi[2] = {0, 0}, off_flags = 0;  // byte offsets in the pool
        const double* pushed = nullptr; // buffer whose boundary rows a producer kernel pushed
                                        // with epoch `epoch` (fused push, not yet waited for)
        bool publish = false;           // a fused push awaits its publish_pushed()
    };
    std::vector<Chan> chans;
    void* halo_pool = nullptr;
    size_t halo_pool_bytes = 0;
    bool p2p = false;                   // TPMG_HALO=nccl selects NCCL send/recv
    char* peer_pool[2] = {nullptr, nullptr};   // [0] lower neighbour's pool, [1] upper's (IPC-mapped)
    std::vector<char*> peer_all;               // every rank's pool (IPC-mapped; mine at [rank])
    bool p2p_reduce = false;                   // allreduces by k_allreduce_p2p (TPMG_ALLREDUCE=nccl: NCCL)
    P2PReduce red{};                           // its slot / flag addresses
    unsigned red_epoch = 0;
    size_t off_red = 0, off_redflags = 0;      // byte offsets in the pool
    // overlap of halo exchanges with interior work (nranks > 1)
    ncclComm_t comm_halo = nullptr;     // halo traffic on its own communicator and stream
    cudaStream_t comm_stream = nullptr;
    cudaEvent_t ev_ready = nullptr, ev_halo = nullptr;
    bool overlap = true;                // P2P halos: interior rows while the halo travels (TPMG_OVERLAP=0 off)
    bool overlap_cg = false;            // the CG direction kernel too (TPMG_OVERLAP_CG=1)
    bool pair_u = false;                // CG: u updated every second iteration (TPMG_PAIR_U=1; r2v: PCG
                                        // -4% time, but the two variants run at 0.86 of the copy peak)
    bool overlap_nccl = false;          // NCCL halos: TPMG_OVERLAP=1 (measured slower at N=4 in round 1:
                                        // the split launches cost more than the NCCL latency they hide)
    int reserve_sms = 4;                // SMs left to NCCL while the interior runs
    int cur_reserve = 0;
    tpmg_stats stats{};
    cudaEvent_t ev0 = nullptr, ev1 = nullptr;
    // profiling (tpmg_profile)
    bool pdl = false;                   // programmatic dependent launches (TPMG_PDL=1)
    bool tmem = true;                   // Thomas g' of the column kernels in Tensor Memory (TPMG_TMEM=0: smem)
    int tm_ctas = 1;                    // their CTAs per SM (TPMG_TM_CTAS; see kernels.cuh)
    int tm_stages = 3;                  // their TMA ring depth (TPMG_TM_STAGES: 3, 4, 5)
    bool pivots = true;                 // per-column fields: precomputed pivots (TPMG_PIVOTS=0: off)
    bool ksplit_cg = false;             // k-split CG preconditioner (TPMG_KSPLIT_CG=1)
    bool halo_off = false;              // TPMG_HALO=off: skip halo exchanges (timing experiments)
    bool fused_push = false;            // P2P: producers push their boundary rows (TPMG_FUSED_PUSH=1)
    bool prof_on = false;
    uint32_t prof_mask = 0;             // kernel classes bracketed with events (bit = tpmg_kernel)
    struct ProfRec { int cls; double cells; cudaEvent_t a, b; const int* skip; };
    std::vector<ProfRec> prof_pending;
    int dbg = 0;                        // LineArgs::dbg (timing experiments)
    bool carveout_fit = false;          // line kernels' carveout sized to their CTAs (TPMG_CARVEOUT=fit)
    bool tma_store = false;             // CGPREC outputs by TMA stores (TPMG_TMA_STORE=1)
    bool dev_publish = false;           // P2P: the push kernel stores the epoch flags (TPMG_DEV_PUBLISH=1)
    bool skip_finish = false;           // P2P: no stream waits after an in-kernel-waiting consumer (TPMG_SKIP_FINISH=1)
    unsigned* d_push_done = nullptr;    // k_halo_push ticket counter (device publish)
    int tma_promo = CU_TENSOR_MAP_L2_PROMOTION_L2_256B;   // TMA L2 promotion (TPMG_TMA_PROMO 0..3: none, 64, 128, 256 B)
    int l2hint = 3;                     // k_line TMA L2 policies (TPMG_L2HINT bits: 1 halo'd evict_last, 2 plain evict_first; r2aj/r2ak)
    int cgdir_ctas = 0;                 // k_line<CGDIR> CTAs per SM (TPMG_CGDIR_CTAS; 0 automatic)
    int band_w = 0;                     // k_line tile bands on wide grids (TPMG_BAND=n; r2ag: slower, off)
    bool prof_detail = false;           // TPMG_PROF_DETAIL=1: per-level breakdown on stderr at tpmg_destroy
    std::map<std::pair<int, double>, std::pair<int64_t, double>> prof_by_size;
    std::vector<cudaEvent_t> prof_pool;
    // TMA descriptors, cached by (address, nx, nz, ny, box x, box rows)
    bool use_tma = true;
    bool sync_debug = false;   // TPMG_SYNC_DEBUG=1: synchronise after every line kernel
    bool fuse_prolong = false; // TPMG_FUSE_PROLONG=1: prolongation fused into the post-smooth (k-split);
                               // off by default: measured slower (the in-smem u + P u_c pass
                               // costs more issue slots than the 16 B/cell it saves)
    int ksplit_cfg_coarse = 0;   // k-split config on levels whose 4x4 tiles do not fill the SMs: 0 = 2x8
                                 // (r2ac: 0.5% per V-cycle; TPMG_KSPLIT_COARSE=-1 keeps ksplit_cfg)
    int ksplit_cfg = 1;        // k-split config (TPMG_KSPLIT: "0" off, "1" 2x8/2 stages, "2" 4x4/3 stages
                               // (default), "3" 2x4/2 stages); -1 = off
    std::map<std::tuple<uintptr_t, int64_t, int, int64_t, int, int>, CUtensorMap> tmaps;
    int64_t prof_launches[TPMG_K_COUNT] = {};
    double prof_ms[TPMG_K_COUNT] = {}, prof_cells[TPMG_K_COUNT] = {};
    std::string err;
};

namespace {

tpmg_status fail(tpmg_ctx* ctx, tpmg_status st, const char* fmt, ...)
{
    char buf[512];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof buf, fmt, ap);
    va_end(ap);
    if (ctx) ctx->err = buf; else g_create_error = buf;
    return st;
}

#define CUDA_TRY(ctx, expr)                                                                  \
    do {                                                                                     \
        cudaError_t e_ = (expr);                                                             \
        if (e_ != cudaSuccess)                                                               \
            return fail((ctx), TPMG_E_CUDA, "%s: %s (%s:%d)", #expr, cudaGetErrorString(e_), \
                        __FILE__, __LINE__);                                                 \
    } while (0)

#define NCCL_TRY(ctx, expr)                                                                  \
    do {                                                                                     \
        ncclResult_t e_ = (expr);                                                            \
        if (e_ != ncclSuccess)                                                               \
            return fail((ctx), TPMG_E_NCCL, "%s: %s (%s:%d)", #expr, ncclGetErrorString(e_), \
                        __FILE__, __LINE__);                                                 \
    } while (0)

#define TRY(expr)                            \
    do {                                     \
        tpmg_status s_ = (expr);             \
        if (s_ != TPMG_OK) return s_;        \
    } while (0)

Launcher launcher(tpmg_ctx* ctx)
{
    Launcher ln;
    ln.stream = ctx->stream;
    ln.num_sms = ctx->num_sms;
    ln.launch_counter = &ctx->stats.kernel_launches;
    ln.reserve_sms = ctx->cur_reserve;
    ln.pdl = ctx->pdl;
    ln.tmem = ctx->tmem;
    ln.tm_ctas = ctx->tm_ctas;
    ln.tm_stages = ctx->tm_stages;
    ln.carveout_fit = ctx->carveout_fit;
    return ln;
}

ReduceSlot slot(tpmg_ctx* ctx, double* result)
{
    return ReduceSlot{ctx->d_partials, ctx->d_ticket, result, 0};
}

tpmg_status dev_alloc(tpmg_ctx* ctx, double** p, size_t n)
{
    if (*p) return TPMG_OK;
    cudaError_t e = cudaMalloc((void**)p, sizeof(double) * (n ? n : 1));
    if (e != cudaSuccess) {
        *p = nullptr;
        return fail(ctx, TPMG_E_OOM, "cudaMalloc(%zu doubles): %s", n, cudaGetErrorString(e));
    }
    return TPMG_OK;
}

tpmg_status check_level(tpmg_ctx* ctx, int level)
{
    if (!ctx) return TPMG_E_PARAM;
    if (level < 1 || level > ctx->L) return fail(ctx, TPMG_E_RANGE, "level %d not in [1, %d]", level, ctx->L);
    return TPMG_OK;
}

// ------------------------------------------------------------------ halos and reductions

// Fill the halo slabs of `level` from the neighbours' boundary rows of x (nranks > 1).
tpmg_status exchange_on(tpmg_ctx* ctx, cudaStream_t st, ncclComm_t comm, size_t plane, int64_t nyl, const double* x,
                        double* lo, double* hi)
{
    const double* first = x;
    const double* last = x + (size_t)(nyl - 1) * plane;
    NCCL_TRY(ctx, ncclGroupStart());
    if (ctx->rank > 0) {
        NCCL_TRY(ctx, ncclSend(first, plane, ncclDouble, ctx->rank - 1, comm, st));
        NCCL_TRY(ctx, ncclRecv(lo, plane, ncclDouble, ctx->rank - 1, comm, st));
    }
    if (ctx->rank < ctx->nranks - 1) {
        NCCL_TRY(ctx, ncclSend(last, plane, ncclDouble, ctx->rank + 1, comm, st));
        NCCL_TRY(ctx, ncclRecv(hi, plane, ncclDouble, ctx->rank + 1, comm, st));
    }
    NCCL_TRY(ctx, ncclGroupEnd());
    ++ctx->stats.halo_exchanges;
    return TPMG_OK;
}

// ---- device-initiated halo exchange over NVLink (P2P mode)
PFN_cuStreamWaitValue32_v11070 g_wait_value = nullptr;
PFN_cuStreamWriteValue32_v11070 g_write_value = nullptr;

bool stream_memops()
{
    static bool tried = false;
    if (!tried) {
        tried = true;
        cudaDriverEntryPointQueryResult q;
        void* p = nullptr;
        if (cudaGetDriverEntryPoint("cuStreamWaitValue32", &p, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            g_wait_value = reinterpret_cast<PFN_cuStreamWaitValue32_v11070>(p);
        p = nullptr;
        if (cudaGetDriverEntryPoint("cuStreamWriteValue32", &p, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            g_write_value = reinterpret_cast<PFN_cuStreamWriteValue32_v11070>(p);
    }
    return g_wait_value != nullptr && g_write_value != nullptr;
}

tpmg_status wait_value(tpmg_ctx* ctx, const void* addr, uint32_t v)
{
    CUresult r = g_wait_value((CUstream)ctx->stream, (CUdeviceptr)addr, v, CU_STREAM_WAIT_VALUE_GEQ);
    if (r != CUDA_SUCCESS) return fail(ctx, TPMG_E_CUDA, "cuStreamWaitValue32 failed (%d)", (int)r);
    return TPMG_OK;
}

// Stream-ordered store of v to addr once all preceding work (and its memory traffic, the
// default write-value fence) has completed.
tpmg_status write_value(tpmg_ctx* ctx, void* addr, uint32_t v)
{
    CUresult r = g_write_value((CUstream)ctx->stream, (CUdeviceptr)addr, v, CU_STREAM_WRITE_VALUE_DEFAULT);
    if (r != CUDA_SUCCESS) return fail(ctx, TPMG_E_CUDA, "cuStreamWriteValue32 failed (%d)", (int)r);
    return TPMG_OK;
}

// Remote destinations of channel c's epoch-E rows: slot E & 1 of the neighbours' slabs.
HaloPush push_desc(tpmg_ctx* ctx, tpmg_ctx::Chan& ch, int E)
{
    const int b = E & 1;
    HaloPush hp{};
    hp.n = (int64_t)ch.plane;
    hp.dst_lo = ctx->rank > 0 ? reinterpret_cast<double*>(ctx->peer_pool[0] + ch.off_hi[b]) : nullptr;
    hp.dst_hi = ctx->rank < ctx->nranks - 1 ? reinterpret_cast<double*>(ctx->peer_pool[1] + ch.off_lo[b]) : nullptr;
    return hp;
}

// Publish epoch E of channel ch to the neighbours: stream write-values into their flags
// ("data from upper" of the lower neighbour, "data from lower" of the upper one), each
// fenced after the preceding kernel's remote stores (CU_STREAM_WRITE_VALUE_DEFAULT).
tpmg_status publish_epoch(tpmg_ctx* ctx, tpmg_ctx::Chan& ch, int E)
{
    if (ctx->rank > 0) TRY(write_value(ctx, ctx->peer_pool[0] + ch.off_flags + 1 * 4, (uint32_t)E));
    if (ctx->rank < ctx->nranks - 1) TRY(write_value(ctx, ctx->peer_pool[1] + ch.off_flags + 0 * 4, (uint32_t)E));
    return TPMG_OK;
}

// Wait until both neighbours' epoch-E rows of channel ch have arrived; point the
// consumers at slot E & 1.
tpmg_status wait_epoch(tpmg_ctx* ctx, tpmg_ctx::Chan& ch, int E)
{
    char* mine = static_cast<char*>(ctx->halo_pool) + ch.off_flags;
    if (ctx->rank > 0) TRY(wait_value(ctx, mine + 0 * 4, (uint32_t)E));
    if (ctx->rank < ctx->nranks - 1) TRY(wait_value(ctx, mine + 1 * 4, (uint32_t)E));
    *ch.cur_lo = ch.lo[E & 1];
    *ch.cur_hi = ch.hi[E & 1];
    ++ctx->stats.halo_exchanges;
    return TPMG_OK;
}

// Channel c exchange, epoch E, slot b = E & 1.  Flags (uint32) of channel c in every
// rank's pool: [0] data from the lower neighbour, [1] data from the upper.
//   push:    my row 0 goes into the lower neighbour's hi[b] slab and my row ny-1 into the
//            upper neighbour's lo[b] slab, by remote stores over NVLink: either the
//            producer kernel of x already did it (fused push, see fused_push) or one
//            k_halo_push kernel does it now;
//   publish: stream write-values store E into both neighbours' flags after that kernel;
//   wait:    stream wait-values until both neighbours' epoch-E flags are set.
// No acknowledgements are needed: a neighbour's epoch E-1 push is stream-ordered after its
// kernels that read epoch E-2 (the slot b that epoch E overwrites), and I push epoch E
// only after my stream saw its epoch E-1 data (every pushed epoch is waited for, in
// order, before the next push).  No kernel spins.
// First half of a P2P exchange: push x's boundary rows and publish the epoch, without
// waiting for the neighbours' rows.  *E_out = the epoch to wait for (0: already waited, the
// producer had pushed x itself).  Work that reads no halo row can run before p2p_finish.
tpmg_status p2p_begin(tpmg_ctx* ctx, tpmg_ctx::Chan& ch, const double* x, int* E_out)
{
    *E_out = 0;
    if (ch.pushed) {
        const bool mine = (ch.pushed == x);
        ch.pushed = nullptr;
        TRY(wait_epoch(ctx, ch, ch.epoch));
        if (mine) return TPMG_OK;   // the producer already pushed x's boundary rows
    }
    const int E = ++ch.epoch;
    HaloPush hp = push_desc(ctx, ch, E);
    hp.src_first = x;
    hp.src_last = x + (size_t)(ch.nyl - 1) * ch.plane;
    if (ctx->dev_publish) {   // the push kernel's last CTA stores the epoch flags itself
        hp.flag_lo = ctx->rank > 0 ? reinterpret_cast<unsigned*>(ctx->peer_pool[0] + ch.off_flags + 1 * 4) : nullptr;
        hp.flag_hi = ctx->rank < ctx->nranks - 1 ? reinterpret_cast<unsigned*>(ctx->peer_pool[1] + ch.off_flags + 0 * 4)
                                                 : nullptr;
        hp.done = ctx->d_push_done;
        hp.epoch = (unsigned)E;
    }
    CUDA_TRY(ctx, launch_halo_push(launcher(ctx), hp));
    if (!ctx->dev_publish) TRY(publish_epoch(ctx, ch, E));
    *E_out = E;
    return TPMG_OK;
}

tpmg_status p2p_finish(tpmg_ctx* ctx, tpmg_ctx::Chan& ch, int E)
{
    return E ? wait_epoch(ctx, ch, E) : TPMG_OK;
}

// p2p_finish after a consumer kernel that waited in the kernel for epoch E (HaloWait): its
// completion implies both flags reached E, so the stream waits are redundant (TPMG_SKIP_FINISH);
// the slab pointers and the stats advance as in wait_epoch.
tpmg_status p2p_finish_waited(tpmg_ctx* ctx, tpmg_ctx::Chan& ch, int E)
{
    if (!E || !ctx->skip_finish) return p2p_finish(ctx, ch, E);
    *ch.cur_lo = ch.lo[E & 1];
    *ch.cur_hi = ch.hi[E & 1];
    ++ctx->stats.halo_exchanges;
    return TPMG_OK;
}

// x with the slabs of epoch E of channel ch (E = 0: the current slabs)
HaloField halo_epoch_view(tpmg_ctx* ctx, tpmg_ctx::Chan& ch, const double* x, int E)
{
    const bool lo = ctx->rank > 0, hi = ctx->rank < ctx->nranks - 1;
    if (!E) return HaloField{x, lo ? *ch.cur_lo : nullptr, hi ? *ch.cur_hi : nullptr};
    return HaloField{x, lo ? ch.lo[E & 1] : nullptr, hi ? ch.hi[E & 1] : nullptr};
}

// The in-kernel wait for epoch E of channel ch: my pool's flags [0] data from the lower
// neighbour, [1] data from the upper one.
HaloWait halo_wait_of(tpmg_ctx* ctx, tpmg_ctx::Chan& ch, int E)
{
    const unsigned* f = reinterpret_cast<const unsigned*>(static_cast<char*>(ctx->halo_pool) + ch.off_flags);
    HaloWait w{};
    w.flag[0] = ctx->rank > 0 ? f + 0 : nullptr;
    w.flag[1] = ctx->rank < ctx->nranks - 1 ? f + 1 : nullptr;
    w.epoch = (unsigned)E;
    return w;
}

tpmg_status exchange_p2p(tpmg_ctx* ctx, tpmg_ctx::Chan& ch, int c, const double* x)
{
    (void)c;
    int E = 0;
    TRY(p2p_begin(ctx, ch, x, &E));
    return p2p_finish(ctx, ch, E);
}

// Fused push for a producer kernel about to write `out` (a field of channel c that will
// be read with its halo next): returns the remote destinations to hand to the kernel
// (empty when halos are not device-initiated); publish_pushed() follows the launch.  A
// pending push of the channel is waited for first, so epochs stay in order.
tpmg_status fused_push(tpmg_ctx* ctx, int c, const double* out, HaloPush* hp)
{
    *hp = HaloPush{};
    if (ctx->nranks == 1 || !ctx->p2p || ctx->halo_off || !ctx->fused_push) return TPMG_OK;
    tpmg_ctx::Chan& ch = ctx->chans[c];
    if (ch.pushed) {
        ch.pushed = nullptr;
        TRY(wait_epoch(ctx, ch, ch.epoch));
    }
    const int E = ++ch.epoch;
    *hp = push_desc(ctx, ch, E);
    ch.pushed = out;
    ch.publish = true;
    return TPMG_OK;
}

// After the producer kernel of a fused push: publish its epoch.
tpmg_status publish_pushed(tpmg_ctx* ctx, int c)
{
    if (ctx->nranks == 1 || c >= (int)ctx->chans.size()) return TPMG_OK;
    tpmg_ctx::Chan& ch = ctx->chans[c];
    if (!ch.publish) return TPMG_OK;
    ch.publish = false;
    return publish_epoch(ctx, ch, ch.epoch);
}

// A public call must not trust buffer identities from an earlier call (the caller may
// have refilled or reallocated a buffer at the same address): pending fused pushes stay
// pending (they are still waited for, in order) but never stand in for an exchange.
const double* const kPendingOnly = reinterpret_cast<const double*>(alignof(double));
void begin_call(tpmg_ctx* ctx)
{
    for (auto& ch : ctx->chans)
        if (ch.pushed) ch.pushed = kPendingOnly;
}

// Fill the current halo slabs of channel c (a level, or the CG z channel) from the
// neighbours' boundary rows of x (nranks > 1), in stream order on the context stream.
tpmg_status exchange_chan(tpmg_ctx* ctx, int c, const double* x)
{
    if (ctx->nranks == 1) return TPMG_OK;
    if (ctx->halo_off) return TPMG_OK;   // TPMG_HALO=off: timing experiments only (wrong results)
    tpmg_ctx::Chan& ch = ctx->chans[c];
    if (ctx->p2p) return exchange_p2p(ctx, ch, c, x);
    return exchange_on(ctx, ctx->stream, ctx->comm, ch.plane, ch.nyl, x, *ch.cur_lo, *ch.cur_hi);
}

tpmg_status exchange(tpmg_ctx* ctx, int level, const double* x) { return exchange_chan(ctx, level, x); }

// Start the exchange on the halo stream once everything enqueued so far on the
// context stream is done; finish_async_exchange() makes the context stream wait for it.
tpmg_status start_async_exchange(tpmg_ctx* ctx, int level, const double* x, double* lo, double* hi)
{
    LevelData& L = ctx->lv[level];
    CUDA_TRY(ctx, cudaEventRecord(ctx->ev_ready, ctx->stream));
    CUDA_TRY(ctx, cudaStreamWaitEvent(ctx->comm_stream, ctx->ev_ready, 0));
    TRY(exchange_on(ctx, ctx->comm_stream, ctx->comm_halo, L.plane(), L.lc.ny, x, lo, hi));
    CUDA_TRY(ctx, cudaEventRecord(ctx->ev_halo, ctx->comm_stream));
    return TPMG_OK;
}

tpmg_status finish_async_exchange(tpmg_ctx* ctx)
{
    CUDA_TRY(ctx, cudaStreamWaitEvent(ctx->stream, ctx->ev_halo, 0));
    return TPMG_OK;
}

HaloField halo_of(tpmg_ctx* ctx, int level, const double* x)
{
    LevelData& L = ctx->lv[level];
    return HaloField{x, ctx->rank > 0 ? L.slab_lo : nullptr, ctx->rank < ctx->nranks - 1 ? L.slab_hi : nullptr};
}

// Exchange x's halo into the level slabs and return the halo'd view.
tpmg_status halo(tpmg_ctx* ctx, int level, const double* x, HaloField* out)
{
    TRY(exchange(ctx, level, x));
    *out = halo_of(ctx, level, x);
    return TPMG_OK;
}

// Global sum of n device doubles over the ranks, in place on the context stream:
// device-initiated over NVLink (k_allreduce_p2p: the GPUs store their values into each
// other's pools and wait on epoch flags, no host and no NCCL kernel) when the P2P pools are
// mapped, else ncclAllReduce.
tpmg_status allreduce(tpmg_ctx* ctx, double* d, int n)
{
    if (ctx->nranks == 1) return TPMG_OK;
    if (ctx->p2p_reduce && n <= 4) {
        CUDA_TRY(ctx, launch_allreduce_p2p(launcher(ctx), d, n, ctx->red, ++ctx->red_epoch));
    } else {
        NCCL_TRY(ctx, ncclAllReduce(d, d, n, ncclDouble, ncclSum, ctx->comm, ctx->stream));
    }
    ++ctx->stats.allreduces;
    return TPMG_OK;
}

// Copy n device doubles to the pinned host buffer and wait.
tpmg_status fetch(tpmg_ctx* ctx, const double* d, int n)
{
    CUDA_TRY(ctx, cudaMemcpyAsync(ctx->h_pinned, d, sizeof(double) * n, cudaMemcpyDeviceToHost, ctx->stream));
    CUDA_TRY(ctx, cudaStreamSynchronize(ctx->stream));
    return TPMG_OK;
}

// ------------------------------------------------------------------ kernels (thin wrappers)

LineArgs line_args(tpmg_ctx* ctx, int level)
{
    LineArgs a{};
    a.L = ctx->lv[level].lc;
    a.rho = ctx->p.rho;
    a.scale = 1.0;
    a.ratio = DevRatio{nullptr, -1, -1};
    a.red = ReduceSlot{ctx->d_partials, ctx->d_ticket, nullptr, 0};
    a.skip = ctx->skip;
    a.dbg = ctx->dbg;
    a.band_w = ctx->band_w;
    a.l2hint = ctx->l2hint;
    a.cgdir_ctas = ctx->cgdir_ctas;
    a.im = (ctx->lv[level].lc.gen >= 2 && ctx->lv[level].im_ok) ? ctx->lv[level].d_im : nullptr;
    return a;
}

// ------------------------------------------------------------------ profiling

cudaEvent_t prof_event(tpmg_ctx* ctx)
{
    if (!ctx->prof_pool.empty()) {
        cudaEvent_t e = ctx->prof_pool.back();
        ctx->prof_pool.pop_back();
        return e;
    }
    cudaEvent_t e = nullptr;
    cudaEventCreate(&e);
    return e;
}

// Bracket one kernel launch (class cls, `cells` grid cells) with events when profiling.
struct ProfScope {
    tpmg_ctx* ctx;
    int cls;
    double cells;
    cudaEvent_t a = nullptr;
    ProfScope(tpmg_ctx* c, int k, double n) : ctx(c), cls(k), cells(n)
    {
        if (ctx->prof_on && ((ctx->prof_mask >> cls) & 1u)) {
            a = prof_event(ctx);
            cudaEventRecord(a, ctx->stream);
        }
    }
    ~ProfScope()
    {
        if (a) {
            cudaEvent_t b = prof_event(ctx);
            cudaEventRecord(b, ctx->stream);
            ctx->prof_pending.push_back({cls, cells, a, b, ctx->skip});
        }
    }
};

// Fold the pending event pairs into the per-class totals.  Launches the solver's run-ahead
// enqueued past convergence returned at once on the device (their skip flag was set):
// they are dropped, so the totals count only launches that did the work.  Called before
// the flags are reset (ensure_flags) and by tpmg_profile_read.
tpmg_status prof_collect(tpmg_ctx* ctx)
{
    if (ctx->prof_pending.empty()) return TPMG_OK;
    CUDA_TRY(ctx, cudaStreamSynchronize(ctx->stream));
    std::vector<int> flags;
    if (ctx->d_flags && ctx->flags_cap > 0) {
        flags.resize(ctx->flags_cap);
        CUDA_TRY(ctx, cudaMemcpy(flags.data(), ctx->d_flags, sizeof(int) * flags.size(), cudaMemcpyDeviceToHost));
    }
    for (auto& r : ctx->prof_pending) {
        bool skipped = false;
        if (r.skip && !flags.empty()) {
            const ptrdiff_t q = r.skip - ctx->d_flags;
            skipped = q >= 0 && q < (ptrdiff_t)flags.size() && flags[q] != 0;
        }
        if (!skipped) {
            float ms = 0;
            CUDA_TRY(ctx, cudaEventElapsedTime(&ms, r.a, r.b));
            ctx->prof_launches[r.cls] += 1;
            ctx->prof_ms[r.cls] += ms;
            ctx->prof_cells[r.cls] += r.cells;
            if (ctx->prof_detail) {   // per (class, cells of the launch) = per level
                auto& d = ctx->prof_by_size[std::make_pair(r.cls, r.cells)];
                d.first += 1;
                d.second += ms;
            }
        }
        ctx->prof_pool.push_back(r.a);
        ctx->prof_pool.push_back(r.b);
    }
    ctx->prof_pending.clear();
    return TPMG_OK;
}

double level_cells(const LevelConst& l) { return (double)l.nx * (double)l.ny * (double)l.nz; }

// ------------------------------------------------------------------ TMA descriptors

PFN_cuTensorMapEncodeTiled_v12000 tensor_map_encoder()
{
    static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
    static bool tried = false;
    if (!tried) {
        tried = true;
        cudaDriverEntryPointQueryResult q;
        void* p = nullptr;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
    }
    return fn;
}

// 3-D tiled map over an fp64 field [ny][nz][nx] (x fastest) with box (bx, KB, by).
bool tensor_map(tpmg_ctx* ctx, const double* base, int64_t nx, int nz, int64_t ny, int bx, int by, CUtensorMap* out,
                int bz = kStageK)
{
    auto key = std::make_tuple((uintptr_t)base, nx, nz, ny, bx, by * 1000 + bz);
    auto it = ctx->tmaps.find(key);
    if (it != ctx->tmaps.end()) {
        *out = it->second;
        return true;
    }
    auto enc = tensor_map_encoder();
    if (!enc) return false;
    cuuint64_t dims[3] = {(cuuint64_t)nx, (cuuint64_t)nz, (cuuint64_t)ny};
    cuuint64_t strides[2] = {(cuuint64_t)nx * 8, (cuuint64_t)nx * (cuuint64_t)nz * 8};
    cuuint32_t box[3] = {(cuuint32_t)bx, (cuuint32_t)bz, (cuuint32_t)by};
    cuuint32_t estr[3] = {1, 1, 1};
    CUtensorMap m;
    CUresult r = enc(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, const_cast<double*>(base), dims, strides, box, estr,
                     CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, (CUtensorMapL2promotion)ctx->tma_promo,
                     CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) return false;
    if (ctx->tmaps.size() > 4096) ctx->tmaps.clear();
    ctx->tmaps.emplace(key, m);
    *out = m;
    return true;
}

void mode_fields(int mode, int* nh, int* np)
{
    static const int NH[10] = {1, 1, 0, 1, 2, 1, 1, 2, 1, 1}, NP[10] = {0, 1, 1, 1, 0, 2, 1, 1, 1, 3};
    *nh = NH[mode];
    *np = NP[mode];
}

// Fill a.tma for the TMA loader; falls back to cp.async when a field cannot be
// described (odd nx: the row stride is not a multiple of 16 bytes; misaligned).
void fill_tma(tpmg_ctx* ctx, int mode, LineArgs& a)
{
    a.use_tma = 0;
    if (!ctx->use_tma) return;
    const int64_t nx = a.L.nx, ny = a.L.ny;
    const int nz = a.L.nz;
    if (nx % 2) return;
    const int TY = line_tile_rows(mode, nz, a.L.gen, ctx->tmem, nx);
    int nh, np;
    mode_fields(mode, &nh, &np);
    const HaloField* H[2] = {&a.h0, &a.h1};
    const double* Q[3] = {a.q0, a.q1, a.q2};
    auto aligned = [](const void* p) { return ((uintptr_t)p & 15) == 0; };
    for (int f = 0; f < nh; ++f) {
        TmaHalo& M = a.tma.h[f];
        const HaloField& hf = *H[f];
        if (!hf.base || !aligned(hf.base)) return;
        if (!tensor_map(ctx, hf.base, nx, nz, ny, kTileX + 4, TY + 2, &M.main)) return;
        if (!tensor_map(ctx, hf.base, nx, nz, ny, kTileX + 4, 1, &M.row)) return;
        M.has_lo = hf.lo != nullptr;
        M.has_hi = hf.hi != nullptr;
        if (hf.lo && (!aligned(hf.lo) || !tensor_map(ctx, hf.lo, nx, nz, 1, kTileX + 4, 1, &M.lo))) return;
        if (hf.hi && (!aligned(hf.hi) || !tensor_map(ctx, hf.hi, nx, nz, 1, kTileX + 4, 1, &M.hi))) return;
        M.has_m1 = (hf.lo || hf.hi) && tensor_map(ctx, hf.base, nx, nz, ny, kTileX + 4, TY + 1, &M.m1) ? 1 : 0;
    }
    for (int f = 0; f < np; ++f) {
        if (!Q[f] || !aligned(Q[f])) return;
        if (!tensor_map(ctx, Q[f], nx, nz, ny, kTileX, TY, &a.tma.q[f])) return;
    }
    // the precomputed pivots of the Thomas modes travel as plain field np
    const bool thomas = mode == MODE_PREC || mode == MODE_SMOOTH || is_cgprec(mode);
    if (thomas && a.im && (!aligned(a.im) || !tensor_map(ctx, a.im, nx, nz, ny, kTileX, TY, &a.tma.q[np]))) a.im = nullptr;
    if (!thomas) a.im = nullptr;
    a.use_tma = 1;
    // TMA stores of the TMEM CG preconditioner (TPMG_TMA_STORE=1): r, u in 4-row boxes, z in rows
    a.tst = 0;
    if (mode == MODE_CGPREC && ctx->tma_store && ctx->tmem && !a.L.gen && TY == 4 && nz % kStageK == 0 &&
        nz >= 2 * kStageK && nz <= 128 && !a.push.dst_lo && !a.push.dst_hi && a.out0 && a.out1 && a.out2 &&
        aligned(a.out0) && aligned(a.out1) && aligned(a.out2) &&
        tensor_map(ctx, a.out0, nx, nz, ny, kTileX, 4, &a.tma.o[0]) &&
        tensor_map(ctx, a.out1, nx, nz, ny, kTileX, 4, &a.tma.o[1]) &&
        tensor_map(ctx, a.out2, nx, nz, ny, kTileX, 1, &a.tma.o[2]))
        a.tst = 1;
}

// The level whose constants a LineArgs carries (by its table pointer).
int level_of(tpmg_ctx* ctx, const LevelConst& lc)
{
    for (int l = 1; l <= ctx->L; ++l)
        if (ctx->lv[l].lc.tab == lc.tab) return l;
    return ctx->L;
}

// TMA descriptors for the k-split kernel (boxes of ksplit_boxes()): a halo'd field
// gets a (TY+2)-row box, a one-row box and one-row slab boxes (strip boundaries).
bool ksplit_halo_maps(tpmg_ctx* ctx, const HaloField& hf, int64_t nx, int nz, int64_t ny, int bx, int rows, int depth,
                      TmaHalo& M)
{
    auto aligned = [](const void* p) { return ((uintptr_t)p & 15) == 0; };
    if (!hf.base || !aligned(hf.base)) return false;
    if (!tensor_map(ctx, hf.base, nx, nz, ny, bx, rows, &M.main, depth)) return false;
    if (!tensor_map(ctx, hf.base, nx, nz, ny, bx, 1, &M.row, depth)) return false;
    M.has_lo = hf.lo != nullptr;
    M.has_hi = hf.hi != nullptr;
    if (hf.lo && (!aligned(hf.lo) || !tensor_map(ctx, hf.lo, nx, nz, 1, bx, 1, &M.lo, depth))) return false;
    if (hf.hi && (!aligned(hf.hi) || !tensor_map(ctx, hf.hi, nx, nz, 1, bx, 1, &M.hi, depth))) return false;
    M.has_m1 = 0;
    if ((hf.lo || hf.hi) && rows > 2) M.has_m1 = tensor_map(ctx, hf.base, nx, nz, ny, bx, rows - 1, &M.m1, depth) ? 1 : 0;
    return true;
}

// k-split configuration of a launch: the context's, or (TPMG_KSPLIT_COARSE=c) config c on the
// coarse levels whose 4 x 4 tiles do not fill the SMs
int ksplit_cfg_of(tpmg_ctx* ctx, const LevelConst& lc)
{
    if (ctx->ksplit_cfg_coarse >= 0) {
        const int64_t tiles = ((lc.nx + kTileX - 1) / kTileX) * ((lc.ny + 3) / 4);
        if (tiles < ctx->num_sms) return ctx->ksplit_cfg_coarse;
    }
    return ctx->ksplit_cfg;
}

bool fill_tma_ksplit(tpmg_ctx* ctx, int mode, LineArgs& a)
{
    const int64_t nx = a.L.nx, ny = a.L.ny;
    const int nz = a.L.nz;
    const KsplitBoxes b = ksplit_boxes(mode, ksplit_cfg_of(ctx, a.L));
    if (mode == MODE_SMOOTH || mode == MODE_RESTRICT || mode == MODE_SMOOTH_PROLONG || mode == MODE_CGPREC)
        if (!ksplit_halo_maps(ctx, a.h0, nx, nz, ny, b.hx, b.ty + 2, b.depth, a.tma.h[0])) return false;
    if (mode == MODE_SMOOTH_PROLONG)
        if (!ksplit_halo_maps(ctx, a.h1, nx / 2, nz, ny / 2, b.hxc, b.ty / 2 + 2, b.depth, a.tma.h[1])) return false;
    if (!a.q0 || ((uintptr_t)a.q0 & 15)) return false;
    if (!tensor_map(ctx, a.q0, nx, nz, ny, kTileX, b.ty, &a.tma.q[0], b.kb)) return false;
    if (mode == MODE_CGPREC) {   // u, the second plain input
        if (!a.q1 || ((uintptr_t)a.q1 & 15)) return false;
        if (!tensor_map(ctx, a.q1, nx, nz, ny, kTileX, b.ty, &a.tma.q[1], b.kb)) return false;
    }
    a.use_tma = 1;
    return true;
}

bool ksplit_usable(tpmg_ctx* ctx, int mode, const LevelConst& lc)
{
    // general vertical profiles: the k-split smoother / preconditioner / restriction only
    if (lc.gen && (mode == MODE_SMOOTH_PROLONG || mode == MODE_CGPREC)) return false;
    if (mode == MODE_CGPREC_D || mode == MODE_CGPREC_P) return false;   // one-thread-per-column kernel only
    // per-column fields: the one-thread-per-column kernel (per-column pivots; a k-split
    // residual->restriction with the face-weighted stencil measured slower, r2ad: 703 vs 642 us)
    if (lc.gen == 2) return false;
    // the k-split CG preconditioner is opt-in (TPMG_KSPLIT_CG=1): measured 4% slower per CG
    // iteration than the one-thread-per-column kernel at 1024^2 x 128
    if (mode == MODE_CGPREC && !ctx->ksplit_cg) return false;
    return ctx->use_tma && ctx->ksplit_cfg >= 0 && ksplit_supported(mode, lc.nz, (int)lc.nx);
}

// Tile rows of the kernel run_line will launch for this mode and level.
int launch_rows(tpmg_ctx* ctx, int mode, const LevelConst& lc)
{
    return ksplit_usable(ctx, mode, lc) ? ksplit_boxes(mode, ksplit_cfg_of(ctx, lc)).ty
                                        : line_tile_rows(mode, lc.nz, lc.gen, ctx->tmem && ctx->use_tma, lc.nx);
}

// Fraction of the level's cells a launch covers (interior / boundary tile rows).
double part_cells(tpmg_ctx* ctx, int mode, const LineArgs& a)
{
    const double all = level_cells(a.L);
    if (a.part == PART_ALL || a.L.ny <= 0) return all;
    const int TY = launch_rows(ctx, mode, a.L);
    const int nty = (int)((a.L.ny + TY - 1) / TY);
    const double rows = (a.part == PART_INTERIOR) ? (double)(nty - 2) * TY : (double)a.L.ny - (double)(nty - 2) * TY;
    return all * rows / (double)a.L.ny;
}

tpmg_status run_line(tpmg_ctx* ctx, int mode, const LineArgs& a0)
{
    LineArgs a = a0;
    if (ksplit_usable(ctx, mode, a.L) && fill_tma_ksplit(ctx, mode, a)) {
        ProfScope ps(ctx, mode == MODE_SMOOTH_PROLONG ? TPMG_K_SMOOTH_PROLONG : mode, part_cells(ctx, mode, a));
        const KTables& kt = ctx->lv[level_of(ctx, a.L)].ktab;
        CUDA_TRY(ctx, launch_line_ksplit(launcher(ctx), mode, ksplit_cfg_of(ctx, a.L), a, kt));
        if (ctx->sync_debug) {
            cudaError_t e = cudaStreamSynchronize(ctx->stream);
            if (e != cudaSuccess)
                return fail(ctx, TPMG_E_CUDA, "k-split kernel mode %d (nx=%lld ny=%lld nz=%d): %s", mode,
                            (long long)a.L.nx, (long long)a.L.ny, a.L.nz, cudaGetErrorString(e));
        }
        return TPMG_OK;
    }
    if (mode == MODE_SMOOTH_PROLONG) return fail(ctx, TPMG_E_PARAM, "fused prolongation-smooth needs the k-split kernel");
    a = a0;
    fill_tma(ctx, mode, a);
    // modes 0..5 = TPMG_K_0..5; the paired-u CG variants count as CG preconditioning with their
    // own bytes expressed in units of MODE_CGPREC's 48 B per cell (32 and 56 B)
    const int pcls = mode == MODE_RESTRICT ? TPMG_K_RESIDUAL_RESTRICT : is_cgprec(mode) ? TPMG_K_CG_PRECONDITION : mode;
    const double pscale = mode == MODE_CGPREC_D ? 32.0 / 48.0 : mode == MODE_CGPREC_P ? 56.0 / 48.0 : 1.0;
    ProfScope ps(ctx, pcls, part_cells(ctx, mode, a) * pscale);
    CUDA_TRY(ctx, launch_line(launcher(ctx), mode, a));
    if (ctx->sync_debug) {
        cudaError_t e = cudaStreamSynchronize(ctx->stream);
        if (e != cudaSuccess)
            return fail(ctx, TPMG_E_CUDA, "line kernel mode %d (%s loader, nx=%lld ny=%lld nz=%d): %s", mode,
                        a.use_tma ? "TMA" : "cp.async", (long long)a.L.nx, (long long)a.L.ny, a.L.nz,
                        cudaGetErrorString(e));
    }
    return TPMG_OK;
}

// A line kernel whose halo'd input x needs an exchange first (channel chan, default the
// level's).  With several ranks the interior tile rows (which read no halo row) run while
// the halo is in flight and the boundary tile rows follow once it has arrived:
//   P2P (default): push x's boundary rows to the neighbours + publish the epoch, interior
//     launch, stream wait for the neighbours' epoch, boundary launch;
//   NCCL (TPMG_HALO=nccl with TPMG_OVERLAP=1): the exchange on the halo stream, leaving
//     reserve_sms SMs to NCCL during the interior launch.
// pre_boundary(a) (optional) runs between the halo's arrival and the boundary launch (e.g.
// the CG p-halo update) and may refresh a's halo views.  TPMG_OVERLAP=0 (or a fused push of
// the output) runs one launch after the exchange.
template <typename PreBoundary>
tpmg_status run_line_halo(tpmg_ctx* ctx, int level, int mode, LineArgs a, const double* x, double* lo, double* hi,
                          PreBoundary pre_boundary, const double* push_out = nullptr, int chan = -1,
                          bool overlap = true)
{
    if (chan < 0) chan = level;
    if (ctx->nranks == 1) {
        TRY(pre_boundary(a));
        return run_line(ctx, mode, a);
    }
    const LevelConst& lc = ctx->lv[level].lc;
    const int TY = launch_rows(ctx, mode, lc);
    const int nty = (int)((lc.ny + TY - 1) / TY);
    const bool fused_out = push_out && ctx->fused_push;
    const bool hw_ok = ksplit_usable(ctx, mode, lc) ? ksplit_halo_wait(mode, ksplit_cfg_of(ctx, lc), lc.gen)
                                                    : line_halo_wait(mode, lc.nz, lc.gen, ctx->use_tma, ctx->tmem);
    if (ctx->p2p && ctx->overlap && overlap && !ctx->halo_off && !fused_out && nty >= 3 && hw_ok) {
        // ONE launch: its CTAs walk the interior tile rows first; the loader of a strip-
        // boundary tile row waits in the kernel (ld.acquire.sys on my pool's epoch flag) for
        // the neighbour's rows, which travel while the interior is computed
        tpmg_ctx::Chan& ch = ctx->chans[chan];
        int E = 0;
        TRY(p2p_begin(ctx, ch, x, &E));
        if (a.h0.base == x) a.h0 = halo_epoch_view(ctx, ch, x, E);
        if (E) a.hw = halo_wait_of(ctx, ch, E);
        TRY(run_line(ctx, mode, a));
        TRY(p2p_finish_waited(ctx, ch, E));   // stream order for the channel's next push (the kernel already waited)
        return pre_boundary(a);
    }
    if (!ctx->overlap_nccl || ctx->p2p || nty < 3) {
        TRY(exchange_chan(ctx, chan, x));
        if (a.h0.base == x && chan == level) a.h0 = halo_of(ctx, level, x);   // P2P: the current slab buffer alternates
        TRY(pre_boundary(a));
        if (push_out) TRY(fused_push(ctx, level, push_out, &a.push));   // after the input's exchange
        TRY(run_line(ctx, mode, a));
        return push_out ? publish_pushed(ctx, level) : TPMG_OK;
    }
    TRY(start_async_exchange(ctx, level, x, lo, hi));
    a.part = PART_INTERIOR;
    ctx->cur_reserve = ctx->reserve_sms;
    tpmg_status st = run_line(ctx, mode, a);
    ctx->cur_reserve = 0;
    TRY(st);
    TRY(finish_async_exchange(ctx));
    TRY(pre_boundary(a));
    a.part = PART_BOUNDARY;
    a.red.accumulate = 1;
    return run_line(ctx, mode, a);
}

tpmg_status run_line_halo(tpmg_ctx* ctx, int level, int mode, const LineArgs& a, const double* x,
                          const double* push_out = nullptr)
{
    LevelData& L = ctx->lv[level];
    return run_line_halo(ctx, level, mode, a, x, L.slab_lo, L.slab_hi, [](LineArgs&) { return TPMG_OK; }, push_out);
}

// out = u + rho M^-1 (f - A u) (out-of-place), optional sum r^2 into result
tpmg_status smooth_once(tpmg_ctx* ctx, int level, const double* u, const double* f, double* out,
                        double* result)
{
    LineArgs a = line_args(ctx, level);
    a.h0 = halo_of(ctx, level, u);
    a.q0 = f;
    a.out0 = out;
    a.red.result = result;
    return run_line_halo(ctx, level, MODE_SMOOTH, a, u, /*push_out=*/out);   // out is read halo'd next
}

// ------------------------------------------------------------------ multigrid

tpmg_status mg_alloc(tpmg_ctx* ctx)
{
    if (ctx->mg_ready) return TPMG_OK;
    for (int l = 1; l <= ctx->L; ++l) {
        LevelData& L = ctx->lv[l];
        if (l < ctx->L) {
            TRY(dev_alloc(ctx, &L.u[0], L.n()));
            TRY(dev_alloc(ctx, &L.f, L.n()));
        }
        TRY(dev_alloc(ctx, &L.u[1], L.n()));
    }
    ctx->mg_ready = true;
    return TPMG_OK;
}

// Kernel RestrictSmooth preceded by the fine residual:
// f^(l) = R (f^(l+1) - A u^(l+1)), u^(l) = rho M^-1 f^(l)   (zero initial guess)
tpmg_status mg_restrict_smooth(tpmg_ctx* ctx, int l)
{
    LevelData& F = ctx->lv[l + 1];
    LevelData& Cc = ctx->lv[l];
    {
        LineArgs r = line_args(ctx, l + 1);
        r.h0 = halo_of(ctx, l + 1, F.u[F.cur]);
        r.q0 = F.f;
        r.out0 = Cc.f;
        TRY(run_line_halo(ctx, l + 1, MODE_RESTRICT, r, F.u[F.cur]));
    }
    LineArgs a = line_args(ctx, l);
    a.q0 = Cc.f;
    a.out0 = Cc.u[0];
    a.scale = ctx->p.rho;
    Cc.cur = 0;
    TRY(fused_push(ctx, l, Cc.u[0], &a.push));   // u_c is read halo'd next (restriction / smooth)
    TRY(run_line(ctx, MODE_PREC, a));
    return publish_pushed(ctx, l);
}

tpmg_status mg_smooth(tpmg_ctx* ctx, int l, double* result = nullptr)
{
    LevelData& L = ctx->lv[l];
    TRY(smooth_once(ctx, l, L.u[L.cur], L.f, L.u[1 - L.cur], result));
    L.cur ^= 1;
    return TPMG_OK;
}

// u^(l+1) += P u^(l) with the coarse halo exchange overlapped (interior coarse rows first).
tpmg_status prolong_overlapped(tpmg_ctx* ctx, int lc_)
{
    LevelData& Cc = ctx->lv[lc_];
    LevelData& F = ctx->lv[lc_ + 1];
    const HaloField uc = halo_of(ctx, lc_, Cc.u[Cc.cur]);
    const double cells = level_cells(F.lc);
    const double fb = Cc.lc.ny > 0 ? 2.0 / (double)Cc.lc.ny : 1.0;   // boundary coarse rows' share
    if (ctx->nranks > 1 && ctx->p2p && ctx->overlap && !ctx->halo_off && !ctx->fused_push && Cc.lc.ny >= 3) {
        // P2P overlap in ONE launch: the blocks of the strip-boundary coarse rows go last and
        // wait in the kernel for the coarse halo rows, which travel meanwhile
        tpmg_ctx::Chan& ch = ctx->chans[lc_];
        int E = 0;
        TRY(p2p_begin(ctx, ch, Cc.u[Cc.cur], &E));
        const HaloField ucE = halo_epoch_view(ctx, ch, Cc.u[Cc.cur], E);
        const HaloWait hw = halo_wait_of(ctx, ch, E);
        {
            ProfScope ps(ctx, TPMG_K_PROLONG_ADD, cells);
            CUDA_TRY(ctx, launch_prolong_add(launcher(ctx), Cc.lc, F.lc, ucE, F.u[F.cur], ctx->skip, PART_ALL, nullptr,
                                             E ? &hw : nullptr));
        }
        return p2p_finish_waited(ctx, ch, E);
    }
    if (ctx->nranks == 1 || !ctx->overlap_nccl || ctx->p2p || Cc.lc.ny < 3) {
        TRY(exchange(ctx, lc_, Cc.u[Cc.cur]));
        const HaloField uc2 = halo_of(ctx, lc_, Cc.u[Cc.cur]);   // current slabs after the exchange
        HaloPush hp;
        TRY(fused_push(ctx, lc_ + 1, F.u[F.cur], &hp));            // u_f is read halo'd by the post-smooth
        ProfScope ps(ctx, TPMG_K_PROLONG_ADD, cells);
        CUDA_TRY(ctx, launch_prolong_add(launcher(ctx), Cc.lc, F.lc, uc2, F.u[F.cur], ctx->skip, PART_ALL, &hp));
        return publish_pushed(ctx, lc_ + 1);
    }
    TRY(start_async_exchange(ctx, lc_, Cc.u[Cc.cur], Cc.slab_lo, Cc.slab_hi));
    {
        ProfScope ps(ctx, TPMG_K_PROLONG_ADD, cells * (1.0 - fb));
        CUDA_TRY(ctx, launch_prolong_add(launcher(ctx), Cc.lc, F.lc, uc, F.u[F.cur], ctx->skip, PART_INTERIOR));
    }
    TRY(finish_async_exchange(ctx));
    ProfScope ps(ctx, TPMG_K_PROLONG_ADD, cells * fb);
    CUDA_TRY(ctx, launch_prolong_add(launcher(ctx), Cc.lc, F.lc, uc, F.u[F.cur], ctx->skip, PART_BOUNDARY));
    return TPMG_OK;
}

// Subroutine VCycle (alg:VCycle) with the readings [R5] of DESIGN.md.
// skip_pre: the first pre-smoothing step of level l has already been done (the MG
// solve fuses it with the convergence test of the previous cycle).
tpmg_status vcycle_rec(tpmg_ctx* ctx, int l, bool skip_pre = false)
{
    const tpmg_params& p = ctx->p;
    if (l == 1) {
        int s0 = 0;
        if (ctx->L > 1) {
            TRY(mg_restrict_smooth(ctx, 1));
            s0 = 1;
        }
        for (int s = s0; s < p.coarse_sweeps; ++s) TRY(mg_smooth(ctx, 1));
        return TPMG_OK;
    }
    if (l == ctx->L) {
        for (int s = skip_pre ? 1 : 0; s < p.pre; ++s) TRY(mg_smooth(ctx, l));
    } else {
        TRY(mg_restrict_smooth(ctx, l));
        for (int s = 1; s < p.pre; ++s) TRY(mg_smooth(ctx, l));
    }
    TRY(vcycle_rec(ctx, l - 1));
    LevelData& Cc = ctx->lv[l - 1];
    LevelData& F = ctx->lv[l];
    HaloField uc = halo_of(ctx, l - 1, Cc.u[Cc.cur]);
    (void)uc;
    const bool fuse = p.post >= 1 && ctx->fuse_prolong && p.boundary == TPMG_BC_GHOST_ZERO &&
                      ksplit_usable(ctx, MODE_SMOOTH_PROLONG, F.lc);   // fused form: zero coarse ghosts, flat box
    if (fuse) {
        TRY(exchange(ctx, l - 1, Cc.u[Cc.cur]));
        uc = halo_of(ctx, l - 1, Cc.u[Cc.cur]);
    }
    int s0 = 0;
    if (fuse) {
        // Prolongate fused with the first post-smooth: u' = S(u + P u_c) without storing
        // u + P u_c.  The halo of u is the one exchanged for the restriction (u has not
        // changed since), the coarse halo was just exchanged.
        LineArgs a = line_args(ctx, l);
        a.h0 = halo_of(ctx, l, F.u[F.cur]);
        a.h1 = uc;
        a.q0 = F.f;
        a.out0 = F.u[1 - F.cur];
        TRY(run_line(ctx, MODE_SMOOTH_PROLONG, a));
        F.cur ^= 1;
        s0 = 1;
    } else {
        TRY(prolong_overlapped(ctx, l - 1));
    }
    for (int s = s0; s < p.post; ++s) TRY(mg_smooth(ctx, l));
    return TPMG_OK;
}

// Bind the caller's fine-level u, f to the hierarchy.
void bind_fine(tpmg_ctx* ctx, double* u, const double* f)
{
    LevelData& F = ctx->lv[ctx->L];
    F.u[0] = u;
    F.f = const_cast<double*>(f);
    F.cur = 0;
}

// Copy the fine iterate back into the caller's u if it ended in the work buffer.
tpmg_status unbind_fine(tpmg_ctx* ctx)
{
    LevelData& F = ctx->lv[ctx->L];
    if (F.cur != 0) CUDA_TRY(ctx, launch_copy(launcher(ctx), F.u[0], F.u[1], (int64_t)F.n(), ctx->skip));
    F.cur = 0;
    return TPMG_OK;
}

// One V-cycle with the caller's fine-level u, f.  Leaves the result in u.
tpmg_status vcycle_fine(tpmg_ctx* ctx, double* u, const double* f)
{
    bind_fine(ctx, u, f);
    TRY(vcycle_rec(ctx, ctx->L));
    return unbind_fine(ctx);
}

// Global ||f - A u||^2 of the fine level (into d_scal[slot]).
tpmg_status fine_residual_norm2(tpmg_ctx* ctx, const double* u, const double* f, double* d_out)
{
    const int l = ctx->L;
    LineArgs a = line_args(ctx, l);
    TRY(halo(ctx, l, u, &a.h0));
    a.q0 = f;
    a.out0 = nullptr;
    a.red.result = d_out;
    TRY(run_line(ctx, MODE_RESID, a));
    return allreduce(ctx, d_out, 1);
}

tpmg_status ensure_scal(tpmg_ctx* ctx, int n)
{
    if (n <= ctx->scal_cap) return TPMG_OK;
    if (ctx->d_scal) cudaFree(ctx->d_scal);
    ctx->d_scal = nullptr;
    TRY(dev_alloc(ctx, &ctx->d_scal, (size_t)n));
    CUDA_TRY(ctx, cudaMemsetAsync(ctx->d_scal, 0, sizeof(double) * n, ctx->stream));
    ctx->scal_cap = n;
    return TPMG_OK;
}

tpmg_status ensure_flags(tpmg_ctx* ctx, int n)
{
    TRY(prof_collect(ctx));   // the pending profile records still refer to the old flags
    if (n > ctx->flags_cap) {
        if (ctx->d_flags) cudaFree(ctx->d_flags);
        if (ctx->h_flags) cudaFreeHost(ctx->h_flags);
        ctx->d_flags = nullptr;
        ctx->h_flags = nullptr;
        CUDA_TRY(ctx, cudaMalloc((void**)&ctx->d_flags, sizeof(int) * n));
        CUDA_TRY(ctx, cudaMallocHost((void**)&ctx->h_flags, sizeof(int) * n));
        CUDA_TRY(ctx, cudaHostGetDevicePointer((void**)&ctx->dh_flags, ctx->h_flags, 0));
        ctx->flags_cap = n;
    }
    for (auto& e : ctx->ev_it)
        if (!e) CUDA_TRY(ctx, cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    CUDA_TRY(ctx, cudaMemsetAsync(ctx->d_flags, 0, sizeof(int) * n, ctx->stream));
    return TPMG_OK;
}

// Copy flag[m] to the host ring and record its event.
// The check kernel stored flags[m] into the mapped pinned h_flags too; the event marks it.
tpmg_status post_flag(tpmg_ctx* ctx, int m)
{
    CUDA_TRY(ctx, cudaEventRecord(ctx->ev_it[m & 7], ctx->stream));
    return TPMG_OK;
}

tpmg_status wait_flag(tpmg_ctx* ctx, int m, int* code)
{
    CUDA_TRY(ctx, cudaEventSynchronize(ctx->ev_it[m & 7]));
    *code = ctx->h_flags[m];
    return TPMG_OK;
}

// Clears the run-ahead predicate on every exit path of a solve.
struct SkipGuard {
    tpmg_ctx* ctx;
    ~SkipGuard() { ctx->skip = nullptr; }
};

void result_init(tpmg_result* res)
{
    if (!res) return;
    res->iterations = 0;
    res->converged = 0;
    res->r0_norm = 0;
    res->rel_residual = 0;
    res->seconds = 0;
}

void record_hist(tpmg_result* res, int it, double v)
{
    if (res && res->history && it < res->history_cap) res->history[it] = v;
}

tpmg_status solve_mg_impl(tpmg_ctx* ctx, const double* f, double* u, double eps, int max_iter,
                          tpmg_result* res)
{
    TRY(mg_alloc(ctx));
    TRY(ensure_scal(ctx, 8 + max_iter + 2));
    const LevelData& F = ctx->lv[ctx->L];
    result_init(res);
    CUDA_TRY(ctx, cudaEventRecord(ctx->ev0, ctx->stream));
    CUDA_TRY(ctx, cudaMemsetAsync(u, 0, sizeof(double) * F.n(), ctx->stream));   // u_0 = 0 [R9]
    // ||r_0|| = ||f - A 0|| = ||f||
    {
        ProfScope ps(ctx, TPMG_K_DOT, (double)F.n());
        CUDA_TRY(ctx, launch_dot(launcher(ctx), f, f, (int64_t)F.n(), slot(ctx, ctx->d_scal)));
    }
    TRY(allreduce(ctx, ctx->d_scal, 1));
    TRY(fetch(ctx, ctx->d_scal, 1));
    const double r0 = std::sqrt(ctx->h_pinned[0]);
    record_hist(res, 0, r0);
    int it = 0;
    bool conv = (r0 == 0.0);
    double rel = conv ? 0.0 : 1.0;
    const bool fused_norm = ctx->L > 1 && ctx->p.pre >= 1;
    if (!fused_norm) {
        while (!conv && it < max_iter) {
            TRY(vcycle_fine(ctx, u, f));
            TRY(fine_residual_norm2(ctx, u, f, ctx->d_scal + 1));
            TRY(fetch(ctx, ctx->d_scal + 1, 1));
            const double rn = std::sqrt(ctx->h_pinned[0]);
            ++it;
            record_hist(res, it, rn);
            rel = rn / r0;
            if (!(rn == rn)) return fail(ctx, TPMG_E_BREAKDOWN, "NaN residual after V-cycle %d", it);
            if (rel < eps) conv = true;
        }
    } else if (!conv && max_iter > 0) {
        // The first fine pre-smooth of cycle n+1 also returns ||f - A u_n||^2 (its input's
        // residual): the convergence test of cycle n costs no extra pass over u and f.  The
        // pre-smooth writes the work buffer, so u_n is still in u when the test passes.
        // Run-ahead: the test is evaluated on the device (k_mg_check -> flags[n]); every
        // later kernel is predicated on it, so the host enqueues the next cycle before it
        // reads flags[n] and the GPU never waits for the host.
        const int LAG = 1;
        SkipGuard guard{ctx};
        TRY(ensure_flags(ctx, max_iter + 2));
        double* norms = ctx->d_scal + 8;          // norms[n] = ||f - A u_n||^2
        bind_fine(ctx, u, f);
        ctx->skip = nullptr;
        TRY(vcycle_rec(ctx, ctx->L));             // cycle 1 (u_0 = 0)
        TRY(unbind_fine(ctx));
        int checked = 0, stop_at = -1, code = 0;
        for (int n = 1; n <= max_iter && stop_at < 0; ++n) {
            ctx->skip = ctx->d_flags + (n - 1);
            bind_fine(ctx, u, f);
            TRY(mg_smooth(ctx, ctx->L, norms + n));
            TRY(allreduce(ctx, norms + n, 1));
            CUDA_TRY(ctx, launch_mg_check(launcher(ctx), norms + n, ctx->d_scal, n, eps, max_iter, ctx->d_flags,
                                          ctx->dh_flags));
            TRY(post_flag(ctx, n));
            ctx->skip = ctx->d_flags + n;
            if (n < max_iter) {                   // cycle n+1 (skipped on the device once flags[n] != 0)
                TRY(vcycle_rec(ctx, ctx->L, /*skip_pre=*/true));
                TRY(unbind_fine(ctx));
            }
            ctx->lv[ctx->L].cur = 0;
            while (checked < n - LAG + 1 && stop_at < 0) {
                ++checked;
                TRY(wait_flag(ctx, checked, &code));
                if (code) stop_at = checked;
            }
        }
        ctx->skip = nullptr;
        it = stop_at > 0 ? stop_at : max_iter;
        // history: one read of the norms
        CUDA_TRY(ctx, cudaStreamSynchronize(ctx->stream));
        std::vector<double> nh(it + 1);
        CUDA_TRY(ctx, cudaMemcpy(nh.data(), norms, sizeof(double) * (it + 1), cudaMemcpyDeviceToHost));
        for (int n = 1; n <= it; ++n) record_hist(res, n, std::sqrt(nh[n]));
        rel = std::sqrt(nh[it]) / r0;
        if (code == 3) return fail(ctx, TPMG_E_BREAKDOWN, "NaN residual after V-cycle %d", it);
        conv = (code == 1);
    }
    CUDA_TRY(ctx, cudaEventRecord(ctx->ev1, ctx->stream));
    CUDA_TRY(ctx, cudaEventSynchronize(ctx->ev1));
    float ms = 0;
    CUDA_TRY(ctx, cudaEventElapsedTime(&ms, ctx->ev0, ctx->ev1));
    if (res) {
        res->iterations = it;
        res->converged = conv ? 1 : 0;
        res->r0_norm = r0;
        res->rel_residual = rel;
        res->seconds = ms * 1e-3;
    }
    return TPMG_OK;
}

// ------------------------------------------------------------------ CG

tpmg_status cg_alloc(tpmg_ctx* ctx)
{
    if (ctx->cg_ready) return TPMG_OK;
    const LevelData& F = ctx->lv[ctx->L];
    TRY(dev_alloc(ctx, &ctx->cg_r, F.n()));
    TRY(dev_alloc(ctx, &ctx->cg_z, F.n()));
    TRY(dev_alloc(ctx, &ctx->cg_p[0], F.n()));
    TRY(dev_alloc(ctx, &ctx->cg_p[1], F.n()));
    if (ctx->nranks > 1) {
        for (int q = 0; q < 2; ++q) {
            TRY(dev_alloc(ctx, &ctx->cg_plo[q], F.plane()));
            TRY(dev_alloc(ctx, &ctx->cg_phi[q], F.plane()));
        }
    }
    ctx->cg_ready = true;
    return TPMG_OK;
}

// scalar slots of iteration n: sigma = 3n, ||r||^2 = 3n+1, zeta = <r, M^-1 r> = 3n+2
inline int S_SIGMA(int n) { return 3 * n; }
inline int S_RR(int n) { return 3 * n + 1; }
inline int S_ZETA(int n) { return 3 * n + 2; }

tpmg_status solve_cg_impl(tpmg_ctx* ctx, const double* f, double* u, double eps, int max_iter,
                          tpmg_result* res)
{
    TRY(cg_alloc(ctx));
    TRY(ensure_scal(ctx, 3 * (max_iter + 2)));
    const int l = ctx->L;
    const LevelData& F = ctx->lv[l];
    const size_t n = F.n(), plane = F.plane();
    result_init(res);
    CUDA_TRY(ctx, cudaEventRecord(ctx->ev0, ctx->stream));
    CUDA_TRY(ctx, cudaMemsetAsync(u, 0, sizeof(double) * n, ctx->stream));          // u_0 = 0 [R9]
    CUDA_TRY(ctx, cudaMemsetAsync(ctx->cg_p[0], 0, sizeof(double) * n, ctx->stream));
    if (ctx->nranks > 1) {
        CUDA_TRY(ctx, cudaMemsetAsync(ctx->cg_plo[0], 0, sizeof(double) * plane, ctx->stream));
        CUDA_TRY(ctx, cudaMemsetAsync(ctx->cg_phi[0], 0, sizeof(double) * plane, ctx->stream));
    }
    const bool has_lo = ctx->rank > 0, has_hi = ctx->rank < ctx->nranks - 1;
    // setup: r = f, z = M^-1 r, rr_0 = <r,r>, zeta_0 = <r,z>  (CGPREC with alpha = 0, p = 0)
    {
        LineArgs a = line_args(ctx, l);
        a.h0 = HaloField{ctx->cg_p[0], nullptr, nullptr};
        a.q0 = f;
        a.q1 = u;
        a.out0 = ctx->cg_r;
        a.out1 = u;
        a.out2 = ctx->cg_z;
        a.red.result = ctx->d_scal + S_RR(0);
        TRY(run_line(ctx, MODE_CGPREC, a));
        TRY(allreduce(ctx, ctx->d_scal + S_RR(0), 2));
        TRY(fetch(ctx, ctx->d_scal + S_RR(0), 2));
    }
    const double r0 = std::sqrt(ctx->h_pinned[0]);
    record_hist(res, 0, r0);
    int it = 0, cur = 0;
    bool conv = (r0 == 0.0);
    double rel = conv ? 0.0 : 1.0;
    if (!conv && !(ctx->h_pinned[1] > 0))
        return fail(ctx, TPMG_E_BREAKDOWN, "CG setup: <r, M^-1 r> = %g", ctx->h_pinned[1]);
    // Run-ahead: iteration m's convergence / breakdown test runs on the device
    // (k_cg_check -> flags[m]); iteration m+1's kernels are predicated on flags[m], so the
    // host enqueues LAG iterations ahead and the GPU never idles waiting for the host.
    const int LAG = 2;
    SkipGuard guard{ctx};
    TRY(ensure_flags(ctx, max_iter + 2));
    int checked = 0, stop_at = -1, code = 0, enq = 0;
    for (int m = 1; !conv && m <= max_iter && stop_at < 0; ++m) {
        ctx->skip = ctx->d_flags + (m - 1);
        // halo of z; the halo of p_old is local: p_halo <- z_halo + beta p_halo (same fma
        // as the neighbour's own rows), so only z crosses NVLink
        HaloField hz{ctx->cg_z, nullptr, nullptr}, hp{ctx->cg_p[cur], nullptr, nullptr};
        const DevRatio beta = (m == 1) ? DevRatio{ctx->d_scal, -1, -1}
                                       : DevRatio{ctx->d_scal, S_ZETA(m - 1), S_ZETA(m - 2)};
        if (ctx->nranks > 1) {
            hz = HaloField{ctx->cg_z, has_lo ? ctx->cg_zlo : nullptr, has_hi ? ctx->cg_zhi : nullptr};
            hp = HaloField{ctx->cg_p[cur], has_lo ? ctx->cg_plo[cur] : nullptr, has_hi ? ctx->cg_phi[cur] : nullptr};
        }
        // (Fused) direction kernel: p = z + beta p, sigma = <p, A p>.  Only z crosses NVLink;
        // the p halo is local: p_halo <- z_halo + beta p_halo (same fma as the neighbour's
        // own rows).  With several ranks the interior tile rows run while z's halo travels
        // (run_line_halo); the p-halo update and the boundary rows follow its arrival.
        {
            LineArgs a = line_args(ctx, l);
            a.h0 = hz;
            a.h1 = hp;
            a.out0 = ctx->cg_p[1 - cur];
            a.ratio = beta;
            a.red.result = ctx->d_scal + S_SIGMA(m);
            auto p_halo = [&](LineArgs& b) -> tpmg_status {
                if (ctx->nranks == 1) return TPMG_OK;
                hz = HaloField{ctx->cg_z, has_lo ? ctx->cg_zlo : nullptr, has_hi ? ctx->cg_zhi : nullptr};
                b.h0 = hz;   // the z slabs of this exchange's epoch
                CUDA_TRY(ctx, launch_cg_halo(launcher(ctx), has_lo ? ctx->cg_plo[1 - cur] : nullptr, hz.lo, hp.lo,
                                             has_hi ? ctx->cg_phi[1 - cur] : nullptr, hz.hi, hp.hi, (int64_t)plane,
                                             beta, ctx->skip));
                return TPMG_OK;
            };
            // (the in-kernel overlap measured 2.5% slower per CG iteration at N = 2, r2t: opt-in)
            TRY(run_line_halo(ctx, l, MODE_CGDIR, a, ctx->cg_z, ctx->cg_zlo, ctx->cg_zhi, p_halo, nullptr, l + 1,
                              ctx->overlap_cg));
            TRY(allreduce(ctx, ctx->d_scal + S_SIGMA(m), 1));
        }
        HaloField hpn{ctx->cg_p[1 - cur], nullptr, nullptr};
        if (ctx->nranks > 1)
            hpn = HaloField{ctx->cg_p[1 - cur], has_lo ? ctx->cg_plo[1 - cur] : nullptr,
                            has_hi ? ctx->cg_phi[1 - cur] : nullptr};
        // (Fused) preconditioner kernel: r -= alpha A p, u += alpha p, z = M^-1 r, ||r||^2, <r,z>.
        // Paired u updates (ctx->pair_u): odd iterations skip u, even ones add alpha_{m-1} p_{m-1}
        // + alpha_m p_m (p_{m-1} is still in the other direction buffer): 68 instead of 72 B per
        // cell per iteration; r, z and the sums -- the whole iteration -- are unchanged.
        {
            LineArgs a = line_args(ctx, l);
            a.h0 = hpn;
            a.q0 = ctx->cg_r;
            a.q1 = u;
            a.out0 = ctx->cg_r;
            a.out1 = u;
            a.out2 = ctx->cg_z;
            a.ratio = DevRatio{ctx->d_scal, S_ZETA(m - 1), S_SIGMA(m)};
            a.red.result = ctx->d_scal + S_RR(m);
            int mode = MODE_CGPREC;
            if (ctx->pair_u && (m & 1)) {
                mode = MODE_CGPREC_D;
                a.q1 = nullptr;
                a.out1 = nullptr;
            } else if (ctx->pair_u) {
                mode = MODE_CGPREC_P;
                a.q2 = ctx->cg_p[cur];   // p_{m-1}
                a.ratio2 = DevRatio{ctx->d_scal, S_ZETA(m - 2), S_SIGMA(m - 1)};
            }
            TRY(run_line(ctx, mode, a));   // z's halo: push kernel (fused measured no faster)
            TRY(allreduce(ctx, ctx->d_scal + S_RR(m), 2));
        }
        CUDA_TRY(ctx, launch_cg_check(launcher(ctx), ctx->d_scal, m, eps, ctx->d_flags, ctx->dh_flags));
        TRY(post_flag(ctx, m));
        enq = m;
        cur ^= 1;
        while (checked < m - LAG && stop_at < 0) {
            ++checked;
            TRY(wait_flag(ctx, checked, &code));
            if (code) stop_at = checked;
        }
    }
    while (stop_at < 0 && checked < enq) {
        ++checked;
        TRY(wait_flag(ctx, checked, &code));
        if (code) stop_at = checked;
    }
    ctx->skip = nullptr;
    if (!conv) {
        it = stop_at > 0 ? stop_at : max_iter;
        CUDA_TRY(ctx, cudaStreamSynchronize(ctx->stream));
        std::vector<double> sc(3 * (it + 1));
        CUDA_TRY(ctx, cudaMemcpy(sc.data(), ctx->d_scal, sizeof(double) * sc.size(), cudaMemcpyDeviceToHost));
        for (int m = 1; m <= it; ++m) record_hist(res, m, std::sqrt(sc[S_RR(m)]));
        rel = std::sqrt(sc[S_RR(it)]) / r0;
        if (code == 2) {
            const double sg = sc[S_SIGMA(it)];
            return fail(ctx, TPMG_E_BREAKDOWN, "CG iteration %d: %s = %g", it,
                        !(sg > 0) ? "<p, A p>" : "<r, M^-1 r>", !(sg > 0) ? sg : sc[S_ZETA(it)]);
        }
        if (code == 3) return fail(ctx, TPMG_E_BREAKDOWN, "CG iteration %d: NaN residual", it);
        conv = (code == 1);
    }
    if (ctx->pair_u && (it & 1)) {
        // the last iteration was odd: its step alpha_it p_it is still to be added to u
        CUDA_TRY(ctx, launch_cg_halo(launcher(ctx), u, u, ctx->cg_p[it & 1], nullptr, nullptr, nullptr, (int64_t)n,
                                     DevRatio{ctx->d_scal, S_ZETA(it - 1), S_SIGMA(it)}, nullptr));
    }
    CUDA_TRY(ctx, cudaEventRecord(ctx->ev1, ctx->stream));
    CUDA_TRY(ctx, cudaEventSynchronize(ctx->ev1));
    float ms = 0;
    CUDA_TRY(ctx, cudaEventElapsedTime(&ms, ctx->ev0, ctx->ev1));
    if (res) {
        res->iterations = it;
        res->converged = conv ? 1 : 0;
        res->r0_norm = r0;
        res->rel_residual = rel;
        res->seconds = ms * 1e-3;
    }
    return TPMG_OK;
}

// All ranks agree on a step's outcome: returns TPMG_OK on every rank only when `local` is OK
// on every rank (an allreduce over ctx->comm), so that no rank enters the next collective
// while another has bailed out (it would wait there forever).
tpmg_status agree(tpmg_ctx* ctx, tpmg_status local)
{
    int* d = nullptr;
    if (cudaMalloc((void**)&d, sizeof(int)) != cudaSuccess) return fail(ctx, TPMG_E_CUDA, "agree: cudaMalloc");
    const int mine = (local == TPMG_OK) ? 0 : 1;
    int any = 1;
    bool ok = cudaMemcpy(d, &mine, sizeof(int), cudaMemcpyHostToDevice) == cudaSuccess &&
              ncclAllReduce(d, d, 1, ncclInt32, ncclMax, ctx->comm, ctx->stream) == ncclSuccess &&
              cudaStreamSynchronize(ctx->stream) == cudaSuccess &&
              cudaMemcpy(&any, d, sizeof(int), cudaMemcpyDeviceToHost) == cudaSuccess;
    cudaFree(d);
    if (local != TPMG_OK) return local;
    if (!ok) return fail(ctx, TPMG_E_NCCL, "agree: allreduce of the step status failed");
    if (any) return fail(ctx, TPMG_E_NCCL, "another rank failed in the same collective step");
    return TPMG_OK;
}

// Halo channels and their pool (nranks > 1).  P2P mode (default): the pool is exported
// with cudaIpcGetMemHandle, the handles are all-gathered over NCCL together with each rank's
// host name and GPU PCI bus id, and each rank maps its two neighbours' pools; the exchanges
// then run as remote stores (exchange_p2p).  P2P is decided collectively: a rank whose
// neighbour is on another host, cannot be reached peer-to-peer, or whose pool cannot be
// mapped votes no, and then EVERY rank falls back to NCCL send/recv.
tpmg_status halo_setup(tpmg_ctx* ctx)
{
    const int L = ctx->L;
    ctx->chans.assign(L + 2, tpmg_ctx::Chan{});
    size_t off = 0;
    auto take = [&](size_t bytes) {
        const size_t o = off;
        off += (bytes + 255) & ~(size_t)255;
        return o;
    };
    for (int c = 1; c <= L + 1; ++c) {
        tpmg_ctx::Chan& ch = ctx->chans[c];
        const LevelData& lv = ctx->lv[c <= L ? c : L];
        ch.plane = lv.plane();
        ch.nyl = lv.lc.ny;
        for (int b = 0; b < 2; ++b) {
            ch.off_lo[b] = take(sizeof(double) * ch.plane);
            ch.off_hi[b] = take(sizeof(double) * ch.plane);
        }
        ch.off_flags = take(4 * sizeof(uint32_t));
    }
    ctx->off_red = take(sizeof(double) * 2 * kMaxP2PRanks * 4);
    ctx->off_redflags = take(sizeof(unsigned) * kMaxP2PRanks);
    const size_t off_pushdone = take(sizeof(unsigned));
    ctx->halo_pool_bytes = off;
    tpmg_status st = TPMG_OK;
    if (cudaMalloc(&ctx->halo_pool, off) != cudaSuccess || cudaMemset(ctx->halo_pool, 0, off) != cudaSuccess)
        st = fail(ctx, TPMG_E_CUDA, "halo pool: cudaMalloc/cudaMemset of %zu bytes", off);
    TRY(agree(ctx, st));
    char* base = static_cast<char*>(ctx->halo_pool);
    ctx->d_push_done = reinterpret_cast<unsigned*>(base + off_pushdone);
    for (int c = 1; c <= L + 1; ++c) {
        tpmg_ctx::Chan& ch = ctx->chans[c];
        for (int b = 0; b < 2; ++b) {
            ch.lo[b] = reinterpret_cast<double*>(base + ch.off_lo[b]);
            ch.hi[b] = reinterpret_cast<double*>(base + ch.off_hi[b]);
        }
        ch.cur_lo = (c <= L) ? &ctx->lv[c].slab_lo : &ctx->cg_zlo;
        ch.cur_hi = (c <= L) ? &ctx->lv[c].slab_hi : &ctx->cg_zhi;
        *ch.cur_lo = ch.lo[0];
        *ch.cur_hi = ch.hi[0];
    }
    const char* hm = std::getenv("TPMG_HALO");
    ctx->halo_off = hm && std::strcmp(hm, "off") == 0;
    const char* fpu = std::getenv("TPMG_FUSED_PUSH");
    ctx->fused_push = fpu && fpu[0] == '1';   // measured no faster than the push kernel
    // the environment and driver capabilities are the same on every rank of a job; the
    // per-neighbour checks below are voted on
    ctx->p2p = !(hm && std::strcmp(hm, "nccl") == 0) && stream_memops();
    if (!ctx->p2p) return TPMG_OK;
    struct PeerRec {
        cudaIpcMemHandle_t h;
        char host[64];
        char bus[32];
        int ok;   // this rank could export its pool
    };
    PeerRec mine{};
    mine.ok = cudaIpcGetMemHandle(&mine.h, ctx->halo_pool) == cudaSuccess &&
              cudaDeviceGetPCIBusId(mine.bus, sizeof mine.bus, ctx->device) == cudaSuccess;
    gethostname(mine.host, sizeof mine.host - 1);
    cudaGetLastError();
    const size_t hb = sizeof(PeerRec);
    std::vector<char> all(hb * ctx->nranks);
    {
        char* d_all = nullptr;
        CUDA_TRY(ctx, cudaMalloc((void**)&d_all, hb * ctx->nranks));
        CUDA_TRY(ctx, cudaMemcpy(d_all + hb * ctx->rank, &mine, hb, cudaMemcpyHostToDevice));
        NCCL_TRY(ctx, ncclAllGather(d_all + hb * ctx->rank, d_all, hb, ncclChar, ctx->comm, ctx->stream));
        CUDA_TRY(ctx, cudaStreamSynchronize(ctx->stream));
        CUDA_TRY(ctx, cudaMemcpy(all.data(), d_all, all.size(), cudaMemcpyDeviceToHost));
        cudaFree(d_all);
    }
    // every rank's pool is mapped (the neighbours' carry the halos, all of them the
    // allreduce slots); every peer must be on my host and reachable peer-to-peer
    int vote = mine.ok ? 1 : 0;
    ctx->peer_all.assign(ctx->nranks, nullptr);
    ctx->peer_all[ctx->rank] = static_cast<char*>(ctx->halo_pool);
    for (int q = 0; q < ctx->nranks && vote; ++q) {
        if (q == ctx->rank) continue;
        PeerRec r;
        std::memcpy(&r, all.data() + hb * q, hb);
        int dev_q = -1, can = 0;
        if (!r.ok || std::strncmp(r.host, mine.host, sizeof r.host) != 0 ||
            cudaDeviceGetByPCIBusId(&dev_q, r.bus) != cudaSuccess || dev_q == ctx->device ||
            cudaDeviceCanAccessPeer(&can, ctx->device, dev_q) != cudaSuccess || !can) {
            vote = 0;
            break;
        }
        void* p = nullptr;
        if (cudaIpcOpenMemHandle(&p, r.h, cudaIpcMemLazyEnablePeerAccess) != cudaSuccess) {
            vote = 0;
            break;
        }
        ctx->peer_all[q] = static_cast<char*>(p);
    }
    if (vote) {
        ctx->peer_pool[0] = ctx->rank > 0 ? ctx->peer_all[ctx->rank - 1] : nullptr;
        ctx->peer_pool[1] = ctx->rank < ctx->nranks - 1 ? ctx->peer_all[ctx->rank + 1] : nullptr;
    }
    cudaGetLastError();   // a failed probe above must not stick to the next call
    // collective decision: P2P only when every rank voted yes
    {
        int* d = nullptr;
        int all_ok = 0;
        CUDA_TRY(ctx, cudaMalloc((void**)&d, sizeof(int)));
        CUDA_TRY(ctx, cudaMemcpy(d, &vote, sizeof(int), cudaMemcpyHostToDevice));
        NCCL_TRY(ctx, ncclAllReduce(d, d, 1, ncclInt32, ncclMin, ctx->comm, ctx->stream));
        CUDA_TRY(ctx, cudaStreamSynchronize(ctx->stream));
        CUDA_TRY(ctx, cudaMemcpy(&all_ok, d, sizeof(int), cudaMemcpyDeviceToHost));
        cudaFree(d);
        if (!all_ok) {
            for (int q = 0; q < (int)ctx->peer_all.size(); ++q)
                if (q != ctx->rank && ctx->peer_all[q]) cudaIpcCloseMemHandle(ctx->peer_all[q]);
            ctx->peer_all.clear();
            ctx->peer_pool[0] = ctx->peer_pool[1] = nullptr;
            ctx->p2p = false;
        }
    }
    // device-initiated allreduce over the mapped pools (TPMG_ALLREDUCE=nccl keeps NCCL)
    const char* ar = std::getenv("TPMG_ALLREDUCE");
    ctx->p2p_reduce = ctx->p2p && ctx->nranks <= kMaxP2PRanks && !(ar && std::strcmp(ar, "nccl") == 0);
    if (ctx->p2p_reduce) {
        ctx->red.me = ctx->rank;
        ctx->red.nranks = ctx->nranks;
        for (int q = 0; q < ctx->nranks; ++q) {
            ctx->red.slots[q] = reinterpret_cast<double*>(ctx->peer_all[q] + ctx->off_red);
            ctx->red.flags[q] = reinterpret_cast<unsigned*>(ctx->peer_all[q] + ctx->off_redflags);
        }
    }
    return TPMG_OK;
}

void params_fill_defaults(tpmg_params* p)
{
    if (p->nz == 0) p->nz = 128;
    if (p->nu_cfl == 0) p->nu_cfl = 8.4;
    if (p->H == 0) p->H = 0.01;
    if (p->lambda == 0) p->lambda = 1.0;
    if (p->levels == 0) p->levels = 5;
    if (p->pre == 0) p->pre = 1;
    if (p->post == 0) p->post = 1;
    if (p->coarse_sweeps == 0) p->coarse_sweeps = 2;
    if (p->rho == 0) p->rho = 2.0 / 3.0;
}

void ctx_free(tpmg_ctx* ctx)
{
    for (size_t l = 1; l < ctx->lv.size(); ++l) {
        LevelData& L = ctx->lv[l];
        cudaFree(L.d_tab);
        cudaFree(L.d_prof);
        cudaFree(L.d_fprof);
        cudaFree(L.d_fld);
        cudaFree(L.d_im);
        if ((int)l < ctx->L) { cudaFree(L.u[0]); cudaFree(L.f); }
        cudaFree(L.u[1]);
    }
    cudaFree(ctx->d_partials);
    cudaFree(ctx->d_ticket);
    cudaFree(ctx->d_scal);
    cudaFree(ctx->scratch);
    cudaFree(ctx->cg_r); cudaFree(ctx->cg_z); cudaFree(ctx->cg_p[0]); cudaFree(ctx->cg_p[1]);
    // cg_zlo / cg_zhi and the level slabs live in the halo pool
    for (int q = 0; q < 2; ++q) { cudaFree(ctx->cg_plo[q]); cudaFree(ctx->cg_phi[q]); }
    cudaFree(ctx->host_f); cudaFree(ctx->host_u); cudaFree(ctx->host_u2);
    if (ctx->copy_stream) cudaStreamDestroy(ctx->copy_stream);
    if (ctx->ev_copy) cudaEventDestroy(ctx->ev_copy);
    if (ctx->h_pinned) cudaFreeHost(ctx->h_pinned);
    cudaFree(ctx->d_flags);
    if (ctx->h_flags) cudaFreeHost(ctx->h_flags);
    for (auto e : ctx->ev_it)
        if (e) cudaEventDestroy(e);
    if (ctx->ev0) cudaEventDestroy(ctx->ev0);
    if (ctx->ev1) cudaEventDestroy(ctx->ev1);
    for (auto& r : ctx->prof_pending) { cudaEventDestroy(r.a); cudaEventDestroy(r.b); }
    for (auto e : ctx->prof_pool) cudaEventDestroy(e);
    for (int q = 0; q < (int)ctx->peer_all.size(); ++q)
        if (q != ctx->rank && ctx->peer_all[q]) cudaIpcCloseMemHandle(ctx->peer_all[q]);
    cudaFree(ctx->halo_pool);
    if (ctx->comm_halo) ncclCommDestroy(ctx->comm_halo);
    if (ctx->comm) ncclCommDestroy(ctx->comm);
    if (ctx->comm_stream) cudaStreamDestroy(ctx->comm_stream);
    if (ctx->ev_ready) cudaEventDestroy(ctx->ev_ready);
    if (ctx->ev_halo) cudaEventDestroy(ctx->ev_halo);
}

}  // namespace

// ====================================================================== C ABI

extern "C" {

int32_t tpmg_version(void) { return TPMG_VERSION_MAJOR * 1000 + TPMG_VERSION_MINOR; }

void tpmg_params_default(tpmg_params* p)
{
    if (!p) return;
    std::memset(p, 0, sizeof *p);
    params_fill_defaults(p);
}

tpmg_status tpmg_nccl_id(void* id128)
{
    if (!id128) return fail(nullptr, TPMG_E_PARAM, "tpmg_nccl_id: NULL id");
    ncclUniqueId id;
    ncclResult_t e = ncclGetUniqueId(&id);
    if (e != ncclSuccess) return fail(nullptr, TPMG_E_NCCL, "ncclGetUniqueId: %s", ncclGetErrorString(e));
    static_assert(sizeof(ncclUniqueId) == 128, "NCCL unique id is 128 bytes");
    std::memcpy(id128, &id, 128);
    return TPMG_OK;
}

namespace {
// Parameter / topology validation shared by tpmg_partition and tpmg_create.
tpmg_status validate(const tpmg_params* params, int32_t rank, int32_t nranks, tpmg_params* out)
{
    if (!params) return fail(nullptr, TPMG_E_PARAM, "NULL params");
    tpmg_params p = *params;
    params_fill_defaults(&p);
    if (p.nx <= 0 || p.ny <= 0 || p.nz <= 0) return fail(nullptr, TPMG_E_PARAM, "grid %lld x %lld x %d must be positive", (long long)p.nx, (long long)p.ny, p.nz);
    if (!(p.nu_cfl > 0) || !(p.H > 0) || !(p.lambda > 0)) return fail(nullptr, TPMG_E_PARAM, "nu_cfl, H, lambda must be > 0");
    if (!(p.rho > 0 && p.rho < 2)) return fail(nullptr, TPMG_E_PARAM, "rho = %g not in (0, 2)", p.rho);
    if (p.levels < 1 || p.levels > 24) return fail(nullptr, TPMG_E_PARAM, "levels = %d not in [1, 24]", p.levels);
    if (p.pre < 0 || p.post < 0 || p.coarse_sweeps < 1) return fail(nullptr, TPMG_E_PARAM, "pre/post >= 0, coarse_sweeps >= 1");
    if (p.boundary != TPMG_BC_GHOST_ZERO && p.boundary != TPMG_BC_FACE)
        return fail(nullptr, TPMG_E_PARAM, "boundary = %d is not a tpmg_boundary", p.boundary);
    if (nranks < 1 || rank < 0 || rank >= nranks) return fail(nullptr, TPMG_E_TOPOLOGY, "rank %d of %d", rank, nranks);
    const int64_t f = (int64_t)1 << (p.levels - 1);
    if (p.nx % f) return fail(nullptr, TPMG_E_SHAPE, "nx = %lld not divisible by 2^(L-1) = %lld", (long long)p.nx, (long long)f);
    if (p.ny % (f * nranks)) return fail(nullptr, TPMG_E_SHAPE, "ny = %lld not divisible by nranks * 2^(L-1) = %lld", (long long)p.ny, (long long)(f * nranks));
    if (p.nz > line_max_nz()) return fail(nullptr, TPMG_E_SHAPE, "nz = %d exceeds the on-chip Thomas buffer (max %d)", p.nz, line_max_nz());
    if (out) *out = p;
    return TPMG_OK;
}
}  // namespace

tpmg_status tpmg_partition(const tpmg_params* params, int32_t rank, int32_t nranks, int32_t level, int64_t* y0,
                           int64_t* ny)
{
    tpmg_params p;
    TRY(validate(params, rank, nranks, &p));
    if (level < 1 || level > p.levels) return fail(nullptr, TPMG_E_RANGE, "level %d not in [1, %d]", level, p.levels);
    const int64_t rows = p.ny / nranks >> (p.levels - level);
    if (y0) *y0 = (int64_t)rank * rows;
    if (ny) *ny = rows;
    return TPMG_OK;
}

// Per-level tables of the column blocks M_T = A_T from the vertical profiles
// (eqn:LocalMatrixStencil; prof == nullptr: the flat box [R2], a = d = 1,
// b_k = -gamma [k > 0], c_k = -gamma [k < nz-1]).  Per level k:
//   diag_k = a_k - b_k - c_k + (4 + nb) c_l d_k   (nb = boundary faces of the column class),
//   m_k = diag_k - b_k c_{k-1} / m_{k-1}  (M = L D L^T, symmetric: b_k = c_{k-1}),
//   1/m_k,  gim_k = -c_k / m_k (backward),  afw_k = -b_k / m_{k-1} (forward),
//   and the k-split propagators over segments of kSegK levels:
//   P_k = prod_{j = k_s..k} afw_j,  Q_k = prod_{j = k..k_e} gim_j.
// One table set per column class (face Dirichlet [R25]: alpha_T = -(4 + nb) c); the
// ghost-zero reading has class 0 only.  With general profiles the stencil also reads the
// per-level couplings (b_k, c_k, c_l d_k) from LevelData::d_prof.
// With per-column fields the line kernels take the profiles raw, [a_k-b_k-c_k][b_k][c_k][d_k]
// (the same on every level), and the level's fields; lc.gen = 2.
tpmg_status fields_profile_tables(tpmg_ctx* ctx)
{
    const int nz = ctx->p.nz;
    const double* a = ctx->prof_abcd.data();
    std::vector<double> t(4 * (size_t)nz);
    for (int k = 0; k < nz; ++k) {
        t[k] = a[k] - a[nz + k] - a[2 * nz + k];
        t[nz + k] = a[nz + k];
        t[2 * nz + k] = a[2 * nz + k];
        t[3 * nz + k] = a[3 * nz + k];
    }
    for (int l = 1; l <= ctx->L; ++l) {
        LevelData& L = ctx->lv[l];
        TRY(dev_alloc(ctx, &L.d_fprof, t.size()));
        CUDA_TRY(ctx, cudaMemcpy(L.d_fprof, t.data(), sizeof(double) * t.size(), cudaMemcpyHostToDevice));
        L.lc.prof = L.d_fprof;
        L.lc.fld = L.d_fld;
        L.lc.gen = 2;
        L.im_ok = false;
    }
    // the Thomas pivots of every column, once per operator: the line kernels stream them with
    // the data instead of running the pivot recurrence (TPMG_PIVOTS=0: recurrence on chip)
    if (ctx->pivots && ctx->use_tma && ctx->tmem && nz <= 128) {
        for (int l = 1; l <= ctx->L; ++l) {
            LevelData& L = ctx->lv[l];
            TRY(dev_alloc(ctx, &L.d_im, L.n()));
            CUDA_TRY(ctx, launch_pivots(launcher(ctx), L.lc, L.d_im));
            L.im_ok = true;
        }
        CUDA_TRY(ctx, cudaStreamSynchronize(ctx->stream));
    }
    return TPMG_OK;
}

tpmg_status build_tables(tpmg_ctx* ctx, const double* const* prof)
{
    const tpmg_params& p = ctx->p;
    const int nz = p.nz;
    const double gamma = ctx->lv[ctx->L].lc.gamma;
    std::vector<double> a(nz), b(nz), c(nz), d(nz);
    for (int k = 0; k < nz; ++k) {
        a[k] = prof ? prof[0][k] : 1.0;
        b[k] = prof ? prof[1][k] : (k > 0 ? -gamma : 0.0);
        c[k] = prof ? prof[2][k] : (k < nz - 1 ? -gamma : 0.0);
        d[k] = prof ? prof[3][k] : 1.0;
    }
    for (int l = 1; l <= ctx->L; ++l) {
        LevelData& L = ctx->lv[l];
        const double cl = L.lc.c;
        const int ncls = (p.boundary == TPMG_BC_FACE) ? kBoundaryClasses : 1;
        std::vector<double> tab(6 * (size_t)nz * ncls);
        for (int cls = 0; cls < ncls; ++cls) {
            double* t_diag = tab.data() + (size_t)cls * 6 * nz;
            double* t_invm = t_diag + nz;
            double* t_gim = t_invm + nz;
            double* t_afw = t_gim + nz;
            double* t_P = t_afw + nz;
            double* t_Q = t_P + nz;
            double mprev = 0.0;
            for (int k = 0; k < nz; ++k) {
                // flat box: 1 + (4 + nb) c + gamma ([k > 0] + [k < nz-1]), the same value
                const double diag = prof ? a[k] - b[k] - c[k] + (4.0 + cls) * cl * d[k]
                                         : 1.0 + (4.0 + cls) * cl + gamma * ((k > 0 ? 1.0 : 0.0) + (k < nz - 1 ? 1.0 : 0.0));
                const double m = (k == 0) ? diag : diag - (-b[k]) * ((-c[k - 1]) / mprev);
                if (m == 0.0 || !std::isfinite(m))
                    return fail(ctx, TPMG_E_SINGULAR, "zero Thomas pivot at level %d, k = %d", l, k);
                t_diag[k] = diag;
                t_invm[k] = 1.0 / m;
                t_gim[k] = (k < nz - 1) ? -c[k] / m : 0.0;
                t_afw[k] = (k > 0) ? -b[k] / mprev : 0.0;
                mprev = m;
            }
            for (int k0 = 0; k0 < nz; k0 += kSegK) {
                const int k1 = std::min(nz, k0 + kSegK) - 1;
                double pr = 1.0;
                for (int k = k0; k <= k1; ++k) { pr *= t_afw[k]; t_P[k] = pr; }
                pr = 1.0;
                for (int k = k1; k >= k0; --k) { pr *= t_gim[k]; t_Q[k] = pr; }
            }
        }
        if (nz <= kKsplitMaxNZ)
            for (int q = 0; q < 6; ++q)
                for (int k = 0; k < nz; ++k) L.ktab.t[q][k] = tab[(size_t)q * nz + k];
        TRY(dev_alloc(ctx, &L.d_tab, tab.size()));
        CUDA_TRY(ctx, cudaMemcpy(L.d_tab, tab.data(), sizeof(double) * tab.size(), cudaMemcpyHostToDevice));
        L.lc.tab = L.d_tab;
        // general profiles: per-level stencil couplings [b_k][c_k][c_l d_k]
        L.lc.gen = prof ? 1 : 0;
        if (prof) {
            std::vector<double> pr(3 * (size_t)nz);
            for (int k = 0; k < nz; ++k) {
                pr[k] = b[k];
                pr[nz + k] = c[k];
                pr[2 * nz + k] = cl * d[k];
            }
            TRY(dev_alloc(ctx, &L.d_prof, pr.size()));
            CUDA_TRY(ctx, cudaMemcpy(L.d_prof, pr.data(), sizeof(double) * pr.size(), cudaMemcpyHostToDevice));
        }
        L.lc.prof = prof ? L.d_prof : nullptr;
    }
    ctx->gen_profiles = prof != nullptr;
    ctx->prof_abcd.resize(4 * (size_t)nz);
    for (int k = 0; k < nz; ++k) {
        ctx->prof_abcd[k] = a[k];
        ctx->prof_abcd[nz + k] = b[k];
        ctx->prof_abcd[2 * nz + k] = c[k];
        ctx->prof_abcd[3 * nz + k] = d[k];
    }
    if (ctx->fields) TRY(fields_profile_tables(ctx));
    return TPMG_OK;
}

tpmg_status tpmg_create(const tpmg_params* params, int32_t rank, int32_t nranks, const void* id128,
                        int32_t device, void* cuda_stream, tpmg_ctx** out)
{
    if (!params || !out) return fail(nullptr, TPMG_E_PARAM, "tpmg_create: NULL argument");
    *out = nullptr;
    tpmg_params p;
    TRY(validate(params, rank, nranks, &p));
    if (nranks > 1 && !id128) return fail(nullptr, TPMG_E_PARAM, "nranks > 1 needs the NCCL id");

    tpmg_ctx* ctx = new tpmg_ctx();
    ctx->p = p;
    ctx->rank = rank;
    ctx->nranks = nranks;
    ctx->device = device;
    ctx->stream = (cudaStream_t)cuda_stream;
    ctx->L = p.levels;
    {
        const char* ld = std::getenv("TPMG_LOADER");   // "cpasync" selects the cp.async loader
        ctx->use_tma = !(ld && std::strcmp(ld, "cpasync") == 0);
        const char* ks = std::getenv("TPMG_KSPLIT");
        ctx->ksplit_cfg = !ks ? 1 : ks[0] == '0' ? -1 : ks[0] == '1' ? 0 : ks[0] == '3' ? 2 : 1;
        const char* ksc = std::getenv("TPMG_KSPLIT_COARSE");   // "0" 2x8 / "2" 2x4 on unfilled levels
        if (ksc) ctx->ksplit_cfg_coarse = std::max(-1, std::min(2, std::atoi(ksc)));
        if (ctx->ksplit_cfg < 0) ctx->ksplit_cfg_coarse = -1;
        const char* ov = std::getenv("TPMG_OVERLAP");
        ctx->overlap = !(ov && ov[0] == '0');        // P2P transport: on by default
        ctx->overlap_nccl = ov && ov[0] == '1';      // NCCL transport: opt-in
        const char* pu = std::getenv("TPMG_PAIR_U");
        ctx->pair_u = pu && pu[0] == '1';
        const char* ovc = std::getenv("TPMG_OVERLAP_CG");
        ctx->overlap_cg = ovc && ovc[0] == '1';
        const char* rs = std::getenv("TPMG_RESERVE_SMS");
        if (rs) ctx->reserve_sms = std::max(0, std::atoi(rs));
        const char* kc = std::getenv("TPMG_KSPLIT_CG");
        ctx->ksplit_cg = kc && kc[0] == '1';
        const char* pd = std::getenv("TPMG_PDL");
        ctx->pdl = pd && pd[0] == '1';
        const char* fp = std::getenv("TPMG_FUSE_PROLONG");
        ctx->fuse_prolong = fp && fp[0] == '1';
        const char* sd = std::getenv("TPMG_SYNC_DEBUG");
        ctx->sync_debug = sd && sd[0] == '1';
        const char* tm = std::getenv("TPMG_TMEM");   // "0": g' of the column kernels in shared memory
        ctx->tmem = !(tm && tm[0] == '0');
        const char* bnd = std::getenv("TPMG_BAND");
        if (bnd) ctx->band_w = std::max(0, std::atoi(bnd));
        const char* cvo = std::getenv("TPMG_CARVEOUT");
        ctx->carveout_fit = cvo && std::strcmp(cvo, "fit") == 0;
        const char* tst = std::getenv("TPMG_TMA_STORE");
        ctx->tma_store = tst && tst[0] == '1';
        const char* dpb = std::getenv("TPMG_DEV_PUBLISH");
        ctx->dev_publish = dpb && dpb[0] == '1';
        const char* skf = std::getenv("TPMG_SKIP_FINISH");
        ctx->skip_finish = skf && skf[0] == '1';
        const char* tpr = std::getenv("TPMG_TMA_PROMO");
        if (tpr) ctx->tma_promo = std::min(3, std::max(0, std::atoi(tpr)));
        const char* l2h = std::getenv("TPMG_L2HINT");
        if (l2h) ctx->l2hint = std::atoi(l2h) & 3;
        const char* cdc = std::getenv("TPMG_CGDIR_CTAS");
        if (cdc) ctx->cgdir_ctas = std::max(0, std::atoi(cdc));
        const char* dpr = std::getenv("TPMG_DBG_PERROW");
        ctx->dbg = (dpr && dpr[0] == '1') ? 1 : 0;
        const char* pdt = std::getenv("TPMG_PROF_DETAIL");
        ctx->prof_detail = pdt && pdt[0] == '1';
        const char* pv = std::getenv("TPMG_PIVOTS");
        ctx->pivots = !(pv && pv[0] == '0');
        const char* ts = std::getenv("TPMG_TM_STAGES");
        if (ts) ctx->tm_stages = std::atoi(ts);
        const char* tc = std::getenv("TPMG_TM_CTAS");
        if (tc) ctx->tm_ctas = std::max(1, std::min(2, std::atoi(tc)));
    }
    ctx->ny_loc = p.ny / nranks;
    ctx->y0 = (int64_t)rank * ctx->ny_loc;
    auto bail = [&](tpmg_status st) {
        g_create_error = ctx->err;
        ctx_free(ctx);
        delete ctx;
        return st;
    };
#define CREATE_TRY(expr)                              \
    do {                                              \
        tpmg_status s__ = (expr);                     \
        if (s__ != TPMG_OK) return bail(s__);         \
    } while (0)
#define CREATE_CUDA(expr)                                                                       \
    do {                                                                                        \
        cudaError_t e__ = (expr);                                                               \
        if (e__ != cudaSuccess)                                                                 \
            return bail(fail(ctx, TPMG_E_CUDA, "%s: %s", #expr, cudaGetErrorString(e__)));      \
    } while (0)

    CREATE_CUDA(cudaSetDevice(device));
    CREATE_CUDA(cudaDeviceGetAttribute(&ctx->num_sms, cudaDevAttrMultiProcessorCount, device));
    CREATE_CUDA(cudaEventCreate(&ctx->ev0));
    CREATE_CUDA(cudaEventCreate(&ctx->ev1));
    CREATE_CUDA(cudaMallocHost((void**)&ctx->h_pinned, 64 * sizeof(double)));
    CREATE_TRY(dev_alloc(ctx, &ctx->d_partials, (size_t)ctx->num_sms * 64 * 2));
    CREATE_CUDA(cudaMalloc((void**)&ctx->d_ticket, sizeof(unsigned)));
    CREATE_CUDA(cudaMemset(ctx->d_ticket, 0, sizeof(unsigned)));

    // Coefficients: h = 1/nx, h_z = H/nz, omega = nu h / 2,
    // c_l = omega^2 / h_l^2 with h_l = 2^(L-l) h [R4], gamma = omega^2 lambda^2 / h_z^2.
    const double h = 1.0 / (double)p.nx;
    const double hz = p.H / (double)p.nz;
    const double omega = 0.5 * p.nu_cfl * h;
    const double gamma = omega * omega * p.lambda * p.lambda / (hz * hz);
    ctx->lv.resize(ctx->L + 1);
    for (int l = 1; l <= ctx->L; ++l) {
        LevelData& L = ctx->lv[l];
        const int64_t fl = (int64_t)1 << (ctx->L - l);
        const double hl = h * (double)fl;
        L.lc.nx = p.nx / fl;
        L.lc.ny = ctx->ny_loc / fl;
        L.lc.nz = p.nz;
        L.lc.c = omega * omega / (hl * hl);
        L.lc.gamma = gamma;
        L.lc.bc = p.boundary;
        L.lc.bnd_lo = (rank == 0) ? 1 : 0;               // local row 0 / ny-1 on the physical boundary
        L.lc.bnd_hi = (rank == nranks - 1) ? 1 : 0;
    }
    CREATE_TRY(build_tables(ctx, nullptr));
    if (nranks > 1) {
        ncclUniqueId id;
        std::memcpy(&id, id128, sizeof id);
        ncclResult_t e = ncclCommInitRank(&ctx->comm, nranks, id, rank);
        if (e != ncclSuccess) return bail(fail(ctx, TPMG_E_NCCL, "ncclCommInitRank: %s", ncclGetErrorString(e)));
        // halo traffic: own communicator (few CTAs) and a high-priority stream
        ncclConfig_t cfg = NCCL_CONFIG_INITIALIZER;
        cfg.minCTAs = 1;
        cfg.maxCTAs = 2;
        e = ncclCommSplit(ctx->comm, 0, rank, &ctx->comm_halo, &cfg);
        if (e != ncclSuccess) return bail(fail(ctx, TPMG_E_NCCL, "ncclCommSplit: %s", ncclGetErrorString(e)));
        int lo_prio = 0, hi_prio = 0;
        tpmg_status st = TPMG_OK;
        if (cudaDeviceGetStreamPriorityRange(&lo_prio, &hi_prio) != cudaSuccess ||
            cudaStreamCreateWithPriority(&ctx->comm_stream, cudaStreamNonBlocking, hi_prio) != cudaSuccess ||
            cudaEventCreateWithFlags(&ctx->ev_ready, cudaEventDisableTiming) != cudaSuccess ||
            cudaEventCreateWithFlags(&ctx->ev_halo, cudaEventDisableTiming) != cudaSuccess)
            st = fail(ctx, TPMG_E_CUDA, "tpmg_create: halo stream / events");
        CREATE_TRY(agree(ctx, st));   // no rank enters halo_setup's collectives alone
        CREATE_TRY(halo_setup(ctx));
    }
#undef CREATE_TRY
#undef CREATE_CUDA
    *out = ctx;
    return TPMG_OK;
}

tpmg_status tpmg_destroy(tpmg_ctx* ctx)
{
    if (!ctx) return TPMG_OK;
    if (ctx->prof_detail)
        for (auto& kv : ctx->prof_by_size)
            std::fprintf(stderr, "tpmg prof rank %d class %d cells %.0f launches %lld ms %.4f avg_us %.1f\n", ctx->rank,
                         kv.first.first, kv.first.second, (long long)kv.second.first, kv.second.second,
                         1e3 * kv.second.second / (double)std::max<int64_t>(kv.second.first, 1));
    cudaSetDevice(ctx->device);
    if (ctx->stream) cudaStreamSynchronize(ctx->stream); else cudaDeviceSynchronize();
    ctx_free(ctx);
    delete ctx;
    return TPMG_OK;
}

tpmg_status tpmg_set_stream(tpmg_ctx* ctx, void* s)
{
    if (!ctx) return TPMG_E_PARAM;
    cudaStream_t ns = (cudaStream_t)s;
    if (ns != ctx->stream) {
        // order the new stream after everything on the old one (shared scratch, reduction
        // tickets, halo slabs)
        cudaEvent_t e = nullptr;
        CUDA_TRY(ctx, cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
        cudaError_t r = cudaEventRecord(e, ctx->stream);
        if (r == cudaSuccess) r = cudaStreamWaitEvent(ns, e, 0);
        cudaEventDestroy(e);
        if (r != cudaSuccess) return fail(ctx, TPMG_E_CUDA, "tpmg_set_stream: %s", cudaGetErrorString(r));
    }
    ctx->stream = ns;
    return TPMG_OK;
}

tpmg_status tpmg_local_box(const tpmg_ctx* cctx, int32_t level, int64_t* y0, int64_t* nx, int64_t* ny,
                           int32_t* nz)
{
    tpmg_ctx* ctx = const_cast<tpmg_ctx*>(cctx);
    TRY(check_level(ctx, level));
    const LevelData& L = ctx->lv[level];
    if (y0) *y0 = ctx->y0 >> (ctx->L - level);
    if (nx) *nx = L.lc.nx;
    if (ny) *ny = L.lc.ny;
    if (nz) *nz = L.lc.nz;
    return TPMG_OK;
}

tpmg_status tpmg_apply(tpmg_ctx* ctx, int32_t level, const double* x, double* y)
{
    if (ctx) begin_call(ctx);
    TRY(check_level(ctx, level));
    if (!x || !y) return fail(ctx, TPMG_E_PARAM, "tpmg_apply: NULL vector");
    if (x == y) return fail(ctx, TPMG_E_SHAPE, "tpmg_apply: x and y must differ");
    LineArgs a = line_args(ctx, level);
    TRY(halo(ctx, level, x, &a.h0));
    a.out0 = y;
    return run_line(ctx, MODE_APPLY, a);
}

tpmg_status tpmg_residual(tpmg_ctx* ctx, int32_t level, const double* u, const double* f, double* r,
                          double* norm2)
{
    if (ctx) begin_call(ctx);
    TRY(check_level(ctx, level));
    if (!u || !f) return fail(ctx, TPMG_E_PARAM, "tpmg_residual: NULL vector");
    if (r == u) return fail(ctx, TPMG_E_SHAPE, "tpmg_residual: r must not alias u");
    if (!r && !norm2) return TPMG_OK;
    TRY(ensure_scal(ctx, 8));
    LineArgs a = line_args(ctx, level);
    TRY(halo(ctx, level, u, &a.h0));
    a.q0 = f;
    a.out0 = r;
    a.red.result = norm2 ? ctx->d_scal + 4 : nullptr;
    TRY(run_line(ctx, MODE_RESID, a));
    if (norm2) {
        TRY(allreduce(ctx, ctx->d_scal + 4, 1));
        TRY(fetch(ctx, ctx->d_scal + 4, 1));
        *norm2 = ctx->h_pinned[0];
    }
    return TPMG_OK;
}

tpmg_status tpmg_precondition(tpmg_ctx* ctx, int32_t level, const double* r, double* z)
{
    if (ctx) begin_call(ctx);
    TRY(check_level(ctx, level));
    if (!r || !z) return fail(ctx, TPMG_E_PARAM, "tpmg_precondition: NULL vector");
    if (r == z) return fail(ctx, TPMG_E_SHAPE, "tpmg_precondition: r and z must differ");
    LineArgs a = line_args(ctx, level);
    a.q0 = r;
    a.out0 = z;
    return run_line(ctx, MODE_PREC, a);
}

tpmg_status tpmg_smooth(tpmg_ctx* ctx, int32_t level, double* u, const double* f, int32_t sweeps)
{
    if (ctx) begin_call(ctx);
    TRY(check_level(ctx, level));
    if (!u || !f) return fail(ctx, TPMG_E_PARAM, "tpmg_smooth: NULL vector");
    if (sweeps < 0) return fail(ctx, TPMG_E_PARAM, "tpmg_smooth: sweeps < 0");
    if (sweeps == 0) return TPMG_OK;
    if (u == f) return fail(ctx, TPMG_E_SHAPE, "tpmg_smooth: u and f must differ");
    const LevelData& L = ctx->lv[level];
    TRY(dev_alloc(ctx, &ctx->scratch, ctx->lv[ctx->L].n()));
    double* bufs[2] = {u, ctx->scratch};
    int cur = 0;
    for (int s = 0; s < sweeps; ++s) {
        TRY(smooth_once(ctx, level, bufs[cur], f, bufs[1 - cur], nullptr));
        cur ^= 1;
    }
    if (cur) CUDA_TRY(ctx, cudaMemcpyAsync(u, ctx->scratch, sizeof(double) * L.n(), cudaMemcpyDeviceToDevice, ctx->stream));
    return TPMG_OK;
}

tpmg_status tpmg_restrict(tpmg_ctx* ctx, int32_t fine_level, const double* r_fine, double* f_coarse)
{
    if (ctx) begin_call(ctx);
    TRY(check_level(ctx, fine_level));
    if (fine_level < 2) return fail(ctx, TPMG_E_RANGE, "tpmg_restrict: fine_level %d < 2", fine_level);
    if (!r_fine || !f_coarse) return fail(ctx, TPMG_E_PARAM, "tpmg_restrict: NULL vector");
    ProfScope ps(ctx, TPMG_K_RESTRICT, level_cells(ctx->lv[fine_level].lc));
    CUDA_TRY(ctx, launch_restrict(launcher(ctx), ctx->lv[fine_level].lc, ctx->lv[fine_level - 1].lc, r_fine, f_coarse));
    return TPMG_OK;
}

tpmg_status tpmg_prolong_add(tpmg_ctx* ctx, int32_t coarse_level, const double* u_coarse, double* u_fine)
{
    if (ctx) begin_call(ctx);
    TRY(check_level(ctx, coarse_level));
    if (coarse_level >= ctx->L) return fail(ctx, TPMG_E_RANGE, "tpmg_prolong_add: coarse_level %d >= L", coarse_level);
    if (!u_coarse || !u_fine) return fail(ctx, TPMG_E_PARAM, "tpmg_prolong_add: NULL vector");
    HaloField uc;
    TRY(halo(ctx, coarse_level, u_coarse, &uc));
    ProfScope ps(ctx, TPMG_K_PROLONG_ADD, level_cells(ctx->lv[coarse_level + 1].lc));
    CUDA_TRY(ctx, launch_prolong_add(launcher(ctx), ctx->lv[coarse_level].lc, ctx->lv[coarse_level + 1].lc, uc, u_fine));
    return TPMG_OK;
}

tpmg_status tpmg_vcycle(tpmg_ctx* ctx, double* u, const double* f)
{
    if (ctx) begin_call(ctx);
    if (!ctx) return TPMG_E_PARAM;
    if (!u || !f) return fail(ctx, TPMG_E_PARAM, "tpmg_vcycle: NULL vector");
    if (u == f) return fail(ctx, TPMG_E_SHAPE, "tpmg_vcycle: u and f must differ");
    TRY(mg_alloc(ctx));
    TRY(vcycle_fine(ctx, u, f));
    CUDA_TRY(ctx, cudaStreamSynchronize(ctx->stream));
    return TPMG_OK;
}

tpmg_status tpmg_solve_mg(tpmg_ctx* ctx, const double* f, double* u, double eps, int32_t max_iter,
                          tpmg_result* res)
{
    if (ctx) begin_call(ctx);
    if (!ctx) return TPMG_E_PARAM;
    if (!u || !f) return fail(ctx, TPMG_E_PARAM, "tpmg_solve_mg: NULL vector");
    if (u == f) return fail(ctx, TPMG_E_SHAPE, "tpmg_solve_mg: u and f must differ");
    if (!(eps > 0) || max_iter < 0) return fail(ctx, TPMG_E_PARAM, "tpmg_solve_mg: eps > 0, max_iter >= 0");
    return solve_mg_impl(ctx, f, u, eps, max_iter, res);
}

tpmg_status tpmg_solve_cg(tpmg_ctx* ctx, const double* f, double* u, double eps, int32_t max_iter,
                          tpmg_result* res)
{
    if (ctx) begin_call(ctx);
    if (!ctx) return TPMG_E_PARAM;
    if (!u || !f) return fail(ctx, TPMG_E_PARAM, "tpmg_solve_cg: NULL vector");
    if (u == f) return fail(ctx, TPMG_E_SHAPE, "tpmg_solve_cg: u and f must differ");
    if (!(eps > 0) || max_iter < 0) return fail(ctx, TPMG_E_PARAM, "tpmg_solve_cg: eps > 0, max_iter >= 0");
    return solve_cg_impl(ctx, f, u, eps, max_iter, res);
}

tpmg_status tpmg_solve_host(tpmg_ctx* ctx, tpmg_solver solver, const double* f_host, double* u_host,
                            double eps, int32_t max_iter, tpmg_result* res)
{
    if (ctx) begin_call(ctx);
    if (!ctx) return TPMG_E_PARAM;
    if (!f_host || !u_host) return fail(ctx, TPMG_E_PARAM, "tpmg_solve_host: NULL buffer");
    const size_t n = ctx->lv[ctx->L].n();
    TRY(dev_alloc(ctx, &ctx->host_f, n));
    TRY(dev_alloc(ctx, &ctx->host_u, n));
    CUDA_TRY(ctx, cudaMemcpyAsync(ctx->host_f, f_host, sizeof(double) * n, cudaMemcpyHostToDevice, ctx->stream));
    tpmg_status st = (solver == TPMG_SOLVER_MG) ? tpmg_solve_mg(ctx, ctx->host_f, ctx->host_u, eps, max_iter, res)
                                                : tpmg_solve_cg(ctx, ctx->host_f, ctx->host_u, eps, max_iter, res);
    if (st != TPMG_OK) return st;
    CUDA_TRY(ctx, cudaMemcpyAsync(u_host, ctx->host_u, sizeof(double) * n, cudaMemcpyDeviceToHost, ctx->stream));
    CUDA_TRY(ctx, cudaStreamSynchronize(ctx->stream));
    return TPMG_OK;
}

tpmg_status tpmg_solve_host_pair(tpmg_ctx* ctx, const double* f_host, double* u_mg_host, double* u_cg_host,
                                 double eps, int32_t max_iter_mg, int32_t max_iter_cg, tpmg_result* res_mg,
                                 tpmg_result* res_cg)
{
    if (ctx) begin_call(ctx);
    if (!ctx) return TPMG_E_PARAM;
    if (!f_host || !u_mg_host || !u_cg_host) return fail(ctx, TPMG_E_PARAM, "tpmg_solve_host_pair: NULL buffer");
    const size_t n = ctx->lv[ctx->L].n();
    TRY(dev_alloc(ctx, &ctx->host_f, n));
    TRY(dev_alloc(ctx, &ctx->host_u, n));
    TRY(dev_alloc(ctx, &ctx->host_u2, n));
    if (!ctx->copy_stream) {
        CUDA_TRY(ctx, cudaStreamCreateWithFlags(&ctx->copy_stream, cudaStreamNonBlocking));
        CUDA_TRY(ctx, cudaEventCreateWithFlags(&ctx->ev_copy, cudaEventDisableTiming));
    }
    CUDA_TRY(ctx, cudaMemcpyAsync(ctx->host_f, f_host, sizeof(double) * n, cudaMemcpyHostToDevice, ctx->stream));
    TRY(tpmg_solve_mg(ctx, ctx->host_f, ctx->host_u, eps, max_iter_mg, res_mg));
    // u_mg leaves on the copy engine while the PCG solve computes (its last writer is ordered by
    // the event; the PCG solve writes host_u2, not host_u)
    CUDA_TRY(ctx, cudaEventRecord(ctx->ev_copy, ctx->stream));
    CUDA_TRY(ctx, cudaStreamWaitEvent(ctx->copy_stream, ctx->ev_copy, 0));
    CUDA_TRY(ctx, cudaMemcpyAsync(u_mg_host, ctx->host_u, sizeof(double) * n, cudaMemcpyDeviceToHost, ctx->copy_stream));
    TRY(tpmg_solve_cg(ctx, ctx->host_f, ctx->host_u2, eps, max_iter_cg, res_cg));
    CUDA_TRY(ctx, cudaMemcpyAsync(u_cg_host, ctx->host_u2, sizeof(double) * n, cudaMemcpyDeviceToHost, ctx->stream));
    CUDA_TRY(ctx, cudaStreamSynchronize(ctx->copy_stream));
    CUDA_TRY(ctx, cudaStreamSynchronize(ctx->stream));
    return TPMG_OK;
}

tpmg_status tpmg_transpose(tpmg_ctx* ctx, int32_t level, int32_t direction, const double* src, double* dst)
{
    if (ctx) begin_call(ctx);
    if (!ctx) return TPMG_E_PARAM;
    TRY(check_level(ctx, level));
    if (direction != TPMG_ZC_TO_LAMBDA && direction != TPMG_LAMBDA_TO_ZC)
        return fail(ctx, TPMG_E_PARAM, "tpmg_transpose: direction must be TPMG_ZC_TO_LAMBDA or TPMG_LAMBDA_TO_ZC");
    if (!src || !dst) return fail(ctx, TPMG_E_PARAM, "tpmg_transpose: NULL buffer");
    if (src == dst) return fail(ctx, TPMG_E_PARAM, "tpmg_transpose: src and dst must not alias");
    const LevelConst& L = ctx->lv[level].lc;
    CUDA_TRY(ctx, launch_transpose(launcher(ctx), direction == TPMG_ZC_TO_LAMBDA, src, dst, L.nx, L.ny, L.nz));
    return TPMG_OK;
}

tpmg_status tpmg_halo_push(tpmg_ctx* ctx, int32_t level, const double* src, double* dst_lo, double* dst_hi)
{
    if (ctx) begin_call(ctx);
    if (!ctx) return TPMG_E_PARAM;
    TRY(check_level(ctx, level));
    if (!src) return fail(ctx, TPMG_E_PARAM, "tpmg_halo_push: NULL src");
    const LevelData& L = ctx->lv[level];
    const double* end = src + L.n();
    for (const double* d : {static_cast<const double*>(dst_lo), static_cast<const double*>(dst_hi)})
        if (d && d + L.plane() > src && d < end)
            return fail(ctx, TPMG_E_PARAM, "tpmg_halo_push: a destination overlaps src");
    HaloPush hp{src, src + (size_t)(L.lc.ny - 1) * L.plane(), dst_lo, dst_hi, (int64_t)L.plane()};
    CUDA_TRY(ctx, launch_halo_push(launcher(ctx), hp));
    return TPMG_OK;
}

tpmg_status tpmg_cg_halo(tpmg_ctx* ctx, double beta, double* out_lo, const double* z_lo, const double* p_lo,
                         double* out_hi, const double* z_hi, const double* p_hi)
{
    if (ctx) begin_call(ctx);
    if (!ctx) return TPMG_E_PARAM;
    if ((out_lo && (!z_lo || !p_lo)) || (out_hi && (!z_hi || !p_hi)))
        return fail(ctx, TPMG_E_PARAM, "tpmg_cg_halo: an output plane needs its z and p planes");
    // beta as the device ratio the kernel reads: s[0] / s[1] = beta / 1
    double* d_beta = nullptr;
    TRY(dev_alloc(ctx, &d_beta, 2));
    const double hb[2] = {beta, 1.0};
    cudaError_t e = cudaMemcpy(d_beta, hb, sizeof hb, cudaMemcpyHostToDevice);
    if (e == cudaSuccess)
        e = launch_cg_halo(launcher(ctx), out_lo, z_lo, p_lo, out_hi, z_hi, p_hi, (int64_t)ctx->lv[ctx->L].plane(),
                           DevRatio{d_beta, 0, 1}, nullptr);
    if (e == cudaSuccess) e = cudaStreamSynchronize(ctx->stream);
    cudaFree(d_beta);
    if (e != cudaSuccess) return fail(ctx, TPMG_E_CUDA, "tpmg_cg_halo: %s", cudaGetErrorString(e));
    return TPMG_OK;
}

tpmg_status tpmg_solve_host_zc(tpmg_ctx* ctx, tpmg_solver solver, const double* f_host, double* u_host,
                               double eps, int32_t max_iter, tpmg_result* res)
{
    if (ctx) begin_call(ctx);
    if (!ctx) return TPMG_E_PARAM;
    if (!f_host || !u_host) return fail(ctx, TPMG_E_PARAM, "tpmg_solve_host_zc: NULL buffer");
    const LevelConst& L = ctx->lv[ctx->L].lc;
    const size_t n = ctx->lv[ctx->L].n();
    TRY(dev_alloc(ctx, &ctx->host_f, n));
    TRY(dev_alloc(ctx, &ctx->host_u, n));
    // host_u stages the z-contiguous f, host_f holds f in the Lambda layout; after the solve
    // (u in host_u) host_f stages the z-contiguous u
    CUDA_TRY(ctx, cudaMemcpyAsync(ctx->host_u, f_host, sizeof(double) * n, cudaMemcpyHostToDevice, ctx->stream));
    CUDA_TRY(ctx, launch_transpose(launcher(ctx), true, ctx->host_u, ctx->host_f, L.nx, L.ny, L.nz));
    tpmg_status st = (solver == TPMG_SOLVER_MG) ? tpmg_solve_mg(ctx, ctx->host_f, ctx->host_u, eps, max_iter, res)
                                                : tpmg_solve_cg(ctx, ctx->host_f, ctx->host_u, eps, max_iter, res);
    if (st != TPMG_OK) return st;
    CUDA_TRY(ctx, launch_transpose(launcher(ctx), false, ctx->host_u, ctx->host_f, L.nx, L.ny, L.nz));
    CUDA_TRY(ctx, cudaMemcpyAsync(u_host, ctx->host_f, sizeof(double) * n, cudaMemcpyDeviceToHost, ctx->stream));
    CUDA_TRY(ctx, cudaStreamSynchronize(ctx->stream));
    return TPMG_OK;
}

tpmg_status tpmg_get_stats(const tpmg_ctx* ctx, tpmg_stats* out)
{
    if (!ctx || !out) return TPMG_E_PARAM;
    *out = ctx->stats;
    out->p2p_halo = ctx->p2p ? 1 : 0;
    out->p2p_allreduce = ctx->p2p_reduce ? 1 : 0;
    return TPMG_OK;
}

tpmg_status tpmg_stats_reset(tpmg_ctx* ctx)
{
    if (!ctx) return TPMG_E_PARAM;
    ctx->stats = tpmg_stats{};
    return TPMG_OK;
}

tpmg_status tpmg_profile(tpmg_ctx* ctx, int32_t enable)
{
    return tpmg_profile_mask(ctx, enable ? ((1u << TPMG_K_COUNT) - 1u) : 0u);
}

tpmg_status tpmg_profile_mask(tpmg_ctx* ctx, uint32_t mask)
{
    if (!ctx) return TPMG_E_PARAM;
    const bool enable = (mask & ((1u << TPMG_K_COUNT) - 1u)) != 0;
    if (enable) {
        TRY(prof_collect(ctx));
        for (int k = 0; k < TPMG_K_COUNT; ++k) {
            ctx->prof_launches[k] = 0;
            ctx->prof_ms[k] = 0;
            ctx->prof_cells[k] = 0;
        }
    }
    ctx->prof_on = enable;
    ctx->prof_mask = mask;
    return TPMG_OK;
}

tpmg_status tpmg_profile_read(tpmg_ctx* ctx, int32_t kernel, int64_t* launches, double* ms, double* cells)
{
    if (!ctx) return TPMG_E_PARAM;
    if (kernel < 0 || kernel >= TPMG_K_COUNT) return fail(ctx, TPMG_E_RANGE, "kernel class %d", kernel);
    TRY(prof_collect(ctx));
    if (launches) *launches = ctx->prof_launches[kernel];
    if (ms) *ms = ctx->prof_ms[kernel];
    if (cells) *cells = ctx->prof_cells[kernel];
    return TPMG_OK;
}

const char* tpmg_last_error(const tpmg_ctx* ctx)
{
    if (!ctx) return g_create_error.c_str();
    return ctx->err.c_str();
}

}  // extern "C"

// Per-column horizontal fields.  Coarse levels by reading [R26]: one level down,
//   |T|_c(I,J)   = (|T|(2I,2J) + |T|(2I+1,2J) + |T|(2I,2J+1) + |T|(2I+1,2J+1)) / 4,
//   alpha_c(x-face I of row J) = (alpha(x-face 2I of row 2J) + alpha(x-face 2I of row 2J+1)) / 8,
//   alpha_c(y-face J of column I) = (alpha(y-face 2J of column 2I) + alpha(y-face 2J of column 2I+1)) / 8
// (the mean face coefficient times the 1/4 of the rediscretisation [R4]).  alpha_T of a column is
// the sum of its 4 face alphas [R1]; the face-Dirichlet reading [R25] counts a boundary face twice.
tpmg_status tpmg_set_fields(tpmg_ctx* ctx, const double* area, const double* ax, const double* ay)
{
    if (!ctx) return TPMG_E_PARAM;
    const int64_t nx = ctx->p.nx, ny = ctx->p.ny;
    const int nz = ctx->p.nz;
    if (!area && !ax && !ay) {
        CUDA_TRY(ctx, cudaStreamSynchronize(ctx->stream));
        ctx->fields = false;
        const double* prof[4] = {ctx->prof_abcd.data(), ctx->prof_abcd.data() + nz, ctx->prof_abcd.data() + 2 * nz,
                                 ctx->prof_abcd.data() + 3 * nz};
        const bool flat = !ctx->gen_profiles;
        for (int l = 1; l <= ctx->L; ++l) {
            ctx->lv[l].lc.fld = nullptr;
            ctx->lv[l].im_ok = false;
        }
        return build_tables(ctx, flat ? nullptr : prof);
    }
    if (!area || !ax || !ay) return fail(ctx, TPMG_E_PARAM, "tpmg_set_fields: give all three fields or none");
    for (int64_t q = 0; q < nx * ny; ++q)
        if (!(area[q] > 0) || !std::isfinite(area[q]))
            return fail(ctx, TPMG_E_PARAM, "tpmg_set_fields: |T| must be positive and finite (column %lld)", (long long)q);
    for (int64_t q = 0; q < (nx + 1) * ny; ++q)
        if (!(ax[q] <= 0) || !std::isfinite(ax[q]))
            return fail(ctx, TPMG_E_PARAM, "tpmg_set_fields: x-face alpha must be <= 0 and finite (face %lld)", (long long)q);
    for (int64_t q = 0; q < nx * (ny + 1); ++q)
        if (!(ay[q] <= 0) || !std::isfinite(ay[q]))
            return fail(ctx, TPMG_E_PARAM, "tpmg_set_fields: y-face alpha must be <= 0 and finite (face %lld)", (long long)q);
    if (!ctx->use_tma) return fail(ctx, TPMG_E_PARAM, "tpmg_set_fields: per-column fields need the TMA loader");
    if (!line_gen_fits(nz, 2)) return fail(ctx, TPMG_E_SHAPE, "tpmg_set_fields: nz = %d too large for per-column fields", nz);
    CUDA_TRY(ctx, cudaStreamSynchronize(ctx->stream));   // queued kernels may still read the fields
    // global fields of the current level, finest first
    std::vector<double> A(area, area + nx * ny), X(ax, ax + (nx + 1) * ny), Y(ay, ay + nx * (ny + 1));
    int64_t gx = nx, gy = ny;
    const bool face = ctx->p.boundary == TPMG_BC_FACE;
    for (int l = ctx->L; l >= 1; --l) {
        LevelData& L = ctx->lv[l];
        const int64_t lnx = L.lc.nx, lny = L.lc.ny, y0 = ctx->y0 >> (ctx->L - l), ncol = lnx * lny;
        std::vector<double> F(6 * (size_t)ncol);
        for (int64_t j = 0; j < lny; ++j)
            for (int64_t i = 0; i < lnx; ++i) {
                const int64_t J = y0 + j, c = j * lnx + i;
                const double w = X[J * (gx + 1) + i], e = X[J * (gx + 1) + i + 1];
                const double s = Y[J * gx + i], n = Y[(J + 1) * gx + i];
                double aT = (w + e) + (s + n);
                if (face) aT += (i == 0 ? w : 0.0) + (i == gx - 1 ? e : 0.0) + (J == 0 ? s : 0.0) + (J == gy - 1 ? n : 0.0);
                F[c] = A[J * gx + i];
                F[ncol + c] = aT;
                F[2 * ncol + c] = w;
                F[3 * ncol + c] = e;
                F[4 * ncol + c] = s;
                F[5 * ncol + c] = n;
            }
        TRY(dev_alloc(ctx, &L.d_fld, F.size()));
        CUDA_TRY(ctx, cudaMemcpy(L.d_fld, F.data(), sizeof(double) * F.size(), cudaMemcpyHostToDevice));
        if (l > 1) {   // [R26] one level down
            const int64_t cx = gx / 2, cy = gy / 2;
            std::vector<double> Ac(cx * cy), Xc((cx + 1) * cy), Yc(cx * (cy + 1));
            for (int64_t J = 0; J < cy; ++J)
                for (int64_t I = 0; I < cx; ++I)
                    Ac[J * cx + I] = 0.25 * ((A[(2 * J) * gx + 2 * I] + A[(2 * J) * gx + 2 * I + 1]) +
                                             (A[(2 * J + 1) * gx + 2 * I] + A[(2 * J + 1) * gx + 2 * I + 1]));
            for (int64_t J = 0; J < cy; ++J)
                for (int64_t I = 0; I <= cx; ++I)
                    Xc[J * (cx + 1) + I] = 0.125 * (X[(2 * J) * (gx + 1) + 2 * I] + X[(2 * J + 1) * (gx + 1) + 2 * I]);
            for (int64_t J = 0; J <= cy; ++J)
                for (int64_t I = 0; I < cx; ++I)
                    Yc[J * cx + I] = 0.125 * (Y[(2 * J) * gx + 2 * I] + Y[(2 * J) * gx + 2 * I + 1]);
            A.swap(Ac);
            X.swap(Xc);
            Y.swap(Yc);
            gx = cx;
            gy = cy;
        }
    }
    ctx->fields = true;
    return fields_profile_tables(ctx);
}

tpmg_status tpmg_set_profiles(tpmg_ctx* ctx, const double* a, const double* b, const double* c, const double* d)
{
    if (!ctx) return TPMG_E_PARAM;
    const int nz = ctx->p.nz;
    if (a || b || c || d) {
        if (!a || !b || !c || !d) return fail(ctx, TPMG_E_PARAM, "tpmg_set_profiles: give all four profiles or none");
        for (int k = 0; k < nz; ++k) {
            if (!(a[k] >= 0) || !(b[k] <= 0) || !(c[k] <= 0) || !(d[k] > 0))
                return fail(ctx, TPMG_E_PARAM, "tpmg_set_profiles: need a >= 0, b <= 0, c <= 0, d > 0 (k = %d)", k);
            if (k + 1 < nz && b[k + 1] != c[k])
                return fail(ctx, TPMG_E_PARAM, "tpmg_set_profiles: b[%d] != c[%d] (A must be symmetric)", k + 1, k);
        }
        if (b[0] != 0.0 || c[nz - 1] != 0.0)
            return fail(ctx, TPMG_E_PARAM, "tpmg_set_profiles: b[0] and c[nz-1] must be 0 (no coupling outside the column)");
        if (!ctx->use_tma) return fail(ctx, TPMG_E_PARAM, "tpmg_set_profiles: general profiles need the TMA loader");
        if (!line_gen_fits(nz)) return fail(ctx, TPMG_E_SHAPE, "tpmg_set_profiles: nz = %d too large for general profiles", nz);
        if (ctx->fields && !line_gen_fits(nz, 2))
            return fail(ctx, TPMG_E_SHAPE, "tpmg_set_profiles: nz = %d too large for per-column fields", nz);
    }
    CUDA_TRY(ctx, cudaStreamSynchronize(ctx->stream));   // queued kernels may still read the tables
    const double* prof[4] = {a, b, c, d};
    return build_tables(ctx, a ? prof : nullptr);
}
