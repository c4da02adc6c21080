// device_util.cuh -- sm_100a device helpers shared by the line kernels:
// cp.async, mbarrier + TMA bulk tensor copies, warp / deterministic grid reductions.
#pragma once
#include <cstdint>
#include <cuda.h>
#include <cuda_runtime.h>

#include "kernels.cuh"

namespace tpmg {
namespace dev {

// Programmatic dependent launch (sm_90+): wait for the previous kernel in the stream to
// complete and flush (a no-op when the kernel was launched without the attribute), and
// allow the next kernel to be scheduled once every CTA of this one has started.
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;\n" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;\n" ::: "memory"); }

// ---- fused halo push (P2P mode): a producer kernel stores its strip-boundary output rows
// straight into the neighbours' halo slabs over NVLink (the stream publishes the epoch).
__device__ __forceinline__ void push_out(const HaloPush& p, int64_t j, int64_t ny, int64_t off, double x)
{
    if (j == 0 && p.dst_lo) p.dst_lo[off] = x;
    if (j == ny - 1 && p.dst_hi) p.dst_hi[off] = x;
}


__device__ __forceinline__ void cp_async8(double* dst, const double* src, bool valid)
{
    unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(dst));
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(s), "l"(src),
                 "r"(valid ? 8 : 0)
                 : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N) : "memory"); }

__device__ __forceinline__ double warp_sum(double v)
{
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

// Deterministic grid reduction of NR values (see ReduceSlot).
template <int NR>
__device__ void grid_reduce(const ReduceSlot& red, const double (&acc)[NR > 0 ? NR : 1], double* scratch)
{
    if constexpr (NR > 0) {
        const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nw = blockDim.x >> 5;
        __shared__ bool is_last;
#pragma unroll
        for (int r = 0; r < NR; ++r) {
            double v = warp_sum(acc[r]);
            if (lane == 0) scratch[r * 32 + warp] = v;
        }
        __syncthreads();
        if (tid == 0) {
#pragma unroll
            for (int r = 0; r < NR; ++r) {
                double s = 0.0;
                for (int w = 0; w < nw; ++w) s += scratch[r * 32 + w];
                red.partials[(size_t)blockIdx.x * NR + r] = s;
            }
            __threadfence();
            unsigned t = atomicAdd(red.ticket, 1u);
            is_last = (t == gridDim.x - 1);
        }
        __syncthreads();
        if (is_last && warp == 0) {
            __threadfence();
#pragma unroll
            for (int r = 0; r < NR; ++r) {
                double s = 0.0;
                for (unsigned b = lane; b < gridDim.x; b += 32) s += __ldcg(red.partials + (size_t)b * NR + r);
                s = warp_sum(s);
                if (lane == 0) red.result[r] = red.accumulate ? s + red.result[r] : s;
            }
            if (lane == 0) *red.ticket = 0u;
        }
    }
}

// ------------------------------------------------------------------ TMA (bulk tensor copies)

__device__ __forceinline__ uint32_t smem_u32(const void* p)
{
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count)
{
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes)
{
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity)
{
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "WAIT_%=:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
        "@!p bra WAIT_%=;\n"
        "}\n" ::"r"(smem_u32(bar)),
        "r"(parity)
        : "memory");
}
__device__ __forceinline__ void tma_load_3d(void* dst, const CUtensorMap* map, int x, int y, int z, uint64_t* bar)
{
    asm volatile(
        "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];\n" ::"r"(
            smem_u32(dst)),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(x), "r"(y), "r"(z), "r"(smem_u32(bar))
        : "memory");
}

// The same load with an L2 eviction-priority policy (createpolicy below): on wide grids the
// halo'd field's lines must survive in L2 until the neighbouring tiles read them again.
__device__ __forceinline__ void tma_load_3d_hint(void* dst, const CUtensorMap* map, int x, int y, int z,
                                                 uint64_t* bar, uint64_t policy)
{
    asm volatile(
        "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes.L2::cache_hint"
        " [%0], [%1, {%2, %3, %4}], [%5], %6;\n" ::"r"(smem_u32(dst)),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(x), "r"(y), "r"(z), "r"(smem_u32(bar)), "l"(policy)
        : "memory");
}
__device__ __forceinline__ uint64_t l2_policy_evict_last()
{
    uint64_t p;
    asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;\n" : "=l"(p));
    return p;
}
__device__ __forceinline__ uint64_t l2_policy_evict_first()
{
    uint64_t p;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;\n" : "=l"(p));
    return p;
}

// TMA store of a box from shared memory (bulk async-group of the issuing thread); the writers
// of the box fence.proxy.async before the barrier that precedes the issue.
__device__ __forceinline__ void tma_store_3d(const CUtensorMap* map, int x, int y, int z, const void* src)
{
    asm volatile("cp.async.bulk.tensor.3d.global.shared::cta.bulk_group [%0, {%1, %2, %3}], [%4];\n" ::"l"(
                     reinterpret_cast<uint64_t>(map)),
                 "r"(x), "r"(y), "r"(z), "r"(smem_u32(src))
                 : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;\n" ::: "memory"); }
template <int N>
__device__ __forceinline__ void bulk_wait_read() { asm volatile("cp.async.bulk.wait_group.read %0;\n" ::"n"(N) : "memory"); }
template <int N>
__device__ __forceinline__ void bulk_wait() { asm volatile("cp.async.bulk.wait_group %0;\n" ::"n"(N) : "memory"); }
__device__ __forceinline__ void fence_proxy_async_smem() { asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory"); }

// ------------------------------------------------------------------ Tensor Memory (TMEM)
// The line kernels use TMEM (512 columns x 128 lanes x 32 bit per SM) as per-thread scratch
// for the Thomas intermediates g'_k: thread t of warp w owns lane 32 w + t, level k sits in
// columns 2k, 2k+1 (lo, hi word of the double).  A warp may only touch its own 32-lane
// quarter (warp w % 4), so the kernels that use it have 4 warps per CTA.  Allocation: one
// warp, power of two >= 32 columns, address written to shared memory; the same warp frees.
template <uint32_t NCOL>
__device__ __forceinline__ void tmem_alloc(uint32_t* slot)
{
    static_assert(NCOL >= 32 && NCOL <= 512 && (NCOL & (NCOL - 1)) == 0, "TMEM columns: power of two in [32, 512]");
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;\n" ::"r"(smem_u32(slot)),
                 "n"(NCOL)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n" ::: "memory");
}
template <uint32_t NCOL>
__device__ __forceinline__ void tmem_dealloc(uint32_t taddr)
{
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;\n" ::"r"(taddr), "n"(NCOL) : "memory");
}
__device__ __forceinline__ void tmem_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory"); }
__device__ __forceinline__ void tmem_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory"); }
// one double into columns col, col+1 of this thread's lane (asynchronous; tmem_wait_st orders it)
__device__ __forceinline__ void tmem_st_f64(uint32_t taddr, double v)
{
    asm volatile("tcgen05.st.sync.aligned.32x32b.x2.b32 [%0], {%1, %2};\n" ::"r"(taddr), "r"(__double2loint(v)),
                 "r"(__double2hiint(v))
                 : "memory");
}
__device__ __forceinline__ void tmem_wait_st() { asm volatile("tcgen05.wait::st.sync.aligned;\n" ::: "memory"); }
// two doubles into columns col .. col+3 of this thread's lane
__device__ __forceinline__ void tmem_st_f64x2(uint32_t taddr, double v0, double v1)
{
    asm volatile("tcgen05.st.sync.aligned.32x32b.x4.b32 [%0], {%1, %2, %3, %4};\n" ::"r"(taddr),
                 "r"(__double2loint(v0)), "r"(__double2hiint(v0)), "r"(__double2loint(v1)), "r"(__double2hiint(v1))
                 : "memory");
}
// 16 doubles from columns col .. col+31 of this thread's lane (wait in the same statement)
__device__ __forceinline__ void tmem_ld_f64x16(uint32_t taddr, double (&v)[16])
{
    uint32_t r[32];
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, "
        "%15, %16, %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, %28, %29, %30, %31}, [%32];\n"
        "tcgen05.wait::ld.sync.aligned;\n"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]), "=r"(r[8]),
          "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]), "=r"(r[16]),
          "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]),
          "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
        : "r"(taddr)
        : "memory");
#pragma unroll
    for (int q = 0; q < 16; ++q) v[q] = __hiloint2double((int)r[2 * q + 1], (int)r[2 * q]);
}
// 8 doubles from columns col .. col+15 of this thread's lane; the wait is in the same asm
// statement, so no use of the registers can be scheduled before the data has arrived
__device__ __forceinline__ void tmem_ld_f64x8(uint32_t taddr, double (&v)[8])
{
    uint32_t r[16];
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, "
        "%15}, [%16];\n"
        "tcgen05.wait::ld.sync.aligned;\n"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]), "=r"(r[8]),
          "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
        : "r"(taddr)
        : "memory");
#pragma unroll
    for (int q = 0; q < 8; ++q) v[q] = __hiloint2double((int)r[2 * q + 1], (int)r[2 * q]);
}
__device__ __forceinline__ double tmem_ld_f64(uint32_t taddr)
{
    uint32_t lo, hi;
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x2.b32 {%0, %1}, [%2];\n"
        "tcgen05.wait::ld.sync.aligned;\n"
        : "=r"(lo), "=r"(hi)
        : "r"(taddr)
        : "memory");
    return __hiloint2double((int)hi, (int)lo);
}

// Wait until a halo epoch flag (written by a neighbour GPU's stream write-value into my
// memory) reaches `epoch`; acquire at system scope, then order later TMA (async-proxy) reads
// of the slab after it.
__device__ __forceinline__ void halo_flag_wait(const unsigned* flag, unsigned epoch)
{
    for (;;) {
        unsigned v;
        asm volatile("ld.acquire.sys.global.u32 %0, [%1];\n" : "=r"(v) : "l"(flag) : "memory");
        if ((int)(v - epoch) >= 0) break;
        __nanosleep(32);
    }
    asm volatile("fence.proxy.async.global;\n" ::: "memory");
}

// The loader of tile row [j0, j0 + ty) waits for the halo slabs it reads (row -1: flag[0], row ny:
// flag[1]); out of line, so the single-GPU hot loop carries no extra registers.
static __device__ __noinline__ void halo_tile_wait(const HaloWait& hw, int j0, int ty, int ny)
{
    if (j0 == 0 && hw.flag[0]) halo_flag_wait(hw.flag[0], hw.epoch);
    if (j0 + ty >= ny && hw.flag[1]) halo_flag_wait(hw.flag[1], hw.epoch);
}

// Dynamic shared memory available to a kernel: the opt-in maximum minus its static smem.
template <typename K>
size_t dyn_smem_limit(K kern)
{
    static int optin = 0;
    if (!optin) {
        int dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
    }
    cudaFuncAttributes fa{};
    cudaFuncGetAttributes(&fa, kern);
    return (size_t)optin > fa.sharedSizeBytes ? (size_t)optin - fa.sharedSizeBytes : 0;
}


}  // namespace dev
}  // namespace tpmg
