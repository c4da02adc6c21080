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
