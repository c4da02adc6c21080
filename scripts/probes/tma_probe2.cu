// Probe: which TMA tiled loads work for fp64 boxes with halo / negative coordinates.
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>
#include <cstdlib>

__device__ __forceinline__ uint32_t su(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__global__ void k(const __grid_constant__ CUtensorMap m, int x, int y, int z, int bytes, double* out, int n, int off)
{
    extern __shared__ __align__(128) double s[];
    __shared__ __align__(8) uint64_t bar;
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(su(&bar)));
        asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(su(&bar)), "r"(bytes) : "memory");
        asm volatile("cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];\n"
                     ::"r"(su(s + off)), "l"(reinterpret_cast<uint64_t>(&m)), "r"(x), "r"(y), "r"(z), "r"(su(&bar)) : "memory");
    }
    asm volatile("{\n.reg .pred p;\nW_%=:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n@!p bra W_%=;\n}\n" ::"r"(su(&bar)) : "memory");
    for (int i = threadIdx.x; i < n; i += blockDim.x) out[i] = s[i + off];
}

int main(int argc, char** argv)
{
    int only = argc > 1 ? atoi(argv[1]) : -1;
    PFN_cuTensorMapEncodeTiled_v12000 enc = nullptr;
    cudaDriverEntryPointQueryResult q;
    cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", (void**)&enc, cudaEnableDefault, &q);
    const int nx = 64, nz = 16, ny = 8;
    double* g; cudaMalloc(&g, sizeof(double) * nx * nz * ny);
    double* h = new double[nx * nz * ny];
    for (int i = 0; i < nx * nz * ny; ++i) h[i] = i + 1;
    cudaMemcpy(g, h, sizeof(double) * nx * nz * ny, cudaMemcpyHostToDevice);
    double* out; cudaMalloc(&out, sizeof(double) * 65536);
    struct Case { int bx, by; int x, y, z; int off; };
    Case cases[] = {{36, 1, -2, 0, 0, 0}, {36, 1, -2, 0, 0, 2}, {36, 1, -2, 0, 0, 6}, {36, 1, -2, 0, 0, 360},
                    {36, 1, -2, 0, 0, 16}, {36, 6, -2, 0, -1, 0}};
    int ci = -1;
    for (auto c : cases) {
        ++ci;
        if (only >= 0 && ci != only) continue;
        CUtensorMap m;
        cuuint64_t dims[3] = {nx, nz, ny};
        cuuint64_t str[2] = {nx * 8, (cuuint64_t)nx * nz * 8};
        cuuint32_t box[3] = {(cuuint32_t)c.bx, 8, (cuuint32_t)c.by};
        cuuint32_t es[3] = {1, 1, 1};
        CUresult r = enc(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, g, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                         CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        int n = c.bx * 8 * c.by;
        cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 100000);
        k<<<1, 128, n * 8 + 128 + c.off * 8>>>(m, c.x, c.y, c.z, n * 8, out, n, c.off);
        cudaError_t e = cudaDeviceSynchronize();
        double o[4] = {0};
        if (e == cudaSuccess) cudaMemcpy(o, out, sizeof o, cudaMemcpyDeviceToHost);
        printf("off=%d box(%d,8,%d) at (%d,%d,%d): encode=%d run=%s first=%g %g %g %g\n", c.off, c.bx, c.by, c.x, c.y, c.z, (int)r,
               cudaGetErrorString(e), o[0], o[1], o[2], o[3]);
        if (e != cudaSuccess) return 1;   // sticky
    }
    return 0;
}
