// splitmix_gpu.cu -- device twin of inputs/splitmix.py (seeded RHS generator).
// Holds none of the solver's arithmetic; bit-identical to the numpy version
// (pure uint64 integer work, then one exact int->double conversion and scaling).
#include <cstdint>
#include <cuda_runtime.h>

namespace {
__global__ void k_fill_rhs(double* __restrict__ dst, int64_t nx_glob, int64_t y0, int64_t ny, int nz,
                           uint64_t seed, int64_t n)
{
    for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < n; q += (int64_t)gridDim.x * blockDim.x) {
        // local Lambda index q = (j*nz + k)*nx + i  ->  global index G with j_g = y0 + j
        const int64_t i = q % nx_glob;
        const int64_t jk = q / nx_glob;
        const int64_t k = jk % nz, j = jk / nz;
        const uint64_t G = ((uint64_t)(y0 + j) * (uint64_t)nz + (uint64_t)k) * (uint64_t)nx_glob + (uint64_t)i;
        const uint64_t GOLDEN = 0x9E3779B97F4A7C15ull;
        uint64_t z = seed * GOLDEN + G + GOLDEN;
        z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
        z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
        z ^= z >> 31;
        dst[q] = (double)(z >> 11) * 0x1.0p-53 * 2.0 - 1.0;
    }
}
}  // namespace

extern "C" int tpmg_inputs_fill_rhs(double* dst, int64_t nx_glob, int64_t y0, int64_t ny, int32_t nz,
                                    uint64_t seed, void* stream)
{
    const int64_t n = nx_glob * ny * (int64_t)nz;
    if (n <= 0) return 0;
    int64_t blocks = (n + 255) / 256;
    if (blocks > 148 * 64) blocks = 148 * 64;
    k_fill_rhs<<<(unsigned)blocks, 256, 0, (cudaStream_t)stream>>>(dst, nx_glob, y0, ny, nz, seed, n);
    return (int)cudaGetLastError();
}
