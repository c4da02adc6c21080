/* Plain-C client of the C ABI (include/tpmg.h): host-only entry points, no GPU needed.
 * Built and run by tests/test_library_cpu.py::test_plain_c_client. */
#include <stdio.h>
#include <string.h>
#include "tpmg.h"

#define CHECK(c)                                                    \
    do {                                                            \
        if (!(c)) {                                                 \
            fprintf(stderr, "check failed: %s (line %d)\n", #c, __LINE__); \
            return 1;                                               \
        }                                                           \
    } while (0)

int main(void)
{
    CHECK(tpmg_version() == 1);
    tpmg_params p;
    memset(&p, 0, sizeof p);
    tpmg_params_default(&p);
    CHECK(p.nz == 128 && p.levels == 5 && p.pre == 1 && p.post == 1 && p.coarse_sweeps == 2);
    CHECK(p.nu_cfl == 8.4 && p.H == 0.01 && p.lambda == 1.0 && p.boundary == TPMG_BC_GHOST_ZERO);
    p.nx = 1024;
    p.ny = 4096;
    /* rank 2 of 4: rows 2048..3071 of the finest level, 64 rows of the coarsest (L = 5) */
    int64_t y0 = -1, ny = -1;
    CHECK(tpmg_partition(&p, 2, 4, 5, &y0, &ny) == TPMG_OK && y0 == 2048 && ny == 1024);
    CHECK(tpmg_partition(&p, 2, 4, 1, &y0, &ny) == TPMG_OK && y0 == 128 && ny == 64);
    CHECK(tpmg_partition(&p, 0, 4, 6, &y0, &ny) == TPMG_E_RANGE);
    /* parameter errors are reported before any device work */
    tpmg_ctx *ctx = NULL;
    tpmg_params bad = p;
    bad.rho = 2.5;
    CHECK(tpmg_create(&bad, 0, 1, NULL, 0, NULL, &ctx) == TPMG_E_PARAM && ctx == NULL);
    bad = p;
    bad.nx = 1000; /* not divisible by 2^(L-1) = 16 */
    CHECK(tpmg_create(&bad, 0, 1, NULL, 0, NULL, &ctx) == TPMG_E_SHAPE);
    bad = p;
    bad.boundary = 7;
    CHECK(tpmg_create(&bad, 0, 1, NULL, 0, NULL, &ctx) == TPMG_E_PARAM);
    CHECK(tpmg_create(&p, 4, 4, NULL, 0, NULL, &ctx) == TPMG_E_TOPOLOGY);
    CHECK(strlen(tpmg_last_error(NULL)) > 0);
    printf("abi_host ok: %s\n", tpmg_last_error(NULL));
    return 0;
}
