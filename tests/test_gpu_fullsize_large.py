"""Sampled parity at the large BASELINE configurations on one GPU: configs[3]'s per-GPU
grid (2048 x 2048 x 128) and configs[4]'s whole grid (4096 x 4096 x 128, 2^31 unknowns,
16 GiB per vector), in the launch configuration bench.py times (same library, default
kernels; the wide-grid CG direction launch included through the sampled CG step).

The oracle evaluates single columns.  It only reads a column's 3 x 3 neighbourhood, so
its input arrays are lazily allocated zero arrays (np.zeros: untouched pages cost no
RAM) into which just those neighbourhoods are copied from the GPU."""
import numpy as np
import pytest

from oracle import oracle as O

from gpu_util import ctx_for, rel_l2

pytestmark = pytest.mark.gpu

SIZES = [2048, 4096]


def sample_columns(n, seed):
    rng = np.random.default_rng(seed)
    ii = list(rng.integers(0, n, 24)) + [0, n - 1, 0, n - 1, 31, 32, n // 2, n - 33, 1]
    jj = list(rng.integers(0, n, 24)) + [0, 0, n - 1, n - 1, 3, 4, n // 2 - 1, n - 5, n - 2]
    return np.array(ii, dtype=np.int64), np.array(jj, dtype=np.int64)


def gpu_cols(t, ii, jj):
    import torch
    ti = torch.as_tensor(ii, device=t.device)
    tj = torch.as_tensor(jj, device=t.device)
    return t[tj, :, ti].cpu().numpy()


def sparse_zc(t, ii, jj, n, nz):
    """Lazy zero array (ny, nx, nz) holding the 3 x 3 column neighbourhoods of the samples."""
    out = np.zeros((n, n, nz))
    for di in (-1, 0, 1):
        for dj in (-1, 0, 1):
            ci, cj = ii + di, jj + dj
            ok = (ci >= 0) & (ci < n) & (cj >= 0) & (cj < n)
            out[cj[ok], ci[ok], :] = gpu_cols(t, ci[ok], cj[ok])
    return out


@pytest.mark.parametrize("n", SIZES)
def test_large_grid_sampled_ops(n):
    import torch
    from inputs import gpu as G
    nz = 128
    P = O.Params(nx=n, ny=n, nz=nz)
    ctx = ctx_for(P)
    u = ctx.empty(5)
    f = ctx.empty(5)
    G.fill_rhs(u, n, seed=21)
    G.fill_rhs(f, n, seed=22)
    torch.cuda.synchronize()
    ii, jj = sample_columns(n, n)
    u_zc = sparse_zc(u, ii, jj, n, nz)
    f_zc = sparse_zc(f, ii, jj, n, nz)
    y = ctx.empty(5)
    ctx.apply(5, u, y)
    assert rel_l2(gpu_cols(y, ii, jj), O.apply_cols(P, u_zc, ii, jj)) < 1e-11
    ctx.precondition(5, f, y)
    assert rel_l2(gpu_cols(y, ii, jj), O.precondition_cols(P, f_zc, ii, jj)) < 1e-11
    ctx.residual(5, u, f, y)
    assert rel_l2(gpu_cols(y, ii, jj), O.residual_cols(P, u_zc, f_zc, ii, jj)) < 1e-11
    ctx.smooth(5, u, f, 1)          # in place: u <- u + rho M^-1 (f - A u)
    assert rel_l2(gpu_cols(u, ii, jj), O.smooth_cols(P, u_zc, f_zc, ii, jj)) < 1e-11
    del u, f, y
    torch.cuda.empty_cache()


@pytest.mark.parametrize("n", SIZES)
def test_large_grid_cg_first_iteration(n):
    """One PCG iteration from u = 0 (the CG direction and preconditioner kernels at this
    width): u_1 = alpha z_0 with z_0 = M^-1 f, alpha = <f, z_0> / <z_0, A z_0>.  Checked
    column-wise against the oracle's M^-1 and A, with the global alpha from the GPU's
    reduction cross-checked by the identity <f, z_0> = sum over columns (host, fp64)."""
    import torch
    from inputs import gpu as G
    nz = 128
    P = O.Params(nx=n, ny=n, nz=nz)
    ctx = ctx_for(P)
    f = ctx.empty(5)
    G.fill_rhs(f, n, seed=23)
    u = ctx.empty(5)
    res = ctx.solve_cg(f, u, max_iter=1)
    assert res.iterations == 1
    z = ctx.empty(5)
    ctx.precondition(5, f, z)
    az = ctx.empty(5)
    ctx.apply(5, z, az)
    num = float(torch.sum(f * z))
    den = float(torch.sum(z * az))
    alpha = num / den
    ii, jj = sample_columns(n, n + 1)
    f_zc = sparse_zc(f, ii, jj, n, nz)
    z_ref = O.precondition_cols(P, f_zc, ii, jj)
    assert rel_l2(gpu_cols(z, ii, jj), z_ref) < 1e-11
    assert rel_l2(gpu_cols(u, ii, jj), alpha * z_ref) < 1e-9
    del f, u, z, az
    torch.cuda.empty_cache()
