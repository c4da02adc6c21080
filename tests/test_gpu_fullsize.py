"""Parity at BASELINE.json's full size (configs[1]: 1024 x 1024 x 128), in the
launch configuration bench.py times (same library, same grid, default TMA
loader), on sampled outputs the oracle computes column by column, and on the
solves via properties that hold at any size plus the oracle's own solve."""
import numpy as np
import pytest

from oracle import oracle as O

from gpu_util import ctx_for, rel_l2

pytestmark = pytest.mark.gpu

N, NZ = 1024, 128
P = O.Params(nx=N, ny=N, nz=NZ)


@pytest.fixture(scope="module")
def setup():
    import torch
    from inputs import gpu as G
    ctx = ctx_for(P)
    u = ctx.empty(5)
    f = ctx.empty(5)
    G.fill_rhs(u, N, seed=11)
    G.fill_rhs(f, N, seed=12)
    torch.cuda.synchronize()
    u_zc = O.from_lambda(u.cpu().numpy())
    f_zc = O.from_lambda(f.cpu().numpy())
    rng = np.random.default_rng(0)
    # random columns plus the domain corners/edges and tile boundaries (tiles are 32 x 4)
    ii = list(rng.integers(0, N, 48)) + [0, N - 1, 0, N - 1, 31, 32, 511, 512, 5, 1000]
    jj = list(rng.integers(0, N, 48)) + [0, 0, N - 1, N - 1, 3, 4, 7, 8, N - 2, 1]
    return ctx, u, f, u_zc, f_zc, np.array(ii), np.array(jj)


def gpu_cols(t, ii, jj):
    """Columns (i, j) of a device field in Lambda layout -> (ncols, nz)."""
    import torch
    ti = torch.as_tensor(ii, device=t.device)
    tj = torch.as_tensor(jj, device=t.device)
    return t[tj, :, ti].cpu().numpy()


def test_fullsize_smooth_sampled(setup):
    ctx, u, f, u_zc, f_zc, ii, jj = setup
    out = u.clone()
    ctx.smooth(5, out, f, 1)
    want = O.smooth_cols(P, u_zc, f_zc, ii, jj)
    assert rel_l2(gpu_cols(out, ii, jj), want) < 1e-11


def test_fullsize_apply_precondition_residual_sampled(setup):
    ctx, u, f, u_zc, f_zc, ii, jj = setup
    y = ctx.empty(5)
    ctx.apply(5, u, y)
    assert rel_l2(gpu_cols(y, ii, jj), O.apply_cols(P, u_zc, ii, jj)) < 1e-11
    ctx.precondition(5, f, y)
    assert rel_l2(gpu_cols(y, ii, jj), O.precondition_cols(P, f_zc, ii, jj)) < 1e-11
    n2 = ctx.residual(5, u, f, y, want_norm2=True)
    assert rel_l2(gpu_cols(y, ii, jj), O.residual_cols(P, u_zc, f_zc, ii, jj)) < 1e-11
    r_full = O.residual(P, u_zc, f_zc)
    assert n2 == pytest.approx(float(np.sum(r_full * r_full)), rel=1e-12)


def test_fullsize_transfers(setup):
    ctx, u, f, u_zc, f_zc, ii, jj = setup
    fc = ctx.empty(4)
    ctx.restrict(5, u, fc)
    want = O.restrict(P, u_zc, 5)
    import torch
    torch.cuda.synchronize()
    assert rel_l2(O.from_lambda(fc.cpu().numpy()), want) < 1e-11
    uf = f.clone()
    ctx.prolong_add(4, fc, uf)
    assert rel_l2(O.from_lambda(uf.cpu().numpy()), O.prolong_add(P, want, f_zc, 4)) < 1e-11


@pytest.mark.parametrize("solver", ["mg", "cg"])
def test_fullsize_solve(setup, solver):
    """Solve of the bench workload: converged to 1e-5 as judged by the oracle's own
    residual of the GPU answer, and the oracle's solve takes the same number of
    iterations (+-1)."""
    ctx, u, f, u_zc, f_zc, ii, jj = setup
    x = ctx.empty(5)
    res = ctx.solve_mg(f, x) if solver == "mg" else ctx.solve_cg(f, x)
    assert res.converged
    x_zc = O.from_lambda(x.cpu().numpy())
    rr = np.linalg.norm(O.residual(P, x_zc, f_zc)) / np.linalg.norm(f_zc)
    assert rr < (1e-5 if solver == "mg" else 1.5e-5)
    ref = O.solve_mg(P, f_zc) if solver == "mg" else O.solve_cg(P, f_zc)
    assert abs(res.iterations - ref.iterations) <= 1
    if res.iterations == ref.iterations:
        assert rel_l2(x_zc, ref.u) < 1e-8
