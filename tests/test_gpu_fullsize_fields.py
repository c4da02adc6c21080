"""Parity with per-column fields (tpmg_set_fields, smooth kind -- the `bench.py --fields
smooth` workload) at BASELINE.json's full size 1024 x 1024 x 128, in the launch
configuration bench.py times: sampled columns of the fused operators against the oracle's
column functions on the same full-size fields, and the MG solve judged by the oracle's own
residual of the GPU answer and its iteration count."""
import numpy as np
import pytest

from oracle import oracle as O
from inputs import horizontal_fields

from gpu_util import ctx_for, rel_l2
from test_gpu_fullsize import gpu_cols
from test_gpu_parity_fields import tol

pytestmark = pytest.mark.gpu

N, NZ = 1024, 128
P = O.Params(nx=N, ny=N, nz=NZ, fields=horizontal_fields(N, N, 8.4 * 8.4 / 4, 1, "smooth"))


@pytest.fixture(scope="module")
def setup():
    import torch
    from inputs import gpu as G
    ctx = ctx_for(P)
    ctx.set_fields(*P.fields)
    u = ctx.empty(5)
    f = ctx.empty(5)
    G.fill_rhs(u, N, seed=21)
    G.fill_rhs(f, N, seed=22)
    torch.cuda.synchronize()
    u_zc = O.from_lambda(u.cpu().numpy())
    f_zc = O.from_lambda(f.cpu().numpy())
    rng = np.random.default_rng(1)
    ii = list(rng.integers(0, N, 40)) + [0, N - 1, 0, N - 1, 31, 32, 511, 512]
    jj = list(rng.integers(0, N, 40)) + [0, 0, N - 1, N - 1, 3, 4, 7, 8]
    return ctx, u, f, u_zc, f_zc, np.array(ii), np.array(jj)


def test_fullsize_fields_ops_sampled(setup):
    ctx, u, f, u_zc, f_zc, ii, jj = setup
    t = tol(P)
    out = u.clone()
    ctx.smooth(5, out, f, 1)
    assert rel_l2(gpu_cols(out, ii, jj), O.smooth_cols(P, u_zc, f_zc, ii, jj)) < t
    y = ctx.empty(5)
    ctx.apply(5, u, y)
    assert rel_l2(gpu_cols(y, ii, jj), O.apply_cols(P, u_zc, ii, jj)) < t
    ctx.precondition(5, f, y)
    assert rel_l2(gpu_cols(y, ii, jj), O.precondition_cols(P, f_zc, ii, jj)) < t
    ctx.residual(5, u, f, y, want_norm2=True)
    assert rel_l2(gpu_cols(y, ii, jj), O.residual_cols(P, u_zc, f_zc, ii, jj)) < t


def test_fullsize_fields_mg_solve(setup):
    ctx, u, f, u_zc, f_zc, ii, jj = setup
    x = ctx.empty(5)
    res = ctx.solve_mg(f, x, max_iter=60)
    assert res.converged
    x_zc = O.from_lambda(x.cpu().numpy())
    assert np.linalg.norm(O.residual(P, x_zc, f_zc)) / np.linalg.norm(f_zc) < 1e-5
    ref = O.solve_mg(P, f_zc, max_iter=60)
    assert abs(res.iterations - ref.iterations) <= 1
