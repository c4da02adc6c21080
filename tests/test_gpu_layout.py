"""The paper's total-solution-time path: z-contiguous host fields, transposed to
the Lambda layout on the GPU (tpmg_transpose), solved, transposed back
(tpmg_solve_host_zc).  The transpose is data movement: bit-exact against numpy."""
import numpy as np
import pytest

from oracle import oracle as O
from inputs import rhs_zc

from gpu_util import ctx_for, lib, rel_l2

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("shape", [(80, 48, 40, 3), (64, 64, 128, 2), (32, 32, 16, 5)],
                         ids=["80x48x40", "64x64x128", "32x32x16"])
def test_transpose_bit_exact(shape):
    import torch
    T = lib()
    nx, ny, nz, L = shape
    p = O.Params(nx=nx, ny=ny, nz=nz, L=L)
    ctx = ctx_for(p)
    for level in (L, max(1, L - 1)):
        s = p.level_shape(level)   # (ny, nx, nz): the oracle's z-contiguous shape
        x = np.random.default_rng(level).standard_normal(s)
        src = torch.from_numpy(x).cuda()
        lam = ctx.empty(level)
        ctx.transpose(level, T.TPMG_ZC_TO_LAMBDA, src, lam)
        torch.cuda.synchronize()
        assert np.array_equal(lam.cpu().numpy(), O.to_lambda(x))
        back = torch.empty_like(src)
        ctx.transpose(level, T.TPMG_LAMBDA_TO_ZC, lam, back)
        torch.cuda.synchronize()
        assert np.array_equal(back.cpu().numpy(), x)
    full = ctx.empty(L)
    with pytest.raises(T.TpmgError, match="TPMG_E_PARAM"):
        ctx.transpose(L, T.TPMG_ZC_TO_LAMBDA, full, full)
    with pytest.raises(T.TpmgError, match="TPMG_E_PARAM"):
        ctx.transpose(L, 7, full, ctx.empty(L))


@pytest.mark.parametrize("solver", ["mg", "cg"])
def test_solve_host_zc_matches_oracle(solver):
    import torch
    T = lib()
    p = O.Params(nx=64, ny=64, nz=32, L=4)
    ctx = ctx_for(p)
    f = rhs_zc(p.nx, p.ny, p.nz, seed=3)
    fh = torch.from_numpy(f).pin_memory()
    uh = torch.empty_like(fh).pin_memory()
    sv = T.TPMG_SOLVER_MG if solver == "mg" else T.TPMG_SOLVER_CG
    res = ctx.solve_host_zc(sv, fh, uh)
    ref = O.solve_mg(p, f) if solver == "mg" else O.solve_cg(p, f)
    assert res.converged and abs(res.iterations - ref.iterations) <= 1
    if res.iterations == ref.iterations:
        assert rel_l2(uh.numpy(), ref.u) < 1e-9
    # and the Lambda-layout host path gives the same answer
    fl = torch.from_numpy(O.to_lambda(f)).pin_memory()
    ul = torch.empty_like(fl).pin_memory()
    ctx.solve_host(sv, fl, ul)
    assert np.array_equal(O.from_lambda(ul.numpy()), uh.numpy())
