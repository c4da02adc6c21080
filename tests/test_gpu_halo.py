"""The multi-rank exchange kernels on ONE GPU (y-strips with halo width 1).

The 2- and 4-rank tests (test_gpu_multirank.py) need as many GPUs; these drive the same
kernels -- the P2P halo push (k_halo_push) and the CG p-halo update (k_cg_halo) -- through
the C ABI (tpmg_halo_push, tpmg_cg_halo) on strips of one global field, and compare the
slabs with the neighbour rows of the global field and with the arithmetic the neighbour
applies to its own rows.
"""
import numpy as np
import pytest

from oracle import oracle as O
from gpu_util import ctx_for, lib

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("nx,ny,nz,L,nstrips", [(64, 32, 16, 3, 2), (96, 64, 40, 3, 4), (32, 16, 128, 2, 2)])
def test_halo_push_delivers_neighbour_rows(nx, ny, nz, L, nstrips):
    import torch
    T = lib()
    rows = ny // nstrips
    ctx = ctx_for(O.Params(nx=nx, ny=rows, nz=nz, L=L))   # one strip's local box
    for level in range(1, L + 1):
        f = 1 << (L - level)
        nyl, nxl = ny // f, nx // f
        g = np.random.default_rng(level).standard_normal((nyl, nz, nxl))   # global field, Lambda order
        ryl = nyl // nstrips
        strips = [torch.from_numpy(np.ascontiguousarray(g[s * ryl:(s + 1) * ryl])).cuda() for s in range(nstrips)]
        lo = [torch.full((nz, nxl), np.nan, dtype=torch.float64, device="cuda") for _ in range(nstrips)]
        hi = [torch.full((nz, nxl), np.nan, dtype=torch.float64, device="cuda") for _ in range(nstrips)]
        for s in range(nstrips):   # strip s pushes row 0 down and row ryl-1 up, as api.cpp's exchange does
            T.tpmg_halo_push(ctx.handle, level, strips[s], hi[s - 1] if s > 0 else None,
                             lo[s + 1] if s < nstrips - 1 else None)
        torch.cuda.synchronize()
        for s in range(nstrips):
            if s > 0:       # my lo slab = the global row just below my strip
                assert np.array_equal(lo[s].cpu().numpy(), g[s * ryl - 1])
            else:           # physical boundary: nothing written
                assert np.isnan(lo[s].cpu().numpy()).all()
            if s < nstrips - 1:
                assert np.array_equal(hi[s].cpu().numpy(), g[(s + 1) * ryl])
            else:
                assert np.isnan(hi[s].cpu().numpy()).all()


def test_halo_push_rejects_bad_arguments():
    import torch
    T = lib()
    ctx = ctx_for(O.Params(nx=32, ny=16, nz=8, L=2))
    x = ctx.empty(2)
    with pytest.raises(T.TpmgError, match="TPMG_E_PARAM"):
        T.tpmg_halo_push(ctx.handle, 2, x, x[0].reshape(-1), None)   # destination inside src
    with pytest.raises(T.TpmgError, match="TPMG_E_RANGE"):
        T.tpmg_halo_push(ctx.handle, 3, x, None, None)
    with pytest.raises(ValueError):
        T.tpmg_halo_push(ctx.handle, 2, x, torch.empty(5, dtype=torch.float64, device="cuda"), None)


@pytest.mark.parametrize("beta", [0.0, 0.37, -1.5e3])
def test_cg_halo_matches_direction_update(beta):
    """out = beta p + z on the halo planes, rounded once (the fma k_line<CGDIR> applies to the
    neighbour's own rows, so the local p halo equals the neighbour's new p row)."""
    import torch
    T = lib()
    nx, ny, nz = 64, 32, 24
    ctx = ctx_for(O.Params(nx=nx, ny=ny, nz=nz, L=2))
    rng = np.random.default_rng(3)
    z_lo, p_lo, z_hi, p_hi = (rng.standard_normal((nz, nx)) for _ in range(4))
    dev = lambda a: torch.from_numpy(a).cuda()
    out_lo = torch.zeros((nz, nx), dtype=torch.float64, device="cuda")
    out_hi = torch.zeros_like(out_lo)
    T.tpmg_cg_halo(ctx.handle, beta, out_lo, dev(z_lo), dev(p_lo), out_hi, dev(z_hi), dev(p_hi))
    for out, z, p in ((out_lo, z_lo, p_lo), (out_hi, z_hi, p_hi)):
        want = (np.longdouble(beta) * p.astype(np.longdouble) + z.astype(np.longdouble)).astype(np.float64)
        got = out.cpu().numpy()
        ulp = np.spacing(np.maximum(np.abs(want), np.finfo(np.float64).tiny))
        assert np.all(np.abs(got - want) <= ulp)
    # one side only (a strip at the physical boundary): the other plane is untouched
    out_hi.fill_(7.0)
    T.tpmg_cg_halo(ctx.handle, beta, out_lo, dev(z_lo), dev(p_lo), None, None, None)
    torch.cuda.synchronize()
    assert (out_hi == 7.0).all()
