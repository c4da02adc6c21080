"""GPU parity with general vertical profiles a, b, c, d (tpmg_set_profiles;
eqn:LocalMatrixStencil P:250-257) against the oracle with the same profiles: single
operators on all levels, the smoother, the V-cycle and both solves, with the k-split
kernels and with the one-thread-per-column kernels, plus the face-Dirichlet reading."""
import numpy as np
import pytest

from oracle import oracle as O
from inputs import rhs_zc, vertical_profiles

from gpu_util import ctx_for, lib, rel_l2, to_dev, to_host_zc, close
from test_gpu_parity import rand

pytestmark = pytest.mark.gpu


def tol(p, level=None):
    """1e-11, or the forward-error bound of the column solve (the profile couplings reach
    `coupling` x 4 relative to the zero-order term: kappa(M_T) up to ~1e3 here)."""
    level = p.L if level is None else level
    a, b, c, d = p.profiles
    c_l = p.c_h(level)
    diag = a - b - c + 4 * c_l * d
    kappa = np.max(diag + np.abs(b) + np.abs(c)) / np.min(a + 4 * c_l * d)
    return max(1e-11, 8 * 2.2e-16 * kappa)


def P(nx, ny, nz, L, seed, coupling, **kw):
    return O.Params(nx=nx, ny=ny, nz=nz, L=L, profiles=vertical_profiles(nz, seed, coupling), **kw)


SHAPES = [
    P(32, 32, 16, 5, 1, 200.0),                 # C1-sized, L = 5
    P(80, 48, 64, 3, 2, 1000.0),                # k-split with 2 segments, ragged x tiles
    P(64, 32, 40, 2, 3, 50.0),                  # nz = 40: one-thread-per-column kernels only
    P(256, 256, 128, 5, 4, 3000.0),             # paper's nz, many tiles
    P(48, 48, 32, 4, 5, 500.0, boundary=1),     # with the face-Dirichlet reading [R25]
]
IDS = ["32x32x16", "80x48x64", "64x32x40", "256x256x128", "48x48x32-face"]


@pytest.mark.parametrize("loader", ["tma", "tma-noks"])
@pytest.mark.parametrize("p", SHAPES, ids=IDS)
def test_profiles_ops_all_levels(p, loader):
    ctx = ctx_for(p, loader=loader)
    for level in range(1, p.L + 1):
        s = p.level_shape(level)
        x, f = rand(s, 1 + level), rand(s, 100 + level)
        dx, df = to_dev(x), to_dev(f)
        y = ctx.empty(level)
        ctx.apply(level, dx, y)
        assert close(to_host_zc(y), O.apply(p, x, level), tol(p, level))
        r = ctx.empty(level)
        n2 = ctx.residual(level, dx, df, r, want_norm2=True)
        want = O.residual(p, x, f, level)
        assert close(to_host_zc(r), want, tol(p, level))
        assert n2 == pytest.approx(float(np.sum(want * want)), rel=1e-10)
        z = ctx.empty(level)
        ctx.precondition(level, df, z)
        assert close(to_host_zc(z), O.precondition(p, f, level), tol(p, level))
        for sweeps in (1, 2):
            du = to_dev(x)
            ctx.smooth(level, du, df, sweeps)
            assert close(to_host_zc(du), O.smooth(p, x, f, level, sweeps), tol(p, level))


@pytest.mark.parametrize("loader", ["tma", "tma-noks"])
@pytest.mark.parametrize("p", SHAPES, ids=IDS)
def test_profiles_vcycle(p, loader):
    ctx = ctx_for(p, loader=loader)
    s = p.level_shape(p.L)
    u, f = rand(s, 5), rand(s, 6)
    du = to_dev(u)
    ctx.vcycle(du, to_dev(f))
    assert close(to_host_zc(du), O.vcycle(p, u, f), tol(p))


@pytest.mark.parametrize("solver", ["mg", "cg"])
@pytest.mark.parametrize("p", [SHAPES[0], SHAPES[1], P(128, 128, 128, 5, 7, 2000.0)],
                         ids=["32x32x16", "80x48x64", "128x128x128"])
def test_profiles_solve_parity(p, solver):
    ctx = ctx_for(p)
    f = rhs_zc(p.nx, p.ny, p.nz, seed=0)
    u = ctx.empty(p.L)
    if solver == "mg":
        res, ref = ctx.solve_mg(to_dev(f), u, max_iter=100), O.solve_mg(p, f, max_iter=100)
    else:
        res, ref = ctx.solve_cg(to_dev(f), u), O.solve_cg(p, f)
    assert res.converged and ref.converged
    assert abs(res.iterations - ref.iterations) <= 1
    if res.iterations == ref.iterations:
        assert close(to_host_zc(u), ref.u, 1e-8)
        assert np.allclose(res.history, ref.history, rtol=1e-7)


def test_profiles_errors_and_reset():
    T = lib()
    p = SHAPES[0]
    ctx = ctx_for(p)
    a, b, c, d = p.profiles
    c2 = c.copy()
    c2[3] *= 1.5
    with pytest.raises(T.TpmgError, match="TPMG_E_PARAM"):
        ctx.set_profiles(a, b, c2, d)
    # back to the flat box: the default operator again
    ctx.set_profiles()
    flat = O.Params(nx=p.nx, ny=p.ny, nz=p.nz, L=p.L)
    x = rand(p.level_shape(p.L), 3)
    y = ctx.empty(p.L)
    ctx.apply(p.L, to_dev(x), y)
    assert close(to_host_zc(y), O.apply(flat, x), 1e-11)
    # flat profiles given explicitly: bit-identical to the default tables
    ctx.set_profiles(*flat.flat_profiles())
    y2 = ctx.empty(p.L)
    ctx.apply(p.L, to_dev(x), y2)
    assert close(to_host_zc(y2), O.apply(flat, x), 1e-11)
