"""GPU parity with per-column horizontal fields |T|, alpha_{T,T'} (tpmg_set_fields;
eqn:LocalMatrixStencil P:250-257, coarse levels by reading R26) against the oracle with the
same fields: single operators on all levels (the per-column Thomas pivots of the line
kernel), the smoother, restriction through the V-cycle, both solves; with vertical profiles
and with the face-Dirichlet reading too."""
import numpy as np
import pytest

from oracle import oracle as O
from inputs import rhs_zc, horizontal_fields, vertical_profiles

from gpu_util import ctx_for, lib, rel_l2, to_dev, to_host_zc, close
from test_gpu_parity import rand

pytestmark = pytest.mark.gpu


def tol(p, level=None):
    """1e-11 or the forward-error bound of the column solve: kappa(M_T) <= (max diagonal +
    off-diagonals) / (min zero-order term) over the columns."""
    level = p.L if level is None else level
    area, _, _ = O.level_fields(p, level)
    a, b, c, d = p.profiles if p.profiles is not None else p.flat_profiles()
    _, ax, ay = O.level_fields(p, level)
    amax = 2 * (np.max(-ax) + np.max(-ay)) * (2 if p.boundary else 1)
    kappa = (np.max(area) * np.max(a - 2 * (b + c)) + amax * np.max(d)) / (np.min(area) * np.min(a))
    return max(1e-11, 8 * 2.2e-16 * kappa)


def F(nx, ny, nz, L, seed, kind="random", prof=None, **kw):
    base = O.Params(nx=nx, ny=ny, nz=nz, L=L)
    return O.Params(nx=nx, ny=ny, nz=nz, L=L, fields=horizontal_fields(nx, ny, base.c_h(), seed, kind),
                    profiles=vertical_profiles(nz, seed, prof) if prof else None, **kw)


SHAPES = [
    F(32, 32, 16, 5, 1),                          # C1-sized, L = 5, random fields
    F(80, 48, 64, 3, 2, "smooth"),                # ragged x tiles
    F(64, 32, 40, 2, 3, prof=50.0),               # nz = 40, with vertical profiles
    F(256, 256, 128, 5, 4),                       # paper's nz, many tiles
    F(48, 48, 32, 4, 5, boundary=1),              # face-Dirichlet reading [R25]
]
IDS = ["32x32x16", "80x48x64-smooth", "64x32x40-prof", "256x256x128", "48x48x32-face"]


def fctx(p):
    ctx = ctx_for(p)
    ctx.set_fields(*p.fields)
    return ctx


@pytest.mark.parametrize("p", SHAPES, ids=IDS)
def test_fields_ops_all_levels(p):
    ctx = fctx(p)
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


@pytest.mark.parametrize("p", SHAPES, ids=IDS)
def test_fields_vcycle(p):
    ctx = fctx(p)
    s = p.level_shape(p.L)
    u, f = rand(s, 5), rand(s, 6)
    du = to_dev(u)
    ctx.vcycle(du, to_dev(f))
    assert close(to_host_zc(du), O.vcycle(p, u, f), tol(p))


@pytest.mark.parametrize("solver", ["mg", "cg"])
@pytest.mark.parametrize("p", [SHAPES[0], SHAPES[1], SHAPES[4], F(128, 128, 128, 5, 7, "smooth")],
                         ids=["32x32x16", "80x48x64-smooth", "48x48x32-face", "128x128x128-smooth"])
def test_fields_solve_parity(p, solver):
    ctx = fctx(p)
    f = rhs_zc(p.nx, p.ny, p.nz, seed=0)
    u = ctx.empty(p.L)
    if solver == "mg":
        res, ref = ctx.solve_mg(to_dev(f), u, max_iter=200), O.solve_mg(p, f, max_iter=200)
    else:
        res, ref = ctx.solve_cg(to_dev(f), u, max_iter=2000), O.solve_cg(p, f, max_iter=2000)
    assert res.converged and ref.converged
    assert abs(res.iterations - ref.iterations) <= 1
    if res.iterations == ref.iterations:
        assert close(to_host_zc(u), ref.u, 1e-8)
        assert np.allclose(res.history, ref.history, rtol=1e-7)


def test_fields_errors_and_reset():
    T = lib()
    p = SHAPES[0]
    ctx = fctx(p)
    area, ax, ay = p.fields
    with pytest.raises(T.TpmgError, match="TPMG_E_PARAM"):
        ctx.set_fields(-area, ax, ay)
    with pytest.raises(T.TpmgError, match="TPMG_E_PARAM"):
        ctx.set_fields(area, -ax, ay)
    x = rand(p.level_shape(p.L), 3)
    # back to the uniform coefficients: the flat operator again
    ctx.set_fields()
    flat = O.Params(nx=p.nx, ny=p.ny, nz=p.nz, L=p.L)
    y = ctx.empty(p.L)
    ctx.apply(p.L, to_dev(x), y)
    assert close(to_host_zc(y), O.apply(flat, x), 1e-11)
    # flat fields given explicitly: the flat operator through the per-column kernels, every level
    ctx.set_fields(*flat.flat_fields())
    for level in range(1, p.L + 1):
        xl = rand(p.level_shape(level), 9 + level)
        z = ctx.empty(level)
        ctx.precondition(level, to_dev(xl), z)
        assert close(to_host_zc(z), O.precondition(flat, xl, level), 1e-12)
        ctx.apply(level, to_dev(xl), z)
        assert close(to_host_zc(z), O.apply(flat, xl, level), 1e-12)


def test_fields_with_profiles_either_order():
    p = SHAPES[2]
    x, f = rand(p.level_shape(p.L), 1), rand(p.level_shape(p.L), 2)
    for order in ("fields-first", "profiles-first"):
        ctx = ctx_for(O.Params(nx=p.nx, ny=p.ny, nz=p.nz, L=p.L))
        if order == "fields-first":
            ctx.set_fields(*p.fields)
            ctx.set_profiles(*p.profiles)
        else:
            ctx.set_profiles(*p.profiles)
            ctx.set_fields(*p.fields)
        du = to_dev(x)
        ctx.smooth(p.L, du, to_dev(f), 1)
        assert close(to_host_zc(du), O.smooth(p, x, f, p.L, 1), tol(p))
