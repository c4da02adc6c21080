"""GPU parity of the face-Dirichlet boundary reading [R25] (params.boundary = 1)
against the CPU oracle: boundary columns carry their own line block (class tables
read per thread in boundary tiles), the prolongation reflects the coarse ghosts.
Same bar as test_gpu_parity.py; plus the sec:Robustness schedules solved on
the GPU with the oracle's iteration counts."""
import numpy as np
import pytest

from oracle import oracle as O
from inputs import mode_face_zc, rhs_zc

from gpu_util import ctx_for, rel_l2, to_dev, to_host_zc, close
from test_gpu_parity import tol, rand

pytestmark = pytest.mark.gpu

SHAPES = [
    O.Params(nx=32, ny=32, nz=16, boundary=1),                       # C1, L = 5 (coarsest 2 x 2)
    O.Params(nx=48, ny=48, nz=3, L=4, boundary=1),                   # ragged tiles, 6 x 6 coarsest
    O.Params(nx=80, ny=48, nz=64, L=3, boundary=1),                  # k-split, 2 segments, ragged x
    O.Params(nx=256, ny=256, nz=128, L=5, boundary=1),               # paper's nz, many tiles
    O.Params(nx=32, ny=16, nz=300, L=1, boundary=1),                 # one-thread-per-column fallback
    O.Params(nx=32, ny=32, nz=32, L=6, boundary=1),                  # coarsest 1 x 1: 4 boundary faces
]
IDS = [f"{p.nx}x{p.ny}x{p.nz}-L{p.L}" for p in SHAPES]
LOADERS = ["tma", "cpasync", "tma-noks", "tma-ks2"]


@pytest.mark.parametrize("loader", LOADERS)
@pytest.mark.parametrize("p", SHAPES, ids=IDS)
def test_face_ops_all_levels(p, loader):
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
        assert n2 == pytest.approx(float(np.sum(want * want)), rel=1e-12)
        z = ctx.empty(level)
        ctx.precondition(level, df, z)
        assert close(to_host_zc(z), O.precondition(p, f, level), tol(p, level))
        for sweeps in (1, 2):
            du = to_dev(x)
            ctx.smooth(level, du, df, sweeps)
            assert close(to_host_zc(du), O.smooth(p, x, f, level, sweeps), tol(p, level))
        if level > 1:
            fc = ctx.empty(level - 1)
            ctx.restrict(level, dx, fc)
            assert close(to_host_zc(fc), O.restrict(p, x, level), 1e-11)
            uc = rand(p.level_shape(level - 1), 30 + level)
            duf = to_dev(f)
            ctx.prolong_add(level - 1, to_dev(uc), duf)
            assert close(to_host_zc(duf), O.prolong_add(p, uc, f, level - 1), 1e-11)


@pytest.mark.parametrize("loader", LOADERS)
@pytest.mark.parametrize("p", SHAPES, ids=IDS)
def test_face_vcycle(p, loader):
    ctx = ctx_for(p, loader=loader)
    s = p.level_shape(p.L)
    u, f = rand(s, 5), rand(s, 6)
    du = to_dev(u)
    ctx.vcycle(du, to_dev(f))
    assert close(to_host_zc(du), O.vcycle(p, u, f), tol(p))


def test_face_eigenmode_closed_form():
    """A v = lambda v for the face sine mode, on the GPU (closed form, no oracle)."""
    import math
    p = O.Params(nx=64, ny=64, nz=32, L=1, boundary=1)
    v = mode_face_zc(64, 64, 32, 3, 5, 2)
    c, g = p.c_h(1), p.gamma()
    lam = 1 + 4 * c * (math.sin(3 * math.pi / 128) ** 2 + math.sin(5 * math.pi / 128) ** 2) + \
        4 * g * math.sin(2 * math.pi / 64) ** 2
    ctx = ctx_for(p)
    y = ctx.empty(1)
    ctx.apply(1, to_dev(v), y)
    assert close(to_host_zc(y), lam * v, 1e-12)


ROB = [(5, 8.4, 2), (5, 84.0, 30), (5, 840.0, 150), (7, 84.0, 5), (7, 840.0, 15)]


@pytest.mark.parametrize("L,nu,cs", ROB, ids=[f"L{a}-nu{b}-cs{c}" for a, b, c in ROB])
@pytest.mark.parametrize("loader", ["tma", "tma-noks"])
def test_face_robustness_solves(L, nu, cs, loader):
    """sec:Robustness schedules: GPU MG matches the oracle's iteration count (+-1)
    and converges in the same handful of cycles for nu from 8.4 to 840."""
    p = O.Params(nx=128, ny=128, nz=32, nu_cfl=nu, L=L, coarse_sweeps=cs, boundary=1)
    ctx = ctx_for(p, loader=loader)
    f = rhs_zc(128, 128, 32, seed=0)
    u = ctx.empty(p.L)
    res, ref = ctx.solve_mg(to_dev(f), u), O.solve_mg(p, f)
    assert res.converged and ref.converged and ref.iterations <= 12
    assert abs(res.iterations - ref.iterations) <= 1
    ug = to_host_zc(u)
    rr = np.linalg.norm(O.residual(p, ug, f)) / np.linalg.norm(f)
    assert rr < 1e-5


@pytest.mark.parametrize("solver", ["mg", "cg"])
def test_face_solve_parity(solver):
    p = O.Params(nx=128, ny=128, nz=128, boundary=1)
    ctx = ctx_for(p)
    f = rhs_zc(128, 128, 128, seed=0)
    u = ctx.empty(p.L)
    if solver == "mg":
        res, ref = ctx.solve_mg(to_dev(f), u), O.solve_mg(p, f)
    else:
        res, ref = ctx.solve_cg(to_dev(f), u), O.solve_cg(p, f)
    assert res.converged and ref.converged
    assert abs(res.iterations - ref.iterations) <= 1
    if res.iterations == ref.iterations:
        assert close(to_host_zc(u), ref.u, 1e-9)
        assert np.allclose(res.history, ref.history, rtol=1e-8)
