"""Pins of the oracle's face-Dirichlet boundary reading [R25] (params.boundary = 1).

[R25]: "homogeneous Dirichlet boundary conditions ... in the horizontal direction"
 on the cell-centred finite-volume grid with the boundary value on
the boundary FACE: a boundary face contributes 2 alpha_{T,T'} to alpha_T
(eqn:LocalMatrixStencil), i.e. ghost = -u, and the prolongation continues
the coarse field linearly through 0 on the face.  sec:Robustness is the
paper's behavioural pin: with 7 or 10 levels, or 5 levels and more coarse sweeps, MG
iterations stay flat up to nu_CFL = 840.

As in test_oracle_pins.py, nothing here re-types an oracle formula: the pins are
closed-form eigenpairs (sine modes vanishing on the faces), dense numpy solves and
spectra on tiny cases, hand-computed prolongation weights, exactness of the bilinear
interpolation on fields that vanish on the faces, and the paper's robustness text.
"""
import math

import numpy as np
import pytest

from oracle import oracle as O
from inputs import mode_face_zc, rhs_zc


def sin2(x):
    return math.sin(x) ** 2


def eig_face(p: O.Params, level, pp, qq, rr):
    """lambda_pqr = 1 + 4c [sin^2(p pi/(2 nx)) + sin^2(q pi/(2 ny))] + 4 gamma sin^2(r pi/(2 nz))
    for the face-Dirichlet cell-centred modes sin(p pi (i+1/2)/nx) ... (0-based i)."""
    ny, nx, nz = p.level_shape(level)
    c, g = p.c_h(level), p.gamma()
    return (1 + 4 * c * (sin2(pp * math.pi / (2 * nx)) + sin2(qq * math.pi / (2 * ny)))
            + 4 * g * sin2(rr * math.pi / (2 * nz)))


def rel(a, b):
    return np.linalg.norm(np.ravel(a) - np.ravel(b)) / max(np.linalg.norm(np.ravel(b)), 1e-300)


def dense(p, fn, level):
    shape = p.level_shape(level)
    n = int(np.prod(shape))
    A = np.empty((n, n))
    e = np.zeros(n)
    for m in range(n):
        e[:] = 0.0
        e[m] = 1.0
        A[:, m] = fn(e.reshape(shape)).ravel()
    return A


def kappa_M(p: O.Params):
    """Condition number bound of the column blocks: error amplification of a stable solve."""
    return (1 + 4 * p.c_h() + 4 * p.gamma()) / (1 + 4 * p.c_h())


def nb_faces(nx, ny):
    """Number of boundary faces of every column, shape (ny, nx)."""
    i = np.arange(nx)[None, :]
    j = np.arange(ny)[:, None]
    return ((i == 0).astype(int) + (i == nx - 1) + (j == 0) + (j == ny - 1))


@pytest.mark.parametrize("nx,ny,nz,nu", [(6, 5, 4, 8.4), (8, 8, 16, 84.0), (12, 7, 3, 2.0), (1, 4, 2, 8.4)])
def test_face_fourier_eigenpairs(nx, ny, nz, nu):
    p = O.Params(nx=nx, ny=ny, nz=nz, nu_cfl=nu, L=1, boundary=1)
    for (pp, qq, rr) in [(1, 1, 0), (nx, ny, nz - 1), (min(2, nx), min(3, ny), min(1, nz - 1))]:
        v = mode_face_zc(nx, ny, nz, pp, qq, rr)
        lam = eig_face(p, 1, pp, qq, rr)
        bound = 1 + 12 * p.c_h() + 4 * p.gamma()
        assert np.max(np.abs(O.apply(p, v) - lam * v)) <= 32 * 2.2e-16 * bound


def test_face_dense_spectrum_spd_and_levels():
    """The assembled operator is symmetric, SPD, and its spectrum is exactly the closed-form
    set; coarse levels use c_h / 4^(L-l) with the same boundary reading."""
    p = O.Params(nx=6, ny=4, nz=3, L=1, boundary=1)
    A = dense(p, lambda x: O.apply(p, x), 1)
    assert np.max(np.abs(A - A.T)) <= 1e-12 * np.max(np.abs(A))
    ev = np.sort(np.linalg.eigvalsh(A))
    cf = np.sort([eig_face(p, 1, a, b, c) for a in range(1, 7) for b in range(1, 5) for c in range(3)])
    assert np.max(np.abs(ev - cf)) < 1e-13 * (1 + 12 * p.c_h() + 4 * p.gamma())
    assert ev[0] > 1.0
    q = O.Params(nx=32, ny=16, nz=8, L=4, boundary=1)
    for level in (1, 2, 3, 4):
        ny, nx, nz = q.level_shape(level)
        v = mode_face_zc(nx, ny, nz, 1, 2, 1)
        assert rel(O.apply(q, v, level), eig_face(q, level, 1, 2, 1) * v) < 1e-12


def test_face_differs_from_ghost_zero_only_on_boundary_columns():
    """A_face x - A_zero x = c * nb(T) * x (one extra alpha_{T,T'} per boundary face)."""
    p1 = O.Params(nx=8, ny=6, nz=5, L=1, boundary=1)
    p0 = O.Params(nx=8, ny=6, nz=5, L=1, boundary=0)
    rng = np.random.default_rng(4)
    x = rng.standard_normal(p1.level_shape(1))
    d = O.apply(p1, x) - O.apply(p0, x)
    want = p1.c_h() * nb_faces(8, 6)[:, :, None] * x
    assert np.max(np.abs(d - want)) < 1e-12 * np.max(np.abs(x)) * p1.c_h() * 8


@pytest.mark.parametrize("nz", [1, 4, 32])
def test_face_precondition_vertical_modes(nz):
    """M is the column block A_T, whose diagonal carries the column's own alpha_T:
    M^-1 (g(i,j) cos_r(k)) = g(i,j) cos_r(k) / (1 + (4 + nb(i,j)) c + 4 gamma sin^2(r pi/(2 nz)))."""
    p = O.Params(nx=7, ny=5, nz=nz, L=1, boundary=1)
    rng = np.random.default_rng(nz)
    g = rng.standard_normal((5, 7))
    nb = nb_faces(7, 5)
    for r in {0, nz // 2, nz - 1}:
        ck = np.cos(r * np.pi * (np.arange(nz) + 0.5) / nz)
        v = g[:, :, None] * ck[None, None, :]
        m = 1 + (4 + nb) * p.c_h() + 4 * p.gamma() * sin2(r * math.pi / (2 * nz))
        assert rel(O.precondition(p, v), v / m[:, :, None]) < 10 * kappa_M(p) * 2.2e-16


def test_face_precondition_is_block_of_A():
    p = O.Params(nx=8, ny=8, nz=12, L=1, boundary=1)
    rng = np.random.default_rng(5)
    z0 = np.zeros(p.level_shape(1))
    mask = np.zeros((8, 8), bool)
    mask[::2, ::2] = True
    mask[7, 7] = mask[7, 1] = mask[1, 7] = True   # boundary and corner columns, isolated
    z0[mask] = rng.standard_normal((mask.sum(), 12))
    Az = O.apply(p, z0)
    Az[~mask] = 0.0
    assert rel(O.precondition(p, Az), z0) < 10 * kappa_M(p) * 2.2e-16


def test_face_prolongation_weights_and_exactness():
    p = O.Params(nx=16, ny=12, nz=2, L=2, boundary=1)
    nyc, nxc, nz = p.level_shape(1)
    nyf, nxf, _ = p.level_shape(2)
    zero_f = np.zeros((nyf, nxf, nz))
    # interior unit: the same (1,3,3,1) x (1,3,3,1) / 16 patch as [R7]
    e = np.zeros((nyc, nxc, nz)); e[2, 3, :] = 1.0
    out = O.prolong_add(p, e, zero_f)
    w1 = np.array([1, 3, 3, 1])
    assert np.array_equal(out[3:7, 5:9, 0] * 16, np.outer(w1, w1))
    # corner unit, hand-computed with ghosts -1 (edges) and +1 (corner): fine (0,0)
    # 9 - 3 - 3 + 1 = 4; fine (i=1, j=0): 9 + 3*0 + 3*(-1) + (-0) = 6; fine (1,1): 9
    e = np.zeros((nyc, nxc, nz)); e[0, 0, :] = 1.0
    out = O.prolong_add(p, e, zero_f)
    assert out[0, 0, 0] * 16 == 4 and out[0, 1, 0] * 16 == 6 and out[1, 1, 0] * 16 == 9
    # bilinear interpolation is exact on a field that vanishes linearly on a face, the fine
    # cells next to that face included (the reflected ghost is the linear continuation):
    # u = X(x) Y(y) with X in {x, 1 - x}, Y in {y, 1 - y} (cell centres, unit square) is
    # reproduced everywhere except next to the two faces where it does not vanish
    X = (np.arange(nxc) + 0.5) / nxc; Y = (np.arange(nyc) + 0.5) / nyc
    x = (np.arange(nxf) + 0.5) / nxf; y = (np.arange(nyf) + 0.5) / nyf
    for flip_x in (False, True):
        for flip_y in (False, True):
            fx = (lambda s: 1 - s) if flip_x else (lambda s: s)
            fy = (lambda s: 1 - s) if flip_y else (lambda s: s)
            uc = np.repeat((fy(Y)[:, None] * fx(X)[None, :])[:, :, None], nz, axis=2)
            want = np.repeat((fy(y)[:, None] * fx(x)[None, :])[:, :, None], nz, axis=2)
            err = np.abs(O.prolong_add(p, uc, zero_f) - want)
            xs = slice(1, None) if flip_x else slice(0, -1)   # drop the column next to the non-zero face
            ys = slice(1, None) if flip_y else slice(0, -1)
            assert np.max(err[ys, xs]) < 1e-14
            assert np.max(err) > 1e-3   # ... where it is not exact


def test_face_restriction_unchanged():
    p1 = O.Params(nx=16, ny=8, nz=3, L=2, boundary=1)
    p0 = O.Params(nx=16, ny=8, nz=3, L=2, boundary=0)
    r = np.random.default_rng(0).standard_normal(p1.level_shape(2))
    assert np.array_equal(O.restrict(p1, r), O.restrict(p0, r))


def test_face_solvers_match_dense_solve():
    p = O.Params(nx=16, ny=16, nz=4, L=3, boundary=1)
    f = rhs_zc(16, 16, 4, seed=1)
    A = dense(p, lambda x: O.apply(p, x), 3)
    ustar = np.linalg.solve(A, f.ravel()).reshape(f.shape)
    cg = O.solve_cg(p, f, eps=1e-12)
    mg = O.solve_mg(p, f, eps=1e-12, max_iter=200)
    assert cg.converged and mg.converged
    assert rel(cg.u, ustar) < 1e-9 and rel(mg.u, ustar) < 1e-9
    assert rel(O.vcycle(p, ustar, f), ustar) < 1e-12   # fixed point


# the coarse-sweep schedules of sec:Robustness: (levels, nu_CFL, coarse sweeps)
ROBUSTNESS = [(5, 8.4, 2), (5, 16.8, 2), (5, 84.0, 30), (5, 840.0, 150),
              (7, 8.4, 2), (7, 84.0, 5), (7, 840.0, 15)]


def test_robustness_schedules_face_boundary():
    """"the number of iterations ... depends only weakly on the CFL number" with
    the stated coarse-sweep counts.  With face Dirichlet the MG iteration count at
    128^2 x 16 stays within 10..12 from nu = 8.4 to 840 for L = 5 and L = 7."""
    f = rhs_zc(128, 128, 16, seed=0)
    its = []
    for L, nu, cs in ROBUSTNESS:
        p = O.Params(nx=128, ny=128, nz=16, nu_cfl=nu, L=L, coarse_sweeps=cs, boundary=1)
        r = O.solve_mg(p, f, eps=1e-5, max_iter=40)
        assert r.converged, (L, nu, cs)
        its.append(r.iterations)
    assert max(its) <= 12 and max(its) - min(its) <= 2, its


def test_robustness_ghost_zero_reading_breaks_down():
    """Why [R25] exists: with ghost-zero Dirichlet [R1] the coarse operators put the boundary
    at a level-dependent position (h_l/2 outside the domain), and at nu = 84 the same
    schedule no longer converges (documented in DESIGN.md)."""
    f = rhs_zc(128, 128, 16, seed=0)
    p = O.Params(nx=128, ny=128, nz=16, nu_cfl=84.0, L=5, coarse_sweeps=30, boundary=0)
    r = O.solve_mg(p, f, eps=1e-5, max_iter=20)
    assert not r.converged and r.history[-1] > r.history[2]
