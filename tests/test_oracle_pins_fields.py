"""Pins of the oracle with per-column horizontal fields (eqn:LocalMatrixStencil, P:250-257:
"the coefficients alpha_{T,T'} and alpha_T are different for each horizontal grid cell T (and
depend on the multigrid level)"): |T| per column and alpha_{T,T'} per face, alpha_T = the sum
over the column's 4 faces [R1] (boundary faces twice under [R25]), coarse levels by [R26].

What pins them (none of it re-runs the oracle's own loops):
  * an explicit edge-list assembly of the dense 3D matrix (column blocks
    |T| T_z - alpha_T D, face blocks alpha_TT' D) with numpy, compared with the oracle's
    stencil applied to unit vectors;
  * the closed-form spectrum of the anisotropic separable case (constant alpha_x != alpha_y);
  * per-column dense solves for M^-1, dense solves for CG / MG;
  * [R26] on constant fields reproduces the flat box's rediscretisation [R4] exactly, and the
    block mean reproduces a field linear in (i, j) at the coarse centres.
"""
import math

import numpy as np
import pytest

from oracle import oracle as O
from inputs import rhs_zc, horizontal_fields, vertical_profiles


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


def rel(a, b):
    return np.linalg.norm(np.ravel(a) - np.ravel(b)) / max(np.linalg.norm(np.ravel(b)), 1e-300)


def profiles_of(p):
    return p.profiles if p.profiles is not None else p.flat_profiles()


def assemble(p, fields, boundary):
    """Dense A from an explicit edge list, z-contiguous unknown order (j, i, k)."""
    area, ax, ay = fields
    ny, nx = area.shape
    nz = p.nz
    a, b, c, d = profiles_of(p)
    Tz = np.diag(a - b - c) + np.diag(b[1:], -1) + np.diag(c[:-1], 1)
    D = np.diag(d)
    n = nx * ny * nz
    A = np.zeros((n, n))
    col = lambda i, j: slice((j * nx + i) * nz, (j * nx + i + 1) * nz)
    # faces: (alpha, column on one side or None, column on the other side or None)
    faces = []
    for j in range(ny):
        for i in range(nx + 1):
            faces.append((ax[j, i], (i - 1, j) if i > 0 else None, (i, j) if i < nx else None))
    for j in range(ny + 1):
        for i in range(nx):
            faces.append((ay[j, i], (i, j - 1) if j > 0 else None, (i, j) if j < ny else None))
    alphaT = np.zeros((ny, nx))
    for al, s, t in faces:
        for cell in (s, t):
            if cell is not None:
                alphaT[cell[1], cell[0]] += al * (2.0 if (boundary and (s is None or t is None)) else 1.0)
        if s is not None and t is not None:
            A[col(*s), col(*t)] += al * D
            A[col(*t), col(*s)] += al * D
    for j in range(ny):
        for i in range(nx):
            A[col(i, j), col(i, j)] += area[j, i] * Tz - alphaT[j, i] * D
    return A


def test_flat_fields_reproduce_default():
    p = O.Params(nx=16, ny=16, nz=8, L=3)
    q = O.Params(nx=16, ny=16, nz=8, L=3, fields=p.flat_fields())
    x = rhs_zc(16, 16, 8, seed=3)
    for l in (3, 2, 1):
        xl = x[: p.level_shape(l)[0], : p.level_shape(l)[1]].copy()
        assert np.array_equal(O.precondition(p, xl, l), O.precondition(q, xl, l))   # same M_T, bitwise
        assert rel(O.apply(q, xl, l), O.apply(p, xl, l)) < 1e-15   # weighted vs plain neighbour sum
    assert rel(O.vcycle(q, np.zeros_like(x), x), O.vcycle(p, np.zeros_like(x), x)) < 1e-14
    assert O.solve_mg(q, x).iterations == O.solve_mg(p, x).iterations
    assert O.solve_cg(q, x).iterations == O.solve_cg(p, x).iterations


def test_coarsening_of_flat_fields_is_rediscretisation():
    p = O.Params(nx=32, ny=16, nz=4, L=4)
    q = O.Params(nx=32, ny=16, nz=4, L=4, fields=p.flat_fields())
    for l in range(1, 5):
        area, ax, ay = O.level_fields(q, l)
        assert np.all(area == 1.0)
        assert np.all(ax == -p.c_h(l)) and np.all(ay == -p.c_h(l))   # c_h / 4^(L-l), [R4]


def test_coarsening_block_mean_and_face_sums():
    nx, ny = 16, 8
    i = np.arange(nx)[None, :]
    j = np.arange(ny)[:, None]
    area = 1.0 + 0.01 * i + 0.02 * j                         # linear in (i, j)
    ax = -(1.0 + 0.1 * np.arange(nx + 1)[None, :] + 0.3 * j)  # varies along and across faces
    ay = -(2.0 + 0.2 * i + 0.05 * np.arange(ny + 1)[:, None])
    p = O.Params(nx=nx, ny=ny, nz=2, L=3, fields=(area, ax, ay))
    a2, ax2, ay2 = O.level_fields(p, 2)
    # the mean of a linear field over a 2x2 block is its value at the block centre
    I = np.arange(nx // 2)[None, :]
    J = np.arange(ny // 2)[:, None]
    assert np.allclose(a2, 1.0 + 0.01 * (2 * I + 0.5) + 0.02 * (2 * J + 0.5), rtol=0, atol=1e-14)
    # coarse x-face I of row J = (fine faces 2I of rows 2J, 2J+1) / 8
    Ix = np.arange(nx // 2 + 1)[None, :]
    assert np.allclose(ax2, -(2 * (1.0 + 0.1 * 2 * Ix) + 0.3 * (4 * J + 1)) / 8, rtol=0, atol=1e-14)
    Jy = np.arange(ny // 2 + 1)[:, None]
    assert np.allclose(ay2, -(2 * 2.0 + 0.2 * (4 * I + 1) + 2 * 0.05 * 2 * Jy) / 8, rtol=0, atol=1e-14)
    a1, _, _ = O.level_fields(p, 1)
    assert np.allclose(a1, 1.0 + 0.01 * (4 * np.arange(4)[None, :] + 1.5) + 0.02 * (4 * np.arange(2)[:, None] + 1.5),
                       rtol=0, atol=1e-14)


@pytest.mark.parametrize("boundary", [0, 1])
@pytest.mark.parametrize("prof", [False, True])
def test_fields_operator_matches_edge_list_assembly(boundary, prof):
    nx, ny, nz = 5, 4, 3
    p0 = O.Params(nx=nx, ny=ny, nz=nz, L=1, boundary=boundary,
                  profiles=vertical_profiles(nz, 2, 5.0) if prof else None)
    fields = horizontal_fields(nx, ny, p0.c_h(), seed=4)
    p = O.Params(nx=nx, ny=ny, nz=nz, L=1, boundary=boundary, profiles=p0.profiles, fields=fields)
    A = dense(p, lambda v: O.apply(p, v), 1)
    B = assemble(p, fields, boundary)
    assert np.max(np.abs(A - B)) <= 1e-13 * np.max(np.abs(B))
    assert np.max(np.abs(A - A.T)) <= 1e-13 * np.max(np.abs(A))
    assert np.linalg.eigvalsh(A).min() > 0


def test_anisotropic_separable_spectrum():
    """|T| = 1, alpha_x = -cx, alpha_y = -cy on every face: A (s_p(i) s_q(j) cos_r(k)) =
    (1 + 4 cx sin^2(p pi/(2(nx+1))) + 4 cy sin^2(q pi/(2(ny+1))) + 4 gamma sin^2(r pi/(2 nz))) v."""
    nx, ny, nz = 6, 5, 4
    base = O.Params(nx=nx, ny=ny, nz=nz, L=1)
    cx, cy, g = 3.0 * base.c_h(), 0.5 * base.c_h(), base.gamma()
    fields = (np.ones((ny, nx)), np.full((ny, nx + 1), -cx), np.full((ny + 1, nx), -cy))
    p = O.Params(nx=nx, ny=ny, nz=nz, L=1, fields=fields)
    A = dense(p, lambda v: O.apply(p, v), 1)
    want = [1 + 4 * cx * math.sin(pp * math.pi / (2 * (nx + 1))) ** 2
            + 4 * cy * math.sin(qq * math.pi / (2 * (ny + 1))) ** 2
            + 4 * g * math.sin(r * math.pi / (2 * nz)) ** 2
            for pp in range(1, nx + 1) for qq in range(1, ny + 1) for r in range(nz)]
    got = np.linalg.eigvalsh(A)
    assert np.max(np.abs(np.sort(got) - np.sort(want))) < 1e-12 * max(want)


@pytest.mark.parametrize("boundary", [0, 1])
def test_fields_precondition_is_column_solve(boundary):
    nx, ny, nz = 6, 5, 9
    base = O.Params(nx=nx, ny=ny, nz=nz, L=1)
    area, ax, ay = horizontal_fields(nx, ny, base.c_h(), seed=9)
    p = O.Params(nx=nx, ny=ny, nz=nz, L=1, boundary=boundary, fields=(area, ax, ay))
    a, b, c, d = p.flat_profiles()
    Tz = np.diag(a - b - c) + np.diag(b[1:], -1) + np.diag(c[:-1], 1)
    r = np.random.default_rng(0).standard_normal(p.level_shape(1))
    z = O.precondition(p, r)
    for j in range(ny):
        for i in range(nx):
            w, e, s, n = ax[j, i], ax[j, i + 1], ay[j, i], ay[j + 1, i]
            aT = w + e + s + n
            if boundary:
                aT += (w if i == 0 else 0) + (e if i == nx - 1 else 0) + (s if j == 0 else 0) + (n if j == ny - 1 else 0)
            M = area[j, i] * Tz - aT * np.eye(nz)
            # both solves are backward stable: agreement to ~ cond(M_T) eps (gamma ~ 5e5 here)
            assert rel(z[j, i], np.linalg.solve(M, r[j, i])) < 10 * np.linalg.cond(M) * 2.2e-16


@pytest.mark.parametrize("kind", ["random", "smooth"])
def test_fields_solvers_match_dense_solve(kind):
    p0 = O.Params(nx=16, ny=16, nz=6, L=3)
    p = O.Params(nx=16, ny=16, nz=6, L=3, fields=horizontal_fields(16, 16, p0.c_h(), seed=2, kind=kind))
    f = rhs_zc(16, 16, 6, seed=5)
    A = dense(p, lambda v: O.apply(p, v), 3)
    ustar = np.linalg.solve(A, f.ravel()).reshape(f.shape)
    cg = O.solve_cg(p, f, eps=1e-12)
    mg = O.solve_mg(p, f, eps=1e-12, max_iter=300)
    assert cg.converged and mg.converged
    assert rel(cg.u, ustar) < 1e-9 and rel(mg.u, ustar) < 1e-9


def test_fields_validation():
    p0 = O.Params(nx=4, ny=4, nz=4, L=1)
    area, ax, ay = horizontal_fields(4, 4, p0.c_h(), seed=1)
    for bad in ((-area, ax, ay), (area, -ax, ay), (area, ax, np.where(ay < 0, np.nan, ay))):
        with pytest.raises(O.OracleError):
            O.apply(O.Params(nx=4, ny=4, nz=4, L=1, fields=bad), np.zeros((4, 4, 4)))
