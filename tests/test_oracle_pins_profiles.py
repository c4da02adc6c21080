"""Pins of the oracle with general vertical profiles a, b, c, d (eqn:LocalMatrixStencil,
P:250-257: "the four vectors a, b, c and d ... derived from the vertical stiffness- and
mass-matrices"), i.e. a non-uniform column shared by every horizontal cell.

The operator is then a Kronecker sum: with zero ghosts [R1] the horizontal sine mode
s_pq (eigenvalue lam_pq = 4 sin^2(p pi/(2(nx+1))) + 4 sin^2(q pi/(2(ny+1))) of the
5-point Laplacian) times a vertical vector w gives A (s_pq w) = s_pq (T + c lam_pq D) w,
with T = tridiag(b, a - b - c, c) and D = diag(d) (nz x nz).  So the spectrum of the
assembled 3D operator is the union over (p, q) of eig(T + c lam_pq D), computed here with
numpy from the profiles alone; M_T = T + 4 c D column by column (numpy dense solves).
"""
import math

import numpy as np
import pytest

from oracle import oracle as O
from inputs import rhs_zc, vertical_profiles


def vertical_matrices(prof):
    a, b, c, d = prof
    nz = len(a)
    T = np.diag(a - b - c) + np.diag(b[1:], -1) + np.diag(c[:-1], 1)
    return T, np.diag(d)


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


def test_flat_profiles_reproduce_default_bitwise():
    p = O.Params(nx=16, ny=16, nz=8, L=3)
    q = O.Params(nx=16, ny=16, nz=8, L=3, profiles=p.flat_profiles())
    x = rhs_zc(16, 16, 8, seed=3)
    for fn in (lambda P: O.apply(P, x), lambda P: O.precondition(P, x), lambda P: O.smooth(P, x, x),
               lambda P: O.vcycle(P, np.zeros_like(x), x)):
        assert np.array_equal(fn(p), fn(q))


@pytest.mark.parametrize("seed,coupling", [(1, 1.0), (2, 50.0), (3, 0.02)])
def test_profile_spectrum_is_kronecker_union(seed, coupling):
    nx, ny, nz = 5, 4, 6
    p = O.Params(nx=nx, ny=ny, nz=nz, L=1, profiles=vertical_profiles(nz, seed, coupling))
    A = dense(p, lambda v: O.apply(p, v), 1)
    assert np.max(np.abs(A - A.T)) <= 1e-12 * np.max(np.abs(A))
    T, D = vertical_matrices(p.profiles)
    c = p.c_h(1)
    want = []
    for pp in range(1, nx + 1):
        for qq in range(1, ny + 1):
            lam = 4 * math.sin(pp * math.pi / (2 * (nx + 1))) ** 2 + 4 * math.sin(qq * math.pi / (2 * (ny + 1))) ** 2
            want.extend(np.linalg.eigvalsh(T + c * lam * D))
    got = np.linalg.eigvalsh(A)
    assert np.max(np.abs(np.sort(got) - np.sort(want))) < 1e-11 * np.max(np.abs(got))
    assert got.min() > 0


def test_profile_precondition_is_column_solve():
    nx, ny, nz = 6, 5, 9
    p = O.Params(nx=nx, ny=ny, nz=nz, L=1, profiles=vertical_profiles(nz, 7, 30.0))
    T, D = vertical_matrices(p.profiles)
    M = T + 4 * p.c_h(1) * D          # A_T = |T| diag(a) - alpha_T diag(d) + tridiag, alpha_T = -4c [R1]
    r = np.random.default_rng(0).standard_normal(p.level_shape(1))
    z = O.precondition(p, r)
    want = np.linalg.solve(M, r.reshape(-1, nz).T).T.reshape(r.shape)
    assert rel(z, want) < 1e-12


def test_profile_solvers_match_dense_solve():
    p = O.Params(nx=16, ny=16, nz=6, L=3, profiles=vertical_profiles(6, 11, 20.0))
    f = rhs_zc(16, 16, 6, seed=5)
    A = dense(p, lambda v: O.apply(p, v), 3)
    ustar = np.linalg.solve(A, f.ravel()).reshape(f.shape)
    cg = O.solve_cg(p, f, eps=1e-12)
    mg = O.solve_mg(p, f, eps=1e-12, max_iter=300)
    assert cg.converged and mg.converged
    assert rel(cg.u, ustar) < 1e-9 and rel(mg.u, ustar) < 1e-9


def test_profile_validation():
    a, b, c, d = vertical_profiles(8, 1)
    c2 = c.copy()
    c2[3] *= 1.5                    # breaks b_{k+1} = c_k (non-symmetric column block)
    with pytest.raises(O.OracleError):
        O.apply(O.Params(nx=4, ny=4, nz=8, L=1, profiles=(a, b, c2, d)), np.zeros((4, 4, 8)))
    d2 = d.copy()
    d2[0] = 0.0
    with pytest.raises(O.OracleError):
        O.apply(O.Params(nx=4, ny=4, nz=8, L=1, profiles=(a, b, c, d2)), np.zeros((4, 4, 8)))
