"""Pins of the CPU oracle against what the paper and the mathematics fix.

None of these tests re-types an oracle formula: each compares the oracle with
a closed form (Fourier eigenpairs of the flat-box operator), a library routine
on a tiny case (numpy dense solves / eigensolvers), an invariant (symmetry,
constants and linear fields under the grid transfers, fixed points, linearity)
or a value the paper prints (tests/golden/paper_values.json).  A dropped term,
a wrong sign, a wrong index or a transposed operand in tpmg_oracle.c fails at
least one of them.
"""
import json
import math
import os

import numpy as np
import pytest
import scipy.linalg

from oracle import oracle as O
from inputs import mode_zc, rhs_zc
from inputs.splitmix import _mix

GOLD = os.path.join(os.path.dirname(__file__), "golden")
PAPER = json.load(open(os.path.join(GOLD, "paper_values.json")))


def sin2(x):
    return math.sin(x) ** 2


def eig_closed_form(p: O.Params, level, pp, qq, rr):
    """Eigenvalue of the flat-box operator for the separable mode (p,q,r):
    1 + 4 c [sin^2(p pi/(2(nx+1))) + sin^2(q pi/(2(ny+1)))] + 4 gamma sin^2(r pi/(2 nz))
    (Dirichlet horizontally with zero ghosts [R1], Neumann vertically)."""
    ny, nx, nz = p.level_shape(level)
    c, g = p.c_h(level), p.gamma()
    return (1 + 4 * c * (sin2(pp * math.pi / (2 * (nx + 1))) + sin2(qq * math.pi / (2 * (ny + 1))))
            + 4 * g * sin2(rr * math.pi / (2 * nz)))


def dense(p: O.Params, fn, level=None):
    """Dense matrix of a linear oracle map by columns (unit vectors)."""
    level = p.L if level is None else level
    shape = p.level_shape(level)
    n = int(np.prod(shape))
    A = np.empty((n, n))
    e = np.zeros(n)
    for m in range(n):
        e[:] = 0.0
        e[m] = 1.0
        A[:, m] = fn(e.reshape(shape)).ravel()
    return A


def abs_bound(p: O.Params, level=None):
    """Upper bound of the row sums |A| (1 + 8c + 4 gamma): the floating-point error of one
    application is a few ulps of this times max|x|, whatever the cancellation."""
    level = p.L if level is None else level
    return 1 + 8 * p.c_h(level) + 4 * p.gamma()


def close_op(p, got, want, x, level=None, ulps=16):
    err = np.max(np.abs(np.ravel(got) - np.ravel(want)))
    return err <= ulps * 2.2e-16 * abs_bound(p, level) * np.max(np.abs(x))


def kappa_M(p: O.Params, level=None):
    """Condition number of the column block M_T: error amplification of a stable solve."""
    level = p.L if level is None else level
    return (1 + 4 * p.c_h(level) + 4 * p.gamma()) / (1 + 4 * p.c_h(level))


def rel(a, b):
    return np.linalg.norm(np.ravel(a) - np.ravel(b)) / max(np.linalg.norm(np.ravel(b)), 1e-300)


# ----------------------------------------------------------------------------- operator

@pytest.mark.parametrize("nx,ny,nz,nu", [(6, 5, 4, 8.4), (8, 8, 16, 8.4), (12, 7, 3, 2.0), (5, 9, 1, 10.0)])
def test_operator_fourier_eigenpairs(nx, ny, nz, nu):
    p = O.Params(nx=nx, ny=ny, nz=nz, nu_cfl=nu, L=1)
    for (pp, qq, rr) in [(1, 1, 0), (nx, ny, nz - 1), (2, 3, min(1, nz - 1)), (nx // 2 + 1, 1, nz // 2)]:
        v = mode_zc(nx, ny, nz, pp, qq, rr)
        lam = eig_closed_form(p, 1, pp, qq, rr)
        assert close_op(p, O.apply(p, v), lam * v, v)
        assert rel(O.apply(p, v), lam * v) < 1e-9


def test_operator_coarse_levels_rediscretised():
    """Level l is the flat-box operator with h_l = 2^(L-l) h [R4]: its eigenvalues use
    c_h^l = c_h / 4^(L-l), the factor-4 reduction of P:229."""
    p = O.Params(nx=32, ny=16, nz=8, L=4)
    for level in (1, 2, 3, 4):
        ny, nx, nz = p.level_shape(level)
        v = mode_zc(nx, ny, nz, 1, 2, 1)
        assert close_op(p, O.apply(p, v, level), eig_closed_form(p, level, 1, 2, 1) * v, v, level)
    assert p.c_h(3) == pytest.approx(p.c_h(4) / PAPER["coarse_kappa_factor"]["value"], rel=1e-15)


def test_dense_spectrum_symmetry_spd():
    """Assembled A is symmetric, its spectrum is exactly the closed-form set, lambda_min > 1 (SPD)."""
    nx, ny, nz = 6, 4, 3
    p = O.Params(nx=nx, ny=ny, nz=nz, L=1)
    A = dense(p, lambda x: O.apply(p, x))
    assert np.max(np.abs(A - A.T)) <= 1e-12 * np.max(np.abs(A))
    ev = np.sort(np.linalg.eigvalsh(A))
    cf = np.sort([eig_closed_form(p, 1, a, b, c) for a in range(1, nx + 1)
                  for b in range(1, ny + 1) for c in range(nz)])
    assert np.max(np.abs(ev - cf)) < 1e-13 * abs_bound(p)
    assert ev[0] > 1.0
    # 7-point structure: at most 7 nonzeros per row
    assert np.max(np.count_nonzero(A, axis=1)) == 7


def test_operator_constant_field_interior():
    """A applied to a constant leaves exactly the zero-order term away from horizontal boundaries."""
    p = O.Params(nx=8, ny=8, nz=5, L=1)
    y = O.apply(p, np.full(p.level_shape(1), 3.0))
    assert np.allclose(y[1:-1, 1:-1, :], 3.0, rtol=1e-12, atol=1e-12 * 4 * p.gamma())


def test_symmetry_random_pairs():
    p = O.Params(nx=16, ny=8, nz=6, L=1)
    rng = np.random.default_rng(3)
    for _ in range(20):
        u = rng.standard_normal(p.level_shape(1)); v = rng.standard_normal(p.level_shape(1))
        a, b = O.dot(p, O.apply(p, u), v, 1), O.dot(p, u, O.apply(p, v), 1)
        assert abs(a - b) <= 1e-13 * (abs(a) + np.linalg.norm(u) * np.linalg.norm(v) * 4 * p.gamma())


def test_residual_definition():
    p = O.Params(nx=8, ny=8, nz=4, L=1)
    rng = np.random.default_rng(0)
    u = rng.standard_normal(p.level_shape(1)); f = rng.standard_normal(p.level_shape(1))
    assert np.array_equal(O.residual(p, np.zeros_like(u), f), f)   # u=0 -> r=f
    r = O.residual(p, u, O.apply(p, u))
    assert np.max(np.abs(r)) <= 1e-12 * np.max(np.abs(O.apply(p, u)))


# ----------------------------------------------------------------------------- Thomas / M^-1

def test_thomas_small_dense():
    rng = np.random.default_rng(1)
    for n in range(1, 9):
        s, t = rng.standard_normal(n), rng.standard_normal(n)
        dg = np.abs(s) + np.abs(t) + 1 + rng.random(n)
        g = rng.standard_normal(n)
        T = np.diag(dg) + np.diag(s[1:], -1) + np.diag(t[:-1], 1)
        assert rel(O.thomas(s, dg, t, g), np.linalg.solve(T, g)) < 1e-14


def test_thomas_examples_and_large():
    # identity and the 3x3 example (2,-1)
    g = np.array([1.0, -2.0, 5.0])
    assert np.array_equal(O.thomas(np.zeros(3), np.ones(3), np.zeros(3), g), g)
    T = np.array([[2.0, -1, 0], [-1, 2, -1], [0, -1, 2]])
    assert rel(O.thomas(-np.ones(3), 2 * np.ones(3), -np.ones(3), g), np.linalg.solve(T, g)) < 1e-15
    rng = np.random.default_rng(2)
    n = 128
    s, t = rng.standard_normal(n), rng.standard_normal(n)
    dg = np.abs(s) + np.abs(t) + 0.5
    b = rng.standard_normal(n)
    x = O.thomas(s, dg, t, b)
    Tx = dg * x; Tx[1:] += s[1:] * x[:-1]; Tx[:-1] += t[:-1] * x[1:]
    assert np.linalg.norm(Tx - b) / np.linalg.norm(b) <= 1e-13


def test_thomas_singular():
    with pytest.raises(O.OracleError):
        O.thomas(np.zeros(2), np.array([0.0, 1.0]), np.zeros(2), np.ones(2))


@pytest.mark.parametrize("nz", [1, 2, 16, 128])
def test_precondition_vertical_modes(nz):
    """M^-1 (g(i,j) cos(r pi (k+1/2)/nz)) = that field / m_r with
    m_r = 1 + 4 c + 4 gamma sin^2(r pi/(2 nz)): M is the column block A_T."""
    p = O.Params(nx=8, ny=6, nz=nz, L=1)
    rng = np.random.default_rng(nz)
    g = rng.standard_normal((6, 8))
    for r in {0, nz // 2, nz - 1}:
        ck = np.cos(r * np.pi * (np.arange(nz) + 0.5) / nz)
        v = g[:, :, None] * ck[None, None, :]
        m_r = 1 + 4 * p.c_h() + 4 * p.gamma() * sin2(r * math.pi / (2 * nz))
        kappa_M = (1 + 4 * p.c_h() + 4 * p.gamma()) / (1 + 4 * p.c_h())  # backward-stable solve bound
        assert rel(O.precondition(p, v), v / m_r) < 10 * kappa_M * 2.2e-16


def test_precondition_is_block_of_A():
    """On fields supported on isolated columns, A acts column-wise as M_T:
    M^-1 (A z0 |support) = z0."""
    p = O.Params(nx=8, ny=8, nz=12, L=1)
    rng = np.random.default_rng(5)
    z0 = np.zeros(p.level_shape(1))
    mask = np.zeros((8, 8), bool)
    mask[::2, ::2] = True   # no two support columns are horizontal neighbours
    z0[mask] = rng.standard_normal((mask.sum(), 12))
    Az = O.apply(p, z0)
    Az[~mask] = 0.0
    assert rel(O.precondition(p, Az), z0) < 10 * kappa_M(p) * 2.2e-16


# ----------------------------------------------------------------------------- smoother

def test_smooth_mode_damping():
    """f = 0, u = mode: u <- (1 - rho lambda_pqr / m_r) u (eqn:MultigridSmoother)."""
    p = O.Params(nx=8, ny=8, nz=8, L=1)
    for (pp, qq, rr) in [(1, 1, 0), (8, 8, 7), (3, 5, 2)]:
        v = mode_zc(8, 8, 8, pp, qq, rr)
        lam = eig_closed_form(p, 1, pp, qq, rr)
        m_r = 1 + 4 * p.c_h() + 4 * p.gamma() * sin2(rr * math.pi / 16)
        out = O.smooth(p, v, np.zeros_like(v))
        assert rel(out, (1 - p.rho * lam / m_r) * v) < 1e-12


def test_smooth_fixed_point_and_jacobi():
    p = O.Params(nx=8, ny=8, nz=4, L=1)
    rng = np.random.default_rng(7)
    u = rng.standard_normal(p.level_shape(1))
    f = O.apply(p, u)
    assert rel(O.smooth(p, u, f), u) < 1e-13     # exact solution is a fixed point
    # Jacobi: the smoother equals u + rho M^-1 (f - A u) evaluated with the OLD u everywhere
    f2 = rng.standard_normal(u.shape)
    want = u + p.rho * O.precondition(p, O.residual(p, u, f2))
    assert rel(O.smooth(p, u, f2), want) < 1e-15


# ----------------------------------------------------------------------------- condition number

def test_kappa_closed_form_and_paper_value():
    """kappa(M^-1 A) = (1 + 4c (smax_x + smax_y)) / (1 + 4c (smin_x + smin_y)); tends to
    1 + 8 omega^2/h^2 = 142.1 for nu = 8.4 (eqn:ConditionNumber)."""
    nx, ny, nz = 6, 6, 4
    p = O.Params(nx=nx, ny=ny, nz=nz, L=1)
    A = dense(p, lambda x: O.apply(p, x))
    Minv = dense(p, lambda x: O.precondition(p, x))
    M = np.linalg.inv(Minv)
    ev = scipy.linalg.eigh(A, 0.5 * (M + M.T), eigvals_only=True)
    c = p.c_h()
    smax, smin = math.cos(math.pi / (2 * (nx + 1))) ** 2, math.sin(math.pi / (2 * (nx + 1))) ** 2
    kappa_cf = (1 + 4 * c * 2 * smax) / (1 + 4 * c * 2 * smin)
    assert ev.max() / ev.min() == pytest.approx(kappa_cf, rel=1e-10)
    big = 1 << 20
    smax, smin = math.cos(math.pi / (2 * (big + 1))) ** 2, math.sin(math.pi / (2 * (big + 1))) ** 2
    kappa_lim = (1 + 8 * c * smax) / (1 + 8 * c * smin)
    assert kappa_lim == pytest.approx(PAPER["kappa_estimate"]["value"], abs=0.5)
    assert math.sqrt(c) == pytest.approx(PAPER["omega_over_h"]["value"], rel=1e-12)


# ----------------------------------------------------------------------------- grid transfers

def test_restrict_invariants():
    p = O.Params(nx=16, ny=8, nz=3, L=2)
    ny, nx, nz = p.level_shape(2)
    # constants are preserved
    assert np.array_equal(O.restrict(p, np.full((ny, nx, nz), 2.5)), np.full((ny // 2, nx // 2, nz), 2.5))
    # cell average of a linear function is its value at the coarse cell centre
    x = (np.arange(nx) + 0.5) / nx; y = (np.arange(ny) + 0.5) / nx
    lin = (1.0 + 2.0 * x[None, :, None] - 3.0 * y[:, None, None]) * np.array([1.0, -1.0, 0.5])[None, None, :]
    X = (np.arange(nx // 2) + 0.5) * 2 / nx; Y = (np.arange(ny // 2) + 0.5) * 2 / nx
    want = (1.0 + 2.0 * X[None, :, None] - 3.0 * Y[:, None, None]) * np.array([1.0, -1.0, 0.5])[None, None, :]
    assert np.max(np.abs(O.restrict(p, lin) - want)) < 1e-14
    # conservation: 4 * sum(coarse) = sum(fine), level by level in k
    rng = np.random.default_rng(0)
    r = rng.standard_normal((ny, nx, nz))
    assert np.allclose(4 * O.restrict(p, r).sum(axis=(0, 1)), r.sum(axis=(0, 1)), rtol=1e-13)
    # children of a coarse cell: indicator of fine (0,1) -> coarse(0,0) = 1/4
    e = np.zeros((ny, nx, nz)); e[1, 0, :] = 1.0
    out = O.restrict(p, e)
    assert out[0, 0, 0] == 0.25 and np.count_nonzero(out) == nz


def test_prolong_invariants():
    p = O.Params(nx=16, ny=12, nz=2, L=2)
    nyc, nxc, nz = p.level_shape(1)
    nyf, nxf, _ = p.level_shape(2)
    zero_f = np.zeros((nyf, nxf, nz))
    # a single interior coarse unit spreads the weights (9,3,3,1)/16 over a 4x4 fine patch
    e = np.zeros((nyc, nxc, nz)); e[2, 3, :] = 1.0
    out = O.prolong_add(p, e, zero_f)
    patch = out[3:7, 5:9, 0] * 16
    w1 = np.array([1, 3, 3, 1])
    assert np.array_equal(patch, np.outer(w1, w1)) and out.sum() == pytest.approx(4 * nz)
    # constants reproduced on interior fine cells; linear functions too (bilinear exactness)
    X = (np.arange(nxc) + 0.5) * 2 / nxf; Y = (np.arange(nyc) + 0.5) * 2 / nxf
    x = (np.arange(nxf) + 0.5) / nxf; y = (np.arange(nyf) + 0.5) / nxf
    for a, bx, by in [(1.0, 0, 0), (0.3, 1.5, -2.0)]:
        uc = np.repeat((a + bx * X[None, :] + by * Y[:, None])[:, :, None], nz, axis=2)
        uf = O.prolong_add(p, uc, zero_f)
        want = np.repeat((a + bx * x[None, :] + by * y[:, None])[:, :, None], nz, axis=2)
        assert np.max(np.abs(uf - want)[1:-1, 1:-1]) < 1e-14
    # adds to the fine field (u_f + P u_c), zero ghost at the boundary [R7]: corner gets 9/16
    base = np.full((nyf, nxf, nz), 1.0)
    out = O.prolong_add(p, np.ones((nyc, nxc, nz)), base)
    assert out[0, 0, 0] == 1 + 9 / 16 and out[0, 3, 0] == 1 + 12 / 16 and out[5, 5, 1] == 2.0


# ----------------------------------------------------------------------------- V-cycle and solvers

def _dense_solve(p, f):
    A = dense(p, lambda x: O.apply(p, x), p.L)
    return np.linalg.solve(A, f.ravel()).reshape(f.shape)


def test_vcycle_fixed_point_and_linearity():
    p = O.Params(nx=16, ny=16, nz=4, L=3)
    rng = np.random.default_rng(11)
    f = rng.standard_normal(p.level_shape(3))
    ustar = _dense_solve(p, f)
    assert rel(O.vcycle(p, ustar, f), ustar) < 1e-12
    u1, u2 = rng.standard_normal(f.shape), rng.standard_normal(f.shape)
    f1, f2 = rng.standard_normal(f.shape), rng.standard_normal(f.shape)
    lhs = O.vcycle(p, u1 + 2 * u2, f1 + 2 * f2)
    rhs = O.vcycle(p, u1, f1) + 2 * O.vcycle(p, u2, f2)
    assert rel(lhs, rhs) < 10 * kappa_M(p) * 2.2e-16


def test_vcycle_single_level_is_coarse_sweeps():
    p = O.Params(nx=8, ny=8, nz=4, L=1, coarse_sweeps=3)
    rng = np.random.default_rng(12)
    u, f = rng.standard_normal(p.level_shape(1)), rng.standard_normal(p.level_shape(1))
    assert rel(O.vcycle(p, u, f), O.smooth(p, u, f, sweeps=3)) < 1e-15


def test_vcycle_two_level_error_reduction():
    """Two-grid/V-cycle error is much smaller than the smoother's alone (coarse correction works)."""
    p = O.Params(nx=32, ny=32, nz=16, L=5)
    f = rhs_zc(32, 32, 16, seed=3)
    u = np.zeros_like(f)
    for _ in range(5):
        u = O.vcycle(p, u, f)
    us = O.smooth(p, np.zeros_like(f), f, sweeps=10)   # same fine-level smoothing work
    r_v = np.linalg.norm(O.residual(p, u, f)); r_s = np.linalg.norm(O.residual(p, us, f))
    assert r_v < 0.05 * r_s and r_v < 1e-2 * np.linalg.norm(f)


def test_cg_eigenmode_one_iteration():
    p = O.Params(nx=16, ny=16, nz=8, L=1)
    v = mode_zc(16, 16, 8, 2, 3, 1)
    res = O.solve_cg(p, v, eps=1e-10)
    assert res.iterations == 1 and res.converged
    assert rel(res.u, v / eig_closed_form(p, 1, 2, 3, 1)) < 1e-13


def test_solvers_zero_rhs():
    p = O.Params(nx=32, ny=32, nz=16)
    z = np.zeros(p.level_shape(p.L))
    for fn in (O.solve_cg, O.solve_mg):
        r = fn(p, z)
        assert r.iterations == 0 and r.converged and not r.u.any()


def test_solvers_match_dense_solve():
    p = O.Params(nx=16, ny=16, nz=4, L=3)
    f = rhs_zc(16, 16, 4, seed=1)
    ustar = _dense_solve(p, f)
    cg = O.solve_cg(p, f, eps=1e-12)
    mg = O.solve_mg(p, f, eps=1e-12, max_iter=200)
    assert cg.converged and mg.converged
    assert rel(cg.u, ustar) < 1e-9 and rel(mg.u, ustar) < 1e-9


def test_manufactured_solution():
    """u* = smooth + rough mode; f = A u* from the closed-form eigenvalues; both solvers recover u*."""
    nx = ny = 32; nz = 16
    p = O.Params(nx=nx, ny=ny, nz=nz)
    m1, m2 = mode_zc(nx, ny, nz, 1, 1, 0), mode_zc(nx, ny, nz, nx // 2, ny // 2, 1)
    ustar = m1 + 0.5 * m2
    f = eig_closed_form(p, p.L, 1, 1, 0) * m1 + 0.5 * eig_closed_form(p, p.L, nx // 2, ny // 2, 1) * m2
    for fn in (O.solve_cg, O.solve_mg):
        r = fn(p, f, eps=1e-10, max_iter=500)
        assert r.converged and rel(r.u, ustar) < 1e-8


def test_iteration_counts_paper_soft_pin():
    """Iterations to 1e-5 at 128^2 x 128, nu = 8.4: the paper prints CG 70 and MG 9 for the
    sphere panel; the flat box must land in the same regime (SPEC AC3: CG 70+-20%...)."""
    p = O.Params(nx=128, ny=128, nz=128)
    f = rhs_zc(128, 128, 128, seed=0)
    mg = O.solve_mg(p, f, eps=PAPER["epsilon"]["value"])
    assert mg.converged and mg.iterations <= 12
    assert abs(mg.iterations - PAPER["mg_iterations_table2"]["value"][0]) <= 2
    # MG convergence rate per cycle (asymptotic) well below 1
    h = mg.history
    assert (h[-1] / h[1]) ** (1 / (len(h) - 2)) < 0.45
    cg = O.solve_cg(p, f, eps=PAPER["epsilon"]["value"])
    assert cg.converged and 40 <= cg.iterations <= 84


def test_cg_iterations_grow_with_cfl():
    """CG iterations grow ~linearly with nu_CFL (kappa ~ nu^2); MG stays flat."""
    its_cg, its_mg = [], []
    for nu in (2.0, 8.4):
        p = O.Params(nx=64, ny=64, nz=32, nu_cfl=nu)
        f = rhs_zc(64, 64, 32, seed=0)
        its_cg.append(O.solve_cg(p, f).iterations)
        its_mg.append(O.solve_mg(p, f).iterations)
    assert 2.0 <= its_cg[1] / its_cg[0] <= 5.5
    assert its_mg[1] <= 1.5 * its_mg[0] + 1


# ----------------------------------------------------------------------------- inputs

def test_splitmix_reference_sequence():
    gold = json.load(open(os.path.join(GOLD, "splitmix64.json")))["outputs_hex"]
    for s, hx in enumerate(gold):
        want = (int(hx, 16) >> 11) * 2.0 ** -53 * 2.0 - 1.0
        assert _mix(np.array([0], dtype=np.uint64), s)[0] == want


def test_rhs_decomposition_independent():
    full = rhs_zc(32, 16, 8, seed=4)
    top = rhs_zc(32, 8, 8, seed=4, y0=8)
    assert np.array_equal(full[8:], top)
    assert full.min() >= -1 and full.max() < 1
