"""Pins of the oracle's V-cycle STRUCTURE (alg:VCycle) -- CPU only.

The V-cycle pins of test_oracle_pins.py (fixed point, linearity, L = 1, beats plain
smoothing) hold for any consistent stationary iteration, so a misreading of alg:VCycle (an
extra smooth, RestrictSmooth without rho, one coarse sweep too many) would pass them.  These
pin the structure itself:

1. the kernel inventory of one cycle, per level, against the order of alg:VCycle and the
   kernel rows of tab:TimingBreakdownMultigrid (tests/golden/paper_values.json);
2. the cycle against a dense re-statement of alg:VCycle in numpy, assembled from the dense
   matrices of A_l, M_l^-1, R and P -- each taken from an oracle operator that has its own
   closed-form pins (test_oracle_pins.py) -- including the explicit two-level case
   u = P (rho M_c^-1 R f);
3. the cycle's error-propagation matrix against the textbook product of factors in
   alg:VCycle order, K_l = S_l^post (I - P B_{l-1} R A_l) S_l^pre with S = I - rho M^-1 A
   and the coarsest level's K_1 = S_1^(coarse sweeps) [R5].

scripts/oracle_mutation.py shows that each of those three mutants of tpmg_oracle.c fails
here (profiles/r2/oracle_mutation.txt).
"""
import json
import os

import numpy as np
import pytest

from oracle import oracle as O

GOLD = os.path.join(os.path.dirname(__file__), "golden")
PAPER = json.load(open(os.path.join(GOLD, "paper_values.json")))
KIND = {k: n for n, k in enumerate(O.TRACE_KINDS)}


def rel(a, b):
    return np.linalg.norm(np.ravel(a) - np.ravel(b)) / max(np.linalg.norm(np.ravel(b)), 1e-300)


def dense_map(shape_in, shape_out, fn):
    n = int(np.prod(shape_in))
    D = np.empty((int(np.prod(shape_out)), n))
    e = np.zeros(n)
    for m in range(n):
        e[:] = 0.0
        e[m] = 1.0
        D[:, m] = np.ravel(fn(e.reshape(shape_in)))
    return D


def factors(p: O.Params):
    """Dense A_l, M_l^-1 (l = 1..L), R_l: level l+1 -> l and P_l: level l -> l+1 (l = 1..L-1),
    each from its pinned oracle operator."""
    A, Minv, R, P = {}, {}, {}, {}
    for l in range(1, p.L + 1):
        s = p.level_shape(l)
        A[l] = dense_map(s, s, lambda x, l=l: O.apply(p, x, level=l))
        Minv[l] = dense_map(s, s, lambda x, l=l: O.precondition(p, x, level=l))
    for l in range(1, p.L):
        sc, sf = p.level_shape(l), p.level_shape(l + 1)
        R[l] = dense_map(sf, sc, lambda x, l=l: O.restrict(p, x, fine_level=l + 1))
        P[l] = dense_map(sc, sf, lambda x, l=l, sf=sf: O.prolong_add(p, x, np.zeros(sf), coarse_level=l))
    return A, Minv, R, P


def vcycle_dense(p: O.Params, F, u, f):
    """alg:VCycle written out with dense matrices, in the algorithm's order:
    level L smooths (pre), every other level starts with RestrictSmooth f_l = R r_{l+1},
    u_l = rho M^-1 f_l and smooths pre-1 more times; then Residual, the recursive
    call, Prolongate (u += P u_c) and the post-smoothing; the coarsest level runs
    RestrictSmooth plus coarse_sweeps-1 smooths (the A^-1 of P:187 replaced by the two
    smoother iterations of P:229, [R5]); a one-level hierarchy runs coarse_sweeps smooths."""
    A, Minv, R, P = F
    rho, L = p.rho, p.L

    def smooth(l, u, f):
        return u + rho * Minv[l] @ (f - A[l] @ u)

    def level(l, u, f):
        if l == 1:
            for _ in range(p.coarse_sweeps - (1 if L > 1 else 0)):
                u = smooth(l, u, f)
            return u
        for _ in range(p.pre - (0 if l == L else 1)):
            u = smooth(l, u, f)
        r = f - A[l] @ u                                     # Residual
        fc = R[l - 1] @ r                                     # RestrictSmooth on level l-1 ...
        uc = level(l - 1, rho * Minv[l - 1] @ fc, fc)         # ... u_c = rho M_c^-1 f_c
        u = u + P[l - 1] @ uc                                 # Prolongate
        for _ in range(p.post):
            u = smooth(l, u, f)
        return u

    return level(L, np.ravel(u).copy(), np.ravel(f))


def error_propagation_product(p: O.Params, F):
    """K_L = I - B_L A_L of the cycle as the textbook product of factors (alg:VCycle order):
    S_l = I - rho M_l^-1 A_l;  K_1 = S_1^(coarse_sweeps) (zero initial guess on a coarse
    level: the RestrictSmooth u = rho M^-1 f is one sweep from 0);
    K_l = S_l^post (I - P_{l-1} (I - K_{l-1}) A_{l-1}^-1 R_{l-1} A_l) S_l^pre_l,
    pre_l = pre (RestrictSmooth counted as the first pre-smooth on l < L)."""
    A, Minv, R, P = F
    I = {l: np.eye(A[l].shape[0]) for l in A}
    S = {l: I[l] - p.rho * Minv[l] @ A[l] for l in A}
    K = {1: np.linalg.matrix_power(S[1], p.coarse_sweeps)}
    for l in range(2, p.L + 1):
        Bc = (I[l - 1] - K[l - 1]) @ np.linalg.inv(A[l - 1])
        CGC = I[l] - P[l - 1] @ Bc @ R[l - 1] @ A[l]
        K[l] = np.linalg.matrix_power(S[l], p.post) @ CGC @ np.linalg.matrix_power(S[l], p.pre)
    return K[p.L]


# ----------------------------------------------------------------------------- 1. inventory

def expected_inventory(L, pre, post, cs):
    """Kernel calls per level of one cycle, read off alg:VCycle with [R5]."""
    want = np.zeros((L + 1, 4), dtype=np.int32)
    if L == 1:
        want[1, KIND["Smooth"]] = cs
        return want
    want[L, KIND["Smooth"]] = pre + post
    for l in range(2, L):
        want[l, KIND["ResSmooth"]] = 1
        want[l, KIND["Smooth"]] = (pre - 1) + post
    want[1, KIND["ResSmooth"]] = 1
    want[1, KIND["Smooth"]] = cs - 1
    for l in range(2, L + 1):
        want[l, KIND["Residual"]] = 1
        want[l, KIND["Prolongate"]] = 1
    return want


@pytest.mark.parametrize("L,pre,post,cs", [(5, 1, 1, 2), (3, 2, 3, 3), (2, 1, 1, 1), (4, 1, 2, 5), (1, 1, 1, 3)])
def test_vcycle_kernel_inventory(L, pre, post, cs):
    p = O.Params(nx=32, ny=32, nz=4, L=L, pre=pre, post=post, coarse_sweeps=cs)
    rng = np.random.default_rng(5)
    _, counts = O.vcycle_trace(p, rng.standard_normal(p.level_shape(L)), rng.standard_normal(p.level_shape(L)))
    assert np.array_equal(counts, expected_inventory(L, pre, post, cs)), counts


def test_vcycle_inventory_matches_paper_breakdown_table():
    """tab:TimingBreakdownMultigrid (L = 5 with 1/1 smoothing and 2 coarse sweeps,
    P:418): which kernels run on which level ("---" = not run)."""
    tab = PAPER["mg_breakdown_kernels"]
    p = O.Params(nx=32, ny=32, nz=4)   # the paper's L, pre, post, coarse_sweeps
    assert (p.L, p.pre, p.post, p.coarse_sweeps) == (5, 1, 1, 2)
    rng = np.random.default_rng(6)
    _, counts = O.vcycle_trace(p, rng.standard_normal(p.level_shape(5)), rng.standard_normal(p.level_shape(5)))
    for kind, runs in tab["runs"].items():
        for l, present in zip(tab["levels"], runs):
            assert (counts[l, KIND[kind]] > 0) == bool(present), (kind, l)
    # one call of each present kernel per level, except the fine level's pre + post smooth
    want = np.array(tab["runs"]["Smooth"]) * 1
    want[tab["levels"].index(5)] = 2
    assert [counts[l, KIND["Smooth"]] for l in tab["levels"]] == list(want)


# ----------------------------------------------------------------------------- 2. dense alg:VCycle

def test_two_level_zero_smoothing_is_P_rho_Minv_R():
    """L = 2, pre = post = 0, coarse_sweeps = 1: from u = 0 the cycle is exactly
    u = P (rho M_c^-1 (R f)) (RestrictSmooth; Prolongate)."""
    p = O.Params(nx=8, ny=8, nz=3, L=2, pre=0, post=0, coarse_sweeps=1)
    A, Minv, R, P = factors(p)
    rng = np.random.default_rng(7)
    f = rng.standard_normal(p.level_shape(2))
    got = O.vcycle(p, np.zeros_like(f), f)
    want = P[1] @ (p.rho * (Minv[1] @ (R[1] @ f.ravel())))
    assert rel(got, want) < 1e-13


@pytest.mark.parametrize("nx,ny,nz,L,pre,post,cs,nu", [
    (8, 8, 2, 3, 1, 1, 2, 8.4), (16, 8, 3, 3, 2, 3, 3, 8.4), (8, 8, 4, 2, 1, 1, 2, 20.0),
    (16, 16, 2, 4, 1, 2, 1, 8.4), (8, 8, 3, 1, 1, 1, 3, 8.4)])
def test_vcycle_matches_dense_algorithm(nx, ny, nz, L, pre, post, cs, nu):
    p = O.Params(nx=nx, ny=ny, nz=nz, L=L, pre=pre, post=post, coarse_sweeps=cs, nu_cfl=nu)
    F = factors(p)
    rng = np.random.default_rng(8)
    for _ in range(2):
        u = rng.standard_normal(p.level_shape(L))
        f = rng.standard_normal(p.level_shape(L))
        assert rel(O.vcycle(p, u, f), vcycle_dense(p, F, u, f)) < 1e-12


@pytest.mark.parametrize("boundary", [0, 1])
def test_vcycle_error_propagation_is_product_of_factors(boundary):
    """8 x 8 x 2, L = 3, the paper's 1/1 smoothing and 2 coarse sweeps: the oracle cycle's
    error-propagation matrix (columns V(e_m, 0)) equals S^post (I - P B_c R A) S^pre."""
    p = O.Params(nx=8, ny=8, nz=2, L=3, boundary=boundary)
    F = factors(p)
    s = p.level_shape(3)
    E = dense_map(s, s, lambda e: O.vcycle(p, e, np.zeros(s)))
    K = error_propagation_product(p, F)
    assert np.max(np.abs(E - K)) < 1e-12 * max(1.0, np.max(np.abs(K)))
    # a convergent cycle: spectral radius well below 1 (MG robust)
    assert max(abs(np.linalg.eigvals(K))) < 0.5
