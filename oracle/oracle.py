"""CPU oracle (ctypes wrapper over oracle/liboracle.so).  TEST INFRASTRUCTURE ONLY.

Only tests/, ``__graft_entry__.smoke()`` and bench.py's ``cpu_baseline`` /
``--impl reference`` legs may import this module.  The product package
(paper_1402_3545_b200/) never imports it and shares no code with it.

Fields are numpy float64 arrays in the oracle's z-contiguous layout, shape
``(ny, nx, nz)`` (index ``[j, i, k]``), the CPU-friendly ordering of P:59.
The GPU library uses the paper's x-contiguous Lambda layout, shape
``(ny, nz, nx)``; convert with :func:`to_lambda` / :func:`from_lambda`.

Each function cites the passage of /root/reference/PAPER.md (``P:n``) whose
arithmetic the C code in ``tpmg_oracle.c`` follows.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from dataclasses import dataclass

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "tpmg_oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")
# scripts/oracle_mutation.py points this at a deliberately broken build of the oracle to
# show that the pins catch the mutation (the default is the real oracle)
_LIB_OVERRIDE = os.environ.get("TPMG_ORACLE_LIB")


def build(force: bool = False) -> str:
    """Compile the oracle (plain C, fp64, -ffp-contract=off, OpenMP over columns)."""
    if _LIB_OVERRIDE:
        return _LIB_OVERRIDE
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        subprocess.check_call(
            ["gcc", "-O2", "-std=c11", "-fPIC", "-shared", "-ffp-contract=off", "-fopenmp",
             "-o", _LIB, _SRC, "-lm"])
    return _LIB


class _Params(C.Structure):
    _fields_ = [("nx", C.c_long), ("ny", C.c_long), ("nz", C.c_int),
                ("nu_cfl", C.c_double), ("H", C.c_double), ("lam", C.c_double),
                ("L", C.c_int), ("pre", C.c_int), ("post", C.c_int),
                ("coarse_sweeps", C.c_int), ("rho", C.c_double), ("boundary", C.c_int),
                ("prof_a", C.POINTER(C.c_double)), ("prof_b", C.POINTER(C.c_double)),
                ("prof_c", C.POINTER(C.c_double)), ("prof_d", C.POINTER(C.c_double)),
                ("field_area", C.POINTER(C.c_double)), ("field_ax", C.POINTER(C.c_double)),
                ("field_ay", C.POINTER(C.c_double))]


@dataclass
class Params:
    """Problem/solver parameters.  Defaults: P:114 (nu=8.4), P:257 (nz=128),
    P:418 (L=5, 1 pre / 1 post, 2 coarse sweeps, rho=2/3), [R3] (H=0.01, lambda=1)."""
    nx: int
    ny: int
    nz: int = 128
    nu_cfl: float = 8.4
    H: float = 0.01
    lam: float = 1.0
    L: int = 5
    pre: int = 1
    post: int = 1
    coarse_sweeps: int = 2
    rho: float = 2.0 / 3.0
    boundary: int = 0   # horizontal Dirichlet reading: 0 ghost zero [R1], 1 face [R25]
    profiles: tuple | None = None   # (a, b, c, d) vertical profiles; None: flat box [R2]
    # (area [ny, nx], ax [ny, nx+1], ay [ny+1, nx]) per-column |T| and face alpha_{T,T'} of the
    # finest level; None: the flat box.  Coarser levels: reading [R26].
    fields: tuple | None = None

    def c(self) -> _Params:
        ptrs = [None] * 4
        fptrs = [None] * 3
        keep = []
        if self.profiles is not None:
            arrs = [np.ascontiguousarray(x, dtype=np.float64) for x in self.profiles]
            assert all(a.shape == (self.nz,) for a in arrs)
            keep += arrs
            ptrs = [a.ctypes.data_as(C.POINTER(C.c_double)) for a in arrs]
        if self.fields is not None:
            shapes = [(self.ny, self.nx), (self.ny, self.nx + 1), (self.ny + 1, self.nx)]
            arrs = [np.ascontiguousarray(x, dtype=np.float64) for x in self.fields]
            assert [a.shape for a in arrs] == shapes, [a.shape for a in arrs]
            keep += arrs
            fptrs = [a.ctypes.data_as(C.POINTER(C.c_double)) for a in arrs]
        self._keep = keep   # the C struct points into these
        return _Params(self.nx, self.ny, self.nz, self.nu_cfl, self.H, self.lam, self.L,
                       self.pre, self.post, self.coarse_sweeps, self.rho, self.boundary, *ptrs, *fptrs)

    def flat_fields(self) -> tuple:
        """The flat box as per-column fields: |T| = 1, alpha_{T,T'} = -c_h on every face."""
        c = self.c_h()
        return (np.ones((self.ny, self.nx)), np.full((self.ny, self.nx + 1), -c),
                np.full((self.ny + 1, self.nx), -c))

    def flat_profiles(self) -> tuple:
        """The flat-box profiles [R2] as arrays (a, b, c, d)."""
        g = self.gamma()
        k = np.arange(self.nz)
        return (np.ones(self.nz), np.where(k > 0, -g, 0.0), np.where(k < self.nz - 1, -g, 0.0), np.ones(self.nz))

    def level_shape(self, level: int) -> tuple[int, int, int]:
        f = 1 << (self.L - level)
        return (self.ny // f, self.nx // f, self.nz)

    # closed-form coefficients (used by tests to state pins; the C code derives its own)
    def c_h(self, level: int | None = None) -> float:
        level = self.L if level is None else level
        h = 1.0 / self.nx
        omega = 0.5 * self.nu_cfl * h
        hl = h * (1 << (self.L - level))
        return omega * omega / (hl * hl)

    def gamma(self) -> float:
        h = 1.0 / self.nx
        omega = 0.5 * self.nu_cfl * h
        hz = self.H / self.nz
        return omega * omega * self.lam * self.lam / (hz * hz)


_lib = None
_dp = np.ctypeslib.ndpointer(dtype=np.float64, flags="C_CONTIGUOUS")
_lp = np.ctypeslib.ndpointer(dtype=np.int64, flags="C_CONTIGUOUS")


def lib():
    global _lib
    if _lib is None:
        _lib = C.CDLL(build())
        P = C.POINTER(_Params)
        sig = {
            "or_api_apply": [P, C.c_int, _dp, _dp],
            "or_api_residual": [P, C.c_int, _dp, _dp, _dp],
            "or_api_precondition": [P, C.c_int, _dp, _dp],
            "or_api_smooth": [P, C.c_int, _dp, _dp, _dp],
            "or_api_dot": [P, C.c_int, _dp, _dp, C.POINTER(C.c_double)],
            "or_api_apply_cols": [P, C.c_int, _dp, C.c_int, _lp, _lp, _dp],
            "or_api_residual_cols": [P, C.c_int, _dp, _dp, C.c_int, _lp, _lp, _dp],
            "or_api_precondition_cols": [P, C.c_int, _dp, C.c_int, _lp, _lp, _dp],
            "or_api_smooth_cols": [P, C.c_int, _dp, _dp, C.c_int, _lp, _lp, _dp],
            "or_api_restrict": [P, C.c_int, _dp, _dp],
            "or_api_prolong_add": [P, C.c_int, _dp, _dp],
            "or_api_thomas": [C.c_int, _dp, _dp, _dp, _dp, _dp],
            "or_vcycle": [P, _dp, _dp],
            "or_api_vcycle_trace": [P, _dp, _dp, np.ctypeslib.ndpointer(dtype=np.int32, flags="C_CONTIGUOUS")],
            "or_solve_mg": [P, _dp, _dp, C.c_double, C.c_int, C.POINTER(C.c_int),
                            C.POINTER(C.c_int), _dp, C.c_int],
            "or_solve_cg": [P, _dp, _dp, C.c_double, C.c_int, C.POINTER(C.c_int),
                            C.POINTER(C.c_int), _dp, C.c_int],
            "or_api_level_fields": [P, C.c_int, _dp, _dp, _dp],
            "or_api_num_threads": [],
            "or_api_set_threads": [C.c_int],
        }
        for name, args in sig.items():
            fn = getattr(_lib, name)
            fn.argtypes = args
            fn.restype = C.c_int
    return _lib


class OracleError(RuntimeError):
    pass


def _check(st: int, what: str):
    if st != 0:
        raise OracleError(f"oracle {what} failed with status {st}")


def _arr(x, shape=None):
    a = np.ascontiguousarray(x, dtype=np.float64)
    if shape is not None and a.shape != tuple(shape):
        raise ValueError(f"expected shape {shape}, got {a.shape}")
    return a


def to_lambda(x_zc: np.ndarray) -> np.ndarray:
    """(ny, nx, nz) z-contiguous -> (ny, nz, nx) x-contiguous Lambda layout."""
    return np.ascontiguousarray(np.transpose(x_zc, (0, 2, 1)))


def from_lambda(x_l: np.ndarray) -> np.ndarray:
    return np.ascontiguousarray(np.transpose(x_l, (0, 2, 1)))


def apply(p: Params, x, level: int | None = None):
    """y = A x, eqn:TridiagonalPDE with eqn:LocalMatrixStencil."""
    level = p.L if level is None else level
    x = _arr(x, p.level_shape(level))
    y = np.empty_like(x)
    _check(lib().or_api_apply(C.byref(p.c()), level, x, y), "apply")
    return y


def residual(p: Params, u, f, level: int | None = None):
    """r = f - A u (Kernel Residual)."""
    level = p.L if level is None else level
    u = _arr(u, p.level_shape(level)); f = _arr(f, p.level_shape(level))
    r = np.empty_like(u)
    _check(lib().or_api_residual(C.byref(p.c()), level, u, f, r), "residual")
    return r


def precondition(p: Params, r, level: int | None = None):
    """z = M^{-1} r, vertical line relaxation by the Thomas algorithm."""
    level = p.L if level is None else level
    r = _arr(r, p.level_shape(level))
    z = np.empty_like(r)
    _check(lib().or_api_precondition(C.byref(p.c()), level, r, z), "precondition")
    return z


def smooth(p: Params, u, f, level: int | None = None, sweeps: int = 1):
    """Block-Jacobi smoother u <- u + rho M^{-1}(f - A u), eqn:MultigridSmoother."""
    level = p.L if level is None else level
    u = _arr(u, p.level_shape(level)).copy(); f = _arr(f, p.level_shape(level))
    out = np.empty_like(u)
    for _ in range(sweeps):
        _check(lib().or_api_smooth(C.byref(p.c()), level, u, f, out), "smooth")
        u, out = out, u
    return u


def dot(p: Params, x, y, level: int | None = None) -> float:
    level = p.L if level is None else level
    out = C.c_double()
    _check(lib().or_api_dot(C.byref(p.c()), level, _arr(x), _arr(y), C.byref(out)), "dot")
    return out.value


def _cols(fn, p, level, arrays, ii, jj):
    ii = np.ascontiguousarray(ii, dtype=np.int64); jj = np.ascontiguousarray(jj, dtype=np.int64)
    out = np.empty((len(ii), p.nz), dtype=np.float64)
    _check(fn(C.byref(p.c()), level, *arrays, len(ii), ii, jj, out), fn.__name__)
    return out


def apply_cols(p: Params, x, ii, jj, level=None):
    """Columns (ii[m], jj[m]) of A x -> array (ncols, nz)."""
    level = p.L if level is None else level
    return _cols(lib().or_api_apply_cols, p, level, [_arr(x, p.level_shape(level))], ii, jj)


def residual_cols(p: Params, u, f, ii, jj, level=None):
    level = p.L if level is None else level
    s = p.level_shape(level)
    return _cols(lib().or_api_residual_cols, p, level, [_arr(u, s), _arr(f, s)], ii, jj)


def precondition_cols(p: Params, r, ii, jj, level=None):
    level = p.L if level is None else level
    return _cols(lib().or_api_precondition_cols, p, level, [_arr(r, p.level_shape(level))], ii, jj)


def smooth_cols(p: Params, u, f, ii, jj, level=None):
    level = p.L if level is None else level
    s = p.level_shape(level)
    return _cols(lib().or_api_smooth_cols, p, level, [_arr(u, s), _arr(f, s)], ii, jj)


def restrict(p: Params, r_fine, fine_level: int | None = None):
    """f_c = R r_f, cell average over the 2x2 horizontal children."""
    fine_level = p.L if fine_level is None else fine_level
    rf = _arr(r_fine, p.level_shape(fine_level))
    fc = np.empty(p.level_shape(fine_level - 1))
    _check(lib().or_api_restrict(C.byref(p.c()), fine_level, rf, fc), "restrict")
    return fc


def prolong_add(p: Params, u_coarse, u_fine, coarse_level: int | None = None):
    """u_f + P u_c, bilinear (9,3,3,1)/16 with zero coarse ghosts ([R7])."""
    coarse_level = p.L - 1 if coarse_level is None else coarse_level
    uc = _arr(u_coarse, p.level_shape(coarse_level))
    uf = _arr(u_fine, p.level_shape(coarse_level + 1)).copy()
    _check(lib().or_api_prolong_add(C.byref(p.c()), coarse_level, uc, uf), "prolong_add")
    return uf


def thomas(s, dg, t, g):
    """Textbook Thomas algorithm."""
    s, dg, t, g = (_arr(v) for v in (s, dg, t, g))
    x = np.empty_like(g)
    _check(lib().or_api_thomas(len(g), s, dg, t, g, x), "thomas")
    return x


def vcycle(p: Params, u, f):
    """One V-cycle, alg:VCycle with the readings [R5]."""
    u = _arr(u, p.level_shape(p.L)).copy(); f = _arr(f, p.level_shape(p.L))
    _check(lib().or_vcycle(C.byref(p.c()), u, f), "vcycle")
    return u


TRACE_KINDS = ("Smooth", "ResSmooth", "Residual", "Prolongate")   # tab:TimingBreakdownMultigrid rows


def vcycle_trace(p: Params, u, f):
    """One V-cycle plus its kernel-call trace: (u_new, counts) with counts[l][kind] the number
    of calls of TRACE_KINDS[kind] on level l (l = 1 coarsest .. L finest; row 0 unused)."""
    u = _arr(u, p.level_shape(p.L)).copy(); f = _arr(f, p.level_shape(p.L))
    counts = np.zeros((p.L + 1, len(TRACE_KINDS)), dtype=np.int32)
    _check(lib().or_api_vcycle_trace(C.byref(p.c()), u, f, counts), "vcycle_trace")
    return u, counts


@dataclass
class SolveResult:
    u: np.ndarray
    iterations: int
    converged: bool
    history: np.ndarray  # ||r_it||, it = 0..iterations


def _solve(fn, p: Params, f, eps, max_iter):
    f = _arr(f, p.level_shape(p.L))
    u = np.empty_like(f)
    it = C.c_int(); conv = C.c_int()
    hist = np.zeros(max_iter + 1)
    _check(fn(C.byref(p.c()), f, u, eps, max_iter, C.byref(it), C.byref(conv), hist,
              max_iter + 1), fn.__name__)
    return SolveResult(u, it.value, bool(conv.value), hist[: it.value + 1].copy())


def solve_mg(p: Params, f, eps: float = 1e-5, max_iter: int = 50) -> SolveResult:
    """Multigrid solve to ||r||/||r_0|| < eps (eqn:epsilonTolerance)."""
    return _solve(lib().or_solve_mg, p, f, eps, max_iter)


def solve_cg(p: Params, f, eps: float = 1e-5, max_iter: int = 1000) -> SolveResult:
    """Line-preconditioned CG, textbook recurrences [R10]."""
    return _solve(lib().or_solve_cg, p, f, eps, max_iter)


def level_fields(p: Params, level: int):
    """(area, ax, ay) of `level` by reading [R26] (block mean of |T|, 8^-s face sums)."""
    ny, nx, _ = p.level_shape(level)
    area = np.empty((ny, nx)); ax = np.empty((ny, nx + 1)); ay = np.empty((ny + 1, nx))
    _check(lib().or_api_level_fields(C.byref(p.c()), level, area, ax, ay), "level_fields")
    return area, ax, ay


def num_threads() -> int:
    return lib().or_api_num_threads()


def set_threads(n: int) -> None:
    """OpenMP threads used over columns (reductions stay deterministic)."""
    lib().or_api_set_threads(int(n))
