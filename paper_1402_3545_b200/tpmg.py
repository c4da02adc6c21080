"""Thin Python binding of libtpmg.so (include/tpmg.h), argument marshalling only.

Every function has the C name and signature; vectors may be torch CUDA
tensors (float64, contiguous, shape ``[ny_l, nz, nx_l]`` in the paper's
Lambda layout) or raw device addresses (int).  Every step of the
solver runs in the library's sm_100a kernels; there is no Python or CPU
fallback: if the shared library is missing or fails to load, importing this
module raises.

``Context`` wraps a ``tpmg_ctx*`` for convenience.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass, field

_PKG = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("TPMG_LIB_PATH") or os.path.join(_PKG, "libtpmg.so")   # (override: A/B builds)

if not os.path.exists(LIB_PATH):
    raise ImportError(
        f"{LIB_PATH} is missing: build it with `python -m paper_1402_3545_b200.build` "
        "(there is no fallback path)")
_lib = C.CDLL(LIB_PATH)

TPMG_OK, TPMG_E_PARAM, TPMG_E_SHAPE, TPMG_E_RANGE, TPMG_E_SINGULAR, TPMG_E_BREAKDOWN, \
    TPMG_E_TOPOLOGY, TPMG_E_CUDA, TPMG_E_NCCL, TPMG_E_OOM = range(10)
STATUS_NAMES = ["TPMG_OK", "TPMG_E_PARAM", "TPMG_E_SHAPE", "TPMG_E_RANGE", "TPMG_E_SINGULAR",
                "TPMG_E_BREAKDOWN", "TPMG_E_TOPOLOGY", "TPMG_E_CUDA", "TPMG_E_NCCL", "TPMG_E_OOM"]
TPMG_SOLVER_CG, TPMG_SOLVER_MG = 0, 1


class tpmg_params(C.Structure):
    _fields_ = [("nx", C.c_int64), ("ny", C.c_int64), ("nz", C.c_int32),
                ("nu_cfl", C.c_double), ("H", C.c_double), ("lambda_", C.c_double),
                ("levels", C.c_int32), ("pre", C.c_int32), ("post", C.c_int32),
                ("coarse_sweeps", C.c_int32), ("rho", C.c_double), ("boundary", C.c_int32)]


class tpmg_result(C.Structure):
    _fields_ = [("iterations", C.c_int32), ("converged", C.c_int32), ("r0_norm", C.c_double),
                ("rel_residual", C.c_double), ("seconds", C.c_double),
                ("history", C.POINTER(C.c_double)), ("history_cap", C.c_int32)]


class tpmg_stats(C.Structure):
    _fields_ = [("kernel_launches", C.c_int64), ("halo_exchanges", C.c_int64),
                ("allreduces", C.c_int64), ("graph_launches", C.c_int64),
                ("p2p_halo", C.c_int64), ("p2p_allreduce", C.c_int64)]


_vp, _i32, _i64, _d = C.c_void_p, C.c_int32, C.c_int64, C.c_double
_P = C.POINTER
_SIGS = {
    "tpmg_version": ([], _i32),
    "tpmg_params_default": ([_P(tpmg_params)], None),
    "tpmg_nccl_id": ([_vp], C.c_int),
    "tpmg_partition": ([_P(tpmg_params), _i32, _i32, _i32, _P(_i64), _P(_i64)], C.c_int),
    "tpmg_create": ([_P(tpmg_params), _i32, _i32, _vp, _i32, _vp, _P(_vp)], C.c_int),
    "tpmg_destroy": ([_vp], C.c_int),
    "tpmg_set_stream": ([_vp, _vp], C.c_int),
    "tpmg_local_box": ([_vp, _i32, _P(_i64), _P(_i64), _P(_i64), _P(_i32)], C.c_int),
    "tpmg_apply": ([_vp, _i32, _vp, _vp], C.c_int),
    "tpmg_residual": ([_vp, _i32, _vp, _vp, _vp, _P(_d)], C.c_int),
    "tpmg_precondition": ([_vp, _i32, _vp, _vp], C.c_int),
    "tpmg_smooth": ([_vp, _i32, _vp, _vp, _i32], C.c_int),
    "tpmg_restrict": ([_vp, _i32, _vp, _vp], C.c_int),
    "tpmg_prolong_add": ([_vp, _i32, _vp, _vp], C.c_int),
    "tpmg_vcycle": ([_vp, _vp, _vp], C.c_int),
    "tpmg_solve_mg": ([_vp, _vp, _vp, _d, _i32, _P(tpmg_result)], C.c_int),
    "tpmg_solve_cg": ([_vp, _vp, _vp, _d, _i32, _P(tpmg_result)], C.c_int),
    "tpmg_solve_host": ([_vp, C.c_int, _vp, _vp, _d, _i32, _P(tpmg_result)], C.c_int),
    "tpmg_solve_host_zc": ([_vp, C.c_int, _vp, _vp, _d, _i32, _P(tpmg_result)], C.c_int),
    "tpmg_transpose": ([_vp, _i32, _i32, _vp, _vp], C.c_int),
    "tpmg_get_stats": ([_vp, _P(tpmg_stats)], C.c_int),
    "tpmg_stats_reset": ([_vp], C.c_int),
    "tpmg_profile": ([_vp, _i32], C.c_int),
    "tpmg_profile_mask": ([_vp, C.c_uint32], C.c_int),
    "tpmg_set_profiles": ([_vp, _P(_d), _P(_d), _P(_d), _P(_d)], C.c_int),
    "tpmg_set_fields": ([_vp, _P(_d), _P(_d), _P(_d)], C.c_int),
    "tpmg_profile_read": ([_vp, _i32, _P(_i64), _P(_d), _P(_d)], C.c_int),
    "tpmg_solve_host_pair": ([_vp, _vp, _vp, _vp, _d, _i32, _i32, _P(tpmg_result), _P(tpmg_result)], C.c_int),
    "tpmg_halo_push": ([_vp, _i32, _vp, _vp, _vp], C.c_int),
    "tpmg_cg_halo": ([_vp, _d, _vp, _vp, _vp, _vp, _vp, _vp], C.c_int),
    "tpmg_last_error": ([_vp], C.c_char_p),
}
for _name, (_args, _ret) in _SIGS.items():
    _fn = getattr(_lib, _name)
    _fn.argtypes = _args
    _fn.restype = _ret


class TpmgError(RuntimeError):
    def __init__(self, status: int, msg: str):
        self.status = status
        super().__init__(f"{STATUS_NAMES[status] if 0 <= status < 10 else status}: {msg}")


_ctx_device: dict = {}   # context handle -> CUDA device index (set by tpmg_create)
_ctx_levels: dict = {}   # context handle -> number of levels L


def _level_numel(ctx, level) -> int:
    _, nx, ny, nz = tpmg_local_box(ctx, level)
    return nx * ny * nz


def _ptr(x, ctx=None, level=None, what="vector"):
    """Device address of a torch tensor or an int (a raw address is passed unchecked).
    A tensor must be a contiguous float64 CUDA tensor on the context's device with exactly
    the cells of `level`'s local box (checked before the C library is called: an undersized
    or host tensor would otherwise be read / written out of bounds by the kernels)."""
    if x is None:
        return None
    if isinstance(x, int):
        return x
    import torch
    if not isinstance(x, torch.Tensor):
        raise TypeError(f"{what}: expected a torch tensor or an address, got {type(x)}")
    if x.dtype != torch.float64 or not x.is_contiguous():
        raise ValueError(f"{what}: vectors must be contiguous float64 tensors (Lambda layout)")
    if not x.is_cuda:
        raise ValueError(f"{what}: expected a CUDA tensor, got one on {x.device}")
    if ctx is not None and ctx in _ctx_device and x.device.index != _ctx_device[ctx]:
        raise ValueError(f"{what}: tensor on cuda:{x.device.index}, context on cuda:{_ctx_device[ctx]}")
    if ctx is not None and level is not None:
        n = _level_numel(ctx, level)
        if x.numel() != n:
            raise ValueError(f"{what}: {x.numel()} elements, level {level}'s local box has {n}")
    return x.data_ptr()


def _lv(ctx, level, lo=1, hi=0):
    """`level` when it lies in [lo, L + hi] (size checks apply), else None: an out-of-range
    level is left to the C library, which reports it (TPMG_E_RANGE)."""
    L = _ctx_levels.get(ctx)
    return level if L is not None and lo <= level <= L + hi else None


def _fine(ctx) -> int:
    """The finest level L of a context (recorded by tpmg_create)."""
    return _ctx_levels[ctx]


def _check(st: int, ctx=None):
    if st != TPMG_OK:
        raise TpmgError(st, _lib.tpmg_last_error(ctx).decode())


# ----------------------------------------------------------------- C-named functions

def tpmg_version() -> int:
    return _lib.tpmg_version()


def tpmg_params_default() -> tpmg_params:
    p = tpmg_params()
    _lib.tpmg_params_default(C.byref(p))
    return p


def tpmg_nccl_id() -> bytes:
    buf = C.create_string_buffer(128)
    _check(_lib.tpmg_nccl_id(buf))
    return buf.raw


def tpmg_partition(params: tpmg_params, rank: int, nranks: int, level: int):
    """(y0, ny) of rank's strip on `level` (host-only, no GPU)."""
    y0, ny = _i64(), _i64()
    _check(_lib.tpmg_partition(C.byref(params), rank, nranks, level, C.byref(y0), C.byref(ny)))
    return y0.value, ny.value


def tpmg_create(params: tpmg_params, rank: int = 0, nranks: int = 1, id128: bytes | None = None,
                device: int = 0, cuda_stream: int | None = None) -> int:
    out = _vp()
    idbuf = C.create_string_buffer(id128, 128) if id128 is not None else None
    _check(_lib.tpmg_create(C.byref(params), rank, nranks, idbuf, device, cuda_stream, C.byref(out)))
    _ctx_device[out.value] = device
    _ctx_levels[out.value] = tpmg_params_levels(params)
    return out.value


def tpmg_destroy(ctx: int) -> None:
    _ctx_device.pop(ctx, None)
    _ctx_levels.pop(ctx, None)
    _check(_lib.tpmg_destroy(ctx))


def tpmg_set_stream(ctx: int, cuda_stream: int | None) -> None:
    _check(_lib.tpmg_set_stream(ctx, cuda_stream), ctx)


def tpmg_local_box(ctx: int, level: int):
    y0, nx, ny, nz = _i64(), _i64(), _i64(), _i32()
    _check(_lib.tpmg_local_box(ctx, level, C.byref(y0), C.byref(nx), C.byref(ny), C.byref(nz)), ctx)
    return y0.value, nx.value, ny.value, nz.value


def tpmg_apply(ctx: int, level: int, x, y) -> None:
    _check(_lib.tpmg_apply(ctx, level, _ptr(x, ctx, _lv(ctx, level), "x"), _ptr(y, ctx, _lv(ctx, level), "y")), ctx)


def tpmg_residual(ctx: int, level: int, u, f, r=None, want_norm2: bool = False):
    n2 = _d()
    _check(_lib.tpmg_residual(ctx, level, _ptr(u, ctx, _lv(ctx, level), "u"), _ptr(f, ctx, _lv(ctx, level), "f"), _ptr(r, ctx, _lv(ctx, level), "r"),
                              C.byref(n2) if want_norm2 else None), ctx)
    return n2.value if want_norm2 else None


def tpmg_precondition(ctx: int, level: int, r, z) -> None:
    _check(_lib.tpmg_precondition(ctx, level, _ptr(r, ctx, _lv(ctx, level), "r"), _ptr(z, ctx, _lv(ctx, level), "z")), ctx)


def tpmg_smooth(ctx: int, level: int, u, f, sweeps: int = 1) -> None:
    _check(_lib.tpmg_smooth(ctx, level, _ptr(u, ctx, _lv(ctx, level), "u"), _ptr(f, ctx, _lv(ctx, level), "f"), sweeps), ctx)


def tpmg_restrict(ctx: int, fine_level: int, r_fine, f_coarse) -> None:
    _check(_lib.tpmg_restrict(ctx, fine_level, _ptr(r_fine, ctx, _lv(ctx, fine_level, 2), "r_fine"),
                              _ptr(f_coarse, ctx, _lv(ctx, fine_level, 2) and fine_level - 1, "f_coarse")), ctx)


def tpmg_prolong_add(ctx: int, coarse_level: int, u_coarse, u_fine) -> None:
    _check(_lib.tpmg_prolong_add(ctx, coarse_level, _ptr(u_coarse, ctx, _lv(ctx, coarse_level, 1, -1), "u_coarse"),
                                 _ptr(u_fine, ctx, _lv(ctx, coarse_level, 1, -1) and coarse_level + 1, "u_fine")), ctx)


def tpmg_vcycle(ctx: int, u, f) -> None:
    L = _fine(ctx)
    _check(_lib.tpmg_vcycle(ctx, _ptr(u, ctx, L, "u"), _ptr(f, ctx, L, "f")), ctx)


@dataclass
class SolveResult:
    iterations: int
    converged: bool
    r0_norm: float
    rel_residual: float
    seconds: float
    history: list = field(default_factory=list)


def _result(max_iter: int):
    hist = (C.c_double * (max_iter + 1))()
    res = tpmg_result()
    res.history = C.cast(hist, C.POINTER(C.c_double))
    res.history_cap = max_iter + 1
    return res, hist


def _to_py(res: tpmg_result, hist) -> SolveResult:
    return SolveResult(res.iterations, bool(res.converged), res.r0_norm, res.rel_residual,
                       res.seconds, list(hist[: res.iterations + 1]))


def tpmg_solve_mg(ctx: int, f, u, eps: float = 1e-5, max_iter: int = 50) -> SolveResult:
    res, hist = _result(max_iter)
    L = _fine(ctx)
    _check(_lib.tpmg_solve_mg(ctx, _ptr(f, ctx, L, "f"), _ptr(u, ctx, L, "u"), eps, max_iter, C.byref(res)), ctx)
    return _to_py(res, hist)


def tpmg_solve_cg(ctx: int, f, u, eps: float = 1e-5, max_iter: int = 1000) -> SolveResult:
    res, hist = _result(max_iter)
    L = _fine(ctx)
    _check(_lib.tpmg_solve_cg(ctx, _ptr(f, ctx, L, "f"), _ptr(u, ctx, L, "u"), eps, max_iter, C.byref(res)), ctx)
    return _to_py(res, hist)


TPMG_ZC_TO_LAMBDA, TPMG_LAMBDA_TO_ZC = 0, 1


def tpmg_transpose(ctx: int, level: int, direction: int, src, dst) -> None:
    """z-contiguous <-> Lambda layout of a level's local box (device tensors)."""
    _check(_lib.tpmg_transpose(ctx, level, direction, _ptr(src, ctx, _lv(ctx, level), "src"), _ptr(dst, ctx, _lv(ctx, level), "dst")), ctx)


def tpmg_solve_host_zc(ctx: int, solver: int, f_host, u_host, eps: float = 1e-5,
                       max_iter: int = 1000) -> SolveResult:
    """tpmg_solve_host with z-contiguous host buffers (the paper's total-time path)."""
    return tpmg_solve_host(ctx, solver, f_host, u_host, eps, max_iter, _fn="tpmg_solve_host_zc")


def tpmg_solve_host(ctx: int, solver: int, f_host, u_host, eps: float = 1e-5,
                    max_iter: int = 1000, _fn: str = "tpmg_solve_host") -> SolveResult:
    """f_host / u_host: CPU float64 torch tensors (pinned or pageable) with the local fine
    box's cells, or host addresses (unchecked)."""
    import torch
    n = _level_numel(ctx, _fine(ctx))

    def hptr(x):
        if isinstance(x, int):
            return x
        if not isinstance(x, torch.Tensor) or x.device.type != "cpu" or not x.is_contiguous():
            raise ValueError("host buffers must be contiguous CPU tensors")
        if x.dtype != torch.float64 or x.numel() != n:
            raise ValueError(f"host buffers must be float64 with {n} elements (got {x.dtype}, {x.numel()})")
        return x.data_ptr()
    res, hist = _result(max_iter)
    _check(getattr(_lib, _fn)(ctx, solver, hptr(f_host), hptr(u_host), eps, max_iter,
                              C.byref(res)), ctx)
    return _to_py(res, hist)


def _plane_ptr(x, ctx, n, what):
    """Address of a device plane of n doubles (checked like _ptr), None passes through."""
    if x is None or isinstance(x, int):
        return x
    p = _ptr(x, ctx, None, what)
    if x.numel() != n:
        raise ValueError(f"{what}: {x.numel()} elements, a plane has {n}")
    return p


def tpmg_halo_push(ctx: int, level: int, src, dst_lo=None, dst_hi=None) -> None:
    """dst_lo <- row 0 of src, dst_hi <- row ny-1 of src (the P2P halo push kernel)."""
    lv = _lv(ctx, level)
    n = None
    if lv is not None:
        _, nx, _, nz = tpmg_local_box(ctx, level)
        n = nx * nz
    _check(_lib.tpmg_halo_push(ctx, level, _ptr(src, ctx, lv, "src"),
                               _plane_ptr(dst_lo, ctx, n, "dst_lo") if n else _ptr(dst_lo),
                               _plane_ptr(dst_hi, ctx, n, "dst_hi") if n else _ptr(dst_hi)), ctx)


def tpmg_cg_halo(ctx: int, beta: float, out_lo=None, z_lo=None, p_lo=None, out_hi=None, z_hi=None, p_hi=None) -> None:
    """out = fma(beta, p, z) on each non-None fine-level halo plane (the CG p-halo update)."""
    _, nx, _, nz = tpmg_local_box(ctx, _fine(ctx))
    n = nx * nz
    args = [_plane_ptr(x, ctx, n, w) for x, w in ((out_lo, "out_lo"), (z_lo, "z_lo"), (p_lo, "p_lo"),
                                                  (out_hi, "out_hi"), (z_hi, "z_hi"), (p_hi, "p_hi"))]
    _check(_lib.tpmg_cg_halo(ctx, float(beta), *args), ctx)


def tpmg_solve_host_pair(ctx: int, f_host, u_mg_host, u_cg_host, eps: float = 1e-5, max_iter_mg: int = 50,
                         max_iter_cg: int = 1000):
    """MG and PCG solves of one host RHS: f copied in once, u_mg's copy out overlapping the PCG
    solve.  Host buffers as tpmg_solve_host.  Returns (SolveResult mg, SolveResult cg)."""
    import torch
    n = _level_numel(ctx, _fine(ctx))

    def hptr(x):
        if isinstance(x, int):
            return x
        if not isinstance(x, torch.Tensor) or x.device.type != "cpu" or not x.is_contiguous():
            raise ValueError("host buffers must be contiguous CPU tensors")
        if x.dtype != torch.float64 or x.numel() != n:
            raise ValueError(f"host buffers must be float64 with {n} elements (got {x.dtype}, {x.numel()})")
        return x.data_ptr()
    rm, hm = _result(max_iter_mg)
    rc, hc = _result(max_iter_cg)
    _check(_lib.tpmg_solve_host_pair(ctx, hptr(f_host), hptr(u_mg_host), hptr(u_cg_host), eps, max_iter_mg,
                                     max_iter_cg, C.byref(rm), C.byref(rc)), ctx)
    return _to_py(rm, hm), _to_py(rc, hc)


def tpmg_get_stats(ctx: int) -> dict:
    s = tpmg_stats()
    _check(_lib.tpmg_get_stats(ctx, C.byref(s)), ctx)
    return {name: getattr(s, name) for name, _ in tpmg_stats._fields_}


def tpmg_stats_reset(ctx: int) -> None:
    _check(_lib.tpmg_stats_reset(ctx), ctx)


KERNEL_CLASSES = ["apply", "residual", "precondition", "smooth", "cg_direction",
                  "cg_precondition", "residual_restrict", "restrict", "prolong_add", "dot",
                  "smooth_prolong"]


def tpmg_profile(ctx: int, enable: bool) -> None:
    _check(_lib.tpmg_profile(ctx, 1 if enable else 0), ctx)


def tpmg_set_profiles(ctx: int, a=None, b=None, c=None, d=None) -> None:
    """General vertical profiles (host float64 arrays of nz), or all None for the flat box."""
    if a is None:
        _check(_lib.tpmg_set_profiles(ctx, None, None, None, None), ctx)
        return
    import numpy as np
    arrs = [np.ascontiguousarray(x, dtype=np.float64) for x in (a, b, c, d)]
    ptrs = [x.ctypes.data_as(_P(_d)) for x in arrs]
    _check(_lib.tpmg_set_profiles(ctx, *ptrs), ctx)


def tpmg_set_fields(ctx: int, area=None, ax=None, ay=None) -> None:
    """Per-column fields |T| [ny, nx], x-face alpha [ny, nx+1], y-face alpha [ny+1, nx] of the
    global finest level (host float64), or all None for the uniform coefficients."""
    if area is None:
        _check(_lib.tpmg_set_fields(ctx, None, None, None), ctx)
        return
    import numpy as np
    arrs = [np.ascontiguousarray(x, dtype=np.float64) for x in (area, ax, ay)]
    ny, nx = arrs[0].shape
    if arrs[1].shape != (ny, nx + 1) or arrs[2].shape != (ny + 1, nx):
        raise ValueError(f"field shapes {[a.shape for a in arrs]} do not match [ny, nx], [ny, nx+1], [ny+1, nx]")
    ptrs = [x.ctypes.data_as(_P(_d)) for x in arrs]
    _check(_lib.tpmg_set_fields(ctx, *ptrs), ctx)


def tpmg_profile_mask(ctx: int, mask: int) -> None:
    _check(_lib.tpmg_profile_mask(ctx, mask), ctx)


def tpmg_profile_read(ctx: int, kernel: int):
    n, ms, cells = _i64(), _d(), _d()
    _check(_lib.tpmg_profile_read(ctx, kernel, C.byref(n), C.byref(ms), C.byref(cells)), ctx)
    return n.value, ms.value, cells.value


def tpmg_last_error(ctx: int | None) -> str:
    return _lib.tpmg_last_error(ctx).decode()


# ----------------------------------------------------------------- convenience wrapper

def make_params(nx: int, ny: int, nz: int = 0, nu_cfl: float = 0.0, H: float = 0.0,
                lam: float = 0.0, levels: int = 0, pre: int = 0, post: int = 0,
                coarse_sweeps: int = 0, rho: float = 0.0, boundary: int = 0) -> tpmg_params:
    """Zero fields select the library defaults (include/tpmg.h); boundary: 0 ghost-zero
    Dirichlet [R1], 1 face Dirichlet [R25]."""
    return tpmg_params(nx, ny, nz, nu_cfl, H, lam, levels, pre, post, coarse_sweeps, rho, boundary)


class Context:
    """Owns one tpmg_ctx.  The stream defaults to torch's current stream on `device`."""

    def __init__(self, params: tpmg_params, rank: int = 0, nranks: int = 1,
                 id128: bytes | None = None, device: int = 0, stream=None):
        import torch
        if stream is None:
            stream = torch.cuda.current_stream(device)
        self.stream = stream
        self.params = params
        self.handle = tpmg_create(params, rank, nranks, id128, device, stream.cuda_stream)
        self.device = device
        self.rank, self.nranks = rank, nranks

    def close(self):
        if self.handle:
            tpmg_destroy(self.handle)
            self.handle = 0

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def local_box(self, level: int):
        return tpmg_local_box(self.handle, level)

    def shape(self, level: int):
        _, nx, ny, nz = self.local_box(level)
        return (ny, nz, nx)

    def empty(self, level: int):
        import torch
        return torch.empty(self.shape(level), dtype=torch.float64, device=f"cuda:{self.device}")

    def zeros(self, level: int):
        import torch
        return torch.zeros(self.shape(level), dtype=torch.float64, device=f"cuda:{self.device}")

    @property
    def L(self) -> int:
        return tpmg_params_levels(self.params)

    def apply(self, level, x, y):
        tpmg_apply(self.handle, level, x, y)

    def residual(self, level, u, f, r=None, want_norm2=False):
        return tpmg_residual(self.handle, level, u, f, r, want_norm2)

    def precondition(self, level, r, z):
        tpmg_precondition(self.handle, level, r, z)

    def smooth(self, level, u, f, sweeps=1):
        tpmg_smooth(self.handle, level, u, f, sweeps)

    def restrict(self, fine_level, r_fine, f_coarse):
        tpmg_restrict(self.handle, fine_level, r_fine, f_coarse)

    def prolong_add(self, coarse_level, u_coarse, u_fine):
        tpmg_prolong_add(self.handle, coarse_level, u_coarse, u_fine)

    def vcycle(self, u, f):
        tpmg_vcycle(self.handle, u, f)

    def solve_mg(self, f, u, eps=1e-5, max_iter=50):
        return tpmg_solve_mg(self.handle, f, u, eps, max_iter)

    def solve_cg(self, f, u, eps=1e-5, max_iter=1000):
        return tpmg_solve_cg(self.handle, f, u, eps, max_iter)

    def solve_host(self, solver, f_host, u_host, eps=1e-5, max_iter=1000):
        return tpmg_solve_host(self.handle, solver, f_host, u_host, eps, max_iter)

    def solve_host_pair(self, f_host, u_mg_host, u_cg_host, eps=1e-5, max_iter_mg=50, max_iter_cg=1000):
        return tpmg_solve_host_pair(self.handle, f_host, u_mg_host, u_cg_host, eps, max_iter_mg, max_iter_cg)

    def solve_host_zc(self, solver, f_host, u_host, eps=1e-5, max_iter=1000):
        return tpmg_solve_host_zc(self.handle, solver, f_host, u_host, eps, max_iter)

    def transpose(self, level, direction, src, dst):
        tpmg_transpose(self.handle, level, direction, src, dst)

    def stats(self):
        return tpmg_get_stats(self.handle)

    def stats_reset(self):
        tpmg_stats_reset(self.handle)

    def set_profiles(self, a=None, b=None, c=None, d=None):
        tpmg_set_profiles(self.handle, a, b, c, d)

    def set_fields(self, area=None, ax=None, ay=None):
        tpmg_set_fields(self.handle, area, ax, ay)

    def profile(self, enable: bool, classes=None):
        """Event-time every kernel class (enable), or only the named classes."""
        if classes is None:
            tpmg_profile(self.handle, enable)
        else:
            tpmg_profile_mask(self.handle, sum(1 << KERNEL_CLASSES.index(c) for c in classes) if enable else 0)

    def profile_read(self) -> dict:
        """{class name: (launches, ms, cells)} for every kernel class with launches."""
        out = {}
        for k, name in enumerate(KERNEL_CLASSES):
            n, ms, cells = tpmg_profile_read(self.handle, k)
            if n:
                out[name] = (n, ms, cells)
        return out


def tpmg_params_levels(p: tpmg_params) -> int:
    return p.levels if p.levels else 5


# exported C symbols (checked by the CPU test that the library exports what the header declares)
EXPORTED = tuple(_SIGS)
