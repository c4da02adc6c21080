"""Helpers shared by the GPU parity tests (test infrastructure)."""
from __future__ import annotations

import numpy as np

from oracle import oracle as O


def lib():
    from paper_1402_3545_b200 import build
    build.build()
    from paper_1402_3545_b200 import tpmg
    return tpmg


def ctx_for(p: O.Params, device: int = 0, loader: str | None = None):
    """loader: None (library defaults: TMA loads, k-split Thomas where supported),
    "tma" (same), "cpasync" (cp.async loads, one-thread-per-column kernel), "tma-noks"
    (TMA, k-split off), "tma-ks2" (TMA, k-split 2x8 config).  Read at tpmg_create."""
    import os
    T = lib()
    for var in ("TPMG_LOADER", "TPMG_KSPLIT", "TPMG_FUSE_PROLONG"):
        os.environ.pop(var, None)
    if loader == "cpasync":
        os.environ["TPMG_LOADER"] = "cpasync"
    elif loader == "tma-noks":
        os.environ["TPMG_KSPLIT"] = "0"
    elif loader == "tma-ks2":
        os.environ["TPMG_KSPLIT"] = "1"   # the non-default k-split config (2 x 8 levels)
    elif loader == "tma-fuse":
        os.environ["TPMG_FUSE_PROLONG"] = "1"
    params = T.make_params(p.nx, p.ny, nz=p.nz, nu_cfl=p.nu_cfl, H=p.H, lam=p.lam, levels=p.L,
                           pre=p.pre, post=p.post, coarse_sweeps=p.coarse_sweeps, rho=p.rho,
                           boundary=p.boundary)
    ctx = T.Context(params, device=device)
    if getattr(p, "profiles", None) is not None:
        ctx.set_profiles(*p.profiles)
    return ctx


def to_dev(x_zc: np.ndarray):
    """oracle layout (ny, nx, nz) -> CUDA tensor in Lambda layout (ny, nz, nx)."""
    import torch
    return torch.from_numpy(O.to_lambda(x_zc)).cuda()


def to_host_zc(t) -> np.ndarray:
    import torch
    torch.cuda.synchronize()
    return O.from_lambda(t.cpu().numpy())


def rel_l2(a, b) -> float:
    a = np.ravel(a); b = np.ravel(b)
    nb = np.linalg.norm(b)
    return float(np.linalg.norm(a - b) / (nb if nb > 0 else 1.0))


COLF = 50.0   # per-column bar = COLF x the whole-field bar


def col_err(a, b) -> float:
    """Largest error of one vertical column (z-contiguous (ny, nx, nz) arrays), relative to the
    RMS column norm of b: a wrong tile seam, boundary column or halo row changes a few columns,
    which the whole-field rel-L2 dilutes by the number of columns."""
    a = np.asarray(a, dtype=np.float64)
    b = np.asarray(b, dtype=np.float64)
    if a.ndim != 3:
        return rel_l2(a, b)
    d = np.linalg.norm(a - b, axis=2)
    w = np.linalg.norm(b, axis=2)
    scale = float(np.sqrt(np.mean(w * w)))
    return float(d.max() / (scale if scale > 0 else 1.0))


def close(got, want, t: float) -> bool:
    """Whole-field rel-L2 < t AND every column within COLF * t (relative to the RMS column)."""
    return rel_l2(got, want) < t and col_err(got, want) < COLF * t
