"""Small-shape driver of every library kernel, for compute-sanitizer.

    compute-sanitizer --tool {memcheck,racecheck,synccheck} python scripts/sanitize_driver.py [variant]

variant selects the loader / kernel family (read by tpmg_create from the environment):
  tma (default: TMA loads, k-split Thomas, TMEM g' buffer), tma3 (TMEM form with the 3-stage ring),
  notmem (g' in shared memory), cpasync (cp.async loads), noks (one-thread-per-column Thomas),
  fuse (fused prolongation + post-smooth), face (face-Dirichlet boundary classes), fields, profiles.
Shapes span several tiles and ragged tails but stay small (sanitizers are ~100x slower)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
variant = sys.argv[1] if len(sys.argv) > 1 else "tma"
env = {"tma3": {"TPMG_TM_STAGES": "3"}, "notmem": {"TPMG_TMEM": "0"}, "cpasync": {"TPMG_LOADER": "cpasync"},
       "noks": {"TPMG_KSPLIT": "0"}, "fuse": {"TPMG_FUSE_PROLONG": "1"}}.get(variant, {})
os.environ.update(env)
import numpy as np
import torch

from paper_1402_3545_b200 import tpmg as T
from inputs import gpu as G

nx, ny, nz, L = 96, 64, 32, 3
p = T.make_params(nx, ny, nz=nz, levels=L, boundary=1 if variant == "face" else 0)
ctx = T.Context(p)
if variant == "profiles":
    from inputs import vertical_profiles
    ctx.set_profiles(*vertical_profiles(nz, 3, 100.0))
if variant == "fields":
    from inputs import horizontal_fields
    ctx.set_fields(*horizontal_fields(nx, ny, 8.4 * 8.4 / 4, 1, "random"))
f = ctx.empty(L)
u = ctx.empty(L)
G.fill_rhs(f, nx, seed=0)
G.fill_rhs(u, nx, seed=1)
w = ctx.empty(L)
ctx.apply(L, u, w)
ctx.residual(L, u, f, w, want_norm2=True)
ctx.precondition(L, f, w)
ctx.smooth(L, u, f, 2)
fc = ctx.empty(L - 1)
ctx.restrict(L, f, fc)
ctx.prolong_add(L - 1, fc, u)
ctx.vcycle(u, f)
r = ctx.solve_mg(f, u, max_iter=3)
r2 = ctx.solve_cg(f, u, max_iter=5)
zc = torch.empty(ny, nx, nz, dtype=torch.float64, device="cuda")
ctx.transpose(L, T.TPMG_LAMBDA_TO_ZC, u, zc)
ctx.transpose(L, T.TPMG_ZC_TO_LAMBDA, zc, w)
lo = torch.zeros(nz, nx, dtype=torch.float64, device="cuda")
hi = torch.zeros_like(lo)
T.tpmg_halo_push(ctx.handle, L, u, lo, hi)
T.tpmg_cg_halo(ctx.handle, 0.5, lo, u[0], u[1], hi, u[2], u[3])
fh = f.cpu().pin_memory()
uh = torch.empty_like(fh).pin_memory()
ctx.solve_host(T.TPMG_SOLVER_MG, fh, uh, max_iter=2)
torch.cuda.synchronize()
print(f"sanitize_driver {variant} ok: mg {r.iterations} cg {r2.iterations} launches {ctx.stats()['kernel_launches']}",
      flush=True)
ctx.close()
