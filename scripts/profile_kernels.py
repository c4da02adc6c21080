"""Launch each hot kernel once at the bench workload (1024 x 1024 x 128) for ncu.

Order of launches (k_line modes: 0 apply, 1 residual, 2 precondition, 3 smooth,
4 CG direction, 5 CG preconditioner):
  smooth(fine) ; precondition(fine) ; residual+norm(fine) ;
  CG solve with max_iter=1: CGPREC(setup), CGDIR, CGPREC ;
  one V-cycle (all levels).
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_1402_3545_b200 import tpmg as T
from inputs import gpu as G

n = int(os.environ.get("PROF_N", "1024"))
ctx = T.Context(T.make_params(n, n, nz=128))
if os.environ.get("PROF_FIELDS"):   # per-column fields (tpmg_set_fields), e.g. PROF_FIELDS=smooth
    from inputs import horizontal_fields
    ctx.set_fields(*horizontal_fields(n, n, 8.4 * 8.4 / 4, 1, os.environ["PROF_FIELDS"]))
f = ctx.empty(5)
if os.environ.get("PROF_CG_ONLY"):   # wide grids: the CG kernels only (fewer buffers)
    G.fill_rhs(f, n, seed=0)
    z = ctx.empty(5)
    ctx.solve_cg(f, z, max_iter=1)
    torch.cuda.synchronize()
    print("profile_kernels done", ctx.stats())
    sys.exit(0)
u = ctx.empty(5)
G.fill_rhs(f, n, seed=0)
G.fill_rhs(u, n, seed=1)
z = ctx.empty(5)
torch.cuda.synchronize()
ctx.smooth(5, u, f, 1)
ctx.precondition(5, f, z)
ctx.residual(5, u, f, None, want_norm2=True)
ctx.solve_cg(f, z, max_iter=1)
ctx.vcycle(u, f)
torch.cuda.synchronize()
print("profile_kernels done", ctx.stats())
