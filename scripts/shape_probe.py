"""CG kernel bandwidth vs grid shape: cg_direction / cg_precondition GB/s from
event-timed CG iterations (max_iter fixed) at several (nx, ny) x 128."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_1402_3545_b200 import tpmg as T
from inputs import gpu as G

BPC = {"cg_direction": 24, "cg_precondition": 48, "smooth": 24, "precondition": 16}
SHAPES = [(1024, 1024), (2048, 512), (4096, 256), (512, 2048), (2048, 2048), (4096, 1024), (4096, 4096)]
if len(sys.argv) > 1:
    SHAPES = [tuple(int(v) for v in a.split("x")) for a in sys.argv[1:]]
for nx, ny in SHAPES:
    ctx = T.Context(T.make_params(nx, ny, nz=128))
    f = ctx.empty(5)
    u = ctx.empty(5)
    G.fill_rhs(f, nx, seed=0)
    ctx.solve_cg(f, u, max_iter=3)
    ctx.profile(True)
    ctx.solve_cg(f, u, max_iter=8)
    prof = ctx.profile_read()
    ctx.profile(False)
    out = {k: round(c * BPC[k] / (ms * 1e-3) / 1e9) for k, (n, ms, c) in prof.items() if k in BPC}
    print(os.environ.get("TPMG_LOADER", "tma"), nx, ny, out, flush=True)
    del ctx, f, u
    torch.cuda.empty_cache()
