"""Per-iteration overhead probe at 1024^2 x 128: solve times with and without the
per-kernel event profiling, and CG/MG with fixed iteration counts."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_1402_3545_b200 import tpmg as T
from inputs import gpu as G

n = 1024
ctx = T.Context(T.make_params(n, n, nz=128))
f = ctx.empty(5)
u = ctx.empty(5)
G.fill_rhs(f, n, seed=0)
torch.cuda.synchronize()


def timed(fn, reps=3):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(ctx.stream)
    for _ in range(reps):
        r = fn()
    e1.record(ctx.stream)
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps, r


for prof in (False, True):
    ctx.profile(prof)
    t_cg, r = timed(lambda: ctx.solve_cg(f, u))
    t_mg, rm = timed(lambda: ctx.solve_mg(f, u))
    t_cg1, _ = timed(lambda: ctx.solve_cg(f, u, max_iter=1))
    t_cg11, _ = timed(lambda: ctx.solve_cg(f, u, max_iter=11))
    t_vc, _ = timed(lambda: ctx.vcycle(u, f), reps=10)
    ctx.profile(False)
    print(f"PDL={os.environ.get('TPMG_PDL', '0')} profile={prof}: CG {t_cg:.2f} ms ({r.iterations} it), per it {(t_cg11 - t_cg1) / 10 * 1e3:.1f} us; "
          f"MG {t_mg:.2f} ms ({rm.iterations} cycles); vcycle {t_vc * 1e3:.1f} us")
