"""A/B of two library builds on one GPU: CG iteration and V-cycle time at 1024^2 x 128.
usage: python scripts/ab_probe.py <package root dir>"""
import os
import sys

root = os.path.abspath(sys.argv[1])
sys.path.insert(0, root)
import torch

from paper_1402_3545_b200 import build, tpmg as T
from inputs import gpu as G

build.build()
assert T.LIB_PATH.startswith(root), T.LIB_PATH
ctx = T.Context(T.make_params(1024, 1024, nz=128))
f = ctx.empty(5)
u = ctx.empty(5)
G.fill_rhs(f, 1024, seed=0)


def timed(fn, reps):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(ctx.stream)
    for _ in range(reps):
        fn()
    e1.record(ctx.stream)
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


t1 = timed(lambda: ctx.solve_cg(f, u, max_iter=1), 3)
t21 = timed(lambda: ctx.solve_cg(f, u, max_iter=21), 3)
tv = timed(lambda: ctx.vcycle(u, f), 10)
ctx.profile(True)
for _ in range(5):
    ctx.vcycle(u, f)
prof = ctx.profile_read()
ctx.profile(False)
per = {k: round(ms / n * 1e3, 1) for k, (n, ms, c) in prof.items()}
print(f"{os.path.basename(root)}: CG iteration {(t21 - t1) / 20 * 1e3:.0f} us, vcycle {tv * 1e3:.0f} us; "
      f"vcycle kernels avg us {per}", flush=True)
