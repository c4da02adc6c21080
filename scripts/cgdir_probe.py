"""One CG iteration at the (nx, ny) x 128 given on the command line (for ncu)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_1402_3545_b200 import tpmg as T
from inputs import gpu as G

nx, ny = int(sys.argv[1]), int(sys.argv[2])
ctx = T.Context(T.make_params(nx, ny, nz=128))
f = ctx.empty(5)
u = ctx.empty(5)
G.fill_rhs(f, nx, seed=0)
ctx.solve_cg(f, u, max_iter=2)
torch.cuda.synchronize()
print("done", nx, ny)
