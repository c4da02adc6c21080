"""Run each line-kernel mode with each loader in its own process (a sticky CUDA
error in one cannot hide the others).  Debug aid for the GPU box."""
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CODE = r'''
import os, sys
sys.path.insert(0, {root!r})
os.environ["TPMG_SYNC_DEBUG"] = "1"
os.environ["TPMG_LOADER"] = {loader!r}
import torch
from paper_1402_3545_b200 import tpmg as T
nx, ny, nz = {shape}
p = T.make_params(nx, ny, nz=nz, levels=1)
ctx = T.Context(p)
a = torch.randn((ny, nz, nx), dtype=torch.float64, device="cuda")
b = torch.randn_like(a); c = torch.empty_like(a)
op = {op!r}
if op == "apply": ctx.apply(1, a, c)
elif op == "residual": print(ctx.residual(1, a, b, c, want_norm2=True))
elif op == "precondition": ctx.precondition(1, a, c)
elif op == "smooth": ctx.smooth(1, a, b, 1)
elif op == "mg": print(ctx.solve_mg(b, c, max_iter=2))
elif op == "cg": print(ctx.solve_cg(b, c, max_iter=2))
torch.cuda.synchronize()
print("OK", op, {loader!r}, {shape})
'''
for shape in [(32, 32, 16), (64, 16, 8)]:
    for loader in ("cpasync", "tma"):
        for op in ("apply", "residual", "precondition", "smooth", "mg", "cg"):
            r = subprocess.run([sys.executable, "-c", CODE.format(root=ROOT, loader=loader, shape=shape, op=op)],
                               capture_output=True, text=True, timeout=120)
            tail = (r.stdout + r.stderr).strip().splitlines()[-1:] 
            print(f"{op:13s} {loader:8s} {shape}: rc={r.returncode} {tail}", flush=True)
