"""Time tpmg_prolong_add per level at 1024^2 x 128 (CUDA events, 20 reps) under the
current environment (TPMG_PROLONG_* tuning knobs)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_1402_3545_b200 import tpmg as T

n = 1024
ctx = T.Context(T.make_params(n, n, nz=128))
out = {}
for coarse in (4, 3, 2):
    uc = torch.randn(ctx.shape(coarse), dtype=torch.float64, device="cuda")
    uf = torch.randn(ctx.shape(coarse + 1), dtype=torch.float64, device="cuda")
    for _ in range(3):
        ctx.prolong_add(coarse, uc, uf)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record(ctx.stream)
    for _ in range(20):
        ctx.prolong_add(coarse, uc, uf)
    e1.record(ctx.stream)
    torch.cuda.synchronize()
    us = e0.elapsed_time(e1) / 20 * 1e3
    out[coarse] = round(us, 1)
    bytes_ = uf.numel() * 16 + uc.numel() * 8
    out[f"{coarse}_gbs"] = round(bytes_ / us / 1e3, 0)
print(os.environ.get("TPMG_PROLONG_WANT"), os.environ.get("TPMG_PROLONG_MINLPT"), out)
