"""Multi-rank timing probe (torchrun, one rank per GPU): per-V-cycle and per-CG-iteration
device time at 1024^2 x 128 per rank, max over ranks, under the current TPMG_* env."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import torch.distributed as dist

from paper_1402_3545_b200 import tpmg as T
from inputs import gpu as G

rank, world, local = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"]), int(os.environ["LOCAL_RANK"])
torch.cuda.set_device(local)
dist.init_process_group("nccl", device_id=torch.device("cuda", local))
obj = [T.tpmg_nccl_id() if rank == 0 else None]
dist.broadcast_object_list(obj, src=0)
n = int(os.environ.get("PROBE_N", "1024"))
stream = torch.cuda.Stream()
ctx = T.Context(T.make_params(n, n * world, nz=128), rank=rank, nranks=world, id128=obj[0], device=local, stream=stream)
f = ctx.empty(5)
u = ctx.empty(5)
with torch.cuda.stream(stream):
    G.fill_rhs(f, n, y0=ctx.local_box(5)[0], seed=0, stream=stream)
stream.synchronize()


def timed(fn, reps):
    fn()
    torch.cuda.synchronize()
    dist.barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(reps):
        fn()
    e1.record(stream)
    torch.cuda.synchronize()
    t = torch.tensor([e0.elapsed_time(e1) / reps], device="cuda")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t)


u.zero_()
t_vc = timed(lambda: ctx.vcycle(u, f), 10)
t_cg1 = timed(lambda: ctx.solve_cg(f, u, max_iter=1), 3)
t_cg11 = timed(lambda: ctx.solve_cg(f, u, max_iter=11), 3)
st = ctx.stats()
if rank == 0:
    print(f"N={world} HALO={os.environ.get('TPMG_HALO', 'default')} OVERLAP={os.environ.get('TPMG_OVERLAP', '0')} "
          f"vcycle {t_vc * 1e3:.0f} us, CG iteration {(t_cg11 - t_cg1) / 10 * 1e3:.0f} us", flush=True)
dist.destroy_process_group()
