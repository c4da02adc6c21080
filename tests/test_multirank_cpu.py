"""World-size-2 (gloo, CPU) tests of the multi-rank host logic: the y-strip
decomposition the library computes (tpmg_partition, no GPU needed), the halo
protocol the library runs with NCCL (row 0 -> rank-1, row ny-1 -> rank+1, zero
slabs at physical boundaries), and the unique-id broadcast bench.py does."""
import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import oracle as O
from inputs import rhs_zc


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _run(fn, world=2):
    port = _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_entry, args=(fn, r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=300) for _ in procs]
    for p in procs:
        p.join(timeout=60)
    errs = [r for r in res if r is not True]
    assert not errs, errs


def _entry(fn, rank, world, port, q):
    import sys
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    try:
        dist.init_process_group("gloo", rank=rank, world_size=world)
        globals()[fn](rank, world)
        dist.barrier()
        dist.destroy_process_group()
        q.put(True)
    except Exception as e:  # report to the parent
        import traceback
        q.put(f"rank {rank}: {e!r}\n{traceback.format_exc()}")


# ---------------------------------------------------------------- workers

def w_partition(rank, world):
    from paper_1402_3545_b200 import build
    build.build()
    from paper_1402_3545_b200 import tpmg as T
    p = T.make_params(64, 128, nz=16)
    for level in range(1, 6):
        y0, ny = T.tpmg_partition(p, rank, world, level)
        boxes = [None] * world
        dist.all_gather_object(boxes, (y0, ny))
        boxes.sort()
        assert boxes[0][0] == 0
        for (a0, an), (b0, _) in zip(boxes, boxes[1:]):
            assert a0 + an == b0                      # contiguous strips
        assert boxes[-1][0] + boxes[-1][1] == 128 >> (5 - level)
    # ny = 64 with L = 5 on 8 ranks: 64 / (8 * 16) is not integral
    with pytest.raises(T.TpmgError, match="TPMG_E_SHAPE"):
        T.tpmg_partition(T.make_params(64, 64, nz=16), rank, 8, 5)


def _exchange(x_loc, rank, world):
    """The library's halo protocol (api.cpp exchange()) with gloo point-to-point."""
    import torch
    ny = x_loc.shape[0]
    lo = torch.zeros_like(x_loc[0]); hi = torch.zeros_like(x_loc[0])
    reqs = []
    if rank > 0:
        reqs.append(dist.isend(x_loc[0].contiguous(), rank - 1))
        reqs.append(dist.irecv(lo, rank - 1))
    if rank < world - 1:
        reqs.append(dist.isend(x_loc[ny - 1].contiguous(), rank + 1))
        reqs.append(dist.irecv(hi, rank + 1))
    for r in reqs:
        r.wait()
    return lo, hi


def w_halo(rank, world):
    """Halos carry the neighbours' boundary rows; a strip-local 7-point stencil with
    those halos reproduces the oracle's global operator on the strip."""
    import torch
    nx, ny, nz = 32, 64, 8
    p = O.Params(nx=nx, ny=ny, nz=nz, L=1)
    u = rhs_zc(nx, ny, nz, seed=5)                           # global, oracle layout (ny, nx, nz)
    want = O.apply(p, u)
    rows = ny // world
    y0 = rank * rows
    loc = torch.from_numpy(O.to_lambda(u)[y0:y0 + rows].copy())   # Lambda layout (rows, nz, nx)
    lo, hi = _exchange(loc, rank, world)
    if rank > 0:
        assert torch.equal(lo, torch.from_numpy(O.to_lambda(u)[y0 - 1]))
    else:
        assert not lo.any()
    if rank < world - 1:
        assert torch.equal(hi, torch.from_numpy(O.to_lambda(u)[y0 + rows]))
    else:
        assert not hi.any()
    # strip-local stencil with halos (independent numpy form of P:150's entries)
    c, g = p.c_h(), p.gamma()
    ext = torch.cat([lo[None], loc, hi[None]]).numpy()       # (rows+2, nz, nx)
    core = ext[1:-1]
    S = ext[:-2] + ext[2:]
    S = S + np.pad(core, ((0, 0), (0, 0), (1, 0)))[:, :, :-1] + np.pad(core, ((0, 0), (0, 0), (0, 1)))[:, :, 1:]
    up = np.pad(core, ((0, 0), (0, 1), (0, 0)))[:, 1:, :]
    dn = np.pad(core, ((0, 0), (1, 0), (0, 0)))[:, :-1, :]
    cnt = np.full(nz, 2.0); cnt[0] -= 1; cnt[-1] -= 1
    y = (1 + 4 * c + g * cnt[None, :, None]) * core - g * (up + dn) - c * S
    got = O.from_lambda(y)
    assert np.max(np.abs(got - want[y0:y0 + rows])) <= 1e-12 * np.max(np.abs(want))


def w_nccl_id_broadcast(rank, world):
    obj = [bytes(range(128)) if rank == 0 else None]
    dist.broadcast_object_list(obj, src=0)
    assert obj[0] == bytes(range(128))


@pytest.mark.parametrize("fn", ["w_partition", "w_halo", "w_nccl_id_broadcast"])
def test_world2_gloo(fn):
    _run(fn, 2)


@pytest.mark.parametrize("nx,ny", [(1024, 8192), (2048, 16384), (4096, 4096)])
def test_partition_world8_bench_shapes(nx, ny):
    # The driver's N = 8 scaling run (bench.py workload(): weak 1024^2 / 2048^2 per GPU,
    # strong 4096^2): every level splits into 8 contiguous y-strips covering the grid.
    from paper_1402_3545_b200 import build
    build.build()
    from paper_1402_3545_b200 import tpmg as T
    p = T.make_params(nx, ny, nz=128)
    for level in range(1, 6):
        boxes = [T.tpmg_partition(p, r, 8, level) for r in range(8)]
        assert boxes[0][0] == 0 and all(n > 0 for _, n in boxes)
        for (a0, an), (b0, _) in zip(boxes, boxes[1:]):
            assert a0 + an == b0
        assert boxes[-1][0] + boxes[-1][1] == ny >> (5 - level)
