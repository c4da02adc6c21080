"""Multi-rank GPU parity worker (run by tests/test_gpu_multirank.py under torchrun).

Every rank owns a y-strip of the global domain; each operator and solve through the
C ABI (NCCL halos and all-reduces) must match the CPU oracle on the GLOBAL problem,
restricted to the rank's strip."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import torch.distributed as dist

from oracle import oracle as O
from inputs import rhs_zc

rank, world, local = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"]), int(os.environ["LOCAL_RANK"])
torch.cuda.set_device(local)
dist.init_process_group("nccl", device_id=torch.device("cuda", local))
from paper_1402_3545_b200 import tpmg as T

failures = []


def check(name, got, want, tol):
    if os.environ.get("TPMG_TEST_FIELDS", "-1") != "-1":
        tol = max(tol, 2e-10)   # random fields: kappa(M_T) ~ 1e5 (tests/test_gpu_parity_fields.py tol)
    err = np.linalg.norm(got - want) / max(np.linalg.norm(want), 1e-300)
    if not err < tol:
        failures.append(f"rank {rank}: {name} rel err {err:.3e} >= {tol}")


obj = [T.tpmg_nccl_id() if rank == 0 else None]
dist.broadcast_object_list(obj, src=0)
nx, ny, nz, L = 64, 64 * world, 16, 5
BC = int(os.environ.get("TPMG_TEST_BOUNDARY", "0"))   # 1: face Dirichlet [R25]
PROF_SEED = int(os.environ.get("TPMG_TEST_PROFILES", "-1"))   # >= 0: general vertical profiles
from inputs import vertical_profiles
PROF = vertical_profiles(nz, PROF_SEED, 300.0) if PROF_SEED >= 0 else None
FIELD_SEED = int(os.environ.get("TPMG_TEST_FIELDS", "-1"))   # >= 0: per-column fields (tpmg_set_fields)
from inputs import horizontal_fields
FIELDS = (horizontal_fields(nx, ny, O.Params(nx=nx, ny=ny, nz=nz, L=L).c_h(), FIELD_SEED)
          if FIELD_SEED >= 0 else None)
P = O.Params(nx=nx, ny=ny, nz=nz, L=L, boundary=BC, profiles=PROF, fields=FIELDS)
ctx = T.Context(T.make_params(nx, ny, nz=nz, levels=L, boundary=BC), rank=rank, nranks=world, id128=obj[0],
                device=local)
if PROF is not None:
    ctx.set_profiles(*PROF)
if FIELDS is not None:
    ctx.set_fields(*FIELDS)


def strip(x_zc, level):
    y0, _, nyl, _ = ctx.local_box(level)
    return x_zc[y0:y0 + nyl]


def dev(x_zc, level):
    return torch.from_numpy(O.to_lambda(strip(x_zc, level))).cuda()


def host(t):
    torch.cuda.synchronize()
    return O.from_lambda(t.cpu().numpy())


rng = np.random.default_rng(0)
for level in range(1, L + 1):
    s = P.level_shape(level)
    u, f = rng.standard_normal(s), rng.standard_normal(s)
    y = ctx.empty(level)
    ctx.apply(level, dev(u, level), y)
    check(f"apply L{level}", host(y), strip(O.apply(P, u, level), level), 1e-11)
    n2 = ctx.residual(level, dev(u, level), dev(f, level), y, want_norm2=True)
    r = O.residual(P, u, f, level)
    check(f"residual L{level}", host(y), strip(r, level), 1e-11)
    if abs(n2 - float(np.sum(r * r))) > 1e-10 * float(np.sum(r * r)):
        failures.append(f"rank {rank}: global norm L{level} {n2} vs {np.sum(r * r)}")
    du = dev(u, level)
    ctx.smooth(level, du, dev(f, level), 2)
    check(f"smooth L{level}", host(du), strip(O.smooth(P, u, f, level, 2), level), 1e-11)
    if level < L:
        uf = rng.standard_normal(P.level_shape(level + 1))
        duf = dev(uf, level + 1)
        ctx.prolong_add(level, dev(u, level), duf)
        check(f"prolong L{level}", host(duf), strip(O.prolong_add(P, u, uf, level), level + 1), 1e-11)
        fc = ctx.empty(level)
        ctx.restrict(level + 1, dev(uf, level + 1), fc)
        check(f"restrict L{level + 1}", host(fc), strip(O.restrict(P, uf, level + 1), level), 1e-11)

u, f = rng.standard_normal(P.level_shape(L)), rng.standard_normal(P.level_shape(L))
du = dev(u, L)
ctx.vcycle(du, dev(f, L))
check("vcycle", host(du), strip(O.vcycle(P, u, f), L), 1e-11)

f = rhs_zc(nx, ny, nz, seed=0)
for name, solve, ref in (("mg", ctx.solve_mg, O.solve_mg(P, f)), ("cg", ctx.solve_cg, O.solve_cg(P, f))):
    x = ctx.empty(L)
    res = solve(dev(f, L), x)
    if not res.converged or abs(res.iterations - ref.iterations) > 1:
        failures.append(f"rank {rank}: {name} iterations {res.iterations} vs oracle {ref.iterations}")
    elif res.iterations == ref.iterations:
        check(f"{name} solution", host(x), strip(ref.u, L), 1e-9)

st = ctx.stats()
if st["halo_exchanges"] == 0 or st["allreduces"] == 0:
    failures.append(f"rank {rank}: no exchange / allreduce traffic recorded {st}")
for key, var in (("p2p_halo", "TPMG_TEST_EXPECT_P2P"), ("p2p_allreduce", "TPMG_TEST_EXPECT_P2PAR")):
    want = os.environ.get(var)
    if want is not None and st[key] != int(want):   # the transport the case asked for is the one used
        failures.append(f"rank {rank}: stats {key} = {st[key]}, expected {want}")
ctx.close()
allf = [None] * world
dist.all_gather_object(allf, failures)
dist.destroy_process_group()
flat = [x for fs in allf for x in fs]
if rank == 0:
    print("\n".join(flat) if flat else f"MULTIRANK OK world={world}")
sys.exit(1 if flat else 0)
