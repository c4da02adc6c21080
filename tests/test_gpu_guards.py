"""Out-of-bounds and race checks of every kernel without compute-sanitizer.

compute-sanitizer is closed on this GPU pool (runs under it left GPUs needing a reset;
profiles/r2/sanitize_closed.txt), so the checks are built in:
  * guard bands: every vector lives in the middle of a larger allocation whose guards hold a
    NaN sentinel.  An out-of-bounds store changes a guard (checked bit for bit); an
    out-of-bounds load of an input's guard puts a NaN into the result (checked: finite);
  * determinism: the same call on the same inputs twice gives bit-identical results (a race
    between the TMA / cp.async pipelines, the k-split segment chaining or the reductions and
    their consumers would show up as run-to-run differences);
  * the Tensor Memory form of the Thomas kernels against the shared-memory form (same
    arithmetic, same grid): bit-identical.
Shapes span several tiles with ragged x tails, nz not a multiple of the k-split segment, and
the multigrid levels down to a handful of columns.
"""
import os

import numpy as np
import pytest

from oracle import oracle as O
from gpu_util import ctx_for, lib

pytestmark = pytest.mark.gpu
G = 4096                              # guard doubles before and after each vector
SENT = 0x7FF80000DEADBEEF              # a quiet-NaN bit pattern


def guarded(shape, init=None, seed=0):
    import torch
    n = int(np.prod(shape))
    base = torch.empty(n + 2 * G, dtype=torch.float64, device="cuda")
    base.view(torch.int64).fill_(SENT)
    v = base[G:G + n].view(shape)
    if init is None:
        v.copy_(torch.from_numpy(np.random.default_rng(seed).standard_normal(shape)))
    else:
        v.copy_(init)
    return base, v


def guards_intact(base):
    import torch
    torch.cuda.synchronize()
    g = torch.cat([base[:G], base[-G:]]).view(torch.int64)
    return bool((g == SENT).all())


def finite(v):
    import torch
    torch.cuda.synchronize()
    return bool(torch.isfinite(v).all())


SHAPES = [(96, 64, 40, 3), (64, 32, 128, 3), (80, 48, 32, 3)]


@pytest.mark.parametrize("shape", SHAPES, ids=["96x64x40", "64x32x128", "80x48x32"])
def test_guard_bands_every_operator(shape):
    import torch
    T = lib()
    nx, ny, nz, L = shape
    p = O.Params(nx=nx, ny=ny, nz=nz, L=L)
    ctx = ctx_for(p)
    bufs = []

    def vec(level, seed=0, init=None):
        b, v = guarded(ctx.shape(level), init, seed)
        bufs.append((b, v))
        return v

    for level in range(1, L + 1):
        x, f = vec(level, 1), vec(level, 2)
        y = vec(level, init=torch.zeros(ctx.shape(level), dtype=torch.float64))
        ctx.apply(level, x, y)
        assert finite(y)
        ctx.residual(level, x, f, y, want_norm2=True)
        assert finite(y)
        ctx.precondition(level, f, y)
        assert finite(y)
        ctx.smooth(level, x, f, 2)
        assert finite(x)
        if level > 1:
            fc = vec(level - 1, init=torch.zeros(ctx.shape(level - 1), dtype=torch.float64))
            ctx.restrict(level, f, fc)
            assert finite(fc)
            ctx.prolong_add(level - 1, fc, x)
            assert finite(x)
    u, f = vec(L, 3), vec(L, 4)
    ctx.vcycle(u, f)
    assert finite(u)
    for solve in (ctx.solve_mg, ctx.solve_cg):
        x = vec(L, 5)
        r = solve(f, x, max_iter=4)
        assert r.iterations >= 1 and finite(x)
    zc_b, zc = guarded((ny, nx, nz))
    bufs.append((zc_b, zc))
    ctx.transpose(L, T.TPMG_LAMBDA_TO_ZC, u, zc)
    ctx.transpose(L, T.TPMG_ZC_TO_LAMBDA, zc, f)
    assert finite(zc) and finite(f)
    for b, _ in bufs:
        assert guards_intact(b)


@pytest.mark.parametrize("shape", SHAPES, ids=["96x64x40", "64x32x128", "80x48x32"])
def test_bitwise_repeatable(shape):
    """Same inputs, same call, twice: bit-identical outputs (smoother, CG, V-cycle, MG)."""
    import torch
    nx, ny, nz, L = shape
    ctx = ctx_for(O.Params(nx=nx, ny=ny, nz=nz, L=L))
    rng = np.random.default_rng(9)
    u0 = torch.from_numpy(rng.standard_normal(ctx.shape(L))).cuda()
    f = torch.from_numpy(rng.standard_normal(ctx.shape(L))).cuda()

    def run():
        out = []
        a = u0.clone()
        ctx.smooth(L, a, f, 3)
        out.append(a)
        b = u0.clone()
        ctx.vcycle(b, f)
        out.append(b)
        for solve in (ctx.solve_mg, ctx.solve_cg):
            x = torch.empty_like(f)
            solve(f, x, max_iter=6)
            out.append(x)
        torch.cuda.synchronize()
        return [o.cpu().numpy() for o in out]

    for a, b in zip(run(), run()):
        assert np.array_equal(a.view(np.int64), b.view(np.int64))


@pytest.mark.parametrize("shape", [(64, 64, 128, 3), (96, 32, 40, 2)], ids=["64x64x128", "96x32x40"])
def test_tmem_form_bit_identical_to_shared_memory_form(shape):
    """k_line's Thomas intermediates in Tensor Memory (TMEM) vs in shared memory: the same
    arithmetic on the same grid (1 CTA per SM) -- every CG iterate bit for bit."""
    import torch
    T = lib()
    nx, ny, nz, L = shape
    outs = []
    for tm in ("1", "0"):
        os.environ["TPMG_TMEM"] = tm
        os.environ["TPMG_TM_CTAS"] = "1"
        os.environ["TPMG_PAIR_U"] = "0"   # (the paired-u variants run other tile rows without TMEM)
        try:
            ctx = ctx_for(O.Params(nx=nx, ny=ny, nz=nz, L=L))
        finally:
            os.environ.pop("TPMG_TMEM")
            os.environ.pop("TPMG_TM_CTAS")
            os.environ.pop("TPMG_PAIR_U")
        f = torch.from_numpy(np.random.default_rng(4).standard_normal(ctx.shape(L))).cuda()
        x = torch.empty_like(f)
        r = ctx.solve_cg(f, x, max_iter=12)
        z = torch.empty_like(f)
        ctx.precondition(L, f, z)
        torch.cuda.synchronize()
        outs.append((x.cpu().numpy(), z.cpu().numpy(), r.history))
        ctx.close()
    (x1, z1, h1), (x0, z0, h0) = outs
    assert np.array_equal(z1.view(np.int64), z0.view(np.int64))
    assert np.array_equal(x1.view(np.int64), x0.view(np.int64))
    assert h1 == h0


@pytest.mark.parametrize("shape", [(64, 64, 128, 3), (80, 44, 64, 1), (96, 36, 16, 2)],
                         ids=["64x64x128", "80x44x64", "96x36x16"])
def test_tma_store_form_bit_identical(shape):
    """The CG preconditioner with its outputs staged in shared memory and written by TMA stores
    (TPMG_TMA_STORE=1) vs the per-thread stores: the same arithmetic on the same grid, so every
    CG iterate and the residual history are bit-identical; ragged x and y tiles (the TMA store
    clips the phantom columns and rows) included."""
    import torch
    nx, ny, nz, L = shape
    outs = []
    for ts in ("1", "0"):
        os.environ["TPMG_TMA_STORE"] = ts
        try:
            ctx = ctx_for(O.Params(nx=nx, ny=ny, nz=nz, L=L))
        finally:
            os.environ.pop("TPMG_TMA_STORE")
        f = torch.from_numpy(np.random.default_rng(8).standard_normal(ctx.shape(L))).cuda()
        x = torch.empty_like(f)
        r = ctx.solve_cg(f, x, eps=1e-10, max_iter=40)
        torch.cuda.synchronize()
        outs.append((x.cpu().numpy(), r.history, r.iterations))
        ctx.close()
    (x1, h1, i1), (x0, h0, i0) = outs
    assert i1 == i0 and h1 == h0
    assert np.array_equal(x1.view(np.int64), x0.view(np.int64))


def test_tma_store_guard_bands():
    """TPMG_TMA_STORE=1: the TMA stores of r, u, z stay inside their vectors (NaN guard bands
    around every CG vector the caller passes, ragged tiles)."""
    import torch
    os.environ["TPMG_TMA_STORE"] = "1"
    try:
        ctx = ctx_for(O.Params(nx=80, ny=44, nz=64, L=1))
    finally:
        os.environ.pop("TPMG_TMA_STORE")
    fb, f = guarded(ctx.shape(1), seed=3)
    xb, x = guarded(ctx.shape(1), seed=4)
    r = ctx.solve_cg(f, x, max_iter=12)
    assert r.iterations >= 1 and finite(x)
    assert guards_intact(fb) and guards_intact(xb)
    ctx.close()


@pytest.mark.parametrize("max_iter", [7, 8, 1000])
def test_paired_u_update_changes_only_u_rounding(max_iter):
    """PCG with the u update paired over two iterations (TPMG_PAIR_U=1) vs every iteration
    (default): r, z and the sums are the same arithmetic on the same grid, so the residual history is
    bit-identical; u differs by rounding only.  Odd and even stops (the last odd step is added
    after the loop)."""
    import torch
    nx, ny, nz, L = 64, 64, 32, 3
    outs = []
    for pu in ("1", "0"):
        os.environ["TPMG_PAIR_U"] = pu
        try:
            ctx = ctx_for(O.Params(nx=nx, ny=ny, nz=nz, L=L))
        finally:
            os.environ.pop("TPMG_PAIR_U")
        f = torch.from_numpy(np.random.default_rng(6).standard_normal(ctx.shape(L))).cuda()
        x = torch.empty_like(f)
        r = ctx.solve_cg(f, x, eps=1e-10, max_iter=max_iter)
        torch.cuda.synchronize()
        outs.append((x.cpu().numpy(), r))
        ctx.close()
    (x1, r1), (x0, r0) = outs
    assert r1.iterations == r0.iterations and r1.history == r0.history
    assert np.linalg.norm(x1 - x0) <= 1e-13 * np.linalg.norm(x0)
