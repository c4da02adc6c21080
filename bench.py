#!/usr/bin/env python
"""Benchmark: MG V-cycle and PCG solves to 1e-5 on B200 (BASELINE.json metric).

One "step" is one pass of the whole hot path over one right-hand side: a
multigrid solve (V-cycles of the fused line smoother, residual->restriction,
RestrictSmooth, prolongation) AND a line-preconditioned CG solve (the two fused
CG kernels with their reductions), both from u = 0 to ||r||/||r_0|| < 1e-5, on
the same device-resident f.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl tpmg|reference]

N = 1: BASELINE configs[1] (1024 x 1024 x 128, fp64).  N > 1 (torchrun, one
rank per GPU, NCCL): weak scaling with the same 1024 x 1024 x 128 per GPU,
global 1024 x 1024N (y-strips); --per-gpu-nx 2048 gives configs[3].
--global-nx G: strong scaling of a fixed G x G x 128 grid (4096 = configs[4]).
Vectors are 1 GiB per GPU, far larger than the 126 MB L2, so no flush is
needed between steps.  Prints ONE JSON line on rank 0.
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "MG V-cycle & PCG time-to-1e-5 and achieved HBM GB/s at 1/2/4/8 B200"
UNIT = "unknowns/s (MG + PCG solves to 1e-5, summed)"

# Algorithmic (compulsory) HBM bytes per processed cell of each kernel class
# (DESIGN.md "Kernels and their rooflines"); cells are level cells, fine cells
# for the transfer kernels.
BYTES_PER_CELL = {
    "apply": 16, "residual": 16, "precondition": 16, "smooth": 24, "cg_direction": 24,
    "cg_precondition": 48, "residual_restrict": 18, "restrict": 10, "prolong_add": 18, "dot": 8,
    "smooth_prolong": 26,
}
PAPER_FLOPS = {"cg": 54.0, "mg": 149.4}  # tab:KernelTable totals per cell per iteration


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["tpmg", "reference"], default="tpmg")
    ap.add_argument("--per-gpu-nx", type=int, default=1024)
    ap.add_argument("--nz", type=int, default=128)
    ap.add_argument("--nu", type=float, default=8.4)
    ap.add_argument("--seed", type=int, default=0)
    ap.add_argument("--eps", type=float, default=1e-5)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--solver", choices=["both", "mg", "cg"], default="both")
    ap.add_argument("--levels", type=int, default=5, help="multigrid levels L (P:418; 7 and 10 in sec:Robustness)")
    ap.add_argument("--coarse-sweeps", type=int, default=2, help="smoother sweeps on the coarsest level (P:456)")
    ap.add_argument("--boundary", type=int, default=0, choices=[0, 1],
                    help="horizontal Dirichlet reading: 0 ghost zero [R1], 1 face [R25] (sec:Robustness runs)")
    ap.add_argument("--profiles", type=int, default=-1,
                    help="general vertical profiles (inputs.vertical_profiles with this seed, couplings of "
                         "the flat box's size); -1: flat box")
    ap.add_argument("--fields", choices=["none", "random", "smooth"], default="none",
                    help="per-column horizontal fields |T|, alpha_TT' (inputs.horizontal_fields, seed 1; "
                         "tpmg_set_fields): none = uniform coefficients")
    ap.add_argument("--global-nx", type=int, default=0,
                    help="strong scaling: a fixed global nx x nx x nz grid split into y-strips (4096 = configs[4])")
    return ap.parse_args()


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


def workload(args, world):
    if args.global_nx:
        g = args.global_nx
        tag = "C5 strong scaling" if g == 4096 else "strong scaling"
        return g, g, f"{tag}: {g}x{g}x{args.nz} global, {world} B200 y-strips of {g}x{g // world}"
    nx = args.per_gpu_nx
    ny = nx * world
    name = ("C2: MG + PCG on 1024x1024x128 fp64, 1 B200" if world == 1 and nx == 1024 else
            f"{'C4 ' if nx == 2048 else ''}weak scaling: {nx}x{nx}x{args.nz} per GPU, global {nx}x{ny}x{args.nz}, "
            f"{world} B200 y-strips")
    return nx, ny, name


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""
    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, device: int):
        self.device = device
        self.proc = None
        self.out = b""

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.device), f"--query-gpu={self.Q}", "--format=csv,noheader,nounits",
                 "-lms", "200"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL)
        except Exception:
            self.proc = None
        return self

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            try:
                self.out, _ = self.proc.communicate(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        rows = []
        for line in self.out.decode(errors="ignore").splitlines():
            f = [x.strip() for x in line.split(",")]
            if len(f) >= 9:
                rows.append(f)
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        sm = sorted(float(r[1]) for r in rows if r[1].replace(".", "").isdigit())
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[q] for r in rows for q in range(4) if r[5 + q].lower() == "active"})
        return {"sm_mhz": sm[len(sm) // 2] if sm else None,
                "sm_max_mhz": float(rows[0][2]) if rows[0][2].replace(".", "").isdigit() else None,
                "reasons": reasons, "samples": len(rows)}


def ncu_traffic(kernel):
    """DRAM bytes per launch of `kernel` at this workload from the committed ncu --set full
    capture (profiles/ncu_traffic.json, written by scripts/ncu_summary.py), or None."""
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_traffic.json")) as fh:
            return json.load(fh)[kernel]["bytes"]
    except Exception:
        return None


def measured_peak():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
            return float(json.load(fh)["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md)"


# ---------------------------------------------------------------------------- oracle legs

def bench_profiles(args):
    """--profiles: synthetic non-uniform column (inputs.vertical_profiles) with couplings of
    the size of the flat box's gamma = omega^2 lambda^2 / h_z^2 at this grid."""
    if args.profiles < 0:
        return None
    from inputs import vertical_profiles
    nx = args.global_nx or args.per_gpu_nx
    h = 1.0 / nx
    omega = 0.5 * args.nu * h
    gamma = omega * omega / (0.01 / args.nz) ** 2
    return vertical_profiles(args.nz, args.profiles, gamma)


def bench_fields(args, nx, ny):
    """--fields: seeded per-column fields (inputs.horizontal_fields) of the global grid, alpha of
    the size of the flat box's c_h = nu^2/4."""
    if args.fields == "none":
        return None
    from inputs import horizontal_fields
    return horizontal_fields(nx, ny, args.nu * args.nu / 4.0, 1, args.fields)


def strip_fields(fields, rows):
    return None if fields is None else (fields[0][:rows], fields[1][:rows], fields[2][:rows + 1])


def oracle_sample(nx, nz, nu, rows, seed, threads=None, levels=5, coarse_sweeps=2, boundary=0, profiles=None,
                  fields=None, mg_iter=1, cg_iter=1, eps=1e-30, f=None):
    """Time the CPU oracle (as it stands) on a y-strip of `rows` rows of the workload (rows =
    ny: the whole grid): an MG solve of at most mg_iter V-cycles (r0 norm + cycles + residual
    each) and a PCG solve of at most cg_iter iterations (setup + iterations).  Returns
    (t_mg, t_cg, threads, mg_iterations, cg_iterations)."""
    from oracle import oracle as O
    from inputs import rhs_zc
    if threads:
        O.set_threads(threads)
    p = O.Params(nx=nx, ny=rows, nz=nz, nu_cfl=nu, L=levels, coarse_sweeps=coarse_sweeps, boundary=boundary,
                 profiles=profiles, fields=fields)
    if f is None:
        f = rhs_zc(nx, rows, nz, seed=seed)
    t0 = time.perf_counter()
    rm = O.solve_mg(p, f, eps=eps, max_iter=mg_iter) if mg_iter else None
    t1 = time.perf_counter()
    rc = O.solve_cg(p, f, eps=eps, max_iter=cg_iter) if cg_iter else None
    t2 = time.perf_counter()
    return t1 - t0, t2 - t1, O.num_threads(), rm and rm.iterations, rc and rc.iterations


def cpu_model():
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def oracle_counts(args, nx, ny):
    """Iterations of the ORACLE's own full MG and PCG solves of this workload to 1e-5
    (tests/golden/oracle_iterations.json, written by scripts/oracle_iterations.py, which calls
    only oracle/): (mg, cg, source) or None when the workload has no entry."""
    key = (f"{nx}x{ny}x{args.nz}_nu{args.nu:g}_L{args.levels}_cs{args.coarse_sweeps}_bc{args.boundary}"
           f"_seed{args.seed}")
    if args.profiles >= 0 or args.fields != "none":
        return None
    try:
        with open(os.path.join(ROOT, "tests", "golden", "oracle_iterations.json")) as fh:
            rec = json.load(fh)[key]
        return rec["mg"]["iterations"], rec["cg"]["iterations"], f"oracle full solves of {key} (tests/golden/oracle_iterations.json)"
    except Exception:
        return None


def _counts(args, nx, ny, gpu_counts):
    cnt = oracle_counts(args, nx, ny)
    if cnt is not None:
        return cnt
    it_mg, it_cg = gpu_counts or (10, 54)
    return it_mg, it_cg, "this run's GPU iteration counts (no oracle full-solve entry for this workload)"


def oracle_step_sample(args, nx, ny, do_mg, do_cg, gpu_counts=None, rows_mg=64, rows_cg=32, threads=None):
    """One bounded sample of the workload for the oracle: the oracle's own full iteration
    counts of the workload (oracle_counts) run on y-strips of it -- an MG solve of exactly
    it_mg V-cycles on nx x rows_mg and a PCG solve of exactly it_cg iterations on nx x rows_cg
    (setup amortised as in the whole solve) -- each scaled by ny/rows in cells.  Returns
    (value, extrapolated seconds per step, description)."""
    it_mg, it_cg, src = _counts(args, nx, ny, gpu_counts)
    t = 0.0
    parts = []
    cores = None
    for on, rows, mg_iter, cg_iter, what in ((do_mg, rows_mg, it_mg, 0, "solve_mg"), (do_cg, rows_cg, 0, it_cg, "solve_cg")):
        if not on:
            continue
        rows = min(rows, ny)
        flds = strip_fields(bench_fields(args, nx, ny), rows)
        a, b, cores, im, ic = oracle_sample(nx, args.nz, args.nu, rows, args.seed, threads=threads,
                                            levels=args.levels, coarse_sweeps=args.coarse_sweeps,
                                            boundary=args.boundary, profiles=bench_profiles(args), fields=flds,
                                            mg_iter=mg_iter, cg_iter=cg_iter, eps=1e-300)
        dt = a + b
        t += dt * ny / rows
        parts.append(f"{what} of exactly {im or ic} iterations on a {nx}x{rows}x{args.nz} y-strip: {dt:.3f} s "
                     f"(x{ny / rows:g} in cells)")
    solves = int(do_mg) + int(do_cg)
    desc = {"cores": cores, "sample": "oracle " + "; ".join(parts) + f"; iteration counts: {src}"}
    return solves * nx * ny * args.nz / t, t, desc


def cpu_baseline_block(args, nx, ny, do_mg, do_cg, gpu_counts=None):
    """cpu_baseline (rank 0, N = 1): the oracle as it stands on all host cores -- the whole MG
    solve of the workload to eps MEASURED (its own iteration count), the PCG solve's full
    iteration count run on a y-strip (oracle_step_sample) -- plus a one-thread sample and the
    CPU model."""
    from oracle import oracle as O
    a = 0.0
    it_mg = None
    cores = O.num_threads()
    if do_mg:
        a, _, cores, it_mg, _ = oracle_sample(nx, args.nz, args.nu, ny, args.seed, levels=args.levels,
                                              coarse_sweeps=args.coarse_sweeps, boundary=args.boundary,
                                              profiles=bench_profiles(args), fields=bench_fields(args, nx, ny),
                                              mg_iter=50, cg_iter=0, eps=args.eps)
    t_cg, d_cg = 0.0, None
    if do_cg:
        _, t_cg, d_cg = oracle_step_sample(args, nx, ny, False, True, gpu_counts)
    t = a + t_cg
    solves = int(do_mg) + int(do_cg)
    v_all = solves * nx * ny * args.nz / t
    v_one, t_one, d_one = oracle_step_sample(args, nx, ny, do_mg, do_cg, gpu_counts, rows_mg=32, rows_cg=16,
                                             threads=1)
    O.set_threads(cores)   # restore
    sample = []
    if do_mg:
        sample.append(f"oracle solve_mg to {args.eps:g} on the whole {nx}x{ny}x{args.nz} grid: {a:.2f} s, "
                      f"{it_mg} V-cycles (measured)")
    if do_cg:
        sample.append(d_cg["sample"] + f" = {t_cg:.2f} s")
    return {"value": v_all, "unit": UNIT, "cores": cores, "kind": "oracle",
            "method": "MG: whole solve measured; PCG: its full iteration count measured on a y-strip, x cells",
            "cpu_model": cpu_model(), "host_threads": os.cpu_count(), "sample": "; ".join(sample),
            "seconds_per_step": round(t, 2),
            "one_thread": {"value": v_one, "unit": UNIT, "cores": 1, "seconds_per_step": round(t_one, 2),
                           "sample": d_one["sample"]},
            "speedup_all_cores_vs_one": round(v_all / v_one, 2)}


def run_reference(args):
    """--impl reference: the oracle, as it stands, on the host cores (rank 0 only).  Each
    step is one bounded sample of the workload (oracle_step_sample: the oracle's whole MG and
    PCG iteration counts on y-strips)."""
    rank, world, _ = dist_env()
    if rank != 0:
        return
    nx, ny, name = workload(args, world)
    do_mg = args.solver in ("both", "mg")
    do_cg = args.solver in ("both", "cg")
    for _ in range(args.warmup):
        oracle_step_sample(args, nx, ny, do_mg, do_cg)
    t = 0.0
    wall = 0.0
    desc = None
    for _ in range(args.steps):
        w0 = time.perf_counter()
        _, ts, desc = oracle_step_sample(args, nx, ny, do_mg, do_cg)
        wall += time.perf_counter() - w0
        t += ts
    solves = int(do_mg) + int(do_cg)
    value = solves * nx * ny * args.nz * args.steps / t
    cpu = {"value": value, "unit": UNIT, "cores": desc["cores"], "kind": "oracle",
           "method": "per step: the oracle's full iteration counts of the workload measured on y-strips, x cells",
           "cpu_model": cpu_model(), "host_threads": os.cpu_count(),
           "seconds_per_step": round(t / args.steps, 2), "sample": "per step: " + desc["sample"]}
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * wall / args.steps,
        "extrapolated_ms_per_step": 1e3 * t / args.steps,
        "higher_is_better": True, "scaling": "strong" if args.global_nx else "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (splitmix64 uniform[-1,1) RHS keyed by global index, seed %d)" % args.seed,
        "config": config_block(args, nx, ny, name, world),
        "cpu_baseline": cpu,
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def config_block(args, nx, ny, name, world):
    return {"workload": name, "nx": nx, "ny": ny, "nz": args.nz, "nu_cfl": args.nu, "eps": args.eps,
            "levels": args.levels, "coarse_sweeps": args.coarse_sweeps, "boundary": args.boundary,
            "solver": args.solver,
            "vertical_profiles": "flat box" if args.profiles < 0 else f"synthetic seed {args.profiles}",
            "horizontal_fields": "uniform" if args.fields == "none" else f"{args.fields} seed 1",
            "parallelism": f"y-strips x{world}" if world > 1 else "single GPU",
            "l2": "vectors 1 GiB/GPU >> 126 MB L2 (no flush needed)"}


# ---------------------------------------------------------------------------- GPU arm

def main():
    args = parse()
    if args.impl == "reference":
        run_reference(args)
        return
    import torch
    import torch.distributed as dist
    from paper_1402_3545_b200 import build as B
    B.build()
    from paper_1402_3545_b200 import tpmg as T
    from inputs import gpu as G

    rank, world, local = dist_env()
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    nx, ny, name = workload(args, world)
    nz = args.nz
    id128 = None
    if world > 1:
        obj = [T.tpmg_nccl_id() if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        id128 = obj[0]
    stream = torch.cuda.Stream(device=local)
    params = T.make_params(nx, ny, nz=nz, nu_cfl=args.nu, levels=args.levels, coarse_sweeps=args.coarse_sweeps,
                           boundary=args.boundary)
    ctx = T.Context(params, rank=rank, nranks=world, id128=id128, device=local, stream=stream)
    prof = bench_profiles(args)
    if prof is not None:
        ctx.set_profiles(*prof)
    flds = bench_fields(args, nx, ny)
    if flds is not None:
        ctx.set_fields(*flds)
    shape = ctx.shape(args.levels)
    f = torch.empty(shape, dtype=torch.float64, device=f"cuda:{local}")
    u = torch.empty_like(f)
    y0 = ctx.local_box(args.levels)[0]
    with torch.cuda.stream(stream):
        G.fill_rhs(f, nx, y0=y0, seed=args.seed, stream=stream)
    stream.synchronize()
    n_glob = nx * ny * nz
    do_mg = args.solver in ("both", "mg")
    do_cg = args.solver in ("both", "cg")

    def step():
        r_mg = ctx.solve_mg(f, u, eps=args.eps) if do_mg else None
        r_cg = ctx.solve_cg(f, u, eps=args.eps) if do_cg else None
        return r_mg, r_cg

    def barrier():
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    if args.warmup < 2:
        step()   # the breakdown step must not be the first (cold: module load, descriptors)
    for w in range(args.warmup):
        if w == args.warmup - 1:
            ctx.profile(True)   # last warm-up step: every kernel class event-timed (breakdown)
        step()
    barrier()
    prof_all = ctx.profile_read()
    ctx.profile(False)
    ms_warm = sum(v[1] for v in prof_all.values())
    # the timed region brackets only the dominant class with events (each event pair
    # serialises the stream for a few microseconds; timing every class costs ~4%)
    dom_class = max(prof_all.items(), key=lambda kv: kv[1][1])[0] if prof_all else None
    ctx.stats_reset()
    if dom_class:
        ctx.profile(True, classes=[dom_class])
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t_mg = t_cg = 0.0
    its = None
    with ClockSampler(local) as clk:
        barrier()
        ev0.record(stream)
        for _ in range(args.steps):
            r_mg, r_cg = step()
            t_mg += r_mg.seconds if r_mg else 0.0
            t_cg += r_cg.seconds if r_cg else 0.0
            its = (r_mg, r_cg)
        ev1.record(stream)
        barrier()
    ms_local = ev0.elapsed_time(ev1)
    prof = ctx.profile_read()
    ctx.profile(False)
    stats = ctx.stats()
    ms = torch.tensor([ms_local], dtype=torch.float64, device=f"cuda:{local}")
    if world > 1:
        dist.all_reduce(ms, op=dist.ReduceOp.MAX)
    ms = float(ms.item())
    solves = (1 if do_mg else 0) + (1 if do_cg else 0)
    value = solves * n_glob * args.steps / (ms * 1e-3)

    # roofline of the dominant kernel class (largest share of device time)
    peak, peak_src = measured_peak()
    dom = max(prof.items(), key=lambda kv: kv[1][1]) if prof else None
    roof = None
    kernels = {}   # breakdown from the last warm-up step (all classes event-timed)
    for kname, (n, kms, cells) in prof_all.items():
        gbs = cells * BYTES_PER_CELL[kname] / (kms * 1e-3) / 1e9 if kms > 0 else None
        kernels[kname] = {"launches": n, "ms_total": round(kms, 4), "gbs": gbs and round(gbs, 1),
                          "share_of_kernel_time": round(kms / ms_warm, 4) if ms_warm > 0 else None}
    if dom:
        kname, (n, kms, cells) = dom
        ach = cells * BYTES_PER_CELL[kname] / (kms * 1e-3) / 1e9
        traffic = ncu_traffic(kname) if (world == 1 and not args.global_nx and args.per_gpu_nx == 1024 and nz == 128) else None
        roof = {"bound": "hbm", "kernel": kname, "achieved": round(ach, 1), "peak": peak, "unit": "GB/s",
                "frac": round(ach / peak, 4), "traffic": traffic,
                "traffic_source": "profiles/ncu_traffic.json (ncu --set full, dram read+write per launch)" if traffic else None,
                "algorithmic_bytes_per_launch": cells / n * BYTES_PER_CELL[kname], "peak_source": peak_src,
                "bytes_per_cell": BYTES_PER_CELL[kname],
                "cells_per_launch": cells / n, "avg_launch_ms": kms / n, "launches_timed": n,
                "timing": "CUDA events around every launch of this class in the timed region"}

    # algorithmic bytes per step of each solver's kernels (the last warm-up step, all classes
    # event-timed), for the "useful" GB/s of each solve
    mg_classes = {"smooth", "precondition", "residual_restrict", "restrict", "prolong_add", "smooth_prolong",
                  "residual", "apply"}
    step_bytes = {"mg": sum(c * BYTES_PER_CELL[k] for k, (n, kms, c) in prof_all.items() if k in mg_classes),
                  "cg": sum(c * BYTES_PER_CELL[k] for k, (n, kms, c) in prof_all.items() if k not in mg_classes)}

    def solver_block(r, t_total, kind):
        if r is None:
            return None
        t = t_total / args.steps
        n_it = r.iterations
        useful = round(step_bytes[kind] / t / 1e9, 1) if t > 0 and step_bytes[kind] > 0 else None
        return {"iterations": n_it, "converged": r.converged, "rel_residual": r.rel_residual,
                "time_to_solution_ms": round(1e3 * t, 3),
                "unknowns_per_s": n_glob / t,
                "paper_gflops": PAPER_FLOPS[kind] * n_glob * n_it / t / 1e9,
                "ms_per_iteration": round(1e3 * t / max(n_it, 1), 4), "useful_gbs": useful}

    line_extra = {"mg": solver_block(its[0], t_mg, "mg"), "pcg": solver_block(its[1], t_cg, "cg")}
    # algorithmic HBM GB/s over the whole step: the bytes of one step's kernels (every class,
    # last warm-up step) / the timed time per step
    alg_bytes = step_bytes["mg"] + step_bytes["cg"]
    hbm_gbs_step = alg_bytes / (ms_local / args.steps * 1e-3) / 1e9

    # end-to-end through the C ABI with host buffers (H2D of f and D2H of u inside the timed region)
    e2e = None
    if not args.no_e2e:
        # through the C ABI with HOST buffers: the step's f in from pinned memory, the step's
        # solution(s) out.  Both solvers: tpmg_solve_host_pair (f copied once, the MG solution's
        # copy out overlapping the PCG solve); one solver: tpmg_solve_host.
        fh = f.cpu().pin_memory()
        uh = torch.empty_like(fh).pin_memory()
        uh2 = torch.empty_like(fh).pin_memory()
        pair = do_mg and do_cg

        def e2e_step():
            if pair:
                ctx.solve_host_pair(fh, uh, uh2, eps=args.eps)
            elif do_mg:
                ctx.solve_host(T.TPMG_SOLVER_MG, fh, uh, eps=args.eps)
            else:
                ctx.solve_host(T.TPMG_SOLVER_CG, fh, uh, eps=args.eps)

        e2e_step()   # untimed: allocates the staging buffers and the copy stream
        barrier()
        t0 = time.perf_counter()
        for _ in range(args.steps):
            e2e_step()
        barrier()
        te = torch.tensor([time.perf_counter() - t0], dtype=torch.float64, device=f"cuda:{local}")
        if world > 1:
            dist.all_reduce(te, op=dist.ReduceOp.MAX)
        te = float(te.item())
        nbytes = fh.numel() * 8 * world
        e2e = {"value": solves * n_glob * args.steps / te, "unit": UNIT,
               "h2d_bytes_per_step": nbytes, "d2h_bytes_per_step": solves * nbytes,
               "api": "tpmg_solve_host_pair (f in once, MG solution out overlapping the PCG solve)" if pair
                      else "tpmg_solve_host"}
        # the paper's "total solution time" (tab:SingleGPUTiming): z-contiguous host
        # fields, H2D + transpose on the GPU + solve + transpose + D2H, one solve of each kind
        fz = fh.view(shape).permute(0, 2, 1).contiguous().pin_memory()
        uz = torch.empty_like(fz).pin_memory()
        tz = {}
        for key, sv, on in (("mg_ms", T.TPMG_SOLVER_MG, do_mg), ("cg_ms", T.TPMG_SOLVER_CG, do_cg)):
            if not on:
                continue
            barrier()
            t0 = time.perf_counter()
            ctx.solve_host_zc(sv, fz, uz, eps=args.eps)
            barrier()
            tz[key] = 1e3 * (time.perf_counter() - t0)
        e2e["total_solution_time_zc"] = dict(tz, note="wall ms per solve through tpmg_solve_host_zc: "
                                             "z-contiguous host f in, transposes on the GPU, u out (P:427)")

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        gpu_counts = (its[0].iterations if its[0] else 0, its[1].iterations if its[1] else 0)
        cpu = cpu_baseline_block(args, nx, ny, do_mg, do_cg, gpu_counts)

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms / args.steps, "higher_is_better": True,
            "scaling": "strong" if args.global_nx else "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (splitmix64 uniform[-1,1) RHS keyed by global index, seed %d)" % args.seed,
            "config": config_block(args, nx, ny, name, world),
            "roofline": roof,
            "cpu_baseline": cpu,
            "e2e": e2e,
            "gpu_launches": stats["kernel_launches"],
            "clocks": clk.summary(),
            "hbm_gbs_step": round(hbm_gbs_step, 1),
            "kernels": kernels,
            **line_extra,
        }
        print(json.dumps(line), flush=True)
    ctx.close()
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
