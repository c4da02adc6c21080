"""Full oracle solves at the benchmark workloads (test/bench infrastructure, CPU only).

Runs the CPU oracle's MG and PCG solves to eps = 1e-5 from u = 0 on the whole grid of a
BASELINE configuration (default C2 = 1024 x 1024 x 128, nu = 8.4, L = 5) with the splitmix64
RHS of inputs/ (seed 0) and writes the iteration counts, final relative residuals and wall
times to tests/golden/oracle_iterations.json.  bench.py's reference arm and cpu_baseline scale
their per-iteration oracle timings by these counts (the oracle's own, not the GPU's).  Calls
only oracle/ and inputs/.

    python scripts/oracle_iterations.py [--nx 1024] [--nz 128] [--threads N]
"""
import argparse
import json
import os
import platform
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
OUT = os.path.join(ROOT, "tests", "golden", "oracle_iterations.json")


def cpu_model():
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return platform.processor() or "unknown"


def key(nx, ny, nz, nu, L, cs, boundary, seed):
    return f"{nx}x{ny}x{nz}_nu{nu:g}_L{L}_cs{cs}_bc{boundary}_seed{seed}"


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--nx", type=int, default=1024)
    ap.add_argument("--ny", type=int, default=0)
    ap.add_argument("--nz", type=int, default=128)
    ap.add_argument("--nu", type=float, default=8.4)
    ap.add_argument("--levels", type=int, default=5)
    ap.add_argument("--coarse-sweeps", type=int, default=2)
    ap.add_argument("--boundary", type=int, default=0)
    ap.add_argument("--seed", type=int, default=0)
    ap.add_argument("--threads", type=int, default=0)
    args = ap.parse_args()
    from oracle import oracle as O
    from inputs import rhs_zc
    if args.threads:
        O.set_threads(args.threads)
    nx = args.nx
    ny = args.ny or nx
    p = O.Params(nx=nx, ny=ny, nz=args.nz, nu_cfl=args.nu, L=args.levels, coarse_sweeps=args.coarse_sweeps,
                 boundary=args.boundary)
    f = rhs_zc(nx, ny, args.nz, seed=args.seed)
    rec = {"nx": nx, "ny": ny, "nz": args.nz, "nu_cfl": args.nu, "levels": args.levels,
           "coarse_sweeps": args.coarse_sweeps, "boundary": args.boundary, "seed": args.seed, "eps": 1e-5,
           "threads": O.num_threads(), "cpu_model": cpu_model(), "when": time.strftime("%Y-%m-%d"),
           "written_by": "scripts/oracle_iterations.py (oracle/ only)"}
    for name, fn in (("mg", O.solve_mg), ("cg", O.solve_cg)):
        t0 = time.perf_counter()
        r = fn(p, f, eps=1e-5)
        dt = time.perf_counter() - t0
        rec[name] = {"iterations": r.iterations, "converged": r.converged,
                     "rel_residual": float(r.history[-1] / r.history[0]), "wall_s": round(dt, 2)}
        print(name, rec[name], flush=True)
        del r
    db = json.load(open(OUT)) if os.path.exists(OUT) else {}
    db[key(nx, ny, args.nz, args.nu, args.levels, args.coarse_sweeps, args.boundary, args.seed)] = rec
    open(OUT, "w").write(json.dumps(db, indent=1, sort_keys=True) + "\n")


if __name__ == "__main__":
    main()
