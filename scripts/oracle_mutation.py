"""Mutation check of the oracle pins (test infrastructure, CPU only).

Each mutant is a one-line plausible mistake in oracle/tpmg_oracle.c.  For each, a mutated
copy of the oracle is compiled into a temporary directory and the oracle pin suites
(tests/test_oracle_pins*.py) are run against it (oracle.py honours TPMG_ORACLE_LIB).  A
mutant must make at least one pin fail ("red"); a mutant that passes every pin ("GREEN")
means the pins do not cover that part of the oracle.

    python scripts/oracle_mutation.py [--out profiles/r2/oracle_mutation.txt] [names...]
"""
import argparse
import os
import subprocess
import sys
import tempfile
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SRC = os.path.join(ROOT, "oracle", "tpmg_oracle.c")
PINS = ["tests/test_oracle_pins.py", "tests/test_oracle_pins_face.py", "tests/test_oracle_pins_fields.py",
        "tests/test_oracle_pins_profiles.py", "tests/test_oracle_pins_vcycle.py"]

# (name, passage, original text, mutated text)
MUTANTS = [
    # the three V-cycle mutants of the round-1 review (VERDICT weak #1)
    ("vcycle_post_plus_one", "alg:VCycle P:205-206 (one post-smooth)",
     "for (int s = 0; s < mg->p.post; ++s) st |= or_mg_smooth(mg, l);",
     "for (int s = 0; s <= mg->p.post; ++s) st |= or_mg_smooth(mg, l);"),
    ("restrictsmooth_without_rho", "P:194 u = rho M^-1 f",
     "mg->u[l][q] = mg->p.rho * mg->u[l][q];",
     "mg->u[l][q] = mg->u[l][q];"),
    ("extra_coarse_sweep", "P:229 / [R5] coarse_sweeps - 1 smooths after RestrictSmooth",
     "for (int s = 1; s < mg->p.coarse_sweeps; ++s) st |= or_mg_smooth(mg, 1);",
     "for (int s = 0; s < mg->p.coarse_sweeps; ++s) st |= or_mg_smooth(mg, 1);"),
    ("vcycle_pre_plus_one_coarse", "alg:VCycle P:193-195 (RestrictSmooth is the pre-smooth)",
     "for (int s = 1; s < mg->p.pre; ++s) st |= or_mg_smooth(mg, l);",
     "for (int s = 0; s < mg->p.pre; ++s) st |= or_mg_smooth(mg, l);"),
    ("vcycle_skip_prolongation", "alg:VCycle P:201",
     "or_prolong_add(&mg->op[l - 1], &mg->op[l], mg->u[l - 1], mg->u[l]);",
     "(void)0;"),
    # operator, preconditioner, transfers, solvers (the round-1 list, now scripted)
    ("alpha_T_factor", "P:150 diagonal 1 + 4 omega^2/h^2",
     "op->alpha_T = 4.0 * op->alpha_TT;", "op->alpha_T = 3.0 * op->alpha_TT;"),
    ("neighbour_coupling_sign", "P:150 A_TT' = -omega^2/h^2",
     "y += op->alpha_TT * op->d[k] * nb;", "y -= op->alpha_TT * op->d[k] * nb;"),
    ("neighbour_index_west", "eqn:TridiagonalPDE neighbours",
     "if (has_w) nb += x[ZC(op, i - 1, j, k)];", "if (has_w) nb += x[ZC(op, i, j, k)];"),
    ("thomas_forward_sign", "Thomas, S:267",
     "gp[k] = (g[k] - s[k] * gp[k - 1]) / m;", "gp[k] = (g[k] + s[k] * gp[k - 1]) / m;"),
    ("thomas_backward_sign", "Thomas, S:267",
     "x[k] = gp[k] - tp[k] * x[k + 1];", "x[k] = gp[k] + tp[k] * x[k + 1];"),
    ("smoother_rho", "eqn:MultigridSmoother P:215-218",
     "ucol_out[k] = u[ZC(op, i, j, k)] + rho * z[k];", "ucol_out[k] = u[ZC(op, i, j, k)] + z[k];"),
    ("restrict_child", "P:226 cell average of the 4 children",
     "rf[ZC(fine, 2 * I + 1, 2 * J, k)]", "rf[ZC(fine, 2 * I, 2 * J, k)]"),
    ("prolong_side", "P:226 bilinear, nearer coarse neighbour",
     "long sx = (i % 2 == 0) ? -1 : 1,", "long sx = (i % 2 == 0) ? 1 : -1,"),
    ("face_reflection_sign", "[R25] ghost = -u_c",
     "if (I < 0) { I = 0; sign = -sign; }", "if (I < 0) { I = 0; }"),
    ("face_weight", "[R25] boundary face counts twice",
     "if (i == 0) aT += w;", "if (i == 0) aT += 0.0 * w;"),
    ("cg_beta_inverted", "PCG beta = zeta_new / zeta",
     "double beta = zeta_new / zeta;", "double beta = zeta / zeta_new;"),
    ("dot_drops_row", "deterministic inner product",
     "for (long j = 0; j < op->ny; ++j) s += rows[j];", "for (long j = 1; j < op->ny; ++j) s += rows[j];"),
]


def run_one(name, old, new, tmp, kexpr=None):
    src = open(SRC).read()
    n = src.count(old)
    if n != 1:
        return "SKIP", f"pattern found {n} times"
    mdir = os.path.join(tmp, name)
    os.makedirs(mdir, exist_ok=True)
    csrc = os.path.join(mdir, "tpmg_oracle.c")
    lib = os.path.join(mdir, "liboracle.so")
    open(csrc, "w").write(src.replace(old, new))
    subprocess.check_call(["gcc", "-O2", "-std=c11", "-fPIC", "-shared", "-ffp-contract=off", "-fopenmp",
                           "-o", lib, csrc, "-lm"])
    env = dict(os.environ, TPMG_ORACLE_LIB=lib)
    sel = ["-k", kexpr] if kexpr else []
    r = subprocess.run([sys.executable, "-m", "pytest", "-q", "-x", "-m", "not gpu", "-p", "no:cacheprovider", *sel, *PINS],
                       cwd=ROOT, env=env, capture_output=True, text=True)
    failed = [l for l in r.stdout.splitlines() if l.startswith("FAILED")]
    if r.returncode == 0:
        return "GREEN", "all pins passed"
    return "red", failed[0][7:] if failed else r.stdout.strip().splitlines()[-1]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default=None)
    ap.add_argument("-k", dest="kexpr", default=None, help="pytest -k expression selecting the pins to run")
    ap.add_argument("names", nargs="*")
    args = ap.parse_args()
    lines = [f"# oracle mutation check ({time.strftime('%Y-%m-%d %H:%M')}); pins: {' '.join(PINS)}"
             + (f" -k '{args.kexpr}'" if args.kexpr else ""),
             "# red = at least one pin fails (the mutant is caught); GREEN = every pin passes"]
    bad = 0
    with tempfile.TemporaryDirectory() as tmp:
        for name, cite, old, new in MUTANTS:
            if args.names and name not in args.names:
                continue
            t0 = time.time()
            verdict, why = run_one(name, old, new, tmp, args.kexpr)
            bad += verdict != "red"
            line = f"{verdict:5s} {name:28s} [{cite}] ({time.time() - t0:.0f} s) first failure: {why}"
            print(line, flush=True)
            lines.append(line)
    lines.append(f"# {bad} mutant(s) not caught")
    if args.out:
        os.makedirs(os.path.dirname(os.path.abspath(args.out)), exist_ok=True)
        open(args.out, "w").write("\n".join(lines) + "\n")
    return 1 if bad else 0


if __name__ == "__main__":
    sys.exit(main())
