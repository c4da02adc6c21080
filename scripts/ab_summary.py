"""Summarise gpurun_out/ab_<tag>_<variant>_<rep>.json files: per variant, MG / PCG ms per
iteration, the dominant kernel's avg launch ms and roofline fraction, the SM clock."""
import glob
import json
import re
import sys

tag = sys.argv[1]
rows = {}
for f in sorted(glob.glob(f"gpurun_out/ab_{tag}_*_*.json")):
    m = re.search(rf"ab_{tag}_(\d+)_(\d+)\.json$", f)
    try:
        d = json.loads(open(f).read().strip().splitlines()[-1])
    except Exception as e:
        print(f, "unreadable", e)
        continue
    r = d.get("roofline") or {}
    k = {n: round(v["ms_total"] / max(v["launches"], 1), 4) for n, v in (d.get("kernels") or {}).items()}
    print(f"v{m.group(1)} rep{m.group(2)}: value {d['value']:.4g} ms/step {d['ms_per_step']:.2f} "
          f"mg {d['mg'] and d['mg']['ms_per_iteration']} pcg {d['pcg'] and d['pcg']['ms_per_iteration']} "
          f"dom {r.get('kernel')} {r.get('avg_launch_ms', 0):.4f} ms frac {r.get('frac')} "
          f"clk {d['clocks'].get('sm_mhz')} kernels {k}")
