"""Summarise an ncu --set full report: per captured kernel, duration, DRAM bytes,
achieved DRAM GB/s, warps active, registers, top stall reasons.  Writes markdown to
stdout and (optionally) a JSON of DRAM traffic per kernel class for bench.py."""
import csv
import json
import re
import subprocess
import sys

MODES = {0: "apply", 1: "residual", 2: "precondition", 3: "smooth", 4: "cg_direction",
         5: "cg_precondition", 6: "residual_restrict"}


TSCALE = {"ms": 1.0, "us": 1e-3, "usecond": 1e-3, "ns": 1e-6, "nsecond": 1e-6, "s": 1e3, "msecond": 1.0}
BSCALE = {"Gbyte": 1.0, "Mbyte": 1e-3, "Kbyte": 1e-6, "byte": 1e-9, "Tbyte": 1e3}


def raw(rep):
    """Rows of `ncu -i rep --page raw --csv` (or of an exported .csv of that page)."""
    if rep.endswith(".csv"):
        out = open(rep).read()
    else:
        out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    return rows[0], rows[1], rows[2:]


def main(rep, traffic_json=None):
    h, units, data = raw(rep)
    c = {n: i for i, n in enumerate(h)}
    stall = [n for n in h if "warps_issue_stalled" in n and n.endswith("_per_issue_active.ratio")]
    print("| kernel | grid | time (us) | DRAM read (GB) | DRAM write (GB) | DRAM GB/s | warps active % | regs | top stalls (cycles/issue) |")
    print("|---|---|---|---|---|---|---|---|---|")
    traffic = {}
    for r in data:
        name = r[c["Kernel Name"]]
        m = re.search(r"k_line(k?)<(\d+), ([\d, ]+)>", name)
        if "k_prolong_add" in name:
            label = "k_prolong_add"
        if m:
            mode = int(m.group(2))
            label = f"k_line{m.group(1)}<{m.group(2)},{m.group(3).replace(' ', '')}> ({MODES.get(mode, '?')})"
        elif "k_prolong_add" not in name:
            label = name.split("(")[0][-30:]
        t = float(r[c["gpu__time_duration.sum"]]) * TSCALE[units[c["gpu__time_duration.sum"]]]  # ms
        rd = float(r[c["dram__bytes_read.sum"]]) * BSCALE[units[c["dram__bytes_read.sum"]]]     # GB
        wr = float(r[c["dram__bytes_write.sum"]]) * BSCALE[units[c["dram__bytes_write.sum"]]]
        gbs = (rd + wr) / (t * 1e-3)
        st = sorted(((float(r[c[n]]) if r[c[n]] not in ("", "n/a") else 0.0,
                      n.replace("smsp__average_warps_issue_stalled_", "").replace("_per_issue_active.ratio", ""))
                     for n in stall), reverse=True)[:3]
        print(f"| {label} | {r[c['Grid Size']]} | {t * 1e3:.1f} | {rd:.3f} | {wr:.3f} | {gbs:.0f} | "
              f"{float(r[c['sm__warps_active.avg.pct_of_peak_sustained_active']]):.1f} | {r[c['launch__registers_per_thread']]} | "
              + ", ".join(f"{n} {v:.2f}" for v, n in st) + " |")
        if "k_prolong_add" in name and "prolong_add" not in traffic:
            traffic["prolong_add"] = {"bytes": 0.0, "time_ms": 0.0, "grid": r[c["Grid Size"]]}
        if "k_prolong_add" in name:   # keep the largest (fine-level) launch
            if (rd + wr) * 1e9 > traffic["prolong_add"]["bytes"]:
                traffic["prolong_add"] = {"bytes": (rd + wr) * 1e9, "time_ms": t, "grid": r[c["Grid Size"]]}
        if m:   # per class, the largest (fine-level) capture
            cls = MODES.get(mode)
            if cls and (cls not in traffic or (rd + wr) * 1e9 > traffic[cls]["bytes"]):
                traffic[cls] = {"bytes": (rd + wr) * 1e9, "time_ms": t, "grid": r[c["Grid Size"]]}
    if traffic_json:
        json.dump(traffic, open(traffic_json, "w"), indent=1)


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2] if len(sys.argv) > 2 else None)
