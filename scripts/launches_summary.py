"""Summarise an ncu --csv launch list (gpu__time_duration.sum per launch) by kernel and grid."""
import collections
import csv
import re
import sys


def load(path):
    rows = list(csv.reader(open(path)))
    hi = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
    h = rows[hi]
    ki, vi, gi = h.index("Kernel Name"), h.index("Metric Value"), h.index("Grid Size")
    out = []
    for r in rows[hi + 1:]:
        if len(r) <= vi:
            continue
        m = re.search(r"k_line\w*<[^>]*>", r[ki]) or re.search(r"(k_\w+)", r[ki])
        out.append((m.group(0) if m else r[ki][:40], r[gi], float(r[vi].replace(",", "")) / 1e3))
    return out


if __name__ == "__main__":
    seq = load(sys.argv[1])
    agg = collections.defaultdict(lambda: [0, 0.0])
    for name, grid, us in seq:
        agg[(name, grid)][0] += 1
        agg[(name, grid)][1] += us
    tot = sum(v for _, v in agg.values())
    print(f"{'kernel':28s} {'grid':16s} {'n':>4s} {'total ms':>9s} {'avg us':>9s} share")
    for (name, grid), (n, us) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        print(f"{name:28s} {grid:16s} {n:4d} {us / 1e3:9.3f} {us / n:9.1f} {us / tot:.3f}")
    print(f"total {tot / 1e3:.3f} ms over {len(seq)} launches")
    if len(sys.argv) > 2:
        for s in seq[: int(sys.argv[2])]:
            print(s)
