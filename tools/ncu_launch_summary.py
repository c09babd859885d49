#!/usr/bin/env python
"""Per-kernel totals of an ncu --csv launch list (gpu__time_duration.sum and,
if present, dram bytes): launches, total and mean duration, share.

    python tools/ncu_launch_summary.py launches.csv [--last N]
"""
import csv
import re
import sys
from collections import defaultdict


def main(path, last=None):
    rows = [r for r in csv.reader(open(path)) if r and not r[0].startswith("==")]
    hdr = rows[0]
    ki, mi, vi, ii = (hdr.index(x) for x in ("Kernel Name", "Metric Name", "Metric Value", "ID"))
    per = defaultdict(dict)
    for r in rows[1:]:
        if len(r) < len(hdr):
            continue
        per[int(r[ii])][r[mi]] = float(r[vi].replace(",", ""))
        per[int(r[ii])]["name"] = r[ki]
    ids = sorted(per)
    if last:
        ids = ids[-last:]
    tot = defaultdict(lambda: [0, 0.0])
    for i in ids:
        d = per[i]
        name = re.sub(r"\(.*", "", d["name"]).replace("void ", "").replace("ppf::<unnamed>::", "")
        name = name.replace("unnamed>::", "")
        tot[name][0] += 1
        tot[name][1] += d.get("gpu__time_duration.sum", 0.0)
    allns = sum(v[1] for v in tot.values())
    for name, (n, ns) in sorted(tot.items(), key=lambda kv: -kv[1][1]):
        print(f"{ns / 1e6:9.3f} ms {100 * ns / allns:5.1f}%  {n:6d} x {ns / n / 1e3:8.2f} us  {name}")
    print(f"{allns / 1e6:9.3f} ms total, {len(ids)} launches")


if __name__ == "__main__":
    a = sys.argv[1:]
    last = int(a[a.index("--last") + 1]) if "--last" in a else None
    main(a[0], last)
