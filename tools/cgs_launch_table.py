#!/usr/bin/env python
"""Summarise an ncu --csv launch list of cgs_kernel launches (gpu__time_duration,
dram bytes) per step: mode 2 = PROJ, 3 = UPD+PROJ, 5 = UPD+NRM.

    python tools/cgs_launch_table.py gpurun_out/r2_cgs_launches.csv
"""
import csv
import re
import sys
from collections import defaultdict


def main(path):
    rows = [r for r in csv.reader(open(path)) if r and not r[0].startswith("==")]
    hdr = rows[0]
    ki, mi, vi, ii = hdr.index("Kernel Name"), hdr.index("Metric Name"), hdr.index("Metric Value"), hdr.index("ID")
    per = defaultdict(dict)
    for r in rows[1:]:
        if len(r) < len(hdr):
            continue
        per[int(r[ii])][r[mi]] = float(r[vi].replace(",", ""))
        per[int(r[ii])]["name"] = r[ki]
    tot = defaultdict(lambda: [0, 0.0, 0.0])
    for i in sorted(per):
        d = per[i]
        m = re.search(r"cgs_kernel<(\w+), (?:\(int\))?(\d+), (?:\(int\))?(\d+)>", d["name"])
        key = (m.group(1), int(m.group(2)), int(m.group(3)))
        ns = d["gpu__time_duration.sum"]
        by = d["dram__bytes_read.sum"] + d["dram__bytes_write.sum"]
        t = tot[key]
        t[0] += 1
        t[1] += ns
        t[2] += by
        print(f"{i:5d} {key} {ns / 1e3:8.1f} us {by / ns:7.0f} GB/s")
    print("per instantiation:")
    for k, (n, ns, by) in sorted(tot.items()):
        print(f"  {k}: {n} launches, {ns / 1e3 / n:.1f} us avg, {by / ns:.0f} GB/s")


if __name__ == "__main__":
    main(sys.argv[1])
