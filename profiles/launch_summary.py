"""Aggregate an ncu launch list (--metrics gpu__time_duration.sum --csv) by kernel and grid.
Usage: launch_summary.py launches.csv [top]"""
import collections
import csv
import re
import sys

rows = list(csv.reader(open(sys.argv[1])))
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
hdr = next(r for r in rows if "Kernel Name" in r)
start = rows.index(hdr)
ki, mv, gi = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Grid Size")
mn = hdr.index("Metric Name")
by_kernel = collections.defaultdict(list)
by_shape = collections.defaultdict(list)
for r in rows[start + 1:]:
    if len(r) <= mv or r[mn] != "gpu__time_duration.sum":
        continue
    try:
        ns = float(r[mv].replace(",", ""))
    except ValueError:
        continue
    name = re.sub(r"\(.*", "", r[ki]).replace("void ", "").replace("ckks::", "")
    by_kernel[name].append(ns)
    by_shape[(name, r[gi])].append(ns)
tot = sum(sum(v) for v in by_kernel.values())
n = sum(len(v) for v in by_kernel.values())
print(f"total {tot / 1e6:.3f} ms serialised over {n} launches")
for k, v in sorted(by_kernel.items(), key=lambda kv: -sum(kv[1])):
    print(f"{k:44s} n={len(v):4d} avg={sum(v) / len(v) / 1e3:8.2f} us  tot={sum(v) / 1e6:7.3f} ms {100 * sum(v) / tot:5.1f}%")
print()
for (k, g), v in sorted(by_shape.items(), key=lambda kv: -sum(kv[1]))[:top]:
    print(f"{k:40s} {g:16s} n={len(v):4d} avg={sum(v) / len(v) / 1e3:8.2f} us  tot={sum(v) / 1e6:7.3f} ms {100 * sum(v) / tot:5.1f}%")
