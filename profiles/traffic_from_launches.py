"""profiles/traffic_<workload>.json from an ncu launch list taken with
--metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --csv:
per kernel class launches, average duration, share of the serialised time and DRAM bytes per launch
(what bench.py reports as roofline.traffic).  Usage: traffic_from_launches.py launches.csv out.json "source note" """
import collections
import csv
import json
import re
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr = next(r for r in rows if "Kernel Name" in r)
ki, mn, mv, idc = hdr.index("Kernel Name"), hdr.index("Metric Name"), hdr.index("Metric Value"), hdr.index("ID")
per = collections.defaultdict(dict)
names = {}
for r in rows[rows.index(hdr) + 1:]:
    if len(r) <= mv:
        continue
    try:
        per[r[idc]][r[mn]] = float(r[mv].replace(",", ""))
    except ValueError:
        continue
    name = re.sub(r"[<(].*", "", r[ki]).replace("void ", "").replace("ckks::", "")
    names[r[idc]] = name
agg = collections.defaultdict(lambda: [0, 0.0, 0.0, 0.0])
for i, m in per.items():
    a = agg[names[i]]
    a[0] += 1
    a[1] += m.get("gpu__time_duration.sum", 0.0)
    a[2] += m.get("dram__bytes_read.sum", 0.0)
    a[3] += m.get("dram__bytes_write.sum", 0.0)
total = sum(a[1] for a in agg.values())
doc = {"source": sys.argv[3], "total_serialised_ms": round(total / 1e6, 3), "launches": sum(a[0] for a in agg.values()), "kernels": {}}
for name, (c, ns, rd, wr) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
    doc["kernels"][name] = {"launches": c, "avg_us": round(ns / c / 1e3, 2), "share": round(ns / total, 3),
                            "dram_read_mb_per_launch": round(rd / c / 1e6, 2), "dram_write_mb_per_launch": round(wr / c / 1e6, 2)}
json.dump(doc, open(sys.argv[2], "w"), indent=1)
print(json.dumps({k: v["share"] for k, v in doc["kernels"].items()}))
