"""In-graph kernel durations of one bootstrap replay through CUPTI (torch.profiler): warm caches,
real concurrency -- unlike the serialised cold-cache ncu launch list.  Prints per-kernel totals,
the sum of kernel time, the union of busy intervals and the replay's span.
Usage: python profiles/graph_trace.py [lanes [chrome_trace.json]]"""
import collections
import json
import re
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2512_18345_b200 import ckks, keyswitch as ks
from paper_2512_18345_b200.bootstrap import BootstrapConfig, Bootstrapper
from paper_2512_18345_b200.engine import get_engine
from paper_2512_18345_b200.params import ParameterSet

lanes = int(sys.argv[1]) if len(sys.argv) > 1 else 8
eng = get_engine()
eng.set_lanes(lanes)
p = ParameterSet.builtin("ks48")
from paper_2512_18345_b200.bootstrap import standard_input, standard_setup

sk, _sparse, boot = standard_setup(p)           # the bench's setup: dense key + sparse encapsulation
_z, ct = standard_input(p, boot, sk, 0)
replay = boot.capture(ct)
for _ in range(3):
    replay.graph.replay()
torch.cuda.synchronize()
from torch.profiler import ProfilerActivity, profile

with profile(activities=[ProfilerActivity.CUDA]) as prof:
    replay.graph.replay()
    torch.cuda.synchronize()
if len(sys.argv) > 2:                          # full timeline (stream, grid, block per kernel) for offline analysis
    prof.export_chrome_trace(sys.argv[2])
evs = [e for e in prof.events() if e.device_type == torch.autograd.DeviceType.CUDA and e.cuda_time_total > 0 or getattr(e, "device_time_total", 0) > 0]
rows = []
for e in prof.events():
    dur = getattr(e, "device_time_total", 0) or getattr(e, "cuda_time_total", 0)
    if dur <= 0 or e.time_range is None:
        continue
    rows.append((e.name, e.time_range.start, e.time_range.end))
agg = collections.defaultdict(lambda: [0, 0.0])
for name, a, b in rows:
    short = re.sub(r"\(.*", "", name).replace("void ", "").replace("ckks::", "")
    short = re.sub(r"<.*", "", short)
    agg[short][0] += 1
    agg[short][1] += b - a
total = sum(v[1] for v in agg.values())
iv = sorted((a, b) for _, a, b in rows)
busy, cur_a, cur_b = 0.0, None, None
for a, b in iv:
    if cur_a is None:
        cur_a, cur_b = a, b
    elif a <= cur_b:
        cur_b = max(cur_b, b)
    else:
        busy += cur_b - cur_a
        cur_a, cur_b = a, b
if cur_a is not None:
    busy += cur_b - cur_a
span = iv[-1][1] - iv[0][0] if iv else 0.0
out = {"lanes": lanes, "kernels": len(rows), "sum_kernel_ms": total / 1e3, "busy_union_ms": busy / 1e3, "span_ms": span / 1e3,
       "by_kernel": {k: {"n": v[0], "ms": round(v[1] / 1e3, 3), "avg_us": round(v[1] / v[0], 2)} for k, v in sorted(agg.items(), key=lambda kv: -kv[1][1])}}
print(json.dumps(out, indent=1))
