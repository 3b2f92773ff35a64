"""Per-kernel microbenchmark on synthetic ks48 limbs (N = 2^16): each primitive timed alone
with CUDA events, inputs rotating through a pool larger than the 126 MB L2 ("cold") and on one
resident buffer ("warm").  Prints one JSON object; used to iterate on single kernels before the
bootstrap bench.  Usage: python profiles/kbench.py [reps]"""
import json
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2512_18345_b200 import keyswitch as ks
from paper_2512_18345_b200.engine import get_engine
from paper_2512_18345_b200.params import ParameterSet

reps = int(sys.argv[1]) if len(sys.argv) > 1 else 20
eng = get_engine()
p = ParameterSet.builtin("ks48")
dev = eng.device
g = torch.Generator(device=dev)
g.manual_seed(1)
LIMB = p.n * 4


def rand_rows(slots_basis, rows):
    basis = [slots_basis[i % len(slots_basis)] for i in range(rows)]
    q = torch.tensor([m.q for m in basis], dtype=torch.float64, device=dev)[:, None]
    u = torch.rand((rows, p.n), generator=g, device=dev, dtype=torch.float64)
    return (u * q).to(torch.int64).to(torch.int32).contiguous(), basis


def timeit(fn, n_variants):
    """Capture `reps` back-to-back calls into one CUDA graph (no host launch gaps), replay it."""
    for i in range(2):
        fn(i % n_variants)
    torch.cuda.synchronize()
    graph = torch.cuda.CUDAGraph()
    side = torch.cuda.Stream()
    side.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(side):
        with torch.cuda.graph(graph, stream=side):
            for i in range(reps):
                fn(i % n_variants)
    torch.cuda.synchronize()
    graph.replay()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    graph.replay()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / reps * 1e3      # us


res = {}
ext = p.ext_basis
for rows in (2, 12, 24, 48, 96, 192):
    pool = max(2, min(12, int(400e6 // (rows * LIMB)) + 1))
    bufs = []
    for _ in range(pool):
        d, basis = rand_rows(ext, rows)
        bufs.append(d)
    slots = eng.row_slots(basis, p.n)
    outs = [eng.empty(rows, p.n) for _ in range(pool)]
    for inv in (False, True):
        name = f"ntt_{'inv' if inv else 'fwd'}_R{rows}"
        cold = timeit(lambda i: eng.ntt(bufs[i], slots, inv, out=outs[i]), pool)
        warm = timeit(lambda i: eng.ntt(bufs[0], slots, inv, out=outs[0]), 1)
        alg = 2 * 2 * rows * LIMB      # two kernels, each one read + one write
        res[name] = {"cold_us": round(cold, 2), "warm_us": round(warm, 2),
                     "cold_gbs": round(alg / cold / 1e3, 0), "bfly_per_clk_sm": round(rows * p.n * 8 / (cold * 1e-6) / 148 / 1.965e9, 2)}
    if rows >= 48:
        for nm, inv, lo, hi in (("fwd_strided", False, 0, 8), ("fwd_contig", False, 8, 16),
                                ("inv_contig", True, 0, 8), ("inv_strided", True, 8, 16)):
            cold = timeit(lambda i: eng.ntt_stages(bufs[i], slots, inv, lo, hi, out=outs[i]), pool)
            res[f"{nm}_R{rows}"] = {"cold_us": round(cold, 2), "cold_gbs": round(2 * rows * LIMB / cold / 1e3, 0),
                                    "bfly_per_clk_sm": round(rows * p.n * 4 / (cold * 1e-6) / 148 / 1.965e9, 2)}
    del bufs, outs

# full-level key switch, stage by stage through the profile counters
n_ct, n_evk = 8, 4
cts = []
for _ in range(n_ct):
    d, _b = rand_rows(p.q_basis, 2 * p.l)
    cts.append(d.view(2, p.l, p.n))
evks = []
for _ in range(n_evk):
    d, _b = rand_rows(ext, p.dnum * 2 * len(ext))
    evks.append(d.view(p.dnum, 2, len(ext), p.n))
outs = [eng.empty(2, p.l, p.n) for _ in range(n_ct)]
plan = ks._tables(p).plan()
res["keyswitch_us"] = round(timeit(lambda i: eng.keyswitch(plan, cts[i % n_ct][0], cts[i % n_ct][1], evks[i % n_evk], out=outs[i % n_ct]), 8), 2)
eng.lib.ckks_profile_enable(1)
for i in range(reps):
    eng.keyswitch(plan, cts[i % n_ct][0], cts[i % n_ct][1], evks[i % n_evk], out=outs[i % n_ct])
buf = torch.zeros(1)  # placeholder to keep torch imported
import ctypes
cbuf = ctypes.create_string_buffer(1 << 16)
eng.lib.ckks_profile_read(cbuf, len(cbuf))
eng.lib.ckks_profile_enable(0)
stages = {}
for line in cbuf.value.decode().splitlines():
    parts = line.split()
    if len(parts) >= 4:
        k, c, ms, nb = parts[0], int(parts[1]), float(parts[2]), float(parts[3])
        stages[k] = {"launches": c / reps, "us_per_launch": round(ms / c * 1e3, 2),
                     "gbs": round(nb / (ms * 1e-3) / 1e9, 0) if ms else None}
res["keyswitch_kernels"] = stages
print(json.dumps(res, indent=1))
