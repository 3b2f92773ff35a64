"""Do an HBM-bound kernel (evaluation-key inner product) and an integer-pipe-bound kernel (batched
NTT) of two different stream lanes overlap on B200, i.e. does co-scheduling the paper's
'complementary' kernel groups (reference costmodel.py:508-541) pay at kernel
granularity?  One CUDA graph per case: A = 8 inner products (ks48, 60 rows, 126 MB key each),
B = 8 forward NTTs of 192 rows, A and B on two streams (with and without a high-priority
stream for B).  Prints device times.  Usage: python profiles/overlap_probe.py"""
import json
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2512_18345_b200 import keyswitch as ks
from paper_2512_18345_b200.engine import get_engine
from paper_2512_18345_b200.params import ParameterSet

eng = get_engine()
dev = eng.device
p = ParameterSet.builtin("ks48")
ext = p.ext_basis
g = torch.Generator(device=dev)
g.manual_seed(1)


def rand_limbs(basis, *lead):
    q = torch.tensor([m.q for m in basis], dtype=torch.float64, device=dev)[:, None]
    u = torch.rand((*lead, len(basis), p.n), generator=g, device=dev, dtype=torch.float64)
    return (u * q).to(torch.int64).clamp_(min=0).to(torch.int32).contiguous()


plan = ks._tables(p).plan()
raised = rand_limbs(ext, p.dnum)
evks = [rand_limbs(ext, p.dnum, 2) for _ in range(4)]
rows = 192
basis = tuple(ext[i % len(ext)] for i in range(rows))
polys = [rand_limbs(basis) for _ in range(3)]
outs = [eng.empty(rows, p.n) for _ in range(3)]
slots = eng.row_slots(basis, p.n)
REPS = 8


def run_a():
    for i in range(REPS):
        eng.ks_stage2(plan, raised, evks[i % 4], 0, p.l + p.alpha)


def run_b():
    for i in range(REPS):
        eng.ntt(polys[i % 3], slots, False, out=outs[i % 3])


def capture(fa, fb, prio_b=0):
    main = torch.cuda.Stream(device=dev)
    side = torch.cuda.Stream(device=dev, priority=prio_b)
    graph = torch.cuda.CUDAGraph()
    torch.cuda.synchronize()
    with torch.cuda.stream(main):
        with torch.cuda.graph(graph, stream=main):
            if fa and fb:
                side.wait_stream(main)
                with torch.cuda.stream(side):
                    fb()
                fa()
                main.wait_stream(side)
            elif fa:
                fa()
            else:
                fb()
    return graph


def time_graph(graph, n=5):
    for _ in range(2):
        graph.replay()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(n):
        graph.replay()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / n * 1e3


run_a()
run_b()
torch.cuda.synchronize()
res = {}
res["A_inner_product_x8_us"] = time_graph(capture(run_a, None))
res["B_ntt192_x8_us"] = time_graph(capture(None, run_b))
res["A_and_B_two_streams_us"] = time_graph(capture(run_a, run_b))
res["A_and_B_B_high_priority_us"] = time_graph(capture(run_a, run_b, prio_b=-1))
res["sum_us"] = res["A_inner_product_x8_us"] + res["B_ntt192_x8_us"]
res["max_us"] = max(res["A_inner_product_x8_us"], res["B_ntt192_x8_us"])
print(json.dumps(res, indent=1))
