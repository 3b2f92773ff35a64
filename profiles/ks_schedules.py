"""Throughput of a batch of independent ks48 key switches under different schedules, each captured
as one CUDA graph (L2-aware batching and complementary pipelining as run-time
schedules): a plain loop, `width` key switches in flight on separate lanes, and the two-lane
ModUp | inner product + ModDown pipeline.  Usage: python profiles/ks_schedules.py [batch]"""
import json
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2512_18345_b200 import keyswitch as ks
from paper_2512_18345_b200.engine import get_engine
from paper_2512_18345_b200.params import ParameterSet
from paper_2512_18345_b200.rns import EVALUATION, Polynomial

batch = int(sys.argv[1]) if len(sys.argv) > 1 else 8
eng = get_engine()
res = {}
for name in ("ks48", "ks24", "ks12"):
    p = ParameterSet.builtin(name)
    rng = np.random.default_rng(3)
    ext = p.q_basis + p.p_basis

    def rand(basis):
        rows = np.stack([rng.integers(0, m.q, p.n, dtype=np.uint64) for m in basis])
        return Polynomial(basis, rows, EVALUATION)

    evk = ks.SwitchingKey(params=p, pairs=tuple(ks.PolyPair(rand(ext), rand(ext)) for _ in range(p.beta)))
    evk.matrix()
    cts = [ks.Ciphertext(a=rand(p.q_basis), b=rand(p.q_basis), scale=1) for _ in range(batch)]
    for ct in cts:
        ct.a.data, ct.b.data

    def graph_time(fn, reps=20):
        fn()
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        side = torch.cuda.Stream(device=eng.device)
        side.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(side):
            fn()
            torch.cuda.synchronize()
            with torch.cuda.graph(g, stream=side):
                out = fn()
        torch.cuda.current_stream().wait_stream(side)
        for _ in range(3):
            g.replay()
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(reps):
            g.replay()
        b.record()
        torch.cuda.synchronize()
        return a.elapsed_time(b) / reps * 1e3 / batch, out

    row = {}
    eng.set_lanes(1)
    row["loop"], want = graph_time(lambda: [ks.keyswitch(ct, evk) for ct in cts])
    row["staged_loop"], _ = graph_time(lambda: ks.keyswitch_pipelined(cts, evk))
    for width in (2, 4):
        eng.set_lanes(width)
        row[f"lanes{width}"], got = graph_time(
            lambda: [o for lo in range(0, batch, width)
                     for o in eng.fork([(lambda ct=ct: ks.keyswitch(ct, evk)) for ct in cts[lo:lo + width]])])
        assert all(torch.equal(g.a.data, w.a.data) and torch.equal(g.b.data, w.b.data) for g, w in zip(got, want))
    eng.set_lanes(2)
    row["pipelined"], got = graph_time(lambda: ks.keyswitch_pipelined(cts, evk))
    assert all(torch.equal(g.a.data, w.a.data) and torch.equal(g.b.data, w.b.data) for g, w in zip(got, want))
    from paper_2512_18345_b200.scheduler import plan_batch
    row["plan_batch"] = plan_batch(p, "ks_full").batch
    eng.set_lanes(8)
    row["keyswitch_batched"], _ = graph_time(lambda: ks.keyswitch_batched(cts, evk))
    res[name] = {k: round(v, 2) for k, v in row.items()}
    del evk, cts, want, got
    torch.cuda.empty_cache()
print(json.dumps({"unit": "us per key switch, batch of %d in one graph" % batch, **res}, indent=1))
