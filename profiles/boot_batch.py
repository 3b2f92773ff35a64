"""Throughput of B independent bootstraps in flight on one GPU (one CUDA graph, each bootstrap
on its own group of lanes, optionally staggered) against the single-bootstrap latency.
Usage: python profiles/boot_batch.py [B] [lanes]"""
import json
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2512_18345_b200 import ckks, keyswitch as ks
from paper_2512_18345_b200.bootstrap import BootstrapConfig, Bootstrapper
from paper_2512_18345_b200.engine import get_engine
from paper_2512_18345_b200.params import ParameterSet

B = int(sys.argv[1]) if len(sys.argv) > 1 else 2
lanes = int(sys.argv[2]) if len(sys.argv) > 2 else 16
eng = get_engine()
eng.set_lanes(lanes)
p = ParameterSet.builtin("ks48")
sk = ks.keygen(p, h=p.h_sparse, seed=1)
boot = Bootstrapper(p, sk, BootstrapConfig())
rng = np.random.default_rng(0)
msgs = [rng.uniform(-1, 1, p.n // 2) + 1j * rng.uniform(-1, 1, p.n // 2) for _ in range(B)]
cts = [ckks.encrypt(ckks.encode(z, p, level=2, scale=boot.delta_in), sk, p, seed=50 + i) for i, z in enumerate(msgs)]


def run_all():
    return eng.fork([(lambda c=c: boot.bootstrap(c)) for c in cts])


outs = run_all()
torch.cuda.synchronize()
g = torch.cuda.CUDAGraph()
side = torch.cuda.Stream(device=eng.device)
side.wait_stream(torch.cuda.current_stream())
with torch.cuda.stream(side):
    run_all()
    torch.cuda.synchronize()
    with torch.cuda.graph(g, stream=side):
        outs = run_all()
torch.cuda.current_stream().wait_stream(side)
g.replay()
torch.cuda.synchronize()
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
reps = 10
a.record()
for _ in range(reps):
    g.replay()
b.record()
torch.cuda.synchronize()
ms = a.elapsed_time(b) / reps
errs = [float(np.log2(np.abs(ckks.decrypt_decode(o, sk, p) - z).max())) for o, z in zip(outs, msgs)]
print(json.dumps({"batch": B, "lanes": lanes, "ms_per_batch": ms, "ms_per_bootstrap": ms / B,
                  "bootstraps_per_s": B / ms * 1e3, "log2_err": errs}))
