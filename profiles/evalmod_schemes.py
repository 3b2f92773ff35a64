"""Latency and precision of the bootstrap under the two EvalMod polynomial schemes.
Usage: python profiles/evalmod_schemes.py"""
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

eng = get_engine()
eng.set_lanes(8)
p = ParameterSet.builtin("ks48")
sk = ks.keygen(p, h=p.h_sparse, seed=1)
rng = np.random.default_rng(0)
z = rng.uniform(-1, 1, p.n // 2) + 1j * rng.uniform(-1, 1, p.n // 2)
for name, cfg in (("tree r=6 d=13", BootstrapConfig()),
                  ("ps r=5 d=15", BootstrapConfig(scheme="ps", squarings=5, degree=15)),
                  ("ps r=5 d=15 K=12", BootstrapConfig(scheme="ps", squarings=5, degree=15, k_bound=12))):
    boot = Bootstrapper(p, sk, cfg)
    ct = ckks.encrypt(ckks.encode(z, p, level=2, scale=boot.delta_in), sk, p, seed=50)
    replay = boot.capture(ct)
    out = replay(ct)
    err = float(np.log2(np.abs(ckks.decrypt_decode(out, sk, p) - z).max()))
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(10):
        replay.graph.replay()
    b.record()
    torch.cuda.synchronize()
    print(json.dumps({"scheme": name, "ms": a.elapsed_time(b) / 10, "log2_err": err, "out_level": boot.out_level}))
    del replay, boot
    torch.cuda.empty_cache()
