"""Latency of the bootstrap for different baby-step counts of the BSGS linear transforms
(BootstrapConfig.n1; default: ~2*sqrt(span), at most 16).  Round 2 made giant steps cheaper (only the
a half of their inner sum is scaled down), which could have moved the optimum.
Usage: python profiles/boot_n1.py [n1 ...]   (0 = the default heuristic)"""
import json
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2512_18345_b200 import ckks
from paper_2512_18345_b200.bootstrap import BootstrapConfig, standard_input, standard_setup
from paper_2512_18345_b200.engine import get_engine
from paper_2512_18345_b200.params import ParameterSet

eng = get_engine()
eng.set_lanes(8)
p = ParameterSet.builtin("ks48")
res = {}
for n1 in [int(a) for a in sys.argv[1:]] or [0, 8, 16]:
    sk, _sparse, boot = standard_setup(p, BootstrapConfig(n1=n1 or None))
    z, ct = standard_input(p, boot, sk, 0)
    run = boot.capture(ct)
    for _ in range(10):
        out = run(ct)
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(20):
        out = run(ct)
    b.record()
    torch.cuda.synchronize()
    got = ckks.decrypt_decode(out, sk, p)
    res[n1] = {"ms": round(a.elapsed_time(b) / 20, 3),
               "log2_max_err": round(float(np.log2(np.abs(got - z).max())), 2),
               "baby_x_giant": [[len(lt.baby), len(lt.giants)] for lt in boot.cts + boot.stc]}
    print(n1, res[n1], flush=True)
    del boot, run, out
    torch.cuda.empty_cache()
print(json.dumps(res, indent=1))
