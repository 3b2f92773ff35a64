"""Latency / output level / precision of the bootstrap for different numbers of stage groups per
linear transform (BootstrapConfig.groups): fewer diagonals per group against more levels spent.
Usage: python profiles/boot_groups.py [groups ...]"""
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
res = {}
for groups in [int(a) for a in sys.argv[1:]] or [3, 4]:
    try:
        boot = Bootstrapper(p, sk, BootstrapConfig(groups=groups))
        ct = ckks.encrypt(ckks.encode(z, p, level=2, scale=boot.delta_in), sk, p, seed=50)
        run = boot.capture(ct)
        for _ in range(3):
            out = run(ct)
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(20):
            out = run(ct)
        b.record()
        torch.cuda.synchronize()
        got = ckks.decrypt_decode(out, sk, p)
        res[groups] = {"ms": round(a.elapsed_time(b) / 20, 3), "out_level": boot.out_level,
                       "log2_max_err": round(float(np.log2(np.abs(got - z).max())), 2),
                       "diagonals": [len(lt.baby) * len(lt.giants) for lt in boot.cts]}
        del boot, run, out
        torch.cuda.empty_cache()
    except Exception as exc:                                  # a configuration the level budget cannot hold
        res[groups] = {"error": f"{type(exc).__name__}: {exc}"}
print(json.dumps(res, indent=1))
