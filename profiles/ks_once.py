"""Tiny driver for ncu: a few ks48 key switches on synthetic limbs (same setup as bench.py)."""
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2512_18345_b200 import keyswitch as ks
from paper_2512_18345_b200.engine import get_engine
from paper_2512_18345_b200.params import ParameterSet

reps = int(sys.argv[1]) if len(sys.argv) > 1 else 3
eng = get_engine()
p = ParameterSet.builtin("ks48")
g = torch.Generator(device=eng.device)
g.manual_seed(1)


def rand_limbs(basis, *lead):
    q = torch.tensor([m.q for m in basis], dtype=torch.float64, device=eng.device)[:, None]
    u = torch.rand((*lead, len(basis), p.n), generator=g, device=eng.device, dtype=torch.float64)
    return (u * q).to(torch.int64).to(torch.int32).contiguous()


ct = rand_limbs(p.q_basis, 2)
evk = rand_limbs(p.ext_basis, p.dnum, 2)
out = eng.empty(2, p.l, p.n)
plan = ks._tables(p).plan()
torch.cuda.synchronize()
for _ in range(reps):
    eng.keyswitch(plan, ct[0], ct[1], evk, out=out)
torch.cuda.synchronize()
print("done")
