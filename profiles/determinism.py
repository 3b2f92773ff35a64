"""Race check: the captured bootstrap graph (8 lanes, nested forks, programmatic dependent
launches) replayed several times on the same input must give bit-identical limbs, and equal the
eager single-lane result.  Usage: python profiles/determinism.py [replays]"""
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2512_18345_b200 import ckks, keyswitch as ks
from paper_2512_18345_b200.bootstrap import BootstrapConfig, Bootstrapper
from paper_2512_18345_b200.engine import get_engine
from paper_2512_18345_b200.params import ParameterSet

reps = int(sys.argv[1]) if len(sys.argv) > 1 else 8
eng = get_engine()
p = ParameterSet.builtin("ks48")
sk = ks.keygen(p, h=p.h_sparse, seed=1)
boot = Bootstrapper(p, sk, BootstrapConfig())
rng = np.random.default_rng(0)
z = rng.uniform(-1, 1, p.n // 2) + 1j * rng.uniform(-1, 1, p.n // 2)
ct = ckks.encrypt(ckks.encode(z, p, level=2, scale=boot.delta_in), sk, p, seed=50)
eng.set_lanes(1)
ref = boot.bootstrap(ct)
ref_t = torch.stack([ref.a.data, ref.b.data]).clone()
torch.cuda.synchronize()
eng.set_lanes(8)
replay = boot.capture(ct)
bad = 0
for i in range(reps):
    out = replay(ct)
    t = torch.stack([out.a.data, out.b.data])
    same = bool(torch.equal(t, ref_t))
    bad += 0 if same else 1
    print(f"replay {i}: equal to the eager single-lane limbs: {same}")
torch.cuda.synchronize()
print("DETERMINISTIC" if bad == 0 else f"MISMATCH in {bad} of {reps} replays")
sys.exit(0 if bad == 0 else 1)
