"""Where a bootstrap's time goes: ModRaise, each CoeffToSlot group, EvalMod, each SlotToCoeff
group captured as separate CUDA graphs (same lanes as bench.py) and replayed alone.
Usage: python profiles/boot_phases.py [lanes]"""
import json
import math
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2512_18345_b200 import ckks, keyswitch as ks
from paper_2512_18345_b200.bootstrap import BootstrapConfig, Bootstrapper
from paper_2512_18345_b200.engine import get_engine
from paper_2512_18345_b200.params import ParameterSet

lanes = int(sys.argv[1]) if len(sys.argv) > 1 else 4
eng = get_engine()
eng.set_lanes(lanes)
p = ParameterSet.builtin("ks48")
sk = ks.keygen(p, h=p.h_sparse, seed=1)
boot = Bootstrapper(p, sk, BootstrapConfig())
rng = np.random.default_rng(0)
z = rng.uniform(-1, 1, p.n // 2) + 1j * rng.uniform(-1, 1, p.n // 2)
ct = ckks.encrypt(ckks.encode(z, p, level=2, scale=boot.delta_in), sk, p, seed=50)


def graph_time(fn, reps=10):
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
    g.replay()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        g.replay()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / reps, out, g


res = {}
keep = []
t, raised, g = graph_time(lambda: boot.mod_raise(ct)); keep.append(g)
res["mod_raise"] = t
x = raised
for i, lt in enumerate(boot.cts):
    t, x, g = graph_time(lambda lt=lt, x=x: lt.apply(x, boot.keys)); keep.append(g)
    res[f"cts_group{i}_L{lt.level}_baby{len(lt.baby)}_giant{len(lt.giants)}"] = t


def split(x):
    conj = ckks.conjugate_fused(x, boot.keys)
    lo, hi = ckks.add(x, conj), ckks.sub(x, conj)
    return ckks.Ciphertext(lo.a, lo.b, boot.eval_scale), ckks.Ciphertext(hi.a, hi.b, boot.eval_scale)


t, (lo, hi), g = graph_time(lambda: split(x)); keep.append(g)
res["cts_conj_split"] = t
kappa = boot.q0 / (4.0 * math.pi * boot.delta_in) / 1j


def evalmod():
    m_lo, m_hi = eng.fork([lambda: boot.eval_mod(lo, boot.coef_lo, kappa),
                           lambda: boot.eval_mod(hi, boot.coef_hi, kappa * 1j)])
    return ckks.mod_drop(ckks.add(m_lo, m_hi), boot.lvl_stc)


t, w, g = graph_time(evalmod); keep.append(g)
res["eval_mod_both"] = t
t, _, g = graph_time(lambda: boot._exp_taylor(lo, boot.coef_lo)); keep.append(g)
res["  taylor_one_branch"] = t
x = w
for i, lt in enumerate(boot.stc):
    t, x, g = graph_time(lambda lt=lt, x=x: lt.apply(x, boot.keys)); keep.append(g)
    res[f"stc_group{i}_L{lt.level}_baby{len(lt.baby)}_giant{len(lt.giants)}"] = t
res["sum"] = sum(v for k, v in res.items() if not k.startswith("  "))
print(json.dumps({k: round(v, 3) for k, v in res.items()}, indent=1))
