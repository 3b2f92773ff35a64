import sys
sys.path.insert(0, '/root/repo')
import torch
from paper_2512_18345_b200 import ckks
from paper_2512_18345_b200.bootstrap import standard_input, standard_setup
from paper_2512_18345_b200.engine import get_engine
from paper_2512_18345_b200.params import ParameterSet
from paper_2512_18345_b200.rns import EVALUATION, Polynomial
eng = get_engine(); eng.set_lanes(8); dev = eng.device
p = ParameterSet.builtin("ks48")
sk, _s, boot = standard_setup(p)
z, ct = standard_input(p, boot, sk, 0)
replay = boot.capture(ct)
low = p.q_basis[:2]
ct_t = torch.stack([ct.a.data, ct.b.data])
host_in = [ct_t.cpu().pin_memory() for _ in range(2)]
host_out = [torch.empty(tuple(replay.static_out.shape), dtype=torch.int32).pin_memory() for _ in range(2)]
def mk(d): return ckks.Ciphertext(a=Polynomial(low, d[0], EVALUATION), b=Polynomial(low, d[1], EVALUATION), scale=boot.delta_in)
def v_graph_only(i): replay.graph.replay()
def v_value(i): replay.static_in.copy_(ct_t); replay.graph.replay()
def v_api(i): replay(mk(ct_t), copy_out=False)
def v_h2d(i): d = host_in[i % 2].to(dev, non_blocking=True); replay(mk(d), copy_out=False)
def v_d2h(i):
    out = replay(mk(ct_t), copy_out=False)
    host_out[i % 2][0].copy_(out.a.data, non_blocking=True); host_out[i % 2][1].copy_(out.b.data, non_blocking=True)
def v_d2h_one(i):
    replay(mk(ct_t), copy_out=False)
    host_out[i % 2].copy_(replay.static_out, non_blocking=True)
def v_full(i):
    d = host_in[i % 2].to(dev, non_blocking=True); out = replay(mk(d), copy_out=False)
    host_out[i % 2][0].copy_(out.a.data, non_blocking=True); host_out[i % 2][1].copy_(out.b.data, non_blocking=True)
for name, fn in [("graph only", v_graph_only), ("value loop", v_value), ("api, device ct", v_api), ("+h2d", v_h2d), ("+d2h (2 copies)", v_d2h), ("+d2h (1 copy)", v_d2h_one), ("full e2e", v_full), ("graph only", v_graph_only)]:
    for i in range(5): fn(i)
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for i in range(30): fn(i)
    b.record(); torch.cuda.synchronize()
    print(f"{name:18s} {a.elapsed_time(b) / 30:.3f} ms")
