import sys
from pathlib import Path
import numpy as np, torch
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2512_18345_b200 import ckks, keyswitch as ks
from paper_2512_18345_b200.engine import get_engine
from paper_2512_18345_b200.params import generate_parameter_set

p = generate_parameter_set(n=2048, l=12, dnum=3, delta=1 << 40, h_dense=32, h_sparse=32)
eng = get_engine()
sk = ks.keygen(p, h=32, seed=1)
keys = ckks.EvaluationKeys(p)
keys.add_rotation(sk, 3, seed=5)
rng = np.random.default_rng(0)
n2 = p.n // 2
z = rng.uniform(-1, 1, n2) + 1j * rng.uniform(-1, 1, n2)
scale = float(p.q_basis[-1].q) * float(p.q_basis[-2].q)
ct = ckks.encrypt(ckks.encode(z, p, scale=scale), sk, p, seed=3)
level = p.l; alpha = p.alpha; ext = level + alpha
plan = eng.ks_plan(p.n, ct.a.basis, p.p_basis, alpha, p.l + alpha, p.l)
raised = eng.ks_stage1(plan, ct.a.data, -(-level // alpha), ext)
k = ckks.galois_element(3, p.n)
evk = keys.galois[k].matrix()
ref = eng.ks_hoisted(plan, raised, k, evk, ct.b.data)
got = ckks.decrypt_decode(ckks.ct_from_tensor(ref, ct.a.basis, ct.scale), sk, p)
print("ks_hoisted err", np.abs(got - np.roll(z, -3)).max())
qp = eng.ks_hoisted_raw(plan, raised, k, evk, ct.b.data, ext)
md = eng.ks_stage3(plan, qp[0, :level], qp[1, :level], qp[0, level:], qp[1, level:])
got = ckks.decrypt_decode(ckks.ct_from_tensor(md, ct.a.basis, ct.scale), sk, p)
print("raw + ModDown err", np.abs(got - np.roll(z, -3)).max())
print("limb diff a", int((md[0] != ref[0]).sum()), "b", int((md[1] != ref[1]).sum()), "max abs diff", int((md.to(torch.int64) - ref.to(torch.int64)).abs().max()))
# pmult in QP then ModDown == pmult after ModDown
w = rng.uniform(-1, 1, n2)
ext_basis = ct.a.basis + p.p_basis
pt_ext = ckks.encode(w, p, scale=scale, basis=ext_basis)
ext_slots = eng.row_slots(ext_basis)
prod = eng.fused_terms([qp], [pt_ext.poly.data], ext_slots)
md2 = eng.ks_stage3(plan, prod[0, :level], prod[1, :level], prod[0, level:], prod[1, level:])
res = ckks.rescale(ckks.ct_from_tensor(md2, ct.a.basis, ct.scale * scale), 2)
got = ckks.decrypt_decode(res, sk, p)
print("QP pmult err", np.abs(got - np.roll(z, -3) * w).max())
# unrotated term lifted to QP
import math
pp = math.prod(m.q for m in p.p_basis)
lift = [pp % m.q for m in ct.a.basis] + [0] * alpha
pt0 = ckks.encode(w, p, scale=scale, basis=ext_basis, row_factors=lift)
x = ckks.ct_tensor(ct)
x_ext = torch.cat([x, torch.zeros((2, alpha, p.n), dtype=x.dtype, device=x.device)], dim=1)
prod = eng.fused_terms([x_ext], [pt0.poly.data], ext_slots)
md3 = eng.ks_stage3(plan, prod[0, :level], prod[1, :level], prod[0, level:], prod[1, level:])
res = ckks.rescale(ckks.ct_from_tensor(md3, ct.a.basis, ct.scale * scale), 2)
print("lifted identity term err", np.abs(ckks.decrypt_decode(res, sk, p) - z * w).max())

# whole linear transform, double-hoisted vs single-hoisted vs plaintext
from paper_2512_18345_b200.bootstrap import LinearTransform, apply_diagonals
for offsets, n1 in (([0], 4), ([1], 4), ([0, 1], 4), ([1, 2], 4), ([0, 1, 2, 3], 4)):
    diags = {d: rng.uniform(-1, 1, n2) + 1j * rng.uniform(-1, 1, n2) for d in offsets}
    want = apply_diagonals(diags, z)
    for dh in (False, True):
        lt = LinearTransform(diags, p, level, n1=n1, limbs=2, double_hoist=dh)
        kk = ckks.EvaluationKeys(p)
        for r in lt.rotations():
            kk.add_rotation(sk, r, seed=100 + r)
        out = lt.apply(ct, kk)
        err = np.abs(ckks.decrypt_decode(out, sk, p) - want).max()
        print(f"LT offsets {offsets} n1={n1} double_hoist={dh}: baby {lt.baby} giants {lt.giants} step {lt.step} err {err:.3e}")
