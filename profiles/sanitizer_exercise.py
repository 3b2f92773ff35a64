# small exercise of every hot kernel for compute-sanitizer: one ks48-shaped key switch at N=2^16 with 12 limbs (ks12),
# small-ring transforms, hoisted + batched ModDown paths, a short BSGS kernel
import sys
sys.path.insert(0, '/root/repo'); sys.path.insert(0, '/root/repo/tests/golden')
import numpy as np, torch
import recipes as R
from paper_2512_18345_b200 import keyswitch as ks, transform, rns, ckks
from paper_2512_18345_b200.engine import get_engine
from paper_2512_18345_b200.params import ParameterSet, generate_parameter_set
eng = get_engine(); eng.set_lanes(4)
p = ParameterSet.builtin("ks12")
s1, s2 = ks.keygen(p, seed=1), ks.keygen(p, seed=2)
msg = np.random.default_rng(0).integers(1, 9, p.n).astype(np.int64) * p.delta
ct = ks.encrypt(msg, s1, p, seed=3)
evk = ks.switching_keygen(s1, s2, p, seed=4)
out = ks.keyswitch(ct, evk)
dec = ks.decrypt(out, s2)
print("ks12 rel err", float((np.abs(dec - msg) / np.abs(msg)).max()))
# engine-level paths at N = 2^16
l = 12; q = p.q_basis[:l]; ext = l + p.alpha
plan = eng.ks_plan(p.n, q, p.p_basis, p.alpha, p.l + p.alpha, p.l)
raised = eng.ks_stage1(plan, ct.a.data, 1, ext)
m = evk.matrix()
raw = eng.ks_hoisted_raw(plan, raised, 5, m, ct.b.data, ext)
qps = torch.stack([raw, raw]).contiguous()
a_md = eng.ks_stage3_batch_a(plan, qps, l)
both = eng.ks_stage3_batch(plan, qps, l)
assert torch.equal(a_md[0], both[0][0])
eng.ks_accumulate_rot_qp(plan, a_md[0], qps[0][1], 25, m, True)
eng.ks_accumulate_rot_qp(plan, a_md[1], qps[1][1], 5, m, False)
fin = eng.ks_finish(plan, 1, None, None, l, p.n)
table = [[raw[0] * 0 + 1, None], [None, raw[0] * 0 + 2]]
bs = eng.bsgs_inner(plan, raised, ct.a.data, ct.b.data, [0, 5], [None, m], table, ext)
# late round 2: a pair through the batched baby-step kernel; both transform policies (single-pass cluster
# kernels at 2 and 3 CTAs per SM with their ModDown-epilogue and product-on-load variants, two-kernel split)
bsb = eng.bsgs_inner_batch(plan, [raised, raised], [ct.a.data, ct.a.data], [ct.b.data, ct.b.data], [0, 5], [None, m], table, ext)
assert torch.equal(bsb[0][0], bs[0]) and torch.equal(bsb[1][1], bs[1])
rlk16 = ckks.relin_keygen(s1, p, seed=9)
ct16 = ckks.Ciphertext(ct.a, ct.b, float(p.delta))
saved = eng.ntt_policy()
prods = []
for pol in ((1 << 20, 2), (1 << 20, 3), (0, 2)):
    eng.ntt_policy(*pol)
    prods.append(ckks.hmult_rescale(ct16, ct16, rlk16, 2))
    x = eng.ntt(ct.a.data, eng.row_slots(q, p.n), True)
    assert torch.equal(eng.ntt(x, eng.row_slots(q, p.n), False), ct.a.data)
assert all(torch.equal(pr.a.data, prods[0].a.data) and torch.equal(pr.b.data, prods[0].b.data) for pr in prods)
eng.ntt_policy(*saved)
# small-ring transform + config 1 product
p1 = generate_parameter_set(n=8192, l=12, dnum=3, delta=1 << 40, h_dense=64, h_sparse=32)
sk = ks.keygen(p1, seed=1); rlk = ckks.relin_keygen(sk, p1, seed=41)
c1 = ks.encrypt(msg[:p1.n] // p.delta * (1 << 20), sk, p1, seed=2)
prod = ckks.rescale(ckks.hmult(c1, c1, rlk), 1)
torch.cuda.synchronize()
print("sanitizer exercise done", int(fin.sum()), int(prod.a.data.sum()))
