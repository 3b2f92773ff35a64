"""Step-by-step diagnostics of the bootstrapping circuit at a small ring (debug aid)."""
import math
import sys
import time
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2512_18345_b200 import ckks, keyswitch as ks
from paper_2512_18345_b200.bootstrap import BootstrapConfig, Bootstrapper
from paper_2512_18345_b200.params import ParameterSet, generate_parameter_set

logn = int(sys.argv[1]) if len(sys.argv) > 1 else 11
N = 1 << logn
p = generate_parameter_set(n=N, l=36, dnum=3, delta=1 << 40, h_dense=32, h_sparse=32) if logn < 16 \
    else ParameterSet.builtin("ks48")
sk = ks.keygen(p, h=32, seed=1)
lanes = int(sys.argv[2]) if len(sys.argv) > 2 else 1
from paper_2512_18345_b200.engine import get_engine
get_engine().set_lanes(lanes)
print('lanes', lanes)
t0 = time.time()
boot = Bootstrapper(p, sk, BootstrapConfig())
print(f"setup {time.time() - t0:.1f}s  levels: cts {boot.lvl_cts} evalmod {boot.lvl_evalmod} stc {boot.lvl_stc} out {boot.out_level}",
      "rotation keys", len(boot.keys.galois))
rng = np.random.default_rng(0)
n = N // 2
z = rng.uniform(-1, 1, n) + 1j * rng.uniform(-1, 1, n)
ct = ckks.encrypt(ckks.encode(z, p, level=2, scale=boot.delta_in), sk, p, seed=5)
print("fresh err", np.abs(ckks.decrypt_decode(ct, sk, p) - z).max())

raised = boot.mod_raise(ct)
# decrypt the raised ciphertext: t = Delta*m + e + Q0*I
d = ckks.decrypt(ckks.mod_drop(raised, 4), sk)
from paper_2512_18345_b200.transform import ntt_polynomial
tco = ckks._centered_coeffs(ntt_polynomial(d.poly, "inverse"))
I = np.rint(tco / boot.q0)
print("ModRaise: max |I| =", np.abs(I).max(), " residual vs Delta*m:",
      np.abs((tco - I * boot.q0) / boot.delta_in - ckks.Embedding(N).to_coeffs(z)).max())

lo, hi = boot.coeff_to_slot(raised)
y_true = 2 * math.pi * tco / (boot.q0 * (1 << boot.cfg.squarings))
def bitrev_perm(n):
    lg = n.bit_length() - 1
    idx = np.arange(n); out = np.zeros(n, dtype=np.int64)
    for b in range(lg): out |= ((idx >> b) & 1) << (lg - 1 - b)
    return out
R = bitrev_perm(n)
got_lo = ckks.decrypt_decode(lo, sk, p)
got_hi = ckks.decrypt_decode(hi, sk, p)
print("CtS: err lo", np.abs(got_lo - y_true[:n][R]).max(), " err hi", np.abs(got_hi - 1j * y_true[n:][R]).max(),
      " max|y|", np.abs(y_true).max(), "level", ckks.level_of(lo))

kappa = boot.q0 / (4.0 * math.pi * boot.delta_in) / 1j
e = boot._exp_taylor(lo, boot.coef_lo)
print("Taylor: err", np.abs(ckks.decrypt_decode(e, sk, p) - np.exp(1j * y_true[:n][R])).max(), "level", ckks.level_of(e))
m_lo = boot.eval_mod(lo, boot.coef_lo, kappa)
m_true = ckks.Embedding(N).to_coeffs(z)
print("EvalMod lo: err", np.abs(ckks.decrypt_decode(m_lo, sk, p) - m_true[:n][R]).max(), "level", ckks.level_of(m_lo))
m_hi = boot.eval_mod(hi, boot.coef_hi, kappa * 1j)
print("EvalMod hi: err", np.abs(ckks.decrypt_decode(m_hi, sk, p) - 1j * m_true[n:][R]).max())
out = boot.slot_to_coeff(ckks.add(m_lo, m_hi))
out = ckks.Ciphertext(out.a, out.b, boot.out_scale)
err = np.abs(ckks.decrypt_decode(out, sk, p) - z).max()
print(f"bootstrap: level {ckks.level_of(out)}  max err {err:.3e} = 2^{math.log2(err):.2f}")
import torch
torch.cuda.synchronize(); t0 = time.time()
out2 = boot.bootstrap(ct); torch.cuda.synchronize()
print(f"bootstrap wall (eager, python-driven): {(time.time() - t0) * 1e3:.1f} ms")

# CUDA-graph replay
t0 = time.time()
replay = boot.capture(ct)
torch.cuda.synchronize()
print(f"capture {time.time() - t0:.1f}s")
out3 = replay(ct)
torch.cuda.synchronize()
print("graph == eager:", bool((out3.a.data == out2.a.data).all() and (out3.b.data == out2.b.data).all()))
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
for _ in range(3):
    replay(ct, copy_out=False)
a.record()
reps = 10
for _ in range(reps):
    replay(ct, copy_out=False)
b.record(); torch.cuda.synchronize()
print(f"bootstrap graph replay: {a.elapsed_time(b) / reps:.2f} ms")
# per-kernel time inside one eager bootstrap
import ctypes
from paper_2512_18345_b200.engine import get_engine
eng = get_engine()
eng.lib.ckks_profile_enable(1)
boot.bootstrap(ct)
buf = ctypes.create_string_buffer(1 << 16)
eng.lib.ckks_profile_read(buf, len(buf))
eng.lib.ckks_profile_enable(0)
tot = 0.0
rows = []
for line in buf.value.decode().splitlines():
    name, cnt, ms = line.split()[:3]
    rows.append((float(ms), name, int(cnt))); tot += float(ms)
for ms, name, cnt in sorted(rows, reverse=True):
    print(f"   {name:22s} {cnt:6d} launches {ms:8.3f} ms  {100 * ms / tot:5.1f}%")
print(f"   sum of kernel time {tot:.2f} ms over {sum(r[2] for r in rows)} launches")

# phase timing (eager, with lanes): CUDA events around each stage
def timed(fn):
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(); r = fn(); b.record(); torch.cuda.synchronize()
    return r, a.elapsed_time(b)
for _ in range(2):
    raised, t_raise = timed(lambda: boot.mod_raise(ct))
    (lo, hi), t_cts = timed(lambda: boot.coeff_to_slot(raised))
    (m_lo, m_hi), t_em = timed(lambda: eng.fork([lambda: boot.eval_mod(lo, boot.coef_lo, kappa),
                                                 lambda: boot.eval_mod(hi, boot.coef_hi, kappa * 1j)]))
    w = ckks.add(m_lo, m_hi)
    out, t_stc = timed(lambda: boot.slot_to_coeff(w))
print(f"phases (eager): mod_raise {t_raise:.2f}  coeff_to_slot {t_cts:.2f}  eval_mod {t_em:.2f}  slot_to_coeff {t_stc:.2f} ms")
for i, lt in enumerate(boot.cts + boot.stc):
    x = raised if i < 3 else w
    if ckks.level_of(x) != lt.level:
        x = ckks.mod_drop(x, lt.level) if ckks.level_of(x) > lt.level else None
    if x is None:
        continue
    _, t = timed(lambda: lt.apply(x, boot.keys))
    print(f"   LT {i}: level {lt.level} diags {sum(len(r) for r in lt.table.values())} baby {len(lt.baby)} giants {len(lt.giants)} step {lt.step}: {t:.2f} ms")

# phase timing under CUDA-graph replay
def graph_time(fn, reps=10):
    fn(); torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    side = torch.cuda.Stream()
    side.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(side):
        fn(); torch.cuda.synchronize()
        with torch.cuda.graph(g, stream=side):
            keep = fn()
    torch.cuda.current_stream().wait_stream(side)
    for _ in range(3):
        g.replay()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        g.replay()
    b.record(); torch.cuda.synchronize()
    return a.elapsed_time(b) / reps
raised = boot.mod_raise(ct)
lo, hi = boot.coeff_to_slot(raised)
t_cts = graph_time(lambda: boot.coeff_to_slot(raised))
t_em = graph_time(lambda: eng.fork([lambda: boot.eval_mod(lo, boot.coef_lo, kappa), lambda: boot.eval_mod(hi, boot.coef_hi, kappa * 1j)]))
m_lo, m_hi = eng.fork([lambda: boot.eval_mod(lo, boot.coef_lo, kappa), lambda: boot.eval_mod(hi, boot.coef_hi, kappa * 1j)])
w = ckks.add(m_lo, m_hi)
t_stc = graph_time(lambda: boot.slot_to_coeff(w))
t_one = graph_time(lambda: boot.eval_mod(lo, boot.coef_lo, kappa))
print(f"graph phases: coeff_to_slot {t_cts:.2f}  eval_mod(both) {t_em:.2f}  eval_mod(one branch) {t_one:.2f}  slot_to_coeff {t_stc:.2f} ms")
for i, lt in enumerate(boot.cts[:1] + boot.stc[:1]):
    x = raised if i == 0 else w
    print(f"   graph LT level {lt.level}: {graph_time(lambda: lt.apply(x, boot.keys)):.2f} ms")
sq_in = lo
print(f"   graph hmult+rescale at level {ckks.level_of(sq_in)}: {graph_time(lambda: boot._mul(sq_in, sq_in)):.3f} ms")
low = ckks.mod_drop(lo, 24)
print(f"   graph hmult+rescale at level 24: {graph_time(lambda: boot._mul(low, low)):.3f} ms")
