"""Key switching below the top level (partial last digit, rows of the full-level key), hoisted
rotations and the ModDown merged with a rescale, against goldens the REFERENCE produced
(tests/golden/make_golden_level.py -> golden_level.json): its own keyswitch() at
l in {12, 24, 36, 48}, compositions of its public primitives elsewhere.

Each case runs twice through the same engine-level calls: on the CPU oracle engine
(oracle/engine_oracle.py, which every oracle bootstrap is built from) and, marked gpu, on the
CUDA engine through the C ABI.  Bit-exact (integer work)."""
import json
from pathlib import Path

import numpy as np
import pytest

import recipes as R

GOLD = json.loads((Path(__file__).resolve().parent / "golden" / "golden_level.json").read_text())
BACKENDS = ["oracle", pytest.param("cuda", marks=pytest.mark.gpu)]


@pytest.fixture(scope="module", params=BACKENDS)
def env(request):
    from paper_2512_18345_b200 import engine
    from paper_2512_18345_b200.params import ParameterSet

    previous = None
    if request.param == "oracle":
        from oracle.engine_oracle import OracleEngine

        previous = engine.use_backend(OracleEngine())
    else:
        import torch

        assert torch.cuda.is_available(), "GPU tests need a CUDA device"
    eng = engine.get_engine()
    p = ParameterSet.builtin("ks48")
    qs = [m.q for m in p.ext_basis]
    evk = np.stack([np.stack([R.level_key_rows(qs, p.n, t, h) for h in range(2)]) for t in range(p.dnum)])
    yield eng, p, eng.upload(evk.astype(np.uint32))
    if request.param == "oracle":
        engine.use_backend(previous)


def words(t):
    return t.cpu().numpy().view(np.uint32)


def ciphertext(eng, p, l):
    qs = [m.q for m in p.q_basis[:l]]
    return (eng.upload(R.rand_rows(qs, p.n, R.LEVEL_CT_SEEDS[0]).astype(np.uint32)),
            eng.upload(R.rand_rows(qs, p.n, R.LEVEL_CT_SEEDS[1]).astype(np.uint32)))


@pytest.mark.parametrize("l", R.LEVEL_FULL_DIGITS + R.LEVEL_PARTIAL)
def test_level_keyswitch_stages(env, l):
    eng, p, evk = env
    g = GOLD["level"][str(l)]
    q = p.q_basis[:l]
    beta, ext = -(-l // p.alpha), l + p.alpha
    plan = eng.ks_plan(p.n, q, p.p_basis, p.alpha, p.l + p.alpha, p.l)
    a, b = ciphertext(eng, p, l)
    raised = eng.ks_stage1(plan, a, beta, ext)
    assert [R.digest(words(raised[t])) for t in range(beta)] == g["stage1_raised"]
    acc = eng.ks_stage2(plan, raised, evk, 0, ext)
    assert R.digest(words(acc[0])) == g["stage2_acc_a"] and R.digest(words(acc[1])) == g["stage2_acc_b"]
    out = eng.keyswitch(plan, a, b, evk)
    assert R.digest(words(out[0])) == g["out_a"] and R.digest(words(out[1])) == g["out_b"]


@pytest.mark.parametrize("l,k", R.HOIST_CASES)
def test_hoisted_keyswitch(env, l, k):
    eng, p, evk = env
    g = GOLD["hoisted"][f"{l}_{k}"]
    q = p.q_basis[:l]
    beta, ext = -(-l // p.alpha), l + p.alpha
    kk = k % (2 * p.n)
    plan = eng.ks_plan(p.n, q, p.p_basis, p.alpha, p.l + p.alpha, p.l)
    a, b = ciphertext(eng, p, l)
    raised = eng.ks_stage1(plan, a, beta, ext)
    raw = eng.ks_hoisted_raw(plan, raised, kk, evk, b, ext)
    assert R.digest(words(raw[0])) == g["raw_a"] and R.digest(words(raw[1])) == g["raw_b"]
    out = eng.ks_hoisted(plan, raised, kk, evk, b)
    assert R.digest(words(out[0])) == g["out_a"] and R.digest(words(out[1])) == g["out_b"]


@pytest.mark.parametrize("l,k", R.MERGED_MODDOWN_CASES)
def test_moddown_merged_with_rescale(env, l, k):
    eng, p, _ = env
    g = GOLD["merged_moddown"][f"{l}_{k}"]
    q = p.q_basis[:l]
    rest, pp = q[:l - k], q[l - k:] + p.p_basis
    qs = [m.q for m in q + p.p_basis]
    xa = eng.upload(R.rand_rows(qs, p.n, R.MERGED_SEEDS[0]).astype(np.uint32))
    xb = eng.upload(R.rand_rows(qs, p.n, R.MERGED_SEEDS[1]).astype(np.uint32))
    md = eng.moddown_plan(p.n, rest, pp)
    out = eng.ks_stage3(md, xa[:l - k], xb[:l - k], xa[l - k:], xb[l - k:])
    assert R.digest(words(out[0])) == g["out_a"] and R.digest(words(out[1])) == g["out_b"]
