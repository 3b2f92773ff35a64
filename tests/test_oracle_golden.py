"""Pin the CPU oracle (oracle/) against outputs of the real reference package
recorded in tests/golden/golden.json (generator: tests/golden/make_golden.py).
CPU only.  The ks48 cases are the largest and take a few seconds each."""
import numpy as np
import pytest

import recipes as R


def _params(oracle_mod, golden, name):
    return oracle_mod.params_from_dict(golden["params"][name])


def _qs(basis):
    return [q for q, _ in basis]


@pytest.fixture(scope="module")
def ctxs(oracle_mod, golden):
    cache = {}

    def get(name):
        if name not in cache:
            p = _params(oracle_mod, golden, name)
            cache[name] = (p, oracle_mod.Oracle(p.n, p.ext_basis))
        return cache[name]

    return get


def test_small_vectors_q17(oracle_mod, golden):
    g = golden["small"]["q17_n4"]
    orc = oracle_mod.Oracle(4, [(17, g["psi"])])
    fwd, inv, n_inv = orc.twiddles(0)
    assert fwd.tolist() == g["fwd"] and inv.tolist() == g["inv"] and n_inv == g["n_inv"]
    rm = np.zeros(1, np.int32)
    assert orc.ntt(np.array([[1, 0, 0, 0]]), rm)[0].tolist() == g["ntt_delta"]
    assert orc.ntt(np.array([[1, 2, 3, 4]]), rm)[0].tolist() == g["ntt_1234"]
    assert orc.ntt(np.array([[1, 2, 3, 4]]), rm, inverse=True)[0].tolist() == g["intt_1234"]


def test_small_vectors_q97_and_otf(oracle_mod, golden):
    g = golden["small"]["q97_n16"]
    orc = oracle_mod.Oracle(16, [(97, g["psi"])])
    fwd, inv, n_inv = orc.twiddles(0)
    assert fwd.tolist() == g["fwd"] and inv.tolist() == g["inv"] and n_inv == g["n_inv"]
    x = np.array([g["x"]])
    rm = np.zeros(1, np.int32)
    assert orc.ntt(x, rm)[0].tolist() == g["ntt"]
    assert orc.ntt(x, rm, inverse=True)[0].tolist() == g["intt"]
    assert [orc.otf_twiddle(0, t) for t in range(16)] == g["otf_fwd"]
    assert [orc.otf_twiddle(0, t) for t in range(16)] == g["fwd"]
    for n1 in (2, 4, 8, 16):
        assert orc.ntt_two_phase(x, rm, n1=n1)[0].tolist() == g["ntt"]
        assert orc.ntt_two_phase(x, rm, inverse=True, n1=n1)[0].tolist() == g["intt"]


def test_prime_and_root_search(oracle_mod, golden):
    for key, want in golden["small"]["primes"].items():
        cnt, bits, n = (int(v) for v in key.split("_"))
        assert [list(m) for m in oracle_mod.find_ntt_primes(cnt, bits, n)] == want
    for name in ("tiny", "n8192"):
        kw = R.PARAM_SETS[name][1]
        p = oracle_mod.generate_parameter_set(**kw)
        assert [list(m) for m in p.q_basis] == golden["params"][name]["q_basis"]
        assert [list(m) for m in p.p_basis] == golden["params"][name]["p_basis"]


def test_bconv_worked_example(oracle_mod, golden):
    g = golden["small"]["bconv_5_7_11"]
    t, inv = oracle_mod.bconv_table([5, 7], [11])
    assert t.tolist() == g["t"] and inv.tolist() == g["inv_qhat"]
    assert oracle_mod.bconv([5, 7], [11], np.array(g["in"])).tolist() == g["out"]


@pytest.mark.parametrize("name", ["tiny", "n8192", "verify_small", "ks12", "ks24", "ks48"])
def test_twiddles_and_ntt(ctxs, golden, name):
    p, orc = ctxs(name)
    ext = p.ext_basis
    g = golden["twiddle"][name]
    tabs = [orc.twiddles(i) for i in range(len(ext))]
    assert R.digest(np.stack([t[0] for t in tabs])) == g["fwd"]
    assert R.digest(np.stack([t[1] for t in tabs])) == g["inv"]
    assert [t[2] for t in tabs] == g["n_inv"]
    x = R.rand_rows(_qs(ext), p.n, golden["ntt"][name]["seed"])
    assert R.digest(x) == golden["ntt"][name]["in"]
    rm = orc.idx(ext)
    fwd = orc.ntt(x, rm)
    assert R.digest(fwd) == golden["ntt"][name]["fwd"]
    assert R.digest(orc.ntt(x, rm, inverse=True)) == golden["ntt"][name]["inv"]
    if p.n <= 8192:
        assert R.digest(orc.ntt_two_phase(x, rm)) == golden["ntt"][name]["fwd"]
        assert np.array_equal(orc.ntt(fwd, rm, inverse=True), x)


@pytest.mark.parametrize("n", [2, 4, 8, 16, 32, 64, 128, 256, 512, 1024, 2048])
def test_ntt_small_degrees(oracle_mod, golden, n):
    g = golden["ntt"][f"n{n}"]
    mods = [tuple(m) for m in g["moduli"]]
    orc = oracle_mod.Oracle(n, mods)
    x = R.rand_rows(_qs(mods), n, g["seed"])
    rm = np.arange(len(mods), dtype=np.int32)
    assert R.digest(orc.ntt(x, rm)) == g["fwd"]
    assert R.digest(orc.ntt(x, rm, inverse=True)) == g["inv"]


@pytest.mark.parametrize("name", ["tiny", "n8192", "verify_small", "ks12", "ks24", "ks48"])
def test_bconv_tables_and_conversion(oracle_mod, ctxs, golden, name):
    p, _ = ctxs(name)
    g = golden["bconv"][name]
    qall = _qs(p.q_basis)
    for t in range(p.dnum):
        digit = qall[t * p.alpha:(t + 1) * p.alpha]
        target = [q for i, q in enumerate(qall) if i // p.alpha != t] + _qs(p.p_basis)
        tab, inv = oracle_mod.bconv_table(digit, target)
        assert R.digest(tab) == g["raise"][t]["t"]
        assert R.digest(inv) == g["raise"][t]["inv_qhat"]
        x = R.rand_rows(digit, p.n, g["raise"][t]["seed"])
        assert R.digest(oracle_mod.bconv(digit, target, x)) == g["raise"][t]["out"]
    x = R.rand_rows(_qs(p.p_basis), p.n, g["moddown"]["seed"])
    assert R.digest(oracle_mod.bconv(_qs(p.p_basis), qall, x)) == g["moddown"]["out"]
    assert R.digest(oracle_mod.gadget(p)) == g["gadget"]


def test_bconv_worst_case_accumulator(oracle_mod, ctxs, golden):
    p, _ = ctxs("ks48")
    qall = _qs(p.q_basis)
    digit = qall[:p.alpha]
    target = qall[p.alpha:] + _qs(p.p_basis)
    x = np.stack([np.full(64, q - 1, dtype=np.uint64) for q in digit])
    assert R.digest(oracle_mod.bconv(digit, target, x)) == golden["bconv"]["ks48_maxres"]["out"]


@pytest.mark.parametrize("name", ["tiny", "verify_small", "n8192", "ks48"])
def test_automorphism_and_elementwise(ctxs, golden, name):
    p, orc = ctxs(name)
    g = golden["automorphism"][name]
    rm = orc.idx(p.q_basis)
    x = R.rand_rows(_qs(p.q_basis), p.n, g["seed"])
    for k in R.AUTOMORPHISM_KS:
        assert R.digest(orc.automorphism_coeff(x, rm, k)) == g["k"][str(k)]["coeff"]
        assert R.digest(orc.automorphism_eval(x, k)) == g["k"][str(k)]["eval"]
    ge = golden["elementwise"][name]
    y = R.rand_rows(_qs(p.q_basis), p.n, ge["seeds"][1])
    for kind in ("add", "sub", "mul"):
        assert R.digest(orc.elementwise(x, y, rm, kind)) == ge[kind]


@pytest.mark.parametrize("case", ["tiny", "verify_small", "n8192", "ks48"])
def test_keyswitch_pipeline(oracle_mod, ctxs, golden, case):
    g = golden["keyswitch"][case]
    p, orc = ctxs(g["params"])
    s1, s2, mseed, cseed, eseed = g["seeds"]
    s_from = oracle_mod.keygen(p.n, p.h_dense, s1)
    s_to = oracle_mod.keygen(p.n, p.h_dense, s2)
    assert R.digest_i64(s_from) == g["s_from"] and R.digest_i64(s_to) == g["s_to"]
    msg = R.message(p.n, p.delta, mseed)
    assert R.digest_i64(msg) == g["msg"]
    a, b = oracle_mod.encrypt(orc, p, msg, s_from, cseed)
    assert R.digest(a) == g["ct_a"] and R.digest(b) == g["ct_b"]
    evk = oracle_mod.switching_keygen(orc, p, s_from, s_to, eseed)
    assert [[R.digest(evk[t, 0]), R.digest(evk[t, 1])] for t in range(p.dnum)] == g["evk"]
    out_a, out_b, raised, acc = orc.keyswitch(p, a, b, evk, dumps=True)
    assert [R.digest(raised[t]) for t in range(p.dnum)] == g["stage1_raised"]
    assert R.digest(acc[0, :p.l]) == g["stage2_acc_q_a"]
    assert R.digest(acc[1, :p.l]) == g["stage2_acc_q_b"]
    assert R.digest(acc[0, p.l:]) == g["stage2_acc_p_a"]
    assert R.digest(acc[1, p.l:]) == g["stage2_acc_p_b"]
    assert R.digest(out_a) == g["out_a"] and R.digest(out_b) == g["out_b"]
    # stage-level entry points agree with the fused call
    assert np.array_equal(orc.ks_stage1(p, a), raised)
    pa, pb = orc.ks_stage2(p, raised, evk, rows=(p.l, p.l + p.alpha))
    assert np.array_equal(pa, acc[0, p.l:]) and np.array_equal(pb, acc[1, p.l:])
    d_a = orc.ks_moddown(p, acc[0, :p.l], acc[0, p.l:])
    assert R.digest(d_a) == g["stage3_out_a"]
    assert R.digest(orc.ks_moddown(p, acc[1, :p.l], acc[1, p.l:])) == g["stage3_out_b"]
    if p.n <= 8192:
        dec = oracle_mod.decrypt(orc, p.q_basis, out_a, out_b, s_to)
        assert R.digest_i64(np.array(dec, dtype=np.int64)) == g["decrypt_switched"]
        assert int(np.abs(np.array(dec, dtype=np.int64) - msg).max()) == g["max_abs_err_switched"]
