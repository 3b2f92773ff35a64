"""Parity of the CUDA path (through the rnscope-compatible Python API, i.e.
through the C ABI) against (1) golden vectors recorded from the real reference
and (2) the CPU oracle on the same seeded inputs.  Bit-exact everywhere: all
work on this path is integer."""
import itertools

import numpy as np
import pytest

import recipes as R

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def pk():
    import torch

    assert torch.cuda.is_available(), "GPU tests need a CUDA device"
    from paper_2512_18345_b200 import baseconv, keyswitch, params, rns, transform, vectors

    class NS:
        pass

    ns = NS()
    ns.baseconv, ns.ks, ns.params, ns.rns, ns.transform, ns.vectors = (
        baseconv, keyswitch, params, rns, transform, vectors)
    return ns


@pytest.fixture(scope="module")
def psets(pk, golden):
    cache = {}

    def get(name):
        if name not in cache:
            cache[name] = pk.params.ParameterSet.from_dict(golden["params"][name])
        return cache[name]

    return get


def qs(basis):
    return [m.q for m in basis]


# ---------------------------------------------------------------- transforms
def test_exhaustive_identity_n4_q17(pk, golden):
    g = golden["small"]["q17_n4"]
    m = pk.rns.Modulus.for_prime(17, 4)
    assert m.psi == g["psi"]
    table = pk.transform.build_twiddle_table(m, 4)
    assert table.fwd.tolist() == g["fwd"] and table.inv.tolist() == g["inv"] and table.n_inv == g["n_inv"]
    rows = np.array(list(itertools.product(range(17), repeat=4)), dtype=np.uint64)
    fwd = pk.transform.ntt(rows, m, table)
    assert np.array_equal(pk.transform.ntt(fwd, m, table, direction="inverse"), rows)
    assert pk.transform.ntt(np.array([1, 0, 0, 0], dtype=np.uint64), m, table).tolist() == g["ntt_delta"]
    assert pk.transform.ntt(np.array([1, 2, 3, 4], dtype=np.uint64), m, table).tolist() == g["ntt_1234"]
    assert pk.transform.ntt(np.array([1, 2, 3, 4], dtype=np.uint64), m, table,
                            direction="inverse").tolist() == g["intt_1234"]
    assert table.dump_text().splitlines()[0] == "# twiddles q=17 n=4 n1=2"


def test_q97_two_phase_and_otf(pk, golden):
    g = golden["small"]["q97_n16"]
    m = pk.rns.Modulus.for_prime(97, 16)
    table = pk.transform.build_twiddle_table(m, 16)
    assert table.fwd.tolist() == g["fwd"] and table.inv.tolist() == g["inv"]
    x = np.array(g["x"], dtype=np.uint64)
    assert pk.transform.ntt(x, m, table).tolist() == g["ntt"]
    assert pk.transform.ntt(x, m, table, direction="inverse").tolist() == g["intt"]
    block = table.seed_block
    assert [pk.transform.generate_twiddle(table, t // block, t % block, m) for t in range(16)] == g["otf_fwd"]
    p = pk.rns.Polynomial((m,), x[None, :], pk.rns.COEFFICIENT)
    for n1 in (2, 4, 8, 16):
        for otf in (False, True):
            two = pk.transform.ntt_two_phase(p, n1=n1, on_the_fly=otf)
            assert two.coeffs[0].tolist() == g["ntt"]
            back = pk.transform.ntt_two_phase(two, "inverse", n1=n1, on_the_fly=otf)
            assert np.array_equal(back.coeffs, p.coeffs)


@pytest.mark.parametrize("n", [2, 4, 8, 16, 32, 64, 128, 256, 512, 1024, 2048])
def test_ntt_small_degrees(pk, golden, n):
    g = golden["ntt"][f"n{n}"]
    mods = tuple(pk.rns.Modulus.for_prime(q, n, psi) for q, psi in g["moduli"])
    x = R.rand_rows(qs(mods), n, g["seed"])
    fwd = pk.transform.ntt_polynomial(pk.rns.Polynomial(mods, x, pk.rns.COEFFICIENT))
    inv = pk.transform.ntt_polynomial(pk.rns.Polynomial(mods, x, pk.rns.EVALUATION), "inverse")
    assert R.digest(fwd.coeffs) == g["fwd"]
    assert R.digest(inv.coeffs) == g["inv"]


@pytest.mark.parametrize("name", ["tiny", "n8192", "verify_small", "ks12", "ks24", "ks48"])
def test_ntt_parameter_sets(pk, psets, golden, name):
    p = psets(name)
    ext = p.ext_basis
    g = golden["ntt"][name]
    x = R.rand_rows(qs(ext), p.n, g["seed"])
    poly = pk.rns.Polynomial(ext, x, pk.rns.COEFFICIENT)
    fwd = pk.transform.ntt_polynomial(poly)
    assert R.digest(fwd.coeffs) == g["fwd"]
    inv = pk.transform.ntt_polynomial(pk.rns.Polynomial(ext, x, pk.rns.EVALUATION), "inverse")
    assert R.digest(inv.coeffs) == g["inv"]
    assert np.array_equal(pk.transform.ntt_polynomial(fwd, "inverse").coeffs, poly.coeffs)
    two = pk.transform.ntt_two_phase(poly)
    assert R.digest(two.coeffs) == g["fwd"]
    assert np.array_equal(pk.transform.ntt_two_phase(two, "inverse").coeffs, poly.coeffs)
    # twiddle tables the kernels read == the reference's tables
    gt = golden["twiddle"][name]
    tabs = [pk.transform.twiddle_table(m, p.n) for m in ext]
    assert R.digest(np.stack([t.fwd for t in tabs])) == gt["fwd"]
    assert R.digest(np.stack([t.inv for t in tabs])) == gt["inv"]
    assert [t.n_inv for t in tabs] == gt["n_inv"]


def test_ntt_matches_oracle_and_linearity_at_2_16(pk, psets, oracle_mod):
    p = psets("ks48")
    ext = p.ext_basis
    orc = oracle_mod.Oracle(p.n, [(m.q, m.psi) for m in ext])
    rng = np.random.default_rng(20240831)
    x = np.stack([rng.integers(0, m.q, p.n, dtype=np.uint64) for m in ext])
    y = np.stack([rng.integers(0, m.q, p.n, dtype=np.uint64) for m in ext])
    # edge rows: all zero, all q-1, delta
    x[0] = 0
    x[1] = ext[1].q - 1
    x[2] = 0
    x[2, 0] = 1
    fx = pk.transform.ntt_polynomial(pk.rns.Polynomial(ext, x, pk.rns.COEFFICIENT)).coeffs
    rm = np.arange(len(ext), dtype=np.int32)
    assert np.array_equal(fx, orc.ntt(x, rm))
    assert not fx[0].any() and np.all(fx[2] == 1)
    ix = pk.transform.ntt_polynomial(pk.rns.Polynomial(ext, x, pk.rns.EVALUATION), "inverse").coeffs
    assert np.array_equal(ix, orc.ntt(x, rm, inverse=True))
    q_col = np.array(qs(ext), dtype=np.uint64)[:, None]
    fy = pk.transform.ntt_polynomial(pk.rns.Polynomial(ext, y, pk.rns.COEFFICIENT)).coeffs
    fxy = pk.transform.ntt_polynomial(pk.rns.Polynomial(ext, (x + y) % q_col, pk.rns.COEFFICIENT)).coeffs
    assert np.array_equal(fxy, (fx + fy) % q_col)


def test_negative_control_corrupted_input_fails(pk, psets, golden):
    """A single flipped residue must change the digest (the harness can fail)."""
    p = psets("verify_small")
    x = R.rand_rows(qs(p.ext_basis), p.n, golden["ntt"]["verify_small"]["seed"])
    x[3, 17] ^= 1
    fwd = pk.transform.ntt_polynomial(pk.rns.Polynomial(p.ext_basis, x, pk.rns.COEFFICIENT))
    assert R.digest(fwd.coeffs) != golden["ntt"]["verify_small"]["fwd"]


def test_transform_errors(pk):
    m = pk.rns.Modulus.for_prime(17, 4)
    t = pk.transform.build_twiddle_table(m, 4)
    with pytest.raises(pk.rns.StructureError):
        pk.transform.ntt(np.zeros(8, dtype=np.uint64), m, t)
    p = pk.rns.Polynomial((m,), np.zeros((1, 4)), pk.rns.EVALUATION)
    with pytest.raises(pk.rns.StructureError):
        pk.transform.ntt_polynomial(p)
    with pytest.raises(ValueError):
        pk.transform.ntt_two_phase(pk.rns.Polynomial((m,), np.zeros((1, 4)), pk.rns.COEFFICIENT), n1=3)
    with pytest.raises(ValueError):
        pk.transform.generate_twiddle(t, 99, 0, m)


# ---------------------------------------------------------------- base conversion
def test_bconv_worked_example(pk, golden):
    g = golden["small"]["bconv_5_7_11"]
    M = pk.rns.Modulus.for_prime
    q5, q7, p11 = M(5, 1), M(7, 1), M(11, 1)
    table = pk.baseconv.build_bconv_table((q5, q7), (p11,))
    assert table.t.tolist() == g["t"] and table.inv_qhat.tolist() == g["inv_qhat"]
    assert table.overflow_free
    a = pk.rns.Polynomial((q5, q7), np.array(g["in"], dtype=np.uint64), pk.rns.COEFFICIENT)
    assert pk.baseconv.bconv(a, table).coeffs.tolist() == g["out"]
    one = pk.baseconv.build_bconv_table((q5,), (p11,))
    assert one.t.tolist() == [[1]] and one.inv_qhat.tolist() == [1]
    ident = pk.rns.Polynomial((q5,), np.array([[0, 1, 2, 3, 4]], dtype=np.uint64), pk.rns.COEFFICIENT)
    assert pk.baseconv.bconv_with_intermediate_reduction(ident, one).coeffs.tolist() == [[0, 1, 2, 3, 4]]
    with pytest.raises(pk.rns.StructureError):
        pk.baseconv.build_bconv_table((q5, q7), (q7,))
    with pytest.raises(pk.rns.StructureError):
        pk.baseconv.build_bconv_table((q5, q5), (p11,))
    with pytest.raises(pk.rns.StructureError):
        pk.baseconv.bconv(pk.rns.Polynomial((q5, q7), np.array(g["in"]), pk.rns.EVALUATION), table)


@pytest.mark.parametrize("name", ["tiny", "n8192", "verify_small", "ks12", "ks24", "ks48"])
def test_bconv_parameter_sets(pk, psets, golden, name):
    p = psets(name)
    g = golden["bconv"][name]
    tabs = pk.ks._tables(p)
    for t in range(p.dnum):
        digit = p.q_basis[p.digit_slice(t)]
        table = tabs.raise_tables[t]
        assert R.digest(table.t) == g["raise"][t]["t"]
        assert R.digest(table.inv_qhat) == g["raise"][t]["inv_qhat"]
        assert table.overflow_free == g["raise"][t]["overflow_free"]
        x = R.rand_rows(qs(digit), p.n, g["raise"][t]["seed"])
        out = pk.baseconv.convert(pk.rns.Polynomial(digit, x, pk.rns.COEFFICIENT), table)
        assert R.digest(out.coeffs) == g["raise"][t]["out"]
    x = R.rand_rows(qs(p.p_basis), p.n, g["moddown"]["seed"])
    out = pk.baseconv.convert(pk.rns.Polynomial(p.p_basis, x, pk.rns.COEFFICIENT), tabs.moddown_table)
    assert R.digest(out.coeffs) == g["moddown"]["out"]
    assert tabs.moddown_table.overflow_free == g["moddown"]["overflow_free"]
    assert [int(v) for v in tabs.p_inv_col.ravel()] == g["moddown"]["p_inv"]
    assert R.digest(tabs.gadget) == g["gadget"]


def test_bconv_worst_case_and_ragged_columns(pk, psets, golden, oracle_mod):
    p = psets("ks48")
    digit = p.q_basis[p.digit_slice(0)]
    table = pk.ks._tables(p).raise_tables[0]
    assert not table.overflow_free
    x = np.stack([np.full(64, m.q - 1, dtype=np.uint64) for m in digit])
    poly = pk.rns.Polynomial(digit, x, pk.rns.COEFFICIENT)
    with pytest.raises(pk.baseconv.OverflowUnsafeError):
        pk.baseconv.bconv(poly, table)
    assert R.digest(pk.baseconv.convert(poly, table).coeffs) == golden["bconv"]["ks48_maxres"]["out"]
    # column counts that are not a multiple of anything
    rng = np.random.default_rng(3)
    for cols in (1, 3, 257, 1000):
        x = np.stack([rng.integers(0, m.q, cols, dtype=np.uint64) for m in digit])
        got = pk.baseconv.convert(pk.rns.Polynomial(digit, x, pk.rns.COEFFICIENT), table).coeffs
        want = oracle_mod.bconv(qs(digit), qs(table.p_basis), x)
        assert np.array_equal(got, want)


def test_bconv_overflow_free_search_and_fast_path(pk, oracle_mod):
    qb, pb = pk.baseconv.search_overflow_free_moduli(6, 8, 1 << 10, 31)
    table = pk.baseconv.build_bconv_table(qb, pb)
    assert table.overflow_free
    rng = np.random.default_rng(20240831)
    x = np.stack([rng.integers(0, m.q, 10_000, dtype=np.uint64) for m in qb])
    a = pk.rns.Polynomial(qb, x, pk.rns.COEFFICIENT)
    fast = pk.baseconv.bconv(a, table)
    slow = pk.baseconv.bconv_with_intermediate_reduction(a, table)
    assert np.array_equal(fast.coeffs, slow.coeffs)
    assert np.array_equal(fast.coeffs, oracle_mod.bconv(qs(qb), qs(pb), x))


# ---------------------------------------------------------------- automorphism / element-wise
@pytest.mark.parametrize("name", ["tiny", "verify_small", "n8192", "ks48"])
def test_automorphism_and_elementwise(pk, psets, golden, name):
    p = psets(name)
    g = golden["automorphism"][name]
    x = R.rand_rows(qs(p.q_basis), p.n, g["seed"])
    pc = pk.rns.Polynomial(p.q_basis, x, pk.rns.COEFFICIENT)
    pe = pk.rns.Polynomial(p.q_basis, x, pk.rns.EVALUATION)
    for k in R.AUTOMORPHISM_KS:
        assert R.digest(pk.rns.automorphism(pc, k).coeffs) == g["k"][str(k)]["coeff"]
        assert R.digest(pk.rns.automorphism(pe, k).coeffs) == g["k"][str(k)]["eval"]
    ge = golden["elementwise"][name]
    y = pk.rns.Polynomial(p.q_basis, R.rand_rows(qs(p.q_basis), p.n, ge["seeds"][1]), pk.rns.EVALUATION)
    for kind in ("add", "sub", "mul"):
        assert R.digest(pk.rns.poly_elementwise(pe, y, kind).coeffs) == ge[kind]


def test_automorphism_properties(pk, psets):
    p = psets("verify_small")
    rng = np.random.default_rng(5)
    x = pk.rns.random_polynomial(p.q_basis, p.n, rng, pk.rns.EVALUATION)
    two_n = 2 * p.n
    k1, k2 = 5, 3
    lhs = pk.rns.automorphism(pk.rns.automorphism(x, k1), k2)
    rhs = pk.rns.automorphism(x, (k1 * k2) % two_n)
    assert np.array_equal(lhs.coeffs, rhs.coeffs)
    back = pk.rns.automorphism(pk.rns.automorphism(x, 5), pow(5, -1, two_n))
    assert np.array_equal(back.coeffs, x.coeffs)
    # evaluation-domain route == coefficient-domain route
    xc = pk.transform.ntt_polynomial(x, "inverse")
    via_coeff = pk.transform.ntt_polynomial(pk.rns.automorphism(xc, 5))
    assert np.array_equal(via_coeff.coeffs, pk.rns.automorphism(x, 5).coeffs)
    with pytest.raises(ValueError):
        pk.rns.automorphism(x, 4)
    with pytest.raises(pk.rns.StructureError):
        pk.rns.poly_elementwise(x, xc, "add")
    with pytest.raises(pk.rns.StructureError):
        pk.rns.poly_elementwise(xc, xc, "mul")
    with pytest.raises(ValueError):
        pk.rns.poly_elementwise(x, x, "div")


def test_elementwise_small_and_32bit_moduli(pk):
    M = pk.rns.Modulus.for_prime
    basis = (M(17, 4), M(97, 16), M(4294967291, 1), M(2147483137, 64))
    rng = np.random.default_rng(1)
    a = np.stack([rng.integers(0, m.q, 37, dtype=np.uint64) for m in basis])
    b = np.stack([rng.integers(0, m.q, 37, dtype=np.uint64) for m in basis])
    a[:, 0] = [m.q - 1 for m in basis]
    b[:, 0] = [m.q - 1 for m in basis]
    q = np.array(qs(basis), dtype=object)[:, None]
    pa = pk.rns.Polynomial(basis, a, pk.rns.EVALUATION)
    pb = pk.rns.Polynomial(basis, b, pk.rns.EVALUATION)
    ao, bo = a.astype(object), b.astype(object)
    assert np.array_equal(pk.rns.poly_elementwise(pa, pb, "add").coeffs.astype(object), (ao + bo) % q)
    assert np.array_equal(pk.rns.poly_elementwise(pa, pb, "sub").coeffs.astype(object), (ao - bo) % q)
    assert np.array_equal(pk.rns.poly_elementwise(pa, pb, "mul").coeffs.astype(object), (ao * bo) % q)


# ---------------------------------------------------------------- key switching
@pytest.mark.parametrize("case", ["tiny", "verify_small", "n8192", "ks48"])
def test_keyswitch_pipeline_golden(pk, psets, golden, case):
    g = golden["keyswitch"][case]
    p = psets(g["params"])
    s1, s2, mseed, cseed, eseed = g["seeds"]
    s_from, s_to = pk.ks.keygen(p, seed=s1), pk.ks.keygen(p, seed=s2)
    assert R.digest_i64(s_from.ternary) == g["s_from"] and R.digest_i64(s_to.ternary) == g["s_to"]
    msg = R.message(p.n, p.delta, mseed)
    ct = pk.ks.encrypt(msg, s_from, p, seed=cseed)
    assert R.digest(ct.a.coeffs) == g["ct_a"] and R.digest(ct.b.coeffs) == g["ct_b"]
    evk = pk.ks.switching_keygen(s_from, s_to, p, seed=eseed)
    assert evk.shape == (2 * p.dnum, p.l + p.alpha)
    assert [[R.digest(pr.a.coeffs), R.digest(pr.b.coeffs)] for pr in evk.pairs] == g["evk"]
    raised = pk.ks.keyswitch_stage1(ct.a, p)
    assert [R.digest(r.coeffs) for r in raised] == g["stage1_raised"]
    for t, r in enumerate(raised):                       # carried limbs equal the input
        sl = p.digit_slice(t)
        assert np.array_equal(r.coeffs[sl], ct.a.coeffs[sl])
    q_part, p_part = pk.ks.keyswitch_stage2(raised, evk)
    assert R.digest(q_part.a.coeffs) == g["stage2_acc_q_a"]
    assert R.digest(q_part.b.coeffs) == g["stage2_acc_q_b"]
    assert R.digest(p_part.a.coeffs) == g["stage2_acc_p_a"]
    assert R.digest(p_part.b.coeffs) == g["stage2_acc_p_b"]
    p_split, q_split = pk.ks.keyswitch_stage2_split(raised, evk)
    assert np.array_equal(p_split.b.coeffs, p_part.b.coeffs)
    assert np.array_equal(q_split.a.coeffs, q_part.a.coeffs)
    delta = pk.ks.keyswitch_stage3(q_part, p_part, p)
    assert R.digest(delta.a.coeffs) == g["stage3_out_a"]
    assert R.digest(delta.b.coeffs) == g["stage3_out_b"]
    out = pk.ks.keyswitch(ct, evk)
    assert R.digest(out.a.coeffs) == g["out_a"] and R.digest(out.b.coeffs) == g["out_b"]
    folded = pk.rns.poly_elementwise(delta.b, ct.b, "add")
    assert np.array_equal(folded.coeffs, out.b.coeffs)
    if p.n <= 8192:
        dec = pk.ks.decrypt(out, s_to)
        assert R.digest_i64(dec) == g["decrypt_switched"]
        assert int(np.abs(dec - msg).max()) == g["max_abs_err_switched"]
        assert R.digest_i64(pk.ks.decrypt(ct, s_from)) == g["decrypt_fresh"]


def test_keyswitch_matches_oracle_many_seeds(pk, psets, oracle_mod):
    """Reference acceptance criterion 3 (tests/test_acceptance.py:103-141) at a
    reduced seed count, checked limb-for-limb against the oracle."""
    p = psets("verify_small")
    op = oracle_mod.OParams(p.n, p.l, p.dnum, p.alpha, p.delta, p.h_dense,
                            tuple((m.q, m.psi) for m in p.q_basis),
                            tuple((m.q, m.psi) for m in p.p_basis))
    orc = oracle_mod.Oracle(p.n, op.ext_basis)
    worst = 0.0
    for seed in range(6):
        master = np.random.default_rng(seed)
        s_from = pk.ks.keygen(p, seed=seed * 7 + 1)
        s_to = pk.ks.keygen(p, seed=seed * 7 + 2)
        msg = master.integers(1, 9, p.n).astype(np.int64)
        msg *= master.choice(np.array([-1, 1], dtype=np.int64), p.n)
        msg *= p.delta
        ct = pk.ks.encrypt(msg, s_from, p, seed=seed * 7 + 3)
        evk = pk.ks.switching_keygen(s_from, s_to, p, seed=seed * 7 + 4)
        out = pk.ks.keyswitch(ct, evk)
        o_a, o_b = oracle_mod.encrypt(orc, op, msg, s_from.ternary, seed * 7 + 3)
        assert np.array_equal(ct.a.coeffs, o_a) and np.array_equal(ct.b.coeffs, o_b)
        o_evk = oracle_mod.switching_keygen(orc, op, s_from.ternary, s_to.ternary, seed * 7 + 4)
        w_a, w_b = orc.keyswitch(op, o_a, o_b, o_evk)
        assert np.array_equal(out.a.coeffs, w_a) and np.array_equal(out.b.coeffs, w_b)
        dec = pk.ks.decrypt(out, s_to)
        worst = max(worst, float((np.abs(dec - msg) / np.abs(msg)).max()))
    assert worst < 2.0 ** -10


def test_keyswitch_batched_and_degenerate_key(pk, psets):
    p = psets("tiny")
    rng = np.random.default_rng(99)
    sk = pk.ks.keygen(p, seed=1)
    evk = pk.ks.switching_keygen(sk, pk.ks.keygen(p, seed=2), p, seed=4)
    cts = [pk.ks.encrypt(R.message(p.n, p.delta, 50 + i), sk, p, seed=100 + i) for i in range(3)]
    for ct, out in zip(cts, pk.ks.keyswitch_batched(cts, evk)):
        solo = pk.ks.keyswitch(ct, evk)
        assert np.array_equal(solo.a.coeffs, out.a.coeffs) and np.array_equal(solo.b.coeffs, out.b.coeffs)
    # beta = 1, evk pair = (0, all-ones): the raised digit lands in b
    p1 = pk.params.generate_parameter_set(n=64, l=4, dnum=1, delta=1 << 25, h_dense=8, h_sparse=4)
    sk1 = pk.ks.keygen(p1, seed=1)
    ct = pk.ks.encrypt(R.message(p1.n, p1.delta, 3), sk1, p1, seed=2)
    ext = p1.ext_basis
    zeros = pk.rns.Polynomial(ext, np.zeros((len(ext), p1.n)), pk.rns.EVALUATION)
    ones = pk.rns.Polynomial(ext, np.ones((len(ext), p1.n)), pk.rns.EVALUATION)
    evk1 = pk.ks.SwitchingKey(pairs=(pk.ks.PolyPair(a=zeros, b=ones),), params=p1)
    raised = pk.ks.keyswitch_stage1(ct.a, p1)
    q_part, p_part = pk.ks.keyswitch_stage2(raised, evk1)
    assert not q_part.a.coeffs.any() and not p_part.a.coeffs.any()
    assert np.array_equal(q_part.b.coeffs, raised[0].coeffs[:p1.l])
    assert np.array_equal(p_part.b.coeffs, raised[0].coeffs[p1.l:])
    with pytest.raises(Exception):
        pk.ks.keyswitch_stage2(raised[:-1] if len(raised) > 1 else [], evk1)
    with pytest.raises(pk.rns.StructureError):
        pk.ks.keyswitch_stage1(pk.transform.ntt_polynomial(ct.a, "inverse"), p1)
    with pytest.raises(pk.rns.RnsError, match="wrong key or overflow"):
        pk.ks.decrypt(cts[0], pk.ks.keygen(p, seed=2))


def test_zero_p_part_moddown_is_scaling(pk, psets):
    p = psets("tiny")
    sk = pk.ks.keygen(p, seed=1)
    ct = pk.ks.encrypt(R.message(p.n, p.delta, 9), sk, p, seed=3)
    evk = pk.ks.switching_keygen(sk, pk.ks.keygen(p, seed=2), p, seed=4)
    q_part, p_part = pk.ks.keyswitch_stage2(pk.ks.keyswitch_stage1(ct.a, p), evk)
    zero = pk.rns.Polynomial(p.p_basis, np.zeros_like(p_part.a.coeffs), pk.rns.EVALUATION)
    out = pk.ks.keyswitch_stage3(q_part, pk.ks.PolyPair(a=zero, b=zero), p)
    tabs = pk.ks._tables(p)
    q_col = q_part.a.q_column()
    assert np.array_equal(out.a.coeffs, q_part.a.coeffs * tabs.p_inv_col % q_col)


def test_rnsv_roundtrip_from_device(pk, psets, tmp_path):
    p = psets("tiny")
    sk = pk.ks.keygen(p, seed=1)
    ct = pk.ks.encrypt(R.message(p.n, p.delta, 9), sk, p, seed=3)
    evk = pk.ks.switching_keygen(sk, pk.ks.keygen(p, seed=2), p, seed=4)
    names = pk.ks.dump_pipeline_vectors(tmp_path, ct, evk)
    assert names[0] == "stage1_input_a.rnsv" and names[-1] == "stage3_out_b.rnsv"
    assert len(names) == 1 + p.beta + 6
    back = pk.vectors.load_polynomial(tmp_path / "stage1_input_a.rnsv")
    assert pk.rns.poly_equal(back, ct.a)
