"""HRot / HMult+relinearize / rescale against the composed-reference goldens
(bit-exact), and encode / decode / level-l key switching / PMult against
tolerances (no reference counterpart: parity unpinned)."""
import numpy as np
import pytest

import recipes as R

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def env(golden):
    import torch

    assert torch.cuda.is_available()
    from paper_2512_18345_b200 import ckks, keyswitch as ks, rns
    from paper_2512_18345_b200.params import ParameterSet

    class E:
        pass

    e = E()
    e.ckks, e.ks, e.rns = ckks, ks, rns
    e.P = {name: ParameterSet.from_dict(golden["params"][name]) for name in ("tiny", "n8192")}
    return e


@pytest.mark.parametrize("pname", ["tiny", "n8192"])
def test_composed_goldens_bit_exact(env, golden, pname):
    """BASELINE config 1 at N = 2^13 (and the N = 64 profile): HRot, then
    HMult + relinearize + rescale, limb-for-limb equal to the reference composition."""
    g = golden["composed"][pname]
    p = env.P[pname]
    ck, ks = env.ckks, env.ks
    sk = ks.keygen(p, seed=g["sk_seed"])
    m1 = np.random.default_rng(g["msg_seeds"][0]).integers(1, 9, p.n).astype(np.int64) << 20
    m2 = np.random.default_rng(g["msg_seeds"][1]).integers(1, 9, p.n).astype(np.int64) << 20
    ct1 = ks.encrypt(m1, sk, p, seed=g["ct_seeds"][0])
    ct2 = ks.encrypt(m2, sk, p, seed=g["ct_seeds"][1])
    for k in (5, 2 * p.n - 1):
        gk = g[f"hrot_k{k}"]
        evk = ck.galois_keygen(sk, p, k, seed=gk["evk_seed"])
        out = ck.apply_galois(ct1, k, evk)
        assert R.digest(out.a.coeffs) == gk["out_a"] and R.digest(out.b.coeffs) == gk["out_b"]
        dest = (np.arange(p.n, dtype=np.int64) * k) % (2 * p.n)
        m_rot = np.zeros(p.n, dtype=np.int64)
        m_rot[dest % p.n] = np.where(dest >= p.n, -m1, m1)
        assert int(np.abs(ks.decrypt(out, sk) - m_rot).max()) == gk["max_abs_err"]
    gm = g["hmult"]
    rlk = ck.relin_keygen(sk, p, seed=gm["rlk_seed"])
    assert [[R.digest(pr.a.coeffs), R.digest(pr.b.coeffs)] for pr in rlk.pairs] == gm["rlk"]
    d0, d1, d2 = ck.tensor(ct1, ct2)
    assert (R.digest(d0.coeffs), R.digest(d1.coeffs), R.digest(d2.coeffs)) == (gm["d0"], gm["d1"], gm["d2"])
    prod = ck.hmult(ct1, ct2, rlk)
    assert R.digest(prod.a.coeffs) == gm["out_a"] and R.digest(prod.b.coeffs) == gm["out_b"]
    res = ck.rescale(prod)
    assert R.digest(res.a.coeffs) == g["rescale"]["out_a"] and R.digest(res.b.coeffs) == g["rescale"]["out_b"]
    assert res.a.num_limbs == p.l - 1
    assert R.digest_i64(ks.decrypt(res, sk)) == g["rescale"]["decrypt"]
    assert res.scale == pytest.approx(ct1.scale * ct2.scale / p.q_basis[-1].q)


def test_rescale_matches_oracle_composition(env, oracle_mod):
    """rescale == INTT(last) -> non-centred 1->L-1 conversion -> NTT -> (x - conv) * q_last^-1
    restated with the oracle's primitives on random limbs."""
    p = env.P["n8192"]
    rns, ck = env.rns, env.ckks
    rng = np.random.default_rng(11)
    basis = p.q_basis
    x = rns.random_polynomial(basis, p.n, rng, rns.EVALUATION)
    y = rns.random_polynomial(basis, p.n, rng, rns.EVALUATION)
    out = ck.rescale(ck.Ciphertext(a=x, b=y, scale=2.0 ** 60))
    orc = oracle_mod.Oracle(p.n, [(m.q, m.psi) for m in basis])
    last, rest = basis[-1], basis[:-1]
    for src, got in ((x, out.a), (y, out.b)):
        c = orc.ntt(src.coeffs[-1:], np.array([len(basis) - 1], np.int32), inverse=True)
        conv = oracle_mod.bconv([last.q], [m.q for m in rest], c)
        conv = orc.ntt(conv, np.arange(len(rest), dtype=np.int32))
        q_col = np.array([m.q for m in rest], dtype=np.uint64)[:, None]
        inv = np.array([pow(last.q, -1, m.q) for m in rest], dtype=np.uint64)[:, None]
        want = (src.coeffs[:-1] + q_col - conv) % q_col * inv % q_col
        assert np.array_equal(got.coeffs, want)


def test_encode_decode_roundtrip(env):
    p = env.P["n8192"]
    ck = env.ckks
    rng = np.random.default_rng(0)
    z = rng.uniform(-1, 1, p.n // 2) + 1j * rng.uniform(-1, 1, p.n // 2)
    pt = ck.encode(z, p, level=3, scale=2.0 ** 40)
    back = ck.decode(pt, p)
    assert np.abs(back - z).max() < 2.0 ** -25
    # a constant encodes to the constant polynomial
    c = ck.encode_constant(0.75, p, 2, 2.0 ** 30)
    assert np.abs(ck.decode(c, p) - 0.75).max() < 2.0 ** -25
    full = ck.encode(0.75, p, 2, 2.0 ** 30)
    assert np.array_equal(full.poly.coeffs, c.poly.coeffs)


def test_slotwise_semantics_rotation_conjugation_mult(env):
    """Decoded slots after HRot / conjugate / PMult / HMult+rescale match the
    plaintext computation (tolerance 2^-20 relative to unit-size slots)."""
    p = env.P["n8192"]
    ck, ks = env.ckks, env.ks
    rng = np.random.default_rng(1)
    sk = ks.keygen(p, seed=1)
    keys = ck.EvaluationKeys(p, relin=ck.relin_keygen(sk, p, seed=2))
    for r in (1, 5, p.n // 2 - 3):
        keys.add_rotation(sk, r, seed=10 + r)
    keys.add_conjugation(sk, seed=9)
    n2 = p.n // 2
    z1 = rng.uniform(-1, 1, n2) + 1j * rng.uniform(-1, 1, n2)
    z2 = rng.uniform(-1, 1, n2) + 1j * rng.uniform(-1, 1, n2)
    scale = float(p.q_basis[-1].q) * float(p.q_basis[-2].q)        # two limbs per level
    ct1 = ck.encrypt(ck.encode(z1, p, scale=scale), sk, p, seed=3)
    ct2 = ck.encrypt(ck.encode(z2, p, scale=scale), sk, p, seed=4)
    tol = 2.0 ** -20
    assert np.abs(ck.decrypt_decode(ct1, sk, p) - z1).max() < tol
    for r in (1, 5, n2 - 3):
        got = ck.decrypt_decode(ck.hrot(ct1, r, keys), sk, p)
        assert np.abs(got - np.roll(z1, -r)).max() < tol
    assert np.abs(ck.decrypt_decode(ck.conjugate(ct1, keys), sk, p) - np.conj(z1)).max() < tol
    assert np.abs(ck.decrypt_decode(ck.add(ct1, ct2), sk, p) - (z1 + z2)).max() < tol
    prod = ck.rescale(ck.hmult(ct1, ct2, keys.relin), 2)
    assert ck.level_of(prod) == p.l - 2
    assert np.abs(ck.decrypt_decode(prod, sk, p) - z1 * z2).max() < tol
    # level-l key switching with a partial last digit (l = 7, alpha = 4)
    low = ck.mod_drop(ct1, 7)
    got = ck.decrypt_decode(ck.hrot(low, 5, keys), sk, p)
    assert np.abs(got - np.roll(z1, -5)).max() < tol
    sq = ck.rescale(ck.hmult(low, ck.mod_drop(ct2, 7), keys.relin), 2)
    assert np.abs(ck.decrypt_decode(sq, sk, p) - z1 * z2).max() < tol
    # relinearisation and rescale merged into one ModDown
    fused = ck.hmult_rescale(ct1, ct2, keys.relin, 2)
    assert ck.level_of(fused) == p.l - 2 and fused.scale == pytest.approx(prod.scale)
    assert np.abs(ck.decrypt_decode(fused, sk, p) - z1 * z2).max() < tol
    fused_low = ck.hmult_rescale(low, ck.mod_drop(ct2, 7), keys.relin, 2)
    assert np.abs(ck.decrypt_decode(fused_low, sk, p) - z1 * z2).max() < tol
    # hoisted rotations (one ModUp shared) decode to the same slots as plain HRot
    hoisted = ck.hrot_hoisted(low, [0, 1, 5], keys)
    for r in (0, 1, 5):
        got = ck.decrypt_decode(ck.ct_from_tensor(hoisted[r], low.a.basis, low.scale), sk, p)
        assert np.abs(got - np.roll(z1, -r)).max() < tol
    # PMult by an encoded vector and by a constant
    w = rng.uniform(-1, 1, n2)
    pm = ck.rescale(ck.mul_plain(ct1, ck.encode(w, p, scale=scale)), 2)
    assert np.abs(ck.decrypt_decode(pm, sk, p) - z1 * w).max() < tol
    half = ck.mul_const(ct1, 0.5, p, drop=2)
    assert half.scale == ct1.scale
    assert np.abs(ck.decrypt_decode(half, sk, p) - 0.5 * z1).max() < tol
    with pytest.raises(env.rns.RnsError):
        ck.add(ct1, prod if ck.level_of(prod) == ck.level_of(ct1) else ck.Ciphertext(ct1.a, ct1.b, 3.0))


def test_captured_product_equals_eager(golden):
    """ckks.capture: HMult + relinearise + rescale at BASELINE config 1 (N = 2^13) recorded as one
    CUDA graph gives the limbs of the eager call, for the captured sample and for fresh operands."""
    import torch

    from paper_2512_18345_b200 import ckks, keyswitch as ks
    from paper_2512_18345_b200.params import generate_parameter_set

    p = generate_parameter_set(n=8192, l=12, dnum=3, delta=1 << 40, h_dense=64, h_sparse=32)
    sk = ks.keygen(p, seed=1)
    rlk = ckks.relin_keygen(sk, p, seed=41)
    msgs = [np.random.default_rng(7 + i).integers(1, 9, p.n).astype(np.int64) << 20 for i in range(4)]
    cts = [ks.encrypt(m, sk, p, seed=2 + 3 * i) for i, m in enumerate(msgs)]
    product = lambda a, b: ckks.rescale(ckks.hmult(a, b, rlk), 1)
    replay = ckks.capture(product, cts[0], cts[1])
    for a, b in ((cts[0], cts[1]), (cts[2], cts[3]), (cts[1], cts[2])):
        want = product(a, b)
        got = replay(a, b)
        torch.cuda.synchronize()
        assert np.array_equal(got.a.coeffs, want.a.coeffs) and np.array_equal(got.b.coeffs, want.b.coeffs)
        assert got.scale == want.scale and got.a.basis == want.a.basis
    with pytest.raises(Exception):
        replay(ckks.mod_drop(cts[0], 6), ckks.mod_drop(cts[1], 6))
