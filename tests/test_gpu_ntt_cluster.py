"""Single-pass N = 2^16 transform over thread-block clusters (csrc/ntt.cu ntt16_*_cluster; the
transform of reference transform.py:203-250 whose two-kernel split is transform.py:290-323).
Integer work: bit-exact against the CPU oracle, against the two-kernel path, and through the
whole key-switch / HMult pipelines that use its row maps, ModDown epilogue and product-on-load."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def env(golden):
    import torch

    assert torch.cuda.is_available(), "GPU tests need a CUDA device"
    from paper_2512_18345_b200 import ckks, keyswitch, params, rns, transform
    from paper_2512_18345_b200.engine import get_engine

    class NS:
        pass

    ns = NS()
    ns.torch, ns.ckks, ns.ks, ns.rns, ns.transform = torch, ckks, keyswitch, rns, transform
    ns.eng = get_engine()
    ns.ks48 = params.ParameterSet.from_dict(golden["params"]["ks48"])
    ns.saved = ns.eng.ntt_policy()
    yield ns
    ns.eng.ntt_policy(*ns.saved)


def _rows(mods, n, seed):
    rng = np.random.default_rng(seed)
    x = np.stack([rng.integers(0, m.q, n, dtype=np.uint64) for m in mods])
    if len(mods) >= 3:
        x[0] = 0
        x[1] = mods[1].q - 1
        x[2] = 0
        x[2, 0] = 1
    return x


def _dev(env, x):
    return env.torch.from_numpy(x.astype(np.uint32).view(np.int32)).to(env.eng.device)


def _host(t):
    return t.cpu().numpy().view(np.uint32).astype(np.uint64)


@pytest.mark.parametrize("occ", [2, 3])
@pytest.mark.parametrize("rows", [1, 5, 60])
def test_cluster_transform_matches_oracle_and_two_kernel_path(env, oracle_mod, rows, occ):
    p = env.ks48
    n = p.n
    mods = tuple((p.q_basis + p.p_basis)[:rows])
    x = _rows(mods, n, 100 + rows)
    slots = env.eng.row_slots(mods, n)
    t = _dev(env, x)
    env.eng.ntt_policy(0, occ)
    f2 = _host(env.eng.ntt(t, slots, False))
    i2 = _host(env.eng.ntt(t, slots, True))
    env.eng.ntt_policy(1 << 20, occ)
    assert env.eng.ntt_policy() == (1 << 20, occ)
    fc = env.eng.ntt(t, slots, False)
    ic = env.eng.ntt(t, slots, True)
    assert np.array_equal(_host(fc), f2)
    assert np.array_equal(_host(ic), i2)
    # round trip, in place (the key-switch pipeline transforms raised digits in place)
    env.eng.ntt(fc, slots, True, out=fc)
    assert np.array_equal(_host(fc), x)
    # the oracle on a few rows (edge rows included)
    k = min(rows, 4)
    orc = oracle_mod.Oracle(n, [(m.q, m.psi) for m in mods[:k]])
    rm = np.arange(k, dtype=np.int32)
    assert np.array_equal(f2[:k], orc.ntt(x[:k], rm))
    assert np.array_equal(i2[:k], orc.ntt(x[:k], rm, inverse=True))
    if rows >= 3:
        assert np.all(f2[2] == 1) and not f2[0].any()


@pytest.mark.parametrize("occ", [2, 3])
def test_pipelines_are_bit_identical_under_the_cluster_policy(env, occ):
    """Key switch (row maps in and out, fused ModDown epilogue) and HMult + relinearise + rescale
    (product-on-load inverse transform, merged ModDown) at ks48 and at a lower level with a partial
    last digit: the same limbs whichever transform kernels run."""
    p = env.ks48
    ckks, ks = env.ckks, env.ks
    sk = ks.keygen(p, seed=11)
    sk2 = ks.keygen(p, seed=12)
    evk = ks.switching_keygen(sk, sk2, p, seed=13)
    relin = ckks.relin_keygen(sk, p, seed=14)
    rng = np.random.default_rng(5)
    z = rng.uniform(-1, 1, p.n // 2) + 1j * rng.uniform(-1, 1, p.n // 2)
    ct = ckks.encrypt(ckks.encode(z, p, level=p.l, scale=2.0 ** 40), sk, p, seed=15)
    low = ckks.mod_drop(ct, 29)

    def run():
        a = ks.keyswitch(ct, evk)
        b = ckks.hmult_rescale(ct, ct, relin, 2)
        c = ckks.hmult_rescale(low, low, relin, 2)
        d = ckks.keyswitch_level(low, evk)
        env.torch.cuda.synchronize()
        return [x.coeffs.copy() for r in (a, b, c, d) for x in (r.a, r.b)]

    env.eng.ntt_policy(0, occ)
    ref = run()
    env.eng.ntt_policy(1 << 20, occ)
    got = run()
    for r, g in zip(ref, got):
        assert np.array_equal(r, g)
