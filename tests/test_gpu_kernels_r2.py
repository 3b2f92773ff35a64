"""Parity of the kernels added in round 2.  All integer work: bit-exact against the CPU oracle
(itself pinned to the reference's golden vectors, tests/test_oracle_golden.py)."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def env(golden):
    import torch

    assert torch.cuda.is_available(), "GPU tests need a CUDA device"
    from paper_2512_18345_b200 import baseconv, keyswitch, params, rns, transform
    from paper_2512_18345_b200.engine import get_engine

    class NS:
        pass

    ns = NS()
    ns.torch, ns.baseconv, ns.ks, ns.rns, ns.transform, ns.params = torch, baseconv, keyswitch, rns, transform, params
    ns.eng = get_engine()
    ns.ks48 = params.ParameterSet.from_dict(golden["params"]["ks48"])
    return ns


def qs(basis):
    return [m.q for m in basis]


# ---------------------------------------------------------------- single-launch small-ring transform
@pytest.mark.parametrize("lg", [1, 2, 3, 5, 8, 11, 12, 13, 14, 15])
def test_small_ring_transform_matches_oracle(env, oracle_mod, lg):
    """ntt_small_kernel (one CTA per limb, N <= 2^15, reference transform.py:203-250): forward and
    inverse against the oracle on mixed 31-bit moduli, edge rows included, in place and out of place."""
    n = 1 << lg
    primes, cand = [], (1 << 31) - 1
    step = 2 * n
    cand -= (cand - 1) % step
    while len(primes) < 5:
        if env.rns.is_prime(cand):
            primes.append(cand)
        cand -= step
    mods = tuple(env.rns.Modulus.for_prime(q, n) for q in primes)
    orc = oracle_mod.Oracle(n, [(m.q, m.psi) for m in mods])
    rng = np.random.default_rng(lg)
    x = np.stack([rng.integers(0, m.q, n, dtype=np.uint64) for m in mods])
    x[0] = 0
    x[1] = mods[1].q - 1
    x[2] = 0
    x[2, 0] = 1
    rm = np.arange(len(mods), dtype=np.int32)
    fwd = env.transform.ntt_polynomial(env.rns.Polynomial(mods, x, env.rns.COEFFICIENT))
    assert np.array_equal(fwd.coeffs, orc.ntt(x, rm))
    assert np.all(fwd.coeffs[2] == 1) and not fwd.coeffs[0].any()
    inv = env.transform.ntt_polynomial(env.rns.Polynomial(mods, x, env.rns.EVALUATION), "inverse")
    assert np.array_equal(inv.coeffs, orc.ntt(x, rm, inverse=True))
    assert np.array_equal(env.transform.ntt_polynomial(fwd, "inverse").coeffs, x)
    # in place through the engine (the key-switch pipeline transforms raised digits in place)
    t = env.torch.from_numpy(x.astype(np.uint32).view(np.int32)).to(env.eng.device)
    slots = env.eng.row_slots(mods, n)
    env.eng.ntt(t, slots, False, out=t)
    assert np.array_equal(t.cpu().numpy().view(np.uint32).astype(np.uint64), orc.ntt(x, rm))


# ---------------------------------------------------------------- negative control (verify.py:51-57)
def _schoolbook_negacyclic(a, b, q):
    n = len(a)
    c = [0] * n
    for i in range(n):
        for j in range(n):
            k = i + j
            if k < n:
                c[k] = (c[k] + int(a[i]) * int(b[j])) % q
            else:
                c[k - n] = (c[k - n] - int(a[i]) * int(b[j])) % q
    return np.array(c, dtype=np.uint64)


@pytest.mark.parametrize("n", [4, 16, 256, 4096, 65536])
def test_twiddle_corruption_is_detected(env, n):
    """The reference's negative control (verify.py:51-57, transform_suite with fault='twiddle'): one
    forward twiddle slot off by one.  `ntt(limb, m, table)` must use the table it is handed, so with
    the corrupted table the round trip / convolution checks fail, and with the clean one they pass:
    the checks above are able to see a wrong device table."""
    T = env.transform
    m = env.rns.find_ntt_primes(1, 31, n)[0]
    good = T.build_twiddle_table(m, n)
    bad = T.build_twiddle_table(m, n)
    slot = n // 2 + 1 if n > 2 else 1
    fwd = bad.fwd.copy()
    fwd[slot] = (fwd[slot] + 1) % m.q
    bad.fwd = fwd
    rng = np.random.default_rng(n)
    rows = rng.integers(0, m.q, size=(8, n), dtype=np.uint64)
    assert np.array_equal(T.ntt(T.ntt(rows, m, good), m, good, direction="inverse"), rows)
    assert not np.array_equal(T.ntt(T.ntt(rows, m, bad), m, bad, direction="inverse"), rows)
    # forward transforms differ exactly where the corrupted slot is used
    assert not np.array_equal(T.ntt(rows, m, bad), T.ntt(rows, m, good))
    if n <= 256:
        a, b = rows[0], rows[1]
        q = np.uint64(m.q)
        want = _schoolbook_negacyclic(a, b, m.q)
        ok = T.ntt(T.ntt(a, m, good) * T.ntt(b, m, good) % q, m, good, direction="inverse")
        ko = T.ntt(T.ntt(a, m, bad) * T.ntt(b, m, bad) % q, m, bad, direction="inverse")
        assert np.array_equal(ok, want) and not np.array_equal(ko, want)
    # the corruption lives in its own slot: the engine's resident tables are untouched
    again = T.build_twiddle_table(m, n)
    assert np.array_equal(again.fwd, good.fwd)


# ---------------------------------------------------------------- giant steps with the b half over Q||P
@pytest.mark.parametrize("l,count", [(48, 4), (42, 3), (21, 1), (19, 5)])
def test_giant_steps_with_b_half_over_qp_match_oracle(env, l, count):
    """ks_stage3_batch_a (ModDown of the a halves of several Q||P accumulators in one set of launches,
    keyswitch.py:387-419 per polynomial) and ks_accumulate_rot_qp (stage 1-2 of the key switch of
    sigma_k(a), keyswitch.py:297-355, plus sigma_k of a b half that stays over Q||P) followed by the
    shared ModDown: the CUDA engine and the oracle engine run the same calls on the same inputs."""
    import recipes as R
    from oracle.engine_oracle import OracleEngine

    eng, p = env.eng, env.ks48
    eng.set_lanes(8)
    try:
        qs = [m.q for m in p.ext_basis]
        evks = [np.stack([np.stack([R.level_key_rows(qs, p.n, t, h) for h in range(2)]) for t in range(p.dnum)])
                .astype(np.uint32) for _ in range(1)]
        q = p.q_basis[:l]
        ext = l + p.alpha
        ext_qs = [m.q for m in q + p.p_basis]
        rng = np.random.default_rng(100 * l + count)
        qps = np.stack([np.stack([np.stack([rng.integers(0, m, p.n, dtype=np.uint64) for m in ext_qs]) for _ in range(2)])
                        for _ in range(count)]).astype(np.uint32)
        ks_idx = [5, 2 * p.n - 1, 25, 3, 125][:count]
        words = lambda t: t.cpu().numpy().view(np.uint32)

        def run(e):
            plan = e.ks_plan(p.n, q, p.p_basis, p.alpha, p.l + p.alpha, p.l)
            t_qps = e.upload(qps.reshape(-1, p.n)).reshape(count, 2, ext, p.n)
            evk = e.upload(evks[0].reshape(-1, p.n)).reshape(evks[0].shape)
            a_md = e.ks_stage3_batch_a(plan, t_qps, l)
            for g in range(count):
                e.ks_accumulate_rot_qp(plan, a_md[g], t_qps[g][1], ks_idx[g], evk, first=(g == 0))
            out = e.ks_finish(plan, 1, None, None, l, p.n)
            return words(a_md).copy(), words(out).copy()

        got_md, got_out = run(eng)
        want_md, want_out = run(OracleEngine())
        assert np.array_equal(got_md, want_md), "batched ModDown of the a halves differs from the oracle"
        assert np.array_equal(got_out, want_out), "accumulated giant steps differ from the oracle"
    finally:
        eng.set_lanes(1)


# ---------------------------------------------------------------- BSGS kernels against the oracle engine
@pytest.mark.parametrize("level", [42, 21])
def test_bsgs_inner_matches_oracle_engine(env, level):
    """The fused baby-step + inner-sum kernel (hoisted rotations + BSGS) against the
    CPU restatement (OracleEngine.bsgs_inner = keyswitch.py:318-332 per rotation through rns.py:268-292's
    permutation, then rns.py:243-258 products): Q||P accumulators bit for bit, including an absent
    diagonal and the unrotated term."""
    from oracle.engine_oracle import OracleEngine
    from paper_2512_18345_b200 import ckks

    p = env.ks48
    basis = p.q_basis[:level]
    ext = level + p.alpha
    ext_basis = basis + p.p_basis
    rng = np.random.default_rng(level)
    rows = lambda mods: np.stack([rng.integers(0, m.q, p.n, dtype=np.uint64) for m in mods]).astype(np.uint32)
    a_h, b_h = rows(basis), rows(basis)
    rots = [0, 1, 3]
    ks_idx = [0 if r == 0 else ckks.galois_element(r, p.n) for r in rots]
    evk_h = [None if r == 0 else np.stack([np.stack([rows(p.ext_basis) for _ in range(2)]) for _ in range(p.dnum)])
             for r in rots]
    ng = 2
    table_h = [[None if (g, b) == (1, 2) else rows(ext_basis) for b in range(len(rots))] for g in range(ng)]

    def run(e):
        plan = e.ks_plan(p.n, basis, p.p_basis, p.alpha, p.l + p.alpha, p.l)
        ct_a, ct_b = e.upload(a_h), e.upload(b_h)
        raised = e.ks_stage1(plan, ct_a, -(-level // p.alpha), ext)
        evks = [None if k is None else e.upload(k.reshape(-1, p.n)).reshape(k.shape) for k in evk_h]
        table = [[None if t is None else e.upload(t) for t in row] for row in table_h]
        out = e.bsgs_inner(plan, raised, ct_a, ct_b, ks_idx, evks, table, ext)
        return [o.cpu().numpy().view(np.uint32).copy() for o in out]

    got, want = run(env.eng), run(OracleEngine())
    for g in range(ng):
        assert np.array_equal(got[g], want[g]), g


# ---------------------------------------------------------------- 64-bit reduction at the top of its range
@pytest.mark.parametrize("count", [1, 3, 4, 5, 8, 13, 16])
def test_accumulating_kernels_at_the_largest_residues(env, count):
    """reduce64 (csrc/common.cuh: x mod q as hi * (2^32 mod q) + lo with one lazy Shoup product) fed the
    largest values its callers can produce: every operand q - 1, so each product is (q-1)^2 = 1 (mod q),
    four of them plus a carried residue sit just below 2^64 in the fused PMult kernels' accumulators and
    the inner product sums beta of them.  Expected residues in closed form: the number of terms
    (poly_elementwise mul / add chains, reference rns.py:243-258; _stage2_accumulate, keyswitch.py:318-332)."""
    p = env.ks48
    torch, eng = env.torch, env.eng
    mods = tuple(p.q_basis[:6]) + tuple(p.p_basis[:2])
    n = p.n
    slots = eng.row_slots(mods, n)
    top = torch.tensor([m.q - 1 for m in mods], dtype=torch.int64, device=eng.device)[:, None].expand(len(mods), n)
    top32 = top.to(torch.int32).contiguous()                       # q - 1 < 2^31
    ct = torch.stack([top32, top32]).contiguous()
    out = eng.fused_terms([ct] * count, [top32] * count, slots)
    assert bool((out == count).all())
    multi = eng.fused_terms_multi([ct] * count, [[top32] * count, [top32] + [None] * (count - 1)], slots)
    assert bool((multi[0] == count).all()) and bool((multi[1] == 1).all())
    prod = eng.elementwise(top32, top32, slots, 2)
    assert bool((prod == 1).all())


def test_inner_product_at_the_largest_residues(env):
    """Stage 2 with every raised digit and every key word q - 1: acc = beta * (q-1)^2 = beta (mod q) on
    both halves and every row of the extended basis (keyswitch.py:318-332)."""
    p = env.ks48
    torch, eng = env.torch, env.eng
    ext = tuple(p.q_basis) + tuple(p.p_basis)
    plan = env.ks._tables(p).plan()
    top = torch.tensor([m.q - 1 for m in ext], dtype=torch.int64, device=eng.device)[:, None].expand(len(ext), p.n).to(torch.int32)
    raised = top.unsqueeze(0).expand(p.dnum, len(ext), p.n).contiguous()
    evk = top.unsqueeze(0).unsqueeze(0).expand(p.dnum, 2, len(ext), p.n).contiguous()
    acc = eng.ks_stage2(plan, raised, evk, 0, len(ext))
    assert bool((acc == p.dnum).all())
