"""Parity of the kernel variants added after the first CUDA path: the FP64 tensor-core
(DMMA) base conversion at ragged shapes, the multi-output fused inner sums, the ModDown
epilogue fused into the last NTT kernel, and the table-twiddle contiguous NTT phase.  All
integer work: bit-exact against the CPU oracle or against the unfused CUDA composition."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def env(golden):
    import torch

    assert torch.cuda.is_available(), "GPU tests need a CUDA device"
    from paper_2512_18345_b200 import baseconv, keyswitch, params, rns
    from paper_2512_18345_b200.engine import get_engine

    class NS:
        pass

    ns = NS()
    ns.torch, ns.baseconv, ns.ks, ns.rns, ns.eng = torch, baseconv, keyswitch, rns, get_engine()
    ns.ks48 = params.ParameterSet.from_dict(golden["params"]["ks48"])
    return ns


def qs(basis):
    return [m.q for m in basis]


def rand_rows(basis, cols, rng):
    return np.stack([rng.integers(0, m.q, cols, dtype=np.uint64) for m in basis])


# l_in not a multiple of 4 (K padding), l_out not a multiple of 8 (M padding), l_out large enough
# to be split over blockIdx.z, column counts that are / are not multiples of 16 (DMMA vs integer path)
@pytest.mark.parametrize("l_in,l_out,cols", [
    (1, 5, 65536), (2, 9, 4096), (3, 8, 65536), (5, 17, 1024), (7, 30, 65536), (12, 48, 65536),
    (13, 33, 2048), (14, 46, 65536), (16, 44, 512), (12, 36, 48), (12, 36, 1000), (9, 3, 16),
])
def test_bconv_shapes_match_oracle(env, oracle_mod, l_in, l_out, cols):
    p = env.ks48
    ext = p.ext_basis
    src, dst = ext[:l_in], ext[l_in:l_in + l_out]
    assert len(dst) == l_out
    table = env.baseconv.build_bconv_table(src, dst)
    rng = np.random.default_rng(1000 * l_in + l_out)
    x = rand_rows(src, cols, rng)
    # edge columns: all-zero and all-maximal residues
    x[:, 0] = 0
    x[:, -1] = [m.q - 1 for m in src]
    got = env.baseconv.convert(env.rns.Polynomial(src, x, env.rns.COEFFICIENT), table).coeffs
    want = oracle_mod.bconv(qs(src), qs(dst), x)
    assert np.array_equal(got, want)


def test_stage1_stacked_conversions_match_plain_calls(env):
    """The stacked conversions of key-switch stage 1 (all digits in one launch, outputs written
    through row maps into the raised layout) agree with one plain convert() call per digit."""
    p = env.ks48
    tabs = env.ks._tables(p)
    rng = np.random.default_rng(77)
    coeff = rand_rows(p.q_basis, p.n, rng)
    poly = env.rns.Polynomial(p.q_basis, coeff, env.rns.COEFFICIENT)
    from paper_2512_18345_b200.transform import ntt_polynomial

    ev = ntt_polynomial(poly, "forward")
    raised = env.ks.keyswitch_stage1(ev, p)
    for t in range(p.dnum):
        digit = p.q_basis[p.digit_slice(t)]
        x = coeff[p.digit_slice(t)]
        conv = env.baseconv.convert(env.rns.Polynomial(digit, x, env.rns.COEFFICIENT), tabs.raise_tables[t])
        want = ntt_polynomial(conv, "forward").coeffs
        rows = [i for i, m in enumerate(p.ext_basis) if m not in digit]
        assert np.array_equal(raised[t].coeffs[rows], want)


def test_fused_terms_multi_matches_single(env):
    eng, torch, p = env.eng, env.torch, env.ks48
    rows, n = 9, p.n
    basis = p.ext_basis[:rows]
    slots = eng.row_slots(basis)
    rng = np.random.default_rng(5)

    def rnd(*lead):
        return eng.upload(np.stack([rng.integers(0, m.q, (*lead, n), dtype=np.uint64) for m in basis], axis=len(lead))
                          .reshape(*lead, rows, n))

    for nb, ng in ((1, 1), (3, 2), (5, 5), (16, 4), (7, 8)):
        xs = [rnd(2) for _ in range(nb)]
        table = [[rnd() if (g + b) % 5 != 3 else None for b in range(nb)] for g in range(ng)]
        outs = eng.fused_terms_multi(xs, table, slots)
        for g in range(ng):
            present = [b for b in range(nb) if table[g][b] is not None]
            if present:
                want = eng.fused_terms([xs[b] for b in present], [table[g][b] for b in present], slots)
            else:
                want = torch.zeros_like(xs[0])
            assert torch.equal(outs[g], want), (nb, ng, g)


def test_fused_moddown_epilogue_matches_reference_composition(env, oracle_mod):
    """keyswitch_stage3 (iNTT -> BConv -> NTT with the ModDown epilogue applied inside the last
    NTT kernel) against the oracle's stage 3 on the same accumulators, at N = 2^16."""
    from oracle import oracle

    p = env.ks48
    rng = np.random.default_rng(11)
    ext = p.ext_basis
    acc = [rand_rows(ext, p.n, rng) for _ in range(2)]
    L = p.l

    def pair(lo, hi):
        basis = ext[lo:hi]
        return env.ks.PolyPair(a=env.rns.Polynomial(basis, acc[0][lo:hi], env.rns.EVALUATION),
                               b=env.rns.Polynomial(basis, acc[1][lo:hi], env.rns.EVALUATION))

    got = env.ks.keyswitch_stage3(pair(0, L), pair(L, L + p.alpha), p)
    op = oracle.OParams(p.n, p.l, p.dnum, p.alpha, p.delta, p.h_dense,
                        tuple((m.q, m.psi) for m in p.q_basis), tuple((m.q, m.psi) for m in p.p_basis))
    orc = oracle.Oracle(p.n, op.ext_basis)
    want_a = orc.ks_moddown(op, acc[0][:L], acc[0][L:])
    want_b = orc.ks_moddown(op, acc[1][:L], acc[1][L:])
    assert np.array_equal(got.a.coeffs, want_a) and np.array_equal(got.b.coeffs, want_b)


def test_ntt_phases_compose_and_invert_at_2_16(env):
    """The two fast kernels of each direction, run one at a time through ntt_stages, equal the
    whole transform; forward then inverse is the identity (table twiddles, 256-bit accesses)."""
    eng, torch, p = env.eng, env.torch, env.ks48
    basis = p.ext_basis
    slots = eng.row_slots(basis, p.n)
    rng = np.random.default_rng(21)
    x = eng.upload(rand_rows(basis, p.n, rng))
    fwd = eng.ntt(x, slots, False)
    half = eng.ntt_stages(x, slots, False, 0, 8)
    assert torch.equal(eng.ntt_stages(half, slots, False, 8, 16), fwd)
    back = eng.ntt(fwd, slots, True)
    assert torch.equal(back, x)
    half = eng.ntt_stages(fwd, slots, True, 0, 8)
    assert torch.equal(eng.ntt_stages(half, slots, True, 8, 16), x)


def test_bsgs_inner_equals_unfused_baby_steps(env):
    """The fused baby-step + inner-sum kernel against ckks_ks_hoisted_raw followed by
    ckks_fused_terms_multi on the same keys, digits and plaintexts: exact modular arithmetic, so
    the Q||P accumulators must agree bit for bit (including an absent diagonal and the
    unrotated term)."""
    eng, torch, p = env.eng, env.torch, env.ks48
    from paper_2512_18345_b200 import ckks

    level = 21                                  # two digits, the second one partial
    basis = p.q_basis[:level]
    ext = level + p.alpha
    ext_basis = basis + p.p_basis
    rng = np.random.default_rng(31)
    ct_a = eng.upload(rand_rows(basis, p.n, rng))
    ct_b = eng.upload(rand_rows(basis, p.n, rng))
    plan = eng.ks_plan(p.n, basis, p.p_basis, p.alpha, p.l + p.alpha, p.l)
    beta = -(-level // p.alpha)
    raised = eng.ks_stage1(plan, ct_a, beta, ext)
    full_ext = p.ext_basis
    rots = [0, 1, 2, 5]
    ks_idx = [0 if r == 0 else ckks.galois_element(r, p.n) for r in rots]
    evks = [None if r == 0 else eng.upload(rand_rows(full_ext, p.dnum * 2 * p.n, rng).reshape(len(full_ext), p.dnum, 2, p.n)
                                           .transpose(1, 2, 0, 3).copy()) for r in rots]
    ng = 3
    table = [[None if (g, b) == (1, 2) else eng.upload(rand_rows(ext_basis, p.n, rng)) for b in range(len(rots))]
             for g in range(ng)]
    fused = eng.bsgs_inner(plan, raised, ct_a, ct_b, ks_idx, evks, table, ext)
    # unfused composition
    accs = []
    for k, evk in zip(ks_idx, evks):
        if k == 0:
            x = torch.stack([ct_a, ct_b])
            accs.append(torch.cat([x, torch.zeros((2, p.alpha, p.n), dtype=x.dtype, device=x.device)], dim=1))
        else:
            accs.append(eng.ks_hoisted_raw(plan, raised, k, evk, ct_b, ext))
    want = eng.fused_terms_multi(accs, table, eng.row_slots(ext_basis))
    for g in range(ng):
        assert torch.equal(fused[g], want[g]), g


@pytest.mark.parametrize("level,k", [(48, 2), (30, 2), (21, 1), (13, 1)])
def test_fused_hmult_equals_tensor_then_relin_rescale(env, level, k):
    """ckks_hmult_relin_rescale (d2 formed while the inverse transform loads, d1 / d0 inside the
    inner product) against ckks_tensor + ckks_ks_relin_rescale on the same operands and key: exact
    modular arithmetic, equal limb for limb (full and partial last digit, 1- and 2-limb rescale)."""
    eng, torch, p = env.eng, env.torch, env.ks48
    basis = p.q_basis[:level]
    rest, dropped = basis[:level - k], basis[level - k:]
    rng = np.random.default_rng(100 + level)
    xa, xb, ya, yb = (eng.upload(rand_rows(basis, p.n, rng)) for _ in range(4))
    full_ext = p.ext_basis
    evk = eng.upload(rand_rows(full_ext, p.dnum * 2 * p.n, rng).reshape(len(full_ext), p.dnum, 2, p.n)
                     .transpose(1, 2, 0, 3).copy())
    ks_plan = eng.ks_plan(p.n, basis, p.p_basis, p.alpha, p.l + p.alpha, p.l)
    md_plan = eng.moddown_plan(p.n, rest, dropped + p.p_basis)
    fused = eng.hmult_relin_rescale(ks_plan, md_plan, xa, xb, ya, yb, evk, level - k)
    d = eng.tensor_halves(xa, xb, ya, yb, eng.row_slots(basis))
    want = eng.ks_relin_rescale(ks_plan, md_plan, d, evk, level - k)
    assert torch.equal(fused, want)
    # squaring: both operands are the same tensors
    fused = eng.hmult_relin_rescale(ks_plan, md_plan, xa, xb, xa, xb, evk, level - k)
    d = eng.tensor_halves(xa, xb, xa, xb, eng.row_slots(basis))
    assert torch.equal(fused, eng.ks_relin_rescale(ks_plan, md_plan, d, evk, level - k))


def test_keyswitch_batched_concurrent_lanes_equals_loop(env, golden):
    """keyswitch_batched with several workspace lanes (scheduler.plan_batch decides how many key
    switches are in flight) returns the limbs of a plain loop of keyswitch()."""
    from paper_2512_18345_b200 import params

    eng, ks = env.eng, env.ks
    p = params.ParameterSet.from_dict(golden["params"]["ks12"])
    s_from, s_to = ks.keygen(p, seed=1), ks.keygen(p, seed=2)
    evk = ks.switching_keygen(s_from, s_to, p, seed=4)
    rng = np.random.default_rng(6)
    cts = [ks.encrypt(rng.integers(1, 9, p.n).astype(np.int64) * p.delta, s_from, p, seed=10 + i) for i in range(5)]
    want = [ks.keyswitch(ct, evk) for ct in cts]
    eng.set_lanes(4)
    try:
        got = ks.keyswitch_batched(cts, evk)
    finally:
        eng.set_lanes(1)
    for g, w in zip(got, want):
        assert np.array_equal(g.a.coeffs, w.a.coeffs) and np.array_equal(g.b.coeffs, w.b.coeffs)


def test_keyswitch_pipelined_equals_loop(env, golden):
    """keyswitch_pipelined (ModUp of ciphertext i + 1 on one lane under the inner product and
    ModDown of ciphertext i on another, stage-2 split) returns the limbs of keyswitch(); also with
    a single lane, where it degenerates to the staged sequence."""
    from paper_2512_18345_b200 import params

    eng, ks = env.eng, env.ks
    p = params.ParameterSet.from_dict(golden["params"]["ks12"])
    s_from, s_to = ks.keygen(p, seed=1), ks.keygen(p, seed=2)
    evk = ks.switching_keygen(s_from, s_to, p, seed=4)
    rng = np.random.default_rng(6)
    cts = [ks.encrypt(rng.integers(1, 9, p.n).astype(np.int64) * p.delta, s_from, p, seed=10 + i) for i in range(5)]
    want = [ks.keyswitch(ct, evk) for ct in cts]
    for lanes in (1, 2, 4):
        eng.set_lanes(lanes)
        try:
            got = ks.keyswitch_pipelined(cts, evk)
            env.torch.cuda.synchronize()
        finally:
            eng.set_lanes(1)
        for g, w in zip(got, want):
            assert np.array_equal(g.a.coeffs, w.a.coeffs) and np.array_equal(g.b.coeffs, w.b.coeffs)


def test_batched_moddown_equals_separate_moddowns(env):
    """ckks_ks_stage3_batch over three accumulators (one set of launches, element g in the arena
    of lane g) against three ckks_ks_stage3 calls: equal limb for limb."""
    eng, torch, p = env.eng, env.torch, env.ks48
    level = 30
    basis = p.q_basis[:level]
    ext = level + p.alpha
    rng = np.random.default_rng(41)
    plan = eng.ks_plan(p.n, basis, p.p_basis, p.alpha, p.l + p.alpha, p.l)
    qps = torch.stack([torch.stack([eng.upload(rand_rows(basis + p.p_basis, p.n, rng)) for _ in range(2)])
                       for _ in range(3)])
    want = [eng.ks_stage3(plan, q[0, :level], q[1, :level], q[0, level:], q[1, level:]) for q in qps]
    eng.set_lanes(3)
    try:
        got = eng.ks_stage3_batch(plan, qps, level)
        torch.cuda.synchronize()
    finally:
        eng.set_lanes(1)
    for g in range(3):
        assert torch.equal(got[g], want[g]), g
