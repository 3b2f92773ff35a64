"""Hybrid (dnum-digit) key switching on the GPU, with the reference's
keygen / encrypt / decrypt harness around it.

API mirror of ``rnscope/keyswitch.py``: value types (:37-93), keygen (:112-121),
encrypt (:124-149), decrypt (:152-183), switching_keygen (:226-253),
keyswitch_stage1/2/3 (:297-441), keyswitch (:444-453), keyswitch_batched
(:456-459), dump_pipeline_vectors (:462-490).

Randomness is drawn on the host with exactly the reference's NumPy calls and
call order (SURVEY 8a'.9), so a seed reproduces the reference's limbs bit for
bit; everything after sampling (transforms, products, the three pipeline
stages) runs in the CUDA kernels.  ``decrypt`` ends with the reference's
big-integer CRT lift on the host (a test harness, not a hot path).
"""
from __future__ import annotations

import functools
import math
from dataclasses import dataclass, field

import numpy as np

from . import baseconv, transform
from .instrument import counters
from .params import ParameterSet
from .rns import (
    COEFFICIENT,
    EVALUATION,
    Modulus,
    Polynomial,
    RnsError,
    StructureError,
    poly_elementwise,
)

NOISE_WIDTH = 3.2  # centred discrete Gaussian width of fresh noise


# ---------------------------------------------------------------------------
# value types
# ---------------------------------------------------------------------------
@dataclass
class SecretKey:
    """Ternary secret with exactly h non-zero coefficients in {-1, +1}."""

    ternary: np.ndarray  # (N,) int8
    n: int
    _eval_cache: dict = field(default_factory=dict, repr=False)

    @property
    def hamming_weight(self) -> int:
        return int(np.count_nonzero(self.ternary))

    def residue_rows(self, basis) -> np.ndarray:
        return _signed_rows(self.ternary, basis)

    def eval_polynomial(self, basis) -> Polynomial:
        """NTT of the secret over ``basis`` (device resident, cached per basis)."""
        key = tuple(m.q for m in basis)
        hit = self._eval_cache.get(key)
        if hit is None:
            coeff = Polynomial(tuple(basis), self.residue_rows(basis), COEFFICIENT)
            hit = self._eval_cache[key] = transform.ntt_polynomial(coeff)
        return hit


@dataclass
class Ciphertext:
    """(a, b) in the evaluation domain; decrypt(ct, s) = b + a*s."""

    a: Polynomial
    b: Polynomial
    scale: int

    def __post_init__(self) -> None:
        if self.a.domain != EVALUATION or self.b.domain != EVALUATION:
            raise StructureError("ciphertext polynomials live in the evaluation domain")


@dataclass
class PolyPair:
    a: Polynomial
    b: Polynomial


@dataclass
class SwitchingKey:
    """dnum gadget-encryption pairs over Q||P.  ``matrix()`` is the contiguous
    device image [dnum][2][L+alpha][N] that stage 2 streams."""

    pairs: tuple[PolyPair, ...]
    params: ParameterSet
    _matrix: object = field(default=None, repr=False, compare=False)

    @property
    def shape(self) -> tuple[int, int]:
        return (2 * len(self.pairs), self.pairs[0].a.num_limbs)

    def matrix(self):
        if self._matrix is None:
            import torch

            self._matrix = torch.stack(
                [torch.stack([pr.a.data, pr.b.data]) for pr in self.pairs]
            ).contiguous()
            # the inner-product kernels prefetch key words ahead of their programmatic-dependency
            # wait: make the freshly stacked matrix globally visible before any of them can start
            if self._matrix.is_cuda:
                torch.cuda.current_stream(self._matrix.device).synchronize()
        return self._matrix


# ---------------------------------------------------------------------------
# sampling (host, NumPy RNG order of the reference)
# ---------------------------------------------------------------------------
def _signed_rows(vals, basis) -> np.ndarray:
    v = np.asarray(vals).astype(np.int64)
    return np.stack([np.mod(v, np.int64(m.q)).astype(np.uint64) for m in basis])


def _gaussian(n: int, rng: np.random.Generator, width: float = NOISE_WIDTH) -> np.ndarray:
    return np.rint(rng.normal(0.0, width, size=n)).astype(np.int64)


def _uniform_rows(basis, n: int, rng: np.random.Generator) -> np.ndarray:
    return np.stack([rng.integers(0, m.q, size=n, dtype=np.uint64) for m in basis])


def keygen(params: ParameterSet, h: int | None = None, seed: int = 0) -> SecretKey:
    h = params.h_dense if h is None else h
    if not 0 < h <= params.n:
        raise RnsError(f"Hamming weight {h} out of range for N={params.n}")
    rng = np.random.default_rng(seed)
    where = rng.choice(params.n, size=h, replace=False)
    s = np.zeros(params.n, dtype=np.int8)
    s[where] = rng.choice(np.array([-1, 1], dtype=np.int8), size=h)
    return SecretKey(ternary=s, n=params.n)


def encrypt(msg, sk: SecretKey, params: ParameterSet, seed: int = 0) -> Ciphertext:
    """b = -a*s + msg + e for a length-N integer row already scaled by delta."""
    msg = np.asarray(msg, dtype=np.int64)
    if msg.shape != (params.n,):
        raise StructureError(f"message must be a length-{params.n} integer row")
    if 4 * int(np.abs(msg).max(initial=0)) >= math.prod(m.q for m in params.q_basis):
        raise RnsError("message magnitude exceeds the modulus budget")
    rng = np.random.default_rng(seed)
    basis = params.q_basis
    a = Polynomial(basis, _uniform_rows(basis, params.n, rng), EVALUATION)
    e = _gaussian(params.n, rng)
    q_col = np.array([m.q for m in basis], dtype=np.uint64)[:, None]
    payload = (_signed_rows(e, basis) + _signed_rows(msg, basis)) % q_col
    payload = transform.ntt_polynomial(Polynomial(basis, payload, COEFFICIENT))
    b = poly_elementwise(payload, poly_elementwise(a, sk.eval_polynomial(basis), "mul"), "sub")
    return Ciphertext(a=a, b=b, scale=params.delta)


@functools.lru_cache(maxsize=32)
def _crt_constants(qs: tuple[int, ...]):
    big = math.prod(qs)
    hats = [big // q for q in qs]
    return big, hats, [pow(h, -1, q) for h, q in zip(hats, qs)]


def _crt_center(rows: np.ndarray, qs: tuple[int, ...]) -> list[int]:
    """Exact CRT lift of every column, centred into (-Q/2, Q/2]."""
    big, hats, invs = _crt_constants(qs)
    total = np.zeros(rows.shape[1], dtype=object)
    for i, q in enumerate(qs):
        total += (rows[i] * np.uint64(invs[i]) % np.uint64(q)).astype(object) * hats[i]
    half = big // 2
    out = []
    for v in total:
        v %= big
        out.append(v - big if v > half else v)
    return out


def decrypt(ct: Ciphertext, sk: SecretKey) -> np.ndarray:
    """Centred integer row b + a*s (message plus noise)."""
    basis = ct.a.basis
    d = poly_elementwise(ct.b, poly_elementwise(ct.a, sk.eval_polynomial(basis), "mul"), "add")
    coeff = transform.ntt_polynomial(d, "inverse")
    vals = _crt_center(coeff.coeffs, tuple(m.q for m in basis))
    if any(abs(v) >= 1 << 62 for v in vals):
        raise RnsError("decrypted value exceeds the int64 range; wrong key or overflow")
    return np.array(vals, dtype=np.int64)


# ---------------------------------------------------------------------------
# per-parameter-set tables
# ---------------------------------------------------------------------------
class _KsTables:
    """Conversion tables and constants of the pipeline (reference :186-218);
    the device copies live in the engine's key-switch plan."""

    def __init__(self, params: ParameterSet):
        self.params = params
        self.ext_basis = ext = params.ext_basis
        alpha = params.alpha
        self.raise_targets = [
            tuple(m for i, m in enumerate(params.q_basis) if i // alpha != t) + params.p_basis
            for t in range(params.dnum)
        ]
        qs = [m.q for m in params.q_basis]
        p_prod = math.prod(m.q for m in params.p_basis)
        big_q = math.prod(qs)
        self.p_inv_col = np.array([pow(p_prod, -1, q) for q in qs], dtype=np.uint64)[:, None]
        self.gadget = np.zeros((params.dnum, len(ext)), dtype=np.uint64)
        for t in range(params.dnum):
            d_t = math.prod(qs[params.digit_slice(t)])
            rest = big_q // d_t
            g = p_prod * rest * pow(rest, -1, d_t)
            self.gadget[t] = [g % m.q for m in ext]
        self._raise_tables = None
        self._moddown_table = None

    @property
    def raise_tables(self):
        if self._raise_tables is None:
            p = self.params
            self._raise_tables = [
                baseconv.build_bconv_table(p.q_basis[p.digit_slice(t)], self.raise_targets[t])
                for t in range(p.dnum)
            ]
        return self._raise_tables

    @property
    def moddown_table(self):
        if self._moddown_table is None:
            self._moddown_table = baseconv.build_bconv_table(self.params.p_basis, self.params.q_basis)
        return self._moddown_table

    def plan(self) -> int:
        from .engine import get_engine

        p = self.params
        return get_engine().ks_plan(p.n, p.q_basis, p.p_basis, p.alpha, p.l + p.alpha, p.l)


@functools.lru_cache(maxsize=8)
def _tables(params: ParameterSet) -> _KsTables:
    return _KsTables(params)


def switching_keygen(s_from: SecretKey, s_to: SecretKey, params: ParameterSet,
                     seed: int = 0) -> SwitchingKey:
    """Pair t satisfies b_t + a_t*s_to = e_t + g_t*s_from over Q||P."""
    tabs = _tables(params)
    ext = tabs.ext_basis
    rng = np.random.default_rng(seed)
    s_to_eval = s_to.eval_polynomial(ext)
    s_from_eval = s_from.eval_polynomial(ext)
    pairs = []
    for t in range(params.dnum):
        a = Polynomial(ext, _uniform_rows(ext, params.n, rng), EVALUATION)
        e = _gaussian(params.n, rng)
        e_eval = transform.ntt_polynomial(Polynomial(ext, _signed_rows(e, ext), COEFFICIENT))
        g_rows = np.broadcast_to(tabs.gadget[t][:, None], (len(ext), params.n))
        g_s = poly_elementwise(Polynomial(ext, g_rows, EVALUATION), s_from_eval, "mul")
        b = poly_elementwise(poly_elementwise(e_eval, g_s, "add"),
                             poly_elementwise(a, s_to_eval, "mul"), "sub")
        pairs.append(PolyPair(a=a, b=b))
    return SwitchingKey(pairs=tuple(pairs), params=params)


# ---------------------------------------------------------------------------
# the three stages
# ---------------------------------------------------------------------------
def _same_basis(p: Polynomial, basis) -> bool:
    return tuple(m.q for m in p.basis) == tuple(m.q for m in basis)


def keyswitch_stage1(d: Polynomial, params: ParameterSet, batch: int | None = None) -> list[Polynomial]:
    """ModUp: raise all beta digits of d to Q||P -> beta polynomials of
    L + alpha limbs, digit limbs carried through.  ``batch`` is accepted for
    API parity: the device pipeline always processes the beta digits as one
    stacked unit and the result is bit-identical for every grouping."""
    if d.domain != EVALUATION:
        raise StructureError("stage 1 input lives in the evaluation domain")
    if not _same_basis(d, params.q_basis):
        raise StructureError("stage 1 input basis must match the parameter q-basis")
    from .engine import get_engine

    tabs = _tables(params)
    ext = tabs.ext_basis
    raised = get_engine().ks_stage1(tabs.plan(), d.data, params.beta, len(ext))
    lg = params.n.bit_length() - 1
    counters.butterflies += (params.l + params.beta * params.l) * (params.n // 2) * lg
    counters.mads += params.beta * params.alpha * params.l * params.n
    return [Polynomial(ext, raised[t], EVALUATION) for t in range(params.beta)]


def _stack_raised(raised: list[Polynomial]):
    import torch

    first = raised[0].data
    step = first.numel() * first.element_size()
    base = getattr(first, "_base", None)
    if base is not None and base.dim() == 3 and base.shape[0] == len(raised) and all(
        r.data.data_ptr() == base.data_ptr() + i * step for i, r in enumerate(raised)
    ):
        return base
    return torch.stack([r.data for r in raised]).contiguous()


def _stage2(raised: list[Polynomial], evk: SwitchingKey, lo: int, hi: int):
    params = evk.params
    if len(raised) != params.beta:
        raise StructureError(f"expected {params.beta} raised digits, got {len(raised)}")
    from .engine import get_engine

    acc = get_engine().ks_stage2(_tables(params).plan(), _stack_raised(raised), evk.matrix(), lo, hi)
    counters.elementwise += 2 * params.beta * (hi - lo) * params.n
    return acc


def keyswitch_stage2(raised: list[Polynomial], evk: SwitchingKey) -> tuple[PolyPair, PolyPair]:
    """Inner product with the key pairs -> ((2, L) Q part, (2, alpha) P part)."""
    p = evk.params
    acc = _stage2(raised, evk, 0, p.l + p.alpha)
    q_part = PolyPair(Polynomial(p.q_basis, acc[0, :p.l], EVALUATION),
                      Polynomial(p.q_basis, acc[1, :p.l], EVALUATION))
    p_part = PolyPair(Polynomial(p.p_basis, acc[0, p.l:], EVALUATION),
                      Polynomial(p.p_basis, acc[1, p.l:], EVALUATION))
    return q_part, p_part


def stage2_p_part(raised: list[Polynomial], evk: SwitchingKey) -> PolyPair:
    p = evk.params
    acc = _stage2(raised, evk, p.l, p.l + p.alpha)
    return PolyPair(Polynomial(p.p_basis, acc[0], EVALUATION), Polynomial(p.p_basis, acc[1], EVALUATION))


def stage2_q_part(raised: list[Polynomial], evk: SwitchingKey) -> PolyPair:
    p = evk.params
    acc = _stage2(raised, evk, 0, p.l)
    return PolyPair(Polynomial(p.q_basis, acc[0], EVALUATION), Polynomial(p.q_basis, acc[1], EVALUATION))


def keyswitch_stage2_split(raised: list[Polynomial], evk: SwitchingKey) -> tuple[PolyPair, PolyPair]:
    """P part first so stage-3 work can start while the Q half is computed."""
    p_part = stage2_p_part(raised, evk)
    return p_part, stage2_q_part(raised, evk)


def keyswitch_stage3(q_part: PolyPair, p_part: PolyPair, params: ParameterSet, batch: int = 2) -> PolyPair:
    """ModDown both accumulator polynomials: (x_Q - NTT(BConv(INTT(x_P)))) * P^-1.
    ``batch`` accepted for parity; both halves always run as one stacked unit."""
    from .engine import get_engine

    out = get_engine().ks_stage3(_tables(params).plan(), q_part.a.data, q_part.b.data,
                                 p_part.a.data, p_part.b.data)
    lg = params.n.bit_length() - 1
    counters.butterflies += 2 * (params.alpha + params.l) * (params.n // 2) * lg
    counters.mads += 2 * params.alpha * params.l * params.n
    counters.elementwise += 4 * params.l * params.n
    return PolyPair(Polynomial(params.q_basis, out[0], EVALUATION),
                    Polynomial(params.q_basis, out[1], EVALUATION))


def keyswitch(ct: Ciphertext, evk: SwitchingKey) -> Ciphertext:
    """All three stages in one call on the plan's device workspace; ct.b is
    folded into the b half inside the ModDown epilogue."""
    params = evk.params
    if not _same_basis(ct.a, params.q_basis):
        raise StructureError("stage 1 input basis must match the parameter q-basis")
    from .engine import get_engine

    out = get_engine().keyswitch(_tables(params).plan(), ct.a.data, ct.b.data, evk.matrix())
    return Ciphertext(a=Polynomial(params.q_basis, out[0], EVALUATION),
                      b=Polynomial(params.q_basis, out[1], EVALUATION), scale=ct.scale)


def keyswitch_batched(cts: list[Ciphertext], evk: SwitchingKey) -> list[Ciphertext]:
    """Independent key switches under one key (reference keyswitch.py:456-459: a plain loop).
    As many as fit the L2 together (scheduler.plan_batch) run concurrently, one workspace lane
    and stream each; every result equals keyswitch(ct, evk) limb for limb."""
    from .engine import get_engine
    from .scheduler import concurrent_keyswitches

    eng = get_engine()
    cts = list(cts)
    width = concurrent_keyswitches(evk.params, eng.lane_count(), len(cts))
    if width <= 1:
        return [keyswitch(ct, evk) for ct in cts]
    out: list[Ciphertext] = []
    for lo in range(0, len(cts), width):
        out += eng.fork([(lambda ct=ct: keyswitch(ct, evk)) for ct in cts[lo:lo + width]])
    return out


def keyswitch_pipelined(cts: list[Ciphertext], evk: SwitchingKey) -> list[Ciphertext]:
    """Independent key switches under one key as a two-lane software pipeline: the ModUp of
    ciphertext i + 1 (transforms and base conversion, cache- and integer-bound) runs on one lane
    while the inner product of ciphertext i streams the key from HBM and its ModDown follows on
    the other -- the complementary pipelining the reference models in costmodel.py:508-541, built
    from the same launches as the fused key switch.  Every result equals keyswitch(ct, evk) limb
    for limb."""
    from .engine import get_engine

    params = evk.params
    eng = get_engine()
    tabs = _tables(params)
    plan, ext, key = tabs.plan(), len(tabs.ext_basis), evk.matrix()
    for ct in cts:
        if not _same_basis(ct.a, params.q_basis):
            raise StructureError("stage 1 input basis must match the parameter q-basis")

    def mod_up(ct):
        return eng.ks_stage1(plan, ct.a.data, params.beta, ext)

    def rest(ct, raised):
        out = eng.ks_hoisted(plan, raised, 1, key, ct.b.data)        # k = 1: no rotation
        return Ciphertext(a=Polynomial(params.q_basis, out[0], EVALUATION),
                          b=Polynomial(params.q_basis, out[1], EVALUATION), scale=ct.scale)

    return eng.pipeline(list(cts), mod_up, rest)


def dump_pipeline_vectors(directory, ct: Ciphertext, evk: SwitchingKey) -> list[str]:
    """Write every stage's polynomials as RNSV files, names as the reference's."""
    from pathlib import Path

    from .vectors import save_polynomial

    directory = Path(directory)
    directory.mkdir(parents=True, exist_ok=True)
    params = evk.params
    raised = keyswitch_stage1(ct.a, params)
    q_part, p_part = keyswitch_stage2(raised, evk)
    delta = keyswitch_stage3(q_part, p_part, params)
    files = [("stage1_input_a.rnsv", ct.a)]
    files += [(f"stage1_raised_digit{t}.rnsv", r) for t, r in enumerate(raised)]
    files += [("stage2_acc_q_a.rnsv", q_part.a), ("stage2_acc_q_b.rnsv", q_part.b),
              ("stage2_acc_p_a.rnsv", p_part.a), ("stage2_acc_p_b.rnsv", p_part.b),
              ("stage3_out_a.rnsv", delta.a), ("stage3_out_b.rnsv", delta.b)]
    for name, poly in files:
        save_polynomial(directory / name, poly)
    return [name for name, _ in files]
