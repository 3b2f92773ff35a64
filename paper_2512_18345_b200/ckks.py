"""CKKS evaluation API on top of the rnscope-compatible primitives:
encode / decode, HAdd, PMult, HMult + relinearize, rescale, HRot, conjugate.

The reference package stops at key switching; these entry points
are the north-star additions.  HRot, HMult+relinearize and rescale are defined
as the compositions of reference primitives validated in SURVEY 8c, so they
have a bit-exact oracle (tests/golden/golden.json["composed"]):

  hrot(ct, k)      = keyswitch(automorphism(a, k), automorphism(b, k); evk_{sigma_k(s) -> s})
  hmult+relin      = tensor (d0, d1, d2) by poly_elementwise, keyswitch((d2, d0); evk_{s^2 -> s}),
                     then a += d1
  rescale          = INTT(last limb) -> convert 1 -> L-1 (non-centred) -> NTT
                     -> (x - conv) * q_last^-1                (ModDown with P = {q_last})

encode / decode (canonical embedding, float) have no reference counterpart:
parity unpinned, tolerance-tested only.

A ciphertext at level l lives over the first l limbs of the parameter set's Q
basis; key switching at l < L runs the same pipeline on the active limbs with
a (possibly partial) last digit and the rows of the full-level key that belong
to active limbs.
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np

from . import keyswitch as ks
from .params import ParameterSet
from .rns import COEFFICIENT, EVALUATION, Polynomial, RnsError, StructureError, automorphism, poly_elementwise
from .transform import ntt_polynomial

Ciphertext = ks.Ciphertext


@dataclass
class Plaintext:
    """An encoded message: evaluation-domain polynomial over the first `level`
    limbs, with the scale it was encoded at."""

    poly: Polynomial
    scale: float

    @property
    def level(self) -> int:
        return self.poly.num_limbs


def level_of(ct: Ciphertext) -> int:
    return ct.a.num_limbs


# ---------------------------------------------------------------------------
# canonical embedding (host, float): slots <-> real coefficient vectors
# ---------------------------------------------------------------------------
class Embedding:
    """Slot j of a degree-N polynomial m is m(zeta^(5^j)), zeta = exp(i*pi/N),
    j < N/2; the other N/2 evaluation points carry the conjugates."""

    _cache: dict = {}

    def __new__(cls, n: int):
        hit = cls._cache.get(n)
        if hit is None:
            hit = super().__new__(cls)
            hit._init(n)
            cls._cache[n] = hit
        return hit

    def _init(self, n: int) -> None:
        self.n = n
        two_n = 2 * n
        rot = np.empty(n // 2, dtype=np.int64)
        g = 1
        for j in range(n // 2):
            rot[j] = g
            g = g * 5 % two_n
        self.pos = (rot - 1) // 2                 # index t with 2t+1 = 5^j
        self.neg = (two_n - rot - 1) // 2         # index t with 2t+1 = -5^j
        k = np.arange(n)
        self.twist = np.exp(1j * np.pi * k / n)   # zeta^k

    def to_coeffs(self, slots: np.ndarray) -> np.ndarray:
        """N/2 complex slots -> N real coefficients (float64)."""
        z = np.asarray(slots, dtype=np.complex128)
        if z.shape != (self.n // 2,):
            raise StructureError(f"expected {self.n // 2} slots, got {z.shape}")
        v = np.empty(self.n, dtype=np.complex128)
        v[self.pos] = z
        v[self.neg] = np.conj(z)
        # v[t] = m(zeta^(2t+1)) = sum_k m_k zeta^k e^{2 pi i t k / N}  =>  m_k zeta^k = fft(v)[k] / N
        return np.real(np.fft.fft(v) / self.n * np.conj(self.twist))

    def to_slots(self, coeffs: np.ndarray) -> np.ndarray:
        m = np.asarray(coeffs, dtype=np.float64)
        v = np.fft.ifft(m * self.twist) * self.n
        return v[self.pos]


def galois_element(r: int, n: int) -> int:
    """Automorphism index that rotates the slot vector left by r."""
    return pow(5, r % (n // 2), 2 * n)


def conjugation_element(n: int) -> int:
    return 2 * n - 1


def _round_to_residues(vals: np.ndarray, basis) -> np.ndarray:
    """Real values (already multiplied by the scale, |v| < 2^126) -> canonical residues
    of round(v) modulo every limb.  Extended precision keeps 64 significant bits."""
    v = np.rint(np.asarray(vals, dtype=np.longdouble))
    neg = v < 0
    mag = np.abs(v)
    two32 = np.longdouble(4294967296.0)
    parts = []
    for _ in range(4):                       # 32-bit digits, little endian
        hi = np.floor(mag / two32)
        parts.append((mag - hi * two32).astype(np.uint64))
        mag = hi
    rows = []
    for m in basis:
        q = np.uint64(m.q)
        base = np.uint64((1 << 32) % m.q)
        acc = np.zeros(v.shape, dtype=np.uint64)
        for digit in reversed(parts):
            acc = (acc * base + digit % q) % q
        rows.append(np.where(neg, (q - acc) % q, acc))
    return np.stack(rows)


def encode(values, params: ParameterSet, level: int | None = None, scale: float | None = None,
           basis=None, row_factors=None) -> Plaintext:
    """Complex (or real) slot vector of length N/2 (a scalar broadcasts) ->
    evaluation-domain plaintext at `level` limbs, coefficients round(scale * m).
    `basis` overrides the limb set (e.g. Q_l || P for double-hoisted linear transforms);
    `row_factors[i]` multiplies limb i by a constant (e.g. P mod q_i)."""
    level = params.l if level is None else level
    scale = float(params.delta) if scale is None else float(scale)
    n = params.n
    z = np.asarray(values, dtype=np.complex128)
    if z.ndim == 0:
        z = np.full(n // 2, z)
    coeffs = Embedding(n).to_coeffs(z)
    basis = params.q_basis[:level] if basis is None else tuple(basis)
    rows = _round_to_residues(coeffs.astype(np.longdouble) * np.longdouble(scale), basis)
    if row_factors is not None:
        for i, (m, f) in enumerate(zip(basis, row_factors)):
            rows[i] = rows[i] * np.uint64(f % m.q) % np.uint64(m.q)
    return Plaintext(ntt_polynomial(Polynomial(basis, rows, COEFFICIENT)), scale)


def encode_constant(value: float, params: ParameterSet, level: int, scale: float) -> Plaintext:
    """A real constant in every slot: the constant polynomial round(scale*value),
    whose evaluation-domain image is that residue in every column (no transform)."""
    basis = params.q_basis[:level]
    c = int(round(value * scale))
    rows = np.stack([np.full(params.n, c % m.q, dtype=np.uint64) for m in basis])
    return Plaintext(Polynomial(basis, rows, EVALUATION), scale)


def _centered_coeffs(poly: Polynomial) -> np.ndarray:
    """Coefficient-domain polynomial -> centred real coefficients (float64) by an
    exact mixed-radix (Garner) lift over all limbs present (callers drop to the few
    limbs that cover the value first)."""
    rows = poly.coeffs
    qs = [m.q for m in poly.basis]
    if len(qs) == 1:
        v = rows[0].astype(np.int64)
        return np.where(v > qs[0] // 2, v - qs[0], v).astype(np.float64)
    value = rows[0].astype(object)
    radix = qs[0]
    for i in range(1, len(qs)):
        q = qs[i]
        inv = pow(radix, -1, q)
        digit = ((rows[i].astype(object) - value) * inv) % q
        value = value + digit * radix
        radix *= q
    half = radix // 2
    return np.array([float(x - radix) if x > half else float(x) for x in value])


def limbs_needed(scale: float, bound: float = 64.0) -> int:
    """Limbs whose product safely exceeds 2 * scale * bound (31-bit limbs)."""
    return max(1, math.ceil((math.log2(scale * bound) + 2) / 30.0))


def decode(pt: Plaintext, params: ParameterSet) -> np.ndarray:
    coeff = ntt_polynomial(pt.poly, "inverse")
    return Embedding(params.n).to_slots(_centered_coeffs(coeff) / pt.scale)


def encrypt(pt: Plaintext, sk: ks.SecretKey, params: ParameterSet, seed: int = 0) -> Ciphertext:
    """Fresh encryption of an encoded plaintext at its level (same sampling
    recipe as the reference's encrypt, keyswitch.py:124-149, on the plaintext's basis)."""
    basis = pt.poly.basis
    rng = np.random.default_rng(seed)
    a = Polynomial(basis, ks._uniform_rows(basis, params.n, rng), EVALUATION)
    e = ks._gaussian(params.n, rng)
    e_eval = ntt_polynomial(Polynomial(basis, ks._signed_rows(e, basis), COEFFICIENT))
    payload = poly_elementwise(pt.poly, e_eval, "add")
    b = poly_elementwise(payload, poly_elementwise(a, sk.eval_polynomial(basis), "mul"), "sub")
    return Ciphertext(a=a, b=b, scale=pt.scale)


def decrypt(ct: Ciphertext, sk: ks.SecretKey) -> Plaintext:
    basis = ct.a.basis
    d = poly_elementwise(ct.b, poly_elementwise(ct.a, sk.eval_polynomial(basis), "mul"), "add")
    return Plaintext(d, ct.scale)


def decrypt_decode(ct: Ciphertext, sk: ks.SecretKey, params: ParameterSet) -> np.ndarray:
    ct = mod_drop(ct, min(level_of(ct), limbs_needed(ct.scale)))
    return decode(decrypt(ct, sk), params)


# ---------------------------------------------------------------------------
# keys
# ---------------------------------------------------------------------------
def rotated_secret(sk: ks.SecretKey, k: int) -> ks.SecretKey:
    """sigma_k(s): the secret under X -> X^k (coefficient i -> i*k mod 2N with sign)."""
    n = sk.n
    dest = (np.arange(n, dtype=np.int64) * (k % (2 * n))) % (2 * n)
    out = np.zeros(n, dtype=np.int8)
    out[dest % n] = np.where(dest >= n, -sk.ternary, sk.ternary)
    return ks.SecretKey(ternary=out, n=n)


def galois_keygen(sk: ks.SecretKey, params: ParameterSet, k: int, seed: int = 0) -> ks.SwitchingKey:
    """Switching key sigma_k(s) -> s for the automorphism X -> X^k."""
    return ks.switching_keygen(rotated_secret(sk, k), sk, params, seed=seed)


def relin_keygen(sk: ks.SecretKey, params: ParameterSet, seed: int = 0) -> ks.SwitchingKey:
    """Switching key s^2 -> s.  s^2 is not ternary, so it is injected as an
    evaluation-domain polynomial (the route validated in SURVEY 8c)."""
    ext = params.ext_basis
    s_ext = sk.eval_polynomial(ext)
    squared = ks.SecretKey(ternary=np.zeros(params.n, dtype=np.int8), n=params.n)
    squared._eval_cache[tuple(m.q for m in ext)] = poly_elementwise(s_ext, s_ext, "mul")
    return ks.switching_keygen(squared, sk, params, seed=seed)


@dataclass
class EvaluationKeys:
    """Relinearisation key plus Galois keys by automorphism index."""

    params: ParameterSet
    relin: ks.SwitchingKey | None = None
    galois: dict = field(default_factory=dict)

    def add_rotation(self, sk, r: int, seed: int = 0) -> None:
        k = galois_element(r, self.params.n)
        if k not in self.galois:
            self.galois[k] = galois_keygen(sk, self.params, k, seed=seed)

    def add_conjugation(self, sk, seed: int = 0) -> None:
        k = conjugation_element(self.params.n)
        if k not in self.galois:
            self.galois[k] = galois_keygen(sk, self.params, k, seed=seed)


# ---------------------------------------------------------------------------
# evaluation
# ---------------------------------------------------------------------------
def _same_level(x, y) -> None:
    if tuple(m.q for m in x.basis) != tuple(m.q for m in y.basis):
        raise StructureError("operands live at different levels")


def _close(s1: float, s2: float) -> bool:
    return abs(s1 - s2) <= 1e-9 * max(abs(s1), abs(s2))


def mod_drop(ct: Ciphertext, level: int) -> Ciphertext:
    """Discard limbs above `level` (message and scale unchanged)."""
    if level == level_of(ct):
        return ct
    if not 0 < level <= level_of(ct):
        raise RnsError(f"cannot drop from level {level_of(ct)} to {level}")
    sl = slice(0, level)
    return Ciphertext(a=ct.a.rows(sl), b=ct.b.rows(sl), scale=ct.scale)


def _drop_plain(pt: Plaintext, level: int) -> Polynomial:
    return pt.poly if pt.level == level else pt.poly.rows(slice(0, level))


def _halves(ct: Ciphertext):
    """The [2, l, n] allocation behind a kernel-produced ciphertext, or None when its halves
    are separate tensors."""
    a, b = ct.a.data, ct.b.data
    base = getattr(a, "_base", None)
    if base is not None and base is getattr(b, "_base", None) and base.dim() == 3 and base.shape[0] == 2 \
            and base.data_ptr() == a.data_ptr() and a.data_ptr() + a.numel() * 4 == b.data_ptr():
        return base
    return None


def _both_halves(x: Ciphertext, y: Ciphertext, kind: str, scale: float) -> Ciphertext:
    """x (op) y on both halves.  When both operands are single [2, l, n] allocations this is
    one launch over 2 l rows and the result is again one allocation (so that the next tensor /
    key switch reads it without a gathering copy); otherwise one launch per half
    (poly_elementwise "add" / "sub", rns.py:243-258)."""
    xt, yt = _halves(x), _halves(y)
    if xt is None or yt is None or x.a.domain != y.a.domain or x.a.domain != x.b.domain:
        return Ciphertext(a=poly_elementwise(x.a, y.a, kind), b=poly_elementwise(x.b, y.b, kind), scale=scale)
    from .engine import get_engine
    from .instrument import counters
    from .rns import _KIND_CODE

    eng = get_engine()
    level, n = xt.shape[1], xt.shape[2]
    out = eng.empty(2, level, n)
    eng.elementwise(xt.view(2 * level, n), yt.view(2 * level, n), eng.row_slots(x.a.basis, repeat=2),
                    _KIND_CODE[kind], out=out.view(2 * level, n))
    counters.elementwise += 2 * level * n
    return Ciphertext(a=Polynomial(x.a.basis, out[0], x.a.domain), b=Polynomial(x.a.basis, out[1], x.a.domain),
                      scale=scale)


def add(x: Ciphertext, y: Ciphertext) -> Ciphertext:
    _same_level(x.a, y.a)
    if not _close(x.scale, y.scale):
        raise RnsError(f"scale mismatch in add: {x.scale} vs {y.scale}")
    return _both_halves(x, y, "add", x.scale)


def sub(x: Ciphertext, y: Ciphertext) -> Ciphertext:
    _same_level(x.a, y.a)
    if not _close(x.scale, y.scale):
        raise RnsError(f"scale mismatch in sub: {x.scale} vs {y.scale}")
    return _both_halves(x, y, "sub", x.scale)


def add_plain(ct: Ciphertext, pt: Plaintext) -> Ciphertext:
    if not _close(ct.scale, pt.scale):
        raise RnsError(f"scale mismatch in add_plain: {ct.scale} vs {pt.scale}")
    return Ciphertext(a=ct.a, b=poly_elementwise(ct.b, _drop_plain(pt, level_of(ct)), "add"), scale=ct.scale)


def mul_plain(ct: Ciphertext, pt: Plaintext) -> Ciphertext:
    """PMult: slot-wise product with an encoded plaintext; scales multiply."""
    p = _drop_plain(pt, level_of(ct))
    xt = _halves(ct)
    if xt is not None and ct.a.domain == EVALUATION and p.domain == EVALUATION and ct.a.n % 4 == 0 \
            and tuple(m.q for m in p.basis) == tuple(m.q for m in ct.a.basis):
        # both halves against the same plaintext in one pass, result in one allocation
        from .engine import get_engine
        from .instrument import counters

        eng = get_engine()
        out = eng.fused_terms([xt], [p.data], eng.row_slots(ct.a.basis))
        counters.elementwise += 2 * xt.shape[1] * xt.shape[2]
        return Ciphertext(a=Polynomial(ct.a.basis, out[0], EVALUATION), b=Polynomial(ct.a.basis, out[1], EVALUATION),
                          scale=ct.scale * pt.scale)
    return Ciphertext(a=poly_elementwise(ct.a, p, "mul"), b=poly_elementwise(ct.b, p, "mul"),
                      scale=ct.scale * pt.scale)


def ct_tensor(ct: Ciphertext):
    """[2, l, n] device tensor of a ciphertext (a view when a and b are adjacent halves
    of one allocation, as every kernel-produced ciphertext is; a copy otherwise)."""
    import torch

    base = _halves(ct)
    return base if base is not None else torch.stack([ct.a.data, ct.b.data])


def ct_term(ct: Ciphertext):
    """A ciphertext as a term of Engine.fused_terms: its [2, l, n] tensor when the halves are adjacent,
    the pair of halves otherwise (the kernel takes them separately: no gathering copy)."""
    base = _halves(ct)
    return base if base is not None else (ct.a.data, ct.b.data)


def ct_from_tensor(t, basis, scale) -> Ciphertext:
    return Ciphertext(a=Polynomial(basis, t[0], EVALUATION), b=Polynomial(basis, t[1], EVALUATION), scale=scale)


def tensor(x: Ciphertext, y: Ciphertext):
    """(d0, d1, d2) with d0 + d1*s + d2*s^2 = (b1 + a1 s)(b2 + a2 s): d0 = b1*b2,
    d1 = a1*b2 + a2*b1, d2 = a1*a2 (each a poly_elementwise product), one fused kernel."""
    _same_level(x.a, y.a)
    from .engine import get_engine

    eng = get_engine()
    basis = x.a.basis
    if x.a.n % 4:
        d0 = poly_elementwise(x.b, y.b, "mul")
        d1 = poly_elementwise(poly_elementwise(x.a, y.b, "mul"), poly_elementwise(y.a, x.b, "mul"), "add")
        return d0, d1, poly_elementwise(x.a, y.a, "mul")
    d = eng.tensor_halves(x.a.data, x.b.data, y.a.data, y.b.data, eng.row_slots(basis))
    return tuple(Polynomial(basis, d[i], EVALUATION) for i in range(3))


def keyswitch_level(ct: Ciphertext, evk: ks.SwitchingKey) -> Ciphertext:
    """keyswitch for a ciphertext over the first l <= L limbs of evk.params."""
    params = evk.params
    level = level_of(ct)
    if level == params.l:
        return ks.keyswitch(ct, evk)
    basis = params.q_basis[:level]
    if tuple(m.q for m in ct.a.basis) != tuple(m.q for m in basis):
        raise StructureError("ciphertext basis is not a prefix of the parameter q-basis")
    from .engine import get_engine

    eng = get_engine()
    plan = eng.ks_plan(params.n, basis, params.p_basis, params.alpha, params.l + params.alpha, params.l)
    out = eng.keyswitch(plan, ct.a.data, ct.b.data, evk.matrix())
    return Ciphertext(a=Polynomial(basis, out[0], EVALUATION), b=Polynomial(basis, out[1], EVALUATION),
                      scale=ct.scale)


def relinearize(d0: Polynomial, d1: Polynomial, d2: Polynomial, rlk: ks.SwitchingKey, scale) -> Ciphertext:
    sw = keyswitch_level(Ciphertext(a=d2, b=d0, scale=scale), rlk)
    return Ciphertext(a=poly_elementwise(sw.a, d1, "add"), b=sw.b, scale=scale)


def hmult(x: Ciphertext, y: Ciphertext, rlk: ks.SwitchingKey) -> Ciphertext:
    """HMult + relinearize (no rescale); scale = x.scale * y.scale."""
    d0, d1, d2 = tensor(x, y)
    return relinearize(d0, d1, d2, rlk, x.scale * y.scale)


def hmult_rescale(x: Ciphertext, y: Ciphertext, rlk: ks.SwitchingKey, k: int = 1,
                  addend: Ciphertext | None = None) -> Ciphertext:
    """rescale(hmult(x, y), k) with the relinearisation ModDown and the rescale merged into
    one division by P * (the k dropped limbs): one base conversion and one NTT fewer per
    multiplication.  Same value as the two-step route up to the rounding of the division."""
    from .engine import get_engine

    _same_level(x.a, y.a)
    eng = get_engine()
    params = rlk.params
    level = level_of(x)
    n = x.a.n
    if addend is not None and (n != 65536 or level <= k):
        # `addend` (a ciphertext at the output level, same scale up to the caller) rides in the
        # ModDown epilogue of the fused pipeline only; elsewhere it is a separate add
        out = hmult_rescale(x, y, rlk, k)
        return add(Ciphertext(a=out.a, b=out.b, scale=addend.scale), addend)
    if n % 4 or level <= k:
        return rescale(hmult(x, y, rlk), k)
    basis = x.a.basis
    if tuple(m.q for m in basis) != tuple(m.q for m in params.q_basis[:level]):
        raise StructureError("ciphertext basis is not a prefix of the parameter q-basis")
    rest, dropped = basis[:level - k], basis[level - k:]
    ks_plan = eng.ks_plan(n, basis, params.p_basis, params.alpha, params.l + params.alpha, params.l)
    md_plan = eng.moddown_plan(n, rest, dropped + params.p_basis)
    if n == 65536:
        # no tensor pass: d2 is formed while the first inverse transform loads, d1 / d0 inside the
        # inner product (same limbs as the two-call route below)
        if addend is not None and level_of(addend) != level - k:
            raise RnsError("addend must live at the output level of hmult_rescale")
        out = eng.hmult_relin_rescale(ks_plan, md_plan, x.a.data, x.b.data, y.a.data, y.b.data,
                                      rlk.matrix(), level - k,
                                      None if addend is None else addend.a.data,
                                      None if addend is None else addend.b.data)
    else:
        d = eng.tensor_halves(x.a.data, x.b.data, y.a.data, y.b.data, eng.row_slots(basis))
        out = eng.ks_relin_rescale(ks_plan, md_plan, d, rlk.matrix(), level - k)
    return Ciphertext(a=Polynomial(rest, out[0], EVALUATION), b=Polynomial(rest, out[1], EVALUATION),
                      scale=x.scale * y.scale / math.prod(m.q for m in dropped))


def hmult_sum_rescale(pairs, rlk: ks.SwitchingKey, k: int = 1) -> Ciphertext:
    """rescale(relinearize(sum_i x_i * y_i), k) with ONE key switch for the whole sum (lazy
    relinearisation): the tensor products (d0, d1, d2) of the pairs are added limb-wise before
    the relinearisation.  All operands at one level, all products at one scale."""
    from .engine import get_engine

    eng = get_engine()
    params = rlk.params
    x0, y0 = pairs[0]
    level, n, basis = level_of(x0), x0.a.n, x0.a.basis
    scale = x0.scale * y0.scale
    for x, y in pairs:
        _same_level(x.a, x0.a)
        _same_level(y.a, x0.a)
        if not _close(x.scale * y.scale, scale):
            raise RnsError(f"scale mismatch in hmult_sum_rescale: {x.scale * y.scale} vs {scale}")
    if n % 4 or level <= k:
        raise RnsError("hmult_sum_rescale needs n % 4 == 0 and more than k limbs")
    if tuple(m.q for m in basis) != tuple(m.q for m in params.q_basis[:level]):
        raise StructureError("ciphertext basis is not a prefix of the parameter q-basis")
    slots3 = eng.row_slots(basis, repeat=3)
    d = None
    for x, y in pairs:
        t = eng.tensor_halves(x.a.data, x.b.data, y.a.data, y.b.data, eng.row_slots(basis))
        if d is None:
            d = t
        else:
            eng.elementwise(d.view(3 * level, n), t.view(3 * level, n), slots3, 0, out=d.view(3 * level, n))
    rest, dropped = basis[:level - k], basis[level - k:]
    ks_plan = eng.ks_plan(n, basis, params.p_basis, params.alpha, params.l + params.alpha, params.l)
    md_plan = eng.moddown_plan(n, rest, dropped + params.p_basis)
    out = eng.ks_relin_rescale(ks_plan, md_plan, d, rlk.matrix(), level - k)
    return Ciphertext(a=Polynomial(rest, out[0], EVALUATION), b=Polynomial(rest, out[1], EVALUATION),
                      scale=scale / math.prod(m.q for m in dropped))


def rescale(ct: Ciphertext, k: int = 1) -> Ciphertext:
    """Drop the last k limbs, dividing message and scale by their product P: one ModDown
    pass with P = the dropped limbs, (x_rest - NTT(BConv_{P -> rest}(INTT(x_P)))) * P^-1.
    For k = 1 this is the single-limb RNS rescale of the reference composition
    (bit-exact); for k > 1 it divides by the product in one pass instead of
    k successive single-limb passes (same value up to the rounding of the floor)."""
    from .engine import get_engine

    if k < 1:
        return ct
    eng = get_engine()
    level = level_of(ct)
    if level <= k:
        raise RnsError("no limb left to rescale by")
    basis = ct.a.basis
    rest, dropped = basis[:level - k], basis[level - k:]
    plan = eng.moddown_plan(ct.a.n, rest, dropped)
    a, b = ct.a.data, ct.b.data
    out = eng.ks_stage3(plan, a[:level - k], b[:level - k], a[level - k:], b[level - k:])
    return Ciphertext(a=Polynomial(rest, out[0], EVALUATION), b=Polynomial(rest, out[1], EVALUATION),
                      scale=ct.scale / math.prod(m.q for m in dropped))


def apply_galois(ct: Ciphertext, k: int, evk: ks.SwitchingKey) -> Ciphertext:
    """Automorphism X -> X^k on both halves, then key switch sigma_k(s) -> s."""
    moved = Ciphertext(a=automorphism(ct.a, k), b=automorphism(ct.b, k), scale=ct.scale)
    return keyswitch_level(moved, evk)


def hrot(ct: Ciphertext, r: int, keys: EvaluationKeys) -> Ciphertext:
    """Rotate the slot vector left by r."""
    n = ct.a.n
    if r % (n // 2) == 0:
        return ct
    k = galois_element(r, n)
    if k not in keys.galois:
        raise RnsError(f"no Galois key for rotation {r}")
    return apply_galois(ct, k, keys.galois[k])


def hrot_hoisted(ct: Ciphertext, rotations, keys: EvaluationKeys) -> dict:
    """Several rotations of one ciphertext sharing a single ModUp (hoisting): returns
    {r: [2, l, n] ciphertext tensor}.  Independent rotations run on the engine's lanes."""
    from .engine import get_engine

    eng = get_engine()
    params = keys.params
    level = level_of(ct)
    n = ct.a.n
    basis = ct.a.basis
    out = {}
    todo = []
    for r in rotations:
        if r % (n // 2) == 0:
            out[r] = ct_tensor(ct)
        else:
            k = galois_element(r, n)
            if k not in keys.galois:
                raise RnsError(f"no Galois key for rotation {r}")
            todo.append((r, k))
    if todo:
        plan = eng.ks_plan(n, basis, params.p_basis, params.alpha, params.l + params.alpha, params.l)
        beta = -(-level // params.alpha)
        raised = eng.ks_stage1(plan, ct.a.data, beta, level + params.alpha)
        b = ct.b.data
        res = eng.fork([(lambda k=k: eng.ks_hoisted(plan, raised, k, keys.galois[k].matrix(), b))
                        for _, k in todo])
        for (r, _), t in zip(todo, res):
            out[r] = t
    return out


def apply_galois_fused(ct: Ciphertext, k: int, evk: ks.SwitchingKey) -> Ciphertext:
    """sigma_k followed by its key switch WITHOUT a separate automorphism pass: ModUp of the
    unrotated a part, the rotation applied as a gather inside the inner product and the ModDown
    (the single-rotation case of hoisting).  sigma_k commutes with ModUp only up to a multiple
    of the digit modulus, so the result equals apply_galois up to key-switch noise, not limb
    for limb: hrot / conjugate keep the reference composition, application circuits use this."""
    from .engine import get_engine

    eng = get_engine()
    params = evk.params
    level, n, basis = level_of(ct), ct.a.n, ct.a.basis
    if n % 4:
        return apply_galois(ct, k, evk)
    plan = eng.ks_plan(n, basis, params.p_basis, params.alpha, params.l + params.alpha, params.l)
    raised = eng.ks_stage1(plan, ct.a.data, -(-level // params.alpha), level + params.alpha)
    out = eng.ks_hoisted(plan, raised, k, evk.matrix(), ct.b.data)
    return ct_from_tensor(out, basis, ct.scale)


def hrot_fused(ct: Ciphertext, r: int, keys: EvaluationKeys) -> Ciphertext:
    """hrot through apply_galois_fused (same message, different noise)."""
    n = ct.a.n
    if r % (n // 2) == 0:
        return ct
    k = galois_element(r, n)
    if k not in keys.galois:
        raise RnsError(f"no Galois key for rotation {r}")
    return apply_galois_fused(ct, k, keys.galois[k])


def conjugate_fused(ct: Ciphertext, keys: EvaluationKeys) -> Ciphertext:
    k = conjugation_element(ct.a.n)
    if k not in keys.galois:
        raise RnsError("no conjugation key")
    return apply_galois_fused(ct, k, keys.galois[k])


def conjugate(ct: Ciphertext, keys: EvaluationKeys) -> Ciphertext:
    k = conjugation_element(ct.a.n)
    if k not in keys.galois:
        raise RnsError("no conjugation key")
    return apply_galois(ct, k, keys.galois[k])


def mul_const(ct: Ciphertext, value: float, params: ParameterSet, out_scale: float | None = None,
              drop: int = 1) -> Ciphertext:
    """Multiply by a real constant and rescale by `drop` limbs so that the
    result has exactly `out_scale` (default: the input scale)."""
    level = level_of(ct)
    out_scale = ct.scale if out_scale is None else out_scale
    dropped = math.prod(m.q for m in ct.a.basis[level - drop:])
    pt = encode_constant(value, params, level, out_scale * dropped / ct.scale)
    out = rescale(mul_plain(ct, pt), drop)
    return Ciphertext(a=out.a, b=out.b, scale=out_scale)


def capture(fn, *sample_cts: Ciphertext):
    """Record `fn(*ciphertexts) -> ciphertext` (any composition of the operations above: key
    switches, HMult + relinearise + rescale chains, rotations) into ONE CUDA graph and return
    replay(*ciphertexts) -> ciphertext with the same result limbs as the eager call.  The
    launch overhead of a many-kernel circuit is what capture removes (SURVEY
    section 7 step 8): at N = 2^13 (BASELINE config 1) an HMult + relinearise + rescale is ~15
    launches of a few microseconds each.  Operands must keep the sample's level, basis and scale.
    Like Bootstrapper.capture, the graph holds pointers into the key-switch workspace arena: a
    replay after the arena moved raises."""
    import torch

    from .engine import get_engine

    eng = get_engine()
    statics = [torch.stack([c.a.data, c.b.data]).clone() for c in sample_cts]
    views = [ct_from_tensor(t, c.a.basis, c.scale) for t, c in zip(statics, sample_cts)]
    fn(*views)                                             # warm-up: plans, tables, constants
    torch.cuda.synchronize()
    graph = torch.cuda.CUDAGraph()
    side = torch.cuda.Stream(device=eng.device)
    side.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(side):
        fn(*views)                                         # settle allocator state on the capture stream
        torch.cuda.synchronize()
        with torch.cuda.graph(graph, stream=side):
            out = fn(*views)
            static_out = ct_tensor(out)
    torch.cuda.current_stream().wait_stream(side)
    out_basis, out_scale = out.a.basis, out.scale
    generation = eng.arena_generation()

    def replay(*cts: Ciphertext, copy_out: bool = True) -> Ciphertext:
        if eng.arena_generation() != generation:
            raise RnsError("the workspace arena was reallocated after this graph was captured: capture again")
        if len(cts) != len(statics):
            raise StructureError(f"captured with {len(statics)} operands, called with {len(cts)}")
        for t, c, s in zip(statics, cts, sample_cts):
            if c.a.basis != s.a.basis or not _close(c.scale, s.scale):
                raise StructureError("operand level / basis / scale differs from the captured sample")
            t[0].copy_(c.a.data, non_blocking=True)
            t[1].copy_(c.b.data, non_blocking=True)
        graph.replay()
        return ct_from_tensor(static_out.clone() if copy_out else static_out, out_basis, out_scale)

    replay.graph, replay.static_in, replay.static_out = graph, statics, static_out
    return replay
