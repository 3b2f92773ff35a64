"""CKKS bootstrapping for fully packed ciphertexts (N/2 complex slots):
ModRaise -> CoeffToSlot -> EvalMod -> SlotToCoeff, every arithmetic step on the
GPU through the kernels of csrc/ (key switching, automorphism, PMult
accumulate, rescale), host code only orchestrates.

The reference ships no bootstrapping; this module has no
reference oracle (parity unpinned) and is checked by decoded-slot
precision against the input message.

Circuit
  * ModRaise: exact centred lift of the two bottom limbs to the full basis.
    The lifted polynomial is t = Delta*m + e + Q0*I with small integer I
    (sparse secret, h = params.h_sparse).
  * CoeffToSlot / SlotToCoeff: the special-FFT factorisation of the canonical
    embedding (the decode map of ckks.Embedding), log2(n) butterfly stages of
    three diagonals each, merged into a few groups and evaluated with
    baby-step/giant-step rotations.  The bit reversal is skipped on both sides
    (EvalMod is slot-wise).  One limb per group (plaintext scale = that limb).
  * EvalMod: E = exp(2*pi*i*t / (Q0 * 2^r)) by a degree-d polynomial (Chebyshev interpolation),
    r squarings, then (Q0 / (2*pi*Delta)) * sin = Im(E) scaled; real and
    imaginary coefficient halves are processed as two ciphertexts.  Two limbs
    per multiplicative level (scale ~ 2^62 on 31-bit limbs).
"""
from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np

from . import ckks
from . import keyswitch as ks
from .params import ParameterSet
from .rns import EVALUATION, Polynomial, RnsError
from .transform import ntt_polynomial


# ---------------------------------------------------------------------------
# diagonal algebra on n-slot vectors (host, float)
# ---------------------------------------------------------------------------
def _rot(v: np.ndarray, d: int) -> np.ndarray:
    """Left rotation: out[p] = v[p + d]."""
    return np.roll(v, -d)


def dft_stage(n: int, ell: int, inverse: bool) -> dict[int, np.ndarray]:
    """Butterfly stage `ell` (block length 2^ell) of the special FFT on n slots,
    or its inverse, as {rotation offset: diagonal}: out = sum_d diag_d * rot(in, d)."""
    length = 1 << ell
    half = length >> 1
    p = np.arange(n)
    j = p % length
    first = j < half
    jj = np.where(first, j, j - half)
    pw = np.ones(half, dtype=np.int64)
    for t in range(1, half):
        pw[t] = pw[t - 1] * 5 % (4 * length)
    xi = np.exp(2j * np.pi * pw[jj] / (4 * length))
    z = np.zeros(n, dtype=np.complex128)
    if not inverse:
        d0 = np.where(first, 1.0 + 0j, -xi)
        dp = np.where(first, xi, z)             # takes in[p + half]
        dm = np.where(first, z, 1.0 + 0j)       # takes in[p - half]
    else:
        d0 = np.where(first, 0.5 + 0j, -0.5 * np.conj(xi))
        dp = np.where(first, 0.5 + 0j, z)
        dm = np.where(first, z, 0.5 * np.conj(xi))
    out = {0: d0}
    for off, vec in ((half % n, dp), ((-half) % n, dm)):
        out[off] = out[off] + vec if off in out else vec
    return out


def compose(a: dict, b: dict, n: int) -> dict:
    """Diagonals of A*B (B applied first)."""
    out: dict[int, np.ndarray] = {}
    for d1, va in a.items():
        for d2, vb in b.items():
            d = (d1 + d2) % n
            term = va * _rot(vb, d1)
            out[d] = out[d] + term if d in out else term
    return {d: v for d, v in out.items() if np.abs(v).max() > 0}


def apply_diagonals(diags: dict, x: np.ndarray) -> np.ndarray:
    return sum(v * _rot(x, d) for d, v in diags.items())


def grouped_dft(n: int, group_sizes: list[int], inverse: bool) -> list[dict]:
    """The n-slot special FFT without its bit reversal (or the inverse), as
    merged groups of stages in application order."""
    lg = n.bit_length() - 1
    assert sum(group_sizes) == lg
    stages = list(range(1, lg + 1))
    groups = []
    at = 0
    if not inverse:                      # S_lg ... S_1: stage 1 first
        for size in group_sizes:
            acc = None
            for ell in stages[at:at + size]:
                st = dft_stage(n, ell, False)
                acc = st if acc is None else compose(st, acc, n)
            groups.append(acc)
            at += size
    else:                                # S_1^-1 ... S_lg^-1: stage lg first
        order = stages[::-1]
        for size in group_sizes:
            acc = None
            for ell in order[at:at + size]:
                st = dft_stage(n, ell, True)
                acc = st if acc is None else compose(st, acc, n)
            groups.append(acc)
            at += size
    return groups


def default_groups(lg: int, count: int = 3) -> list[int]:
    base, extra = divmod(lg, count)
    return [base + (1 if i < extra else 0) for i in range(count)]


# ---------------------------------------------------------------------------
# homomorphic linear transform (BSGS)
# ---------------------------------------------------------------------------
ct_tensor = ckks.ct_tensor
ct_from_tensor = ckks.ct_from_tensor


def p_ok(lt) -> bool:
    """The merged finish (ks_finish_rescale) is available: vector kernels need n % 4 == 0."""
    return lt.double_hoist and lt.params.n % 4 == 0 and lt.level > lt.limbs


class LinearTransform:
    """y = sum_d diag_d * rot(x, d) with offsets d = g*n1*step + b*step (mod n):
    inner_g = sum_b rot(diag_d, -g*n1*step) * rot(x, b*step);  y = sum_g rot(inner_g, g*n1*step).
    Diagonals are encoded once at `level` limbs with scale = the product of the last
    `limbs` of them, so PMult + rescale by those limbs leaves the ciphertext scale
    unchanged (two limbs where 2^-31 relative plaintext precision is not enough)."""

    def __init__(self, diags: dict, params: ParameterSet, level: int, n1: int | None = None,
                 factor: complex = 1.0, limbs: int = 1, double_hoist: bool = True, fuse_baby_steps: bool = True,
                 keep_b_qp: bool = True):
        n = params.n // 2
        self.fuse_baby_steps = fuse_baby_steps
        # moving giant steps: scale down only the a half of the inner sum, keep the b half over Q||P
        # (False: ModDown both halves and lift the b half again, the round-1 schedule)
        self.keep_b_qp = keep_b_qp
        self.params, self.level, self.n, self.limbs = params, level, n, limbs
        self.double_hoist = double_hoist
        offs = sorted(diags)
        signed = [d if d <= n // 2 else d - n for d in offs]
        nz = [abs(d) for d in signed if d]
        step = math.gcd(*nz) if nz else 1
        units = [d // step for d in signed]
        span = max(units) - min(units) + 1
        if n1 is None:
            n1 = 1 << max(0, round(math.log2(math.sqrt(span))))
            if double_hoist:
                # baby steps cost one inner product each (no ModUp, no ModDown), giant steps a
                # ModUp + inner product + a ModDown of (half of) their inner sum: favour more baby
                # steps, up to the 16 the fused kernel takes (measured at ks48, profiles/boot_n1.py:
                # 16 everywhere 8.79 ms, 8 in the first / last group 8.87, 8 everywhere 10.2)
                n1 = min(4 * n1, 16)
        self.step, self.n1 = step, n1
        self.pt_scale = float(math.prod(m.q for m in params.q_basis[level - limbs:level]))
        ext_basis = params.q_basis[:level] + params.p_basis
        p_prod = math.prod(m.q for m in params.p_basis)
        lift = [p_prod % m.q for m in params.q_basis[:level]] + [0] * len(params.p_basis)
        table: dict[int, dict[int, ckks.Plaintext]] = {}
        for d, u in zip(offs, units):
            g, b = divmod(u, n1)                      # floor division: b in [0, n1)
            vec = _rot(diags[d] * factor, -g * n1 * step)
            if double_hoist:
                # plaintexts over Q_l || P; the unrotated term multiplies the ciphertext lifted to
                # Q||P, i.e. times P on the Q limbs and zero on the P limbs: fold that into it
                pt = ckks.encode(vec, params, scale=self.pt_scale, basis=ext_basis,
                                 row_factors=lift if b == 0 else None)
            else:
                pt = ckks.encode(vec, params, level=level, scale=self.pt_scale)
            table.setdefault(g, {})[b] = pt
        self.table = table
        self.baby = sorted({b for row in table.values() for b in row})
        self.giants = sorted(table)

    def _fused_ok(self, eng) -> bool:
        """The fused baby-step kernel (bsgs_inner) takes this transform."""
        beta = -(-self.level // self.params.alpha)
        return self.params.n % 2 == 0 and len(self.baby) <= 16 and beta <= 4 and self.fuse_baby_steps

    def _bsgs_prepare(self, ct, keys, eng):
        """ModUp of the input and the argument lists of the fused baby-step kernel (everything of a
        double-hoisted transform that precedes the bsgs_inner launch)."""
        p = self.params
        n_ring, level, alpha = p.n, self.level, p.alpha
        ext = level + alpha
        plan = eng.ks_plan(n_ring, ct.a.basis, p.p_basis, alpha, p.l + alpha, p.l)
        raised = eng.ks_stage1(plan, ct.a.data, -(-level // alpha), ext)
        babies = list(self.baby)
        ks_idx, evks = [], []
        for b in babies:
            if b == 0:
                ks_idx.append(0)
                evks.append(None)
                continue
            k = ckks.galois_element(b * self.step, n_ring)
            if k not in keys.galois:
                raise RnsError(f"no Galois key for rotation {b * self.step}")
            ks_idx.append(k)
            evks.append(keys.galois[k].matrix())
        # the unrotated giant step first, the moving ones after it in one allocation (so that a
        # batched ModDown can take them as one [count, 2, ext, n] slice)
        order = [g for g in self.giants if g == 0] + [g for g in self.giants if g != 0]
        chunks = []
        for g0 in range(0, len(order), 8):
            chunk = order[g0:g0 + 8]
            chunks.append((chunk, [[self.table[g][b].poly.data if b in self.table[g] else None for b in babies]
                                   for g in chunk]))
        return {"plan": plan, "raised": raised, "ks": ks_idx, "evks": evks, "chunks": chunks, "ext": ext}

    def _double_hoisted_inner(self, ct, keys, eng, qps=None):
        """Baby steps as raw Q||P accumulators sharing one ModUp; returns inner_sum(g) that
        forms sum_b pt_{g,b} * u_b over Q||P in one fused pass and scales it down once.
        `qps`: the giant steps' Q||P accumulators when a batched launch (apply_batch) has already
        formed them."""
        import torch

        p = self.params
        n_ring, level, alpha = p.n, self.level, p.alpha
        ext = level + alpha
        basis = ct.a.basis
        plan = eng.ks_plan(n_ring, basis, p.p_basis, alpha, p.l + alpha, p.l)
        giants = self.giants
        if qps is not None:
            pass
        elif self._fused_ok(eng):
            # baby steps and inner sums in ONE pass: each rotated accumulator is formed in
            # registers and multiplied into every giant step's sum, never written
            pre = self._bsgs_prepare(ct, keys, eng)
            qps = {}
            for chunk, table in pre["chunks"]:
                qps.update(zip(chunk, eng.bsgs_inner(plan, pre["raised"], ct.a.data, ct.b.data, pre["ks"], pre["evks"],
                                                     table, ext)))
        else:
            ext_slots = eng.row_slots(basis + p.p_basis)
            raised = eng.ks_stage1(plan, ct.a.data, -(-level // alpha), ext)
            b_half = ct.b.data
            moving = [b for b in self.baby if b]

            def raw(b):
                k = ckks.galois_element(b * self.step, n_ring)
                if k not in keys.galois:
                    raise RnsError(f"no Galois key for rotation {b * self.step}")
                return eng.ks_hoisted_raw(plan, raised, k, keys.galois[k].matrix(), b_half, ext)

            qps = {}
            acc = dict(zip(moving, eng.fork([(lambda b=b: raw(b)) for b in moving])))
            if 0 in self.baby:
                x = ckks.ct_tensor(ct)
                acc[0] = torch.cat([x, torch.zeros((2, alpha, n_ring), dtype=x.dtype, device=x.device)], dim=1)
            # every giant step's inner sum over Q||P in one pass (each baby step read once) ...
            babies = sorted(acc)
            for g0 in range(0, len(giants), 8):
                chunk = giants[g0:g0 + 8]
                table = [[self.table[g][b].poly.data if b in self.table[g] else None for b in babies] for g in chunk]
                qps.update(zip(chunk, eng.fused_terms_multi([acc[b] for b in babies], table, ext_slots)))

        def inner_sum(g):
            # ... then one ModDown per giant step
            qp = qps[g]
            return eng.ks_stage3(plan, qp[0, :level], qp[1, :level], qp[0, level:], qp[1, level:])

        inner_sum.raw = qps          # the Q||P accumulators themselves (giant step 0 needs no ModDown)

        def inner_sums(gs):
            """ModDown of several giant steps' inner sums; one set of launches per run of up to
            four accumulators that are adjacent in memory, over that many of the caller's lanes."""
            out = {}
            width = min(4, eng.lane_count())
            i = 0
            while i < len(gs):
                run = [gs[i]]
                while (len(run) < width and i + len(run) < len(gs) and n_ring == 65536 and
                       qps[gs[i + len(run)]].data_ptr() == qps[run[-1]].data_ptr() + 2 * ext * n_ring * 4):
                    run.append(gs[i + len(run)])
                if len(run) == 1:
                    out[run[0]] = inner_sum(run[0])
                else:
                    first = qps[run[0]]
                    base = first._base if first._base is not None else first
                    at = (first.data_ptr() - base.data_ptr()) // (2 * ext * n_ring * 4)
                    res = eng.ks_stage3_batch(plan, base[at:at + len(run)], level)
                    for j, g in enumerate(run):
                        out[g] = res[j]
                i += len(run)
            return out

        def inner_sums_a(gs):
            """The a halves only of several giant steps' inner sums, scaled down (one batched set of
            launches per run of up to eight adjacent accumulators); their b halves stay over Q||P.
            Returns {g: (a over Q_l [level, n], b over Q||P [ext, n])}."""
            out = {}
            width = min(8, eng.lane_count())
            i = 0
            while i < len(gs):
                run = [gs[i]]
                while (len(run) < width and i + len(run) < len(gs) and
                       qps[gs[i + len(run)]].data_ptr() == qps[run[-1]].data_ptr() + 2 * ext * n_ring * 4):
                    run.append(gs[i + len(run)])
                first = qps[run[0]]
                if len(run) == 1:
                    stack = first.unsqueeze(0)
                else:
                    base = first._base if first._base is not None else first
                    at = (first.data_ptr() - base.data_ptr()) // (2 * ext * n_ring * 4)
                    stack = base[at:at + len(run)]
                res = eng.ks_stage3_batch_a(plan, stack, level)
                for j, g in enumerate(run):
                    out[g] = (res[j], qps[g][1])
                i += len(run)
            return out

        inner_sum.many = inner_sums
        if n_ring == 65536 and self.keep_b_qp:      # the batched a-half ModDown is an N = 2^16 kernel path
            inner_sum.many_a = inner_sums_a
        return inner_sum

    def rotations(self) -> set[int]:
        out = {(b * self.step) % self.n for b in self.baby if b}
        out |= {(g * self.n1 * self.step) % self.n for g in self.giants if g}
        return out

    def apply_batch(self, cts, keys: ckks.EvaluationKeys):
        """The transform of several independent ciphertexts at once (BASELINE config 5: batches of
        independent bootstraps).  Each ciphertext keeps its own lanes for ModUp, giant steps and
        ModDown; what the batch shares is the traffic of the fused baby-step kernel, 27 % of a
        bootstrap: pairs go through one launch that reads every rotation key and every plaintext
        diagonal once for both (Engine.bsgs_inner_batch).  Results equal apply() per ciphertext bit
        for bit."""
        from .engine import get_engine

        eng = get_engine()
        cts = list(cts)
        if len(cts) == 1 or not (self.double_hoist and self._fused_ok(eng)):
            return eng.fork([(lambda ct=ct: self.apply(ct, keys)) for ct in cts]) if len(cts) > 1 else [self.apply(cts[0], keys)]
        for ct in cts:
            if ckks.level_of(ct) != self.level:
                raise RnsError(f"linear transform encoded for level {self.level}, ciphertext at {ckks.level_of(ct)}")
        pre = eng.fork([(lambda ct=ct: self._bsgs_prepare(ct, keys, eng)) for ct in cts])
        first = pre[0]
        qps = [{} for _ in cts]
        for chunk, table in first["chunks"]:
            outs = eng.bsgs_inner_batch(first["plan"], [q["raised"] for q in pre], [ct.a.data for ct in cts],
                                        [ct.b.data for ct in cts], first["ks"], first["evks"], table, first["ext"])
            for mine, o in zip(qps, outs):
                mine.update(zip(chunk, o))
        out = eng.fork([(lambda ct=ct, q=q: self.apply(ct, keys, _qps=q)) for ct, q in zip(cts, qps)])
        del pre                                   # raised digits stay referenced until the joins above
        return out

    def apply(self, ct, keys: ckks.EvaluationKeys, _qps=None):
        from .engine import get_engine

        eng = get_engine()
        if ckks.level_of(ct) != self.level:
            raise RnsError(f"linear transform encoded for level {self.level}, ciphertext at {ckks.level_of(ct)}")
        basis = ct.a.basis
        slots = eng.row_slots(basis)
        if self.double_hoist:
            inner_sum = self._double_hoisted_inner(ct, keys, eng, qps=_qps)
        else:
            # baby steps: rotations of the same input sharing one ModUp, spread over the lanes
            hoisted = ckks.hrot_hoisted(ct, [b * self.step for b in self.baby], keys)
            rotated = {b: hoisted[b * self.step] for b in self.baby}

            def inner_sum(g):
                row = self.table[g]
                return eng.fused_terms([rotated[b] for b in row], [pt.poly.data for pt in row.values()], slots)

        moving = [g for g in self.giants if g]
        # with rotated giant steps the unrotated inner sum joins their shared Q||P accumulator as
        # it is: no ModDown of its own
        base_raw = getattr(inner_sum, "raw", {}).get(0) if moving and p_ok(self) else None
        todo = [g for g in self.giants if not (g == 0 and base_raw is not None)]
        qp_b = hasattr(inner_sum, "many_a") and base_raw is not None and all(g != 0 for g in todo)
        if qp_b:
            # double hoisting in full: only the a half of a moving giant step's inner sum is scaled
            # down (it has to be decomposed again); the b half stays over Q||P and joins the shared
            # accumulator through the rotation as it is
            inners = inner_sum.many_a(todo)
        elif hasattr(inner_sum, "many"):
            inners = inner_sum.many(todo)              # batched ModDowns (adjacent accumulators)
        else:
            inners = dict(zip(todo, eng.fork([(lambda g=g: inner_sum(g)) for g in todo])))
        base = inners.get(0)
        scale = ct.scale * self.pt_scale
        if not moving:
            total = ct_from_tensor(base, basis, scale)
        else:
            # giant steps: rotate each inner sum, run stages 1-2 of its key switch into the
            # lane's Q||P accumulator, and scale everything down with ONE ModDown at the end
            p = self.params
            n_ring = p.n
            plan = eng.ks_plan(n_ring, basis, p.p_basis, p.alpha, p.l + p.alpha, p.l)

            def giant(lane, nth, g):
                k = ckks.galois_element(g * self.n1 * self.step, n_ring)
                if k not in keys.galois:
                    raise RnsError(f"no Galois key for rotation {g * self.n1 * self.step}")
                # the rotation is never materialised: gather inside the inner product, b part lifted
                acc_rot = eng.ks_accumulate_rot_qp if qp_b else eng.ks_accumulate_rot
                acc_rot(plan, inners[g][0], inners[g][1], k, keys.galois[k].matrix(), first=(nth == 0))

            eng.fork([(lambda lane, nth, g=g: giant(lane, nth, g)) for g in moving], with_lane=True)
            lanes_used = min(eng.lane_count(), len(moving))
            if n_ring % 4 == 0 and self.level > self.limbs:
                # the shared ModDown and the rescale by the plaintext limbs as one division
                rest, dropped = basis[:self.level - self.limbs], basis[self.level - self.limbs:]
                md_plan = eng.moddown_plan(n_ring, rest, dropped + p.p_basis)
                out_t = eng.ks_finish_rescale(plan, md_plan, lanes_used, None if base is None else base[0],
                                              None if base is None else base[1], self.level - self.limbs, n_ring,
                                              raw_qp=base_raw)
                return ct_from_tensor(out_t, rest, ct.scale)
            out_t = eng.ks_finish(plan, lanes_used, None if base is None else base[0],
                                  None if base is None else base[1], self.level, n_ring)
            total = ct_from_tensor(out_t, basis, scale)
        out = ckks.rescale(total, self.limbs)
        return ckks.Ciphertext(a=out.a, b=out.b, scale=ct.scale)


# ---------------------------------------------------------------------------
# bootstrapping
# ---------------------------------------------------------------------------
@dataclass
class BootstrapConfig:
    scheme: str = "ps"            # polynomial evaluation: "ps" (Paterson-Stockmeyer, degree <= 15, five
                                  # limb pairs deep, lazy relinearisation: six key switches) or "tree"
                                  # (balanced power tree, depth ceil(log2(degree+1)), one key switch per
                                  # product: nine for degree 13)
    squarings: int = 5            # r: exp(i*theta / 2^r) is squared r times
    degree: int = 15              # degree of the polynomial for exp on |x| <= 2*pi*K / 2^r
    approx: str = "chebyshev"     # "chebyshev": interpolation at the Chebyshev nodes of that interval
                                  # (near-minimax); "taylor": the truncated series.  The approximation
                                  # error is a deterministic function of I, so SlotToCoeff adds it up
                                  # coherently (x sqrt(slots)): it has to sit ~8 bits below the target
                                  # precision.  Degree 15 on K = 12 errs 2^-28 on the message.
    k_bound: int = 12             # |I| <= K for the polynomial's interval.  I is a sum of h + 1 terms
                                  # uniform in [-1/2, 1/2): standard deviation 1.66 at h = 32, K = 12 is
                                  # 7.2 sigma (6e-14 per coefficient); the absolute bound is (h + 1) / 2
    log_delta_in: int = 54        # input scale 2^log_delta_in at two limbs (Q0 ~ 2^62).  Errors made before
                                  # EvalMod return to the message amplified by Q0 * 2^r / (2 pi Delta): every
                                  # bit of Delta is a bit of precision until the sine's cubic term (Delta |m| /
                                  # Q0)^2 takes over.  Measured at ks48, slots in the unit square
                                  # (profiles/boot_delta.py): 2^-17.1 / -19.1 / -21.0 / -22.2 / -18.6 at
                                  # 50 / 52 / 54 / 56 / 58; 54 keeps a factor 4 of headroom in |m|
    groups: int = 3               # stage groups per linear transform
    n1: int | None = None         # baby-step count (default ~ sqrt of the diagonal span)


def exp_coefficients(cfg: BootstrapConfig):
    """Monomial coefficients a_k of a degree-`cfg.degree` polynomial for exp(i*y) on
    |y| <= 2*pi*K / 2^r, and c_k = a_k / i^k of the same polynomial in x = i*y."""
    d = cfg.degree
    if cfg.approx == "taylor":
        a = [(1j ** k) / math.factorial(k) for k in range(d + 1)]
    elif cfg.approx == "chebyshev":
        from numpy.polynomial import chebyshev as cheb

        bound = 2.0 * math.pi * cfg.k_bound / float(1 << cfg.squarings)

        def fit(f):
            mono = np.zeros(d + 1)
            m = cheb.cheb2poly(cheb.chebinterpolate(lambda t: f(bound * t), d))
            mono[:len(m)] = m
            return [mono[k] / bound ** k for k in range(d + 1)]

        cos_c, sin_c = fit(np.cos), fit(np.sin)
        # cos is even and sin odd: drop the interpolation's rounding dust in the other parity
        a = [complex(cos_c[k], 0.0) if k % 2 == 0 else complex(0.0, sin_c[k]) for k in range(d + 1)]
    else:
        raise RnsError(f"unknown approximation {cfg.approx!r}")
    return a, [a[k] / (1j ** k) for k in range(d + 1)]


class Bootstrapper:
    """Keys, encoded DFT diagonals and constants for one parameter set; bootstrap(ct)
    refreshes a level-2 ciphertext of scale 2^log_delta_in to `out_level` limbs."""

    def __init__(self, params: ParameterSet, sk: ks.SecretKey, config: BootstrapConfig | None = None,
                 seed: int = 7000, sk_sparse: ks.SecretKey | None = None):
        """`sk` is the key the ciphertexts live under and every evaluation key is generated
        for.  With `sk_sparse` (sparse-secret encapsulation, PAPER.md / ks48.json h_sparse):
        `sk` may be dense; the input is key-switched to `sk_sparse` on its two bottom limbs,
        raised there (so that |I| stays within k_bound), and switched back to `sk` at the
        top level: two extra key switches, one of them on two limbs only."""
        self.params, self.cfg = params, config or BootstrapConfig()
        cfg = self.cfg
        n = params.n // 2
        lg = n.bit_length() - 1
        L = params.l
        self.q0 = params.q_basis[0].q * params.q_basis[1].q
        self.delta_in = float(1 << cfg.log_delta_in)
        sizes = default_groups(lg, cfg.groups)
        # ---- level plan -----------------------------------------------------------
        self.lvl_cts = L                                   # CoeffToSlot: two limbs per group (its error
        self.lvl_evalmod = L - 2 * cfg.groups              # is amplified by Q0*2^r/(2*pi*Delta) ~ 2^13)
        depth = 5 if cfg.scheme == "ps" else math.ceil(math.log2(cfg.degree + 1))   # polynomial depth
        self.lvl_after_evalmod = self.lvl_evalmod - 2 * (depth + cfg.squarings) - 1
        self.lvl_stc = self.lvl_after_evalmod
        self.out_level = self.lvl_stc - cfg.groups
        if self.out_level < 3:
            raise RnsError(f"parameter set too shallow for bootstrapping: would end at level {self.out_level}")
        self.eval_scale = float(params.q_basis[self.lvl_evalmod - 1].q) * float(params.q_basis[self.lvl_evalmod - 2].q)
        self.out_scale = float(params.q_basis[self.out_level - 1].q) * float(params.q_basis[self.out_level - 2].q)
        # After ModRaise the plaintext polynomial is t; tagging it with scale
        # Q0 * 2^r / (2*pi) makes CoeffToSlot deliver y = 2*pi*t / (Q0 * 2^r) in the slots.
        self.raise_scale = self.q0 * float(1 << cfg.squarings) / (2.0 * math.pi)
        # ---- linear transforms ----------------------------------------------------
        cts = grouped_dft(n, sizes, inverse=True)
        stc = grouped_dft(n, sizes, inverse=False)
        # last CoeffToSlot group also renormalises the scale tag to eval_scale / 2
        # (the factor 2 is absorbed by W +/- conj(W) below)
        renorm = (self.eval_scale / 2.0) / self.raise_scale
        self.cts = [LinearTransform(g, params, self.lvl_cts - 2 * i, cfg.n1,
                                    factor=renorm if i == len(cts) - 1 else 1.0, limbs=2)
                    for i, g in enumerate(cts)]
        self.stc = [LinearTransform(g, params, self.lvl_stc - i, cfg.n1) for i, g in enumerate(stc)]
        # ---- keys -----------------------------------------------------------------
        self.keys = ckks.EvaluationKeys(params, relin=ckks.relin_keygen(sk, params, seed=seed))
        self.keys.add_conjugation(sk, seed=seed + 1)
        self.to_sparse = self.to_dense = None
        if sk_sparse is not None:
            self.to_sparse = ks.switching_keygen(sk, sk_sparse, params, seed=seed + 900_001)
            self.to_dense = ks.switching_keygen(sk_sparse, sk, params, seed=seed + 900_002)
        rots = set()
        for lt in self.cts + self.stc:
            rots |= lt.rotations()
        for i, r in enumerate(sorted(rots)):
            self.keys.add_rotation(sk, r, seed=seed + 2 + i)
        # coefficients of exp(i*y) (real-part branch, input y) and exp(x) (input x = i*y)
        self.coef_lo, self.coef_hi = exp_coefficients(cfg)
        self._consts: dict = {}

    def _const(self, value: complex, level: int, scale: float) -> ckks.Plaintext:
        """Encoded constant, cached: levels and scales are the same on every call."""
        key = (complex(value), level, float(scale))
        hit = self._consts.get(key)
        if hit is None:
            hit = self._consts[key] = ckks.encode(value, self.params, level=level, scale=scale)
        return hit

    # -- steps ---------------------------------------------------------------------
    def mod_raise(self, ct):
        """Level-2 ciphertext -> full level, plaintext t = Delta*m + e + Q0*I."""
        from .engine import get_engine

        eng = get_engine()
        p = self.params
        if ckks.level_of(ct) != 2:
            raise RnsError("bootstrap input must live on the two bottom limbs")
        low = p.q_basis[:2]
        full = p.q_basis
        s0, s1 = eng.slot(low[0], p.n), eng.slot(low[1], p.n)
        slots_full = eng.row_slots(full, p.n)
        halves = []
        for poly in (ct.a, ct.b):
            coeff = ntt_polynomial(poly, "inverse")
            lifted = eng.lift2_centered(coeff.data, s0, s1, slots_full, len(full))
            halves.append(eng.ntt(lifted, slots_full, False))
        return ckks.Ciphertext(a=Polynomial(full, halves[0], EVALUATION),
                               b=Polynomial(full, halves[1], EVALUATION), scale=self.raise_scale)

    def coeff_to_slot(self, ct):
        for lt in self.cts:
            ct = lt.apply(ct, self.keys)
        # W holds (y_lo + i*y_hi) / 2 in bit-reversed slot order, scale tag eval_scale / 2
        conj = ckks.conjugate_fused(ct, self.keys)
        lo = ckks.add(ct, conj)        # y_lo   at tag eval_scale
        hi = ckks.sub(ct, conj)        # i*y_hi at tag eval_scale
        lo = ckks.Ciphertext(lo.a, lo.b, self.eval_scale)
        hi = ckks.Ciphertext(hi.a, hi.b, self.eval_scale)
        return lo, hi

    def _pair(self, x, c0: complex, c1: complex, target_scale: float, level: int):
        """c0 + c1*x at `level` limbs and scale `target_scale` (x two limbs above)."""
        p = self.params
        lvl = ckks.level_of(x)
        dropped = math.prod(m.q for m in x.a.basis[lvl - 2:])
        pt = self._const(c1, lvl, target_scale * dropped / x.scale)
        t = ckks.rescale(ckks.mul_plain(x, pt), 2)
        t = ckks.mod_drop(ckks.Ciphertext(t.a, t.b, target_scale), level)
        return ckks.add_plain(t, self._const(c0, level, target_scale))

    def _mul(self, x, y, addend=None):
        """x * y, relinearised and rescaled by two limbs; `addend` (at the result's level and
        scale) is added inside the same pipeline."""
        lvl = min(ckks.level_of(x), ckks.level_of(y))
        return ckks.hmult_rescale(ckks.mod_drop(x, lvl), ckks.mod_drop(y, lvl), self.keys.relin, 2, addend=addend)

    def _exp_ps(self, x, coef):
        """sum_k coef[k] x^k, degree <= 15, Paterson-Stockmeyer with baby powers x, x^2, x^3 and
        giant powers x^4, x^8, x^12:  p = q_0 + q_1 x^4 + q_2 x^8 + q_3 x^12,  q_j = sum_{i<4}
        coef[4j+i] x^i.  Each q_j is ONE fused plaintext pass over (x, x^2, x^3) + one rescale; the
        three products are tensor products summed before a single relinearisation.  Five limb pairs
        deep (one more than the balanced tree), six key switches instead of nine to ten."""
        from .engine import get_engine

        eng = get_engine()
        d = len(coef) - 1
        if d > 15:
            raise RnsError("Paterson-Stockmeyer evaluation here covers degree <= 15")
        c = list(coef) + [0.0] * (16 - len(coef))
        q = self.params.q_basis
        dd = lambda lvl: float(q[lvl - 1].q) * float(q[lvl - 2].q)      # the two limbs a rescale at `lvl` drops
        L0 = ckks.level_of(x)
        x2 = self._mul(x, x)                           # L0 - 2
        x3, x4 = eng.fork([lambda: self._mul(x2, x), lambda: self._mul(x2, x2)])      # L0 - 4
        x8 = self._mul(x4, x4)                         # L0 - 6
        x12 = self._mul(x8, x4)                        # L0 - 8
        lq = L0 - 4                                    # level the baby polynomials are formed at
        lt = L0 - 8                                    # level of the three products
        out_level = lt - 2
        s_f = self.eval_scale_at(out_level)
        sigma = s_f * dd(lt)                           # scale of every tensor product
        xs = [ckks.mod_drop(x, lq), ckks.mod_drop(x2, lq), x3]
        giants = {1: ckks.mod_drop(x4, lt), 2: ckks.mod_drop(x8, lt), 3: x12}
        slots = eng.row_slots(xs[0].a.basis)
        xts = [ckks.ct_term(v) for v in xs]            # mod-dropped halves go to the kernel as they lie

        def baby(j):
            """q_j at level lq - 2 with the exact scale that makes q_j * x^(4j) land on sigma
            (q_0: directly on s_f)."""
            want = s_f if j == 0 else sigma / giants[j].scale
            pre = want * dd(lq)                        # scale before the rescale
            terms, pts = [], []
            for i in (1, 2, 3):
                ck = c[4 * j + i]
                if ck == 0:
                    continue
                terms.append(xts[i - 1])
                pts.append(self._const(ck, lq, pre / xs[i - 1].scale).poly.data)
            if not terms:
                raise RnsError("degenerate baby polynomial")
            acc = eng.fused_terms(terms, pts, slots)
            t = ckks.ct_from_tensor(acc, xs[0].a.basis, pre)
            if c[4 * j] != 0:
                t = ckks.add_plain(t, self._const(c[4 * j], lq, pre))
            r = ckks.rescale(t, 2)
            return ckks.Ciphertext(r.a, r.b, want)

        top = max(j for j in range(4) if any(c[4 * j + i] != 0 for i in range(4)))
        qs = eng.fork([(lambda j=j: baby(j)) for j in range(top + 1)])
        pairs = [(ckks.mod_drop(qs[j], lt), giants[j]) for j in range(1, top + 1)]
        prod = ckks.hmult_sum_rescale(pairs, self.keys.relin, 2)
        prod = ckks.Ciphertext(prod.a, prod.b, s_f)
        return ckks.add(prod, ckks.mod_drop(qs[0], out_level))

    def _exp_taylor(self, x, coef):
        """sum_k coef[k] x^k by a balanced power tree (depth ceil(log2(degree+1))), or by
        Paterson-Stockmeyer when the configuration asks for it."""
        if self.cfg.scheme == "ps":
            return self._exp_ps(x, coef)
        from .engine import get_engine

        eng = get_engine()
        d = len(coef) - 1
        depth = math.ceil(math.log2(d + 1))
        powers = {1: x}
        for j in range(1, depth):
            powers[1 << j] = self._mul(powers[1 << (j - 1)], powers[1 << (j - 1)])

        def build(lo: int, span: int):
            """Polynomial sum_{k<span} coef[lo+k] x^k; returns None when all coefficients vanish."""
            if lo > d:
                return None
            if span == 2:
                c0 = coef[lo]
                c1 = coef[lo + 1] if lo + 1 <= d else 0.0
                return ("pair", c0, c1)
            half = span // 2
            return ("node", build(lo, half), build(lo + half, half), half)

        def realise(node, want_scale, want_level):
            """Materialise a subtree at exactly (want_scale, want_level)."""
            if node[0] == "pair":
                return self._pair(x, node[1], node[2], want_scale, want_level)
            _, left, right, half = node
            xp = powers[half]
            if right is None:
                return realise(left, want_scale, want_level)
            lvl_in = want_level + 2
            xp_d = ckks.mod_drop(xp, lvl_in) if ckks.level_of(xp) > lvl_in else xp
            dropped = math.prod(m.q for m in self.params.q_basis[want_level:lvl_in])

            # the two halves are independent: spread them over the lanes this branch owns; the low
            # half then rides in the ModDown epilogue of the product (no separate add)
            r, low = eng.fork([lambda: realise(right, want_scale * dropped / xp_d.scale, lvl_in),
                               lambda: realise(left, want_scale, want_level)])
            prod = self._mul(r, xp_d, addend=low)
            return ckks.Ciphertext(prod.a, prod.b, want_scale)

        tree = build(0, 1 << depth)
        out_level = ckks.level_of(x) - 2 * depth
        return realise(tree, self.eval_scale_at(out_level), out_level)

    def eval_scale_at(self, level: int) -> float:
        q = self.params.q_basis
        return float(q[level - 1].q) * float(q[level - 2].q)

    def eval_mod(self, x, coef, kappa: complex):
        """x: slots y (or i*y) with |y| <= 2*pi*K/2^r.  Returns kappa * (E - conj E), E = exp(i*theta)."""
        e = self._exp_taylor(x, coef)
        for _ in range(self.cfg.squarings):
            e = self._mul(e, e)
        diff = ckks.sub(e, ckks.conjugate_fused(e, self.keys))
        lvl = ckks.level_of(diff)
        pt_scale = float(self.params.q_basis[lvl - 1].q)
        # message scale folded so the result carries tag out_scale
        pt = self._const(kappa, lvl, self.out_scale * pt_scale / diff.scale)
        out = ckks.rescale(ckks.mul_plain(diff, pt), 1)
        return ckks.Ciphertext(out.a, out.b, self.out_scale)

    def slot_to_coeff(self, ct):
        for lt in self.stc:
            ct = lt.apply(ct, self.keys)
        return ct

    def bootstrap_batch(self, cts):
        """Several independent bootstraps at once (BASELINE config 5: batches of independent
        bootstraps on one GPU).  Every ciphertext runs the circuit of bootstrap() on its own share
        of the engine's lanes; the six linear transforms go through LinearTransform.apply_batch,
        which reads each rotation key and plaintext diagonal once per PAIR of ciphertexts.  The
        results equal bootstrap() per ciphertext limb for limb."""
        from .engine import get_engine

        eng = get_engine()
        cts = list(cts)
        if len(cts) == 1:
            return [self.bootstrap(cts[0])]
        for ct in cts:
            if not ckks._close(ct.scale, self.delta_in):
                raise RnsError(f"bootstrap expects scale 2^{self.cfg.log_delta_in}, got {ct.scale}")

        def lift(ct):
            if self.to_sparse is not None:
                ct = ckks.keyswitch_level(ct, self.to_sparse)
            raised = self.mod_raise(ct)
            if self.to_dense is not None:
                back = ckks.keyswitch_level(ckks.Ciphertext(raised.a, raised.b, raised.scale), self.to_dense)
                raised = ckks.Ciphertext(a=back.a, b=back.b, scale=raised.scale)
            return raised

        def split(ct):
            conj = ckks.conjugate_fused(ct, self.keys)
            lo, hi = ckks.add(ct, conj), ckks.sub(ct, conj)
            return ckks.Ciphertext(lo.a, lo.b, self.eval_scale), ckks.Ciphertext(hi.a, hi.b, self.eval_scale)

        xs = eng.fork([(lambda ct=ct: lift(ct)) for ct in cts])
        for lt in self.cts:
            xs = lt.apply_batch(xs, self.keys)
        halves = eng.fork([(lambda x=x: split(x)) for x in xs])
        kappa = self.q0 / (4.0 * math.pi * self.delta_in) / 1j
        jobs = []
        for lo, hi in halves:
            jobs.append(lambda lo=lo: self.eval_mod(lo, self.coef_lo, kappa))
            jobs.append(lambda hi=hi: self.eval_mod(hi, self.coef_hi, kappa * 1j))
        ms = eng.fork(jobs)
        ws = [ckks.mod_drop(ckks.add(ms[2 * i], ms[2 * i + 1]), self.lvl_stc) for i in range(len(cts))]
        for lt in self.stc:
            ws = lt.apply_batch(ws, self.keys)
        return [ckks.Ciphertext(w.a, w.b, self.out_scale) for w in ws]

    def capture_batch(self, sample_cts):
        """bootstrap_batch recorded as one CUDA graph: replay(cts) -> list of ciphertexts."""
        import torch

        from .engine import get_engine

        eng = get_engine()
        count = len(sample_cts)
        basis, scale = sample_cts[0].a.basis, sample_cts[0].scale
        static_in = torch.stack([torch.stack([ct.a.data, ct.b.data]) for ct in sample_cts]).clone()
        views = [ct_from_tensor(static_in[i], basis, scale) for i in range(count)]
        self.bootstrap_batch(views)                           # warm-up: plans, constants, caches
        torch.cuda.synchronize()
        graph = torch.cuda.CUDAGraph()
        side = torch.cuda.Stream(device=eng.device)
        side.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(side):
            self.bootstrap_batch(views)                       # settle allocator state on the side stream
            torch.cuda.synchronize()
            with torch.cuda.graph(graph, stream=side):
                outs = self.bootstrap_batch(views)
                static_out = torch.stack([torch.stack([o.a.data, o.b.data]) for o in outs])
        torch.cuda.current_stream().wait_stream(side)
        out_basis, out_scale = outs[0].a.basis, outs[0].scale
        generation = eng.arena_generation()

        def replay(cts, copy_out: bool = True):
            if eng.arena_generation() != generation:
                raise RnsError("the workspace arena was reallocated after this graph was captured (lane count "
                               "changed or a larger key-switch plan was created): capture again")
            if len(cts) != count:
                raise RnsError(f"graph was captured for {count} ciphertexts, got {len(cts)}")
            for i, ct in enumerate(cts):
                static_in[i, 0].copy_(ct.a.data)
                static_in[i, 1].copy_(ct.b.data)
            graph.replay()
            res = static_out.clone() if copy_out else static_out
            return [ct_from_tensor(res[i], out_basis, out_scale) for i in range(count)]

        replay.graph, replay.static_in, replay.static_out = graph, static_in, static_out
        replay.valid = lambda: eng.arena_generation() == generation
        return replay

    def capture(self, sample_ct):
        """Record one whole bootstrap (ModRaise .. SlotToCoeff, ~2.5k kernel launches) into a
        CUDA graph and return replay(ct) -> ciphertext.  The eager run that precedes
        the capture creates every key-switch plan, workspace and encoded constant, so
        nothing allocates or touches the host inside the graph (launch
        overhead of the ~1.5k-kernel bootstrap is what graph capture removes)."""
        import torch

        from .engine import get_engine

        eng = get_engine()
        basis = sample_ct.a.basis
        static_in = torch.stack([sample_ct.a.data, sample_ct.b.data]).clone()
        view = ct_from_tensor(static_in, basis, sample_ct.scale)
        self.bootstrap(view)                                  # warm-up: plans, constants, caches
        torch.cuda.synchronize()
        graph = torch.cuda.CUDAGraph()
        side = torch.cuda.Stream(device=eng.device)
        side.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(side):
            self.bootstrap(view)                              # settle allocator state on the side stream
            torch.cuda.synchronize()
            with torch.cuda.graph(graph, stream=side):
                out = self.bootstrap(view)
                static_out = torch.stack([out.a.data, out.b.data])
        torch.cuda.current_stream().wait_stream(side)
        out_basis, out_scale = out.a.basis, out.scale
        generation = eng.arena_generation()

        def replay(ct, copy_out: bool = True):
            if eng.arena_generation() != generation:
                # the graph holds raw pointers into the key-switch workspace arena as it was
                raise RnsError("the workspace arena was reallocated after this graph was captured (lane count "
                               "changed or a larger key-switch plan was created): capture again")
            static_in[0].copy_(ct.a.data)
            static_in[1].copy_(ct.b.data)
            graph.replay()
            res = static_out.clone() if copy_out else static_out
            return ct_from_tensor(res, out_basis, out_scale)

        replay.graph, replay.static_in, replay.static_out = graph, static_in, static_out
        replay.valid = lambda: eng.arena_generation() == generation
        return replay

    def bootstrap(self, ct, trace=None):
        """`trace(name, ciphertext)`, when given, is called after every phase (eager runs only:
        it reads limbs back, so never under graph capture)."""
        note = trace if trace is not None else (lambda name, c: None)
        if not ckks._close(ct.scale, self.delta_in):
            raise RnsError(f"bootstrap expects scale 2^{self.cfg.log_delta_in}, got {ct.scale}")
        if self.to_sparse is not None:
            ct = ckks.keyswitch_level(ct, self.to_sparse)       # two limbs: cheap
        raised = self.mod_raise(ct)
        if self.to_dense is not None:
            back = ckks.keyswitch_level(ckks.Ciphertext(raised.a, raised.b, raised.scale), self.to_dense)
            raised = ckks.Ciphertext(a=back.a, b=back.b, scale=raised.scale)
        note("mod_raise", raised)
        lo, hi = self.coeff_to_slot(raised)
        note("coeff_to_slot_lo", lo)
        note("coeff_to_slot_hi", hi)
        # (Q0 / (2*pi*Delta)) * sin(theta) = kappa * (E - conj E),  kappa = Q0 / (4*pi*i*Delta)
        kappa = self.q0 / (4.0 * math.pi * self.delta_in) / 1j
        from .engine import get_engine

        m_lo, m_hi = get_engine().fork([lambda: self.eval_mod(lo, self.coef_lo, kappa),
                                        lambda: self.eval_mod(hi, self.coef_hi, kappa * 1j)])
        w = ckks.add(m_lo, m_hi)                       # m_lo + i*m_hi (bit-reversed slots)
        w = ckks.mod_drop(w, self.lvl_stc)
        note("eval_mod", w)
        out = self.slot_to_coeff(w)
        out = ckks.Ciphertext(out.a, out.b, self.out_scale)
        note("slot_to_coeff", out)
        return out


def standard_setup(params: ParameterSet, config: BootstrapConfig | None = None, h_dense: int | None = None,
                   seed: int = 1):
    """The key regime of the paper's bootstrapping table: a dense application
    key of Hamming weight h_dense that every evaluation key is generated for, and a sparse key
    of weight h_sparse used only around ModRaise (sparse-secret encapsulation).  Returns
    (sk, sk_sparse, Bootstrapper); bench.py, the tests and the oracle replay all build the
    headline workload through this one function."""
    sk = ks.keygen(params, h=params.h_dense if h_dense is None else h_dense, seed=seed)
    sk_sparse = ks.keygen(params, h=params.h_sparse, seed=seed + 1000)
    return sk, sk_sparse, Bootstrapper(params, sk, config or BootstrapConfig(), sk_sparse=sk_sparse)


def standard_input(params: ParameterSet, boot: "Bootstrapper", sk, index: int = 0):
    """Synthetic input `index` of the headline workload: uniform slots in the unit square,
    encoded on two limbs at the bootstrap's input scale.  Returns (slots, ciphertext)."""
    rng = np.random.default_rng(index)
    z = rng.uniform(-1, 1, params.n // 2) + 1j * rng.uniform(-1, 1, params.n // 2)
    return z, ckks.encrypt(ckks.encode(z, params, level=2, scale=boot.delta_in), sk, params, seed=50 + index)
