"""HELR-style logistic-regression iteration on packed ciphertexts (BASELINE config 5,
SURVEY 8d: "a fixed sequence of HMult / HRot / rescale iterations on small L"; the paper's HELR
workload spends 82 % of its time at L <= 20).  An application circuit on top of the
public CKKS operations of ckks.py -- nothing here touches the kernels directly.

Layout: `samples` x `features` values row-major in the N/2 slots (one sample per row of
`features` slots, both powers of two, samples * features = N/2).  One iteration of gradient
descent on the cross-entropy loss with a cubic sigmoid:

    ip   = rowsum(Z * W)                      HMult, log2(features) rotations
    ip   = replicate(mask * ip)               PMult, log2(features) rotations
    s    = 0.5 + ip * (c1 + c3 * ip^2)        2 HMult, 1 PMult
    g    = colsum(s * Z)                      HMult, log2(samples) rotations
    W'   = W - (lr / samples) * g             PMult

Z holds the label-folded samples (y_i * x_i), W the weight vector replicated in every row.
Single-limb scale (~2^31): seven limbs per iteration.  `plain_iteration` is the same arithmetic in
NumPy and is what the tests compare decrypted weights against."""
from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np

from . import ckks
from . import keyswitch as ks
from .params import ParameterSet
from .rns import RnsError

SIGMOID_C1 = 0.15012
SIGMOID_C3 = -0.0015930078125           # degree-3 least-squares sigmoid on [-8, 8] (HELR)


def _rot(v: np.ndarray, r: int) -> np.ndarray:
    return np.roll(v, -r)


@dataclass
class HelrShape:
    samples: int
    features: int

    @property
    def slots(self) -> int:
        return self.samples * self.features


def plain_iteration(z: np.ndarray, w: np.ndarray, shape: HelrShape, lr: float) -> np.ndarray:
    """The iteration on slot vectors (length samples * features), same order of operations."""
    f, s = shape.features, shape.samples
    m = z * w
    for k in range(int(math.log2(f))):
        m = m + _rot(m, 1 << k)
    mask = np.zeros(shape.slots)
    mask[::f] = 1.0
    m = m * mask
    for k in range(int(math.log2(f))):
        m = m + _rot(m, -(1 << k))
    sig = 0.5 + m * (SIGMOID_C1 + SIGMOID_C3 * m * m)
    g = sig * z
    for k in range(int(math.log2(s))):
        g = g + _rot(g, f << k)
    return w - (lr / s) * g


class HelrTrainer:
    """Keys, masks and constants for iterations that start at `level` limbs."""

    LIMBS_PER_ITERATION = 7

    def __init__(self, params: ParameterSet, sk: ks.SecretKey, shape: HelrShape, level: int = 20,
                 lr: float = 1.0, seed: int = 9000):
        if shape.slots != params.n // 2:
            raise RnsError(f"samples * features must fill the {params.n // 2} slots")
        for v in (shape.samples, shape.features):
            if v & (v - 1):
                raise RnsError("samples and features must be powers of two")
        if level - self.LIMBS_PER_ITERATION < 1 or level > params.l:
            raise RnsError(f"an iteration needs {self.LIMBS_PER_ITERATION} limbs below level {level}")
        self.params, self.shape, self.level, self.lr = params, shape, level, lr
        self.scale = float(params.q_basis[level - 1].q)          # working scale: the limb dropped first
        self.keys = ckks.EvaluationKeys(params, relin=ckks.relin_keygen(sk, params, seed=seed))
        f, s = shape.features, shape.samples
        rots = [1 << k for k in range(int(math.log2(f)))]
        rots += [-(1 << k) for k in range(int(math.log2(f)))]
        rots += [f << k for k in range(int(math.log2(s)))]
        for i, r in enumerate(rots):
            self.keys.add_rotation(sk, r, seed=seed + 1 + i)
        mask = np.zeros(shape.slots)
        mask[::f] = 1.0
        # encoded at the scale of the limb its rescale drops, so the ciphertext scale is unchanged
        self.mask = ckks.encode(mask, params, level=level - 1, scale=float(params.q_basis[level - 2].q))

        self._consts: dict = {}

    def _const(self, value: float, level: int, scale: float) -> ckks.Plaintext:
        """Encoded constant, cached (levels and scales repeat every iteration; nothing is
        uploaded in the steady state, so an iteration is CUDA-graph capturable)."""
        key = (float(value), level, float(scale))
        hit = self._consts.get(key)
        if hit is None:
            hit = self._consts[key] = ckks.encode_constant(value, self.params, level, scale)
            hit.poly.data                                   # upload now
        return hit

    def _mul_const(self, ct, value: float, out_scale: float):
        """ct * value, rescaled by one limb to exactly `out_scale` (ckks.mul_const with cached plaintexts)."""
        level = ckks.level_of(ct)
        dropped = float(ct.a.basis[level - 1].q)
        out = ckks.rescale(ckks.mul_plain(ct, self._const(value, level, out_scale * dropped / ct.scale)), 1)
        return ckks.Ciphertext(a=out.a, b=out.b, scale=out_scale)

    def encrypt(self, slots: np.ndarray, sk: ks.SecretKey, seed: int = 0):
        return ckks.encrypt(ckks.encode(slots, self.params, level=self.level, scale=self.scale), sk,
                            self.params, seed=seed)

    def _rot_sum(self, ct, rotations):
        for r in rotations:
            ct = ckks.add(ct, ckks.hrot_fused(ct, r, self.keys))
        return ct

    def iteration(self, z, w):
        """One gradient step; z, w at `level` limbs, result at level - 7 with w's scale."""
        keys = self.keys
        f, s = self.shape.features, self.shape.samples
        lf, ls = int(math.log2(f)), int(math.log2(s))
        if ckks.level_of(z) != self.level or ckks.level_of(w) != self.level:
            raise RnsError(f"iteration expects operands at level {self.level}")
        m = ckks.hmult_rescale(z, w, keys.relin, 1)                               # level - 1
        m = self._rot_sum(m, [1 << k for k in range(lf)])
        kept = m.scale
        m = ckks.rescale(ckks.mul_plain(m, self.mask), 1)                         # level - 2
        m = ckks.Ciphertext(a=m.a, b=m.b, scale=kept)
        m = self._rot_sum(m, [-(1 << k) for k in range(lf)])
        x2 = ckks.hmult_rescale(m, m, keys.relin, 1)                              # level - 3
        t = self._mul_const(x2, SIGMOID_C3, m.scale)                              # level - 4
        u = ckks.add_plain(t, self._const(SIGMOID_C1, ckks.level_of(t), t.scale))
        y = ckks.hmult_rescale(ckks.mod_drop(m, ckks.level_of(u)), u, keys.relin, 1)   # level - 5
        sig = ckks.add_plain(y, self._const(0.5, ckks.level_of(y), y.scale))
        g = ckks.hmult_rescale(sig, ckks.mod_drop(z, ckks.level_of(sig)), keys.relin, 1)   # level - 6
        g = self._rot_sum(g, [f << k for k in range(ls)])
        upd = self._mul_const(g, self.lr / s, w.scale)                            # level - 7
        return ckks.sub(ckks.mod_drop(w, ckks.level_of(upd)), upd)
