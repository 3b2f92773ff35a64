"""RNS data model of the B200 engine: word-size NTT-friendly moduli, the
device-resident limb matrix, element-wise arithmetic and the ring automorphism.

Mirrors the names and error behaviour of the reference module
``rnscope/rns.py`` (Modulus :85-125, find_ntt_primes :141-170, Polynomial
:173-212, poly_elementwise :243-258, automorphism :295-320) so its callers and
tests can be pointed here, but residues live in HBM as a contiguous
``[L, N]`` matrix of 32-bit words (the RNSV wire layout, vectors.py:3-14) and
all arithmetic runs in the sm_100a kernels behind ``csrc/libckks_b200.so``.
Host code in this file is setup only (prime search, root search, checks).
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .instrument import counters

COEFFICIENT = "coefficient"
EVALUATION = "evaluation"


class RnsError(Exception):
    """Base class for engine errors (reference rns.py:21)."""


class InsufficientPrimesError(RnsError):
    """Prime search ran out of candidates (reference rns.py:25)."""


class StructureError(RnsError):
    """Operands disagree on basis, degree or domain (reference rns.py:29)."""


# ---------------------------------------------------------------------------
# number theory (host, setup only)
# ---------------------------------------------------------------------------
# Bases {2,3,5,7,11,13,17} are a deterministic Miller-Rabin certificate for
# every n < 3.4e14, which covers the 32-bit moduli this engine admits and the
# 64-bit products formed while building conversion tables.
_MR_BASES = (2, 3, 5, 7, 11, 13, 17, 19, 23, 29, 31, 37)


def is_prime(n: int) -> bool:
    n = int(n)
    if n < 2:
        return False
    for b in _MR_BASES:
        if n == b:
            return True
        if n % b == 0:
            return False
    odd, twos = n - 1, 0
    while not odd & 1:
        odd >>= 1
        twos += 1
    for b in _MR_BASES:
        x = pow(b, odd, n)
        if x == 1 or x == n - 1:
            continue
        for _ in range(twos - 1):
            x = x * x % n
            if x == n - 1:
                break
        else:
            return False
    return True


def minimal_primitive_root_2n(q: int, n: int) -> int:
    """Smallest psi >= 2 of multiplicative order exactly 2n modulo the prime q
    (n a power of two).  The reference fixes this choice of root
    (rns.py:61-82); a different root would permute every evaluation-domain
    limb, so it is parity critical.

    All roots are the odd powers of any one of them; they are enumerated with
    a vectorised cumulative product in uint64 (q < 2^32 keeps it exact).
    """
    cofactor = (q - 1) // (2 * n)
    seed = 0
    for g in range(2, q):
        cand = pow(g, cofactor, q)
        if pow(cand, n, q) == q - 1:
            seed = cand
            break
    if seed == 0:
        raise RnsError(f"no primitive {2 * n}-th root of unity mod {q}")
    if n == 1:
        return seed
    step = seed * seed % q
    # doubling construction of seed * step^j for j in [0, n)
    vals = np.array([seed], dtype=np.uint64)
    mult = np.uint64(step)
    qq = np.uint64(q)
    while len(vals) < n:
        vals = np.concatenate([vals, vals * mult % qq])
        mult = mult * mult % qq
    return int(vals[:n].min())


@dataclass(frozen=True)
class Modulus:
    """A word-size NTT-friendly prime q < 2^32, q = 1 (mod 2n), with psi a
    primitive 2n-th root of unity and scalar Barrett constants
    (reference rns.py:85-125)."""

    q: int
    n: int
    psi: int
    barrett_mu: int
    barrett_shift: int

    @classmethod
    def for_prime(cls, q: int, n: int, psi: int | None = None) -> "Modulus":
        q, n = int(q), int(n)
        if not is_prime(q):
            raise RnsError(f"{q} is not prime")
        if q >> 32:
            raise RnsError(f"{q} does not fit the 32-bit element representation")
        if (q - 1) % (2 * n):
            raise RnsError(f"{q} is not NTT-friendly for ring degree {n}")
        if psi is None:
            psi = minimal_primitive_root_2n(q, n)
        else:
            psi = int(psi)
            if pow(psi, n, q) != q - 1 or pow(psi, 2 * n, q) != 1:
                raise RnsError(f"{psi} is not a primitive {2 * n}-th root mod {q}")
        width = 2 * q.bit_length()
        return cls(q, n, psi, (1 << width) // q, width)

    @property
    def bits(self) -> int:
        return self.q.bit_length()

    def reduce(self, x: int) -> int:
        """Barrett reduction of x < 2^barrett_shift into [0, q)."""
        r = x - ((x * self.barrett_mu) >> self.barrett_shift) * self.q
        while r >= self.q:
            r -= self.q
        return r

    def root_for_degree(self, n: int) -> int:
        """psi squared down to order exactly 2n (reference transform.py:88-96)."""
        root, order = self.psi, 2 * self.n
        while order > 2 * n:
            root = root * root % self.q
            order //= 2
        if order != 2 * n or (n >= 1 and pow(root, n, self.q) != self.q - 1):
            raise StructureError(f"cannot derive a primitive {2 * n}-th root for q={self.q}")
        return root


def mod_arith(x: int, y: int, m: Modulus, kind: str) -> int:
    """Scalar (x op y) mod q on canonical inputs (reference rns.py:128-138)."""
    if kind == "add":
        s = x + y
        return s - m.q if s >= m.q else s
    if kind == "sub":
        d = x - y
        return d + m.q if d < 0 else d
    if kind == "mul":
        return m.reduce(x * y)
    raise ValueError(f"unknown arithmetic kind {kind!r}")


def find_ntt_primes(count: int, bitwidth: int, n: int, floor_bits: int | None = None) -> list[Modulus]:
    """``count`` primes below 2^bitwidth congruent to 1 mod 2n, largest first
    (reference rns.py:141-170; same scan order, so the same moduli)."""
    if count < 1:
        raise ValueError("count must be positive")
    if n < 1 or n & (n - 1):
        raise ValueError("ring degree must be a power of two")
    if bitwidth > 32:
        raise ValueError("bitwidth must be at most 32")
    stride = 2 * n
    if stride > (1 << bitwidth):
        raise ValueError("2n must divide 2^bitwidth")
    lowest = 1 << (bitwidth - 2 if floor_bits is None else floor_bits)
    cand = ((1 << bitwidth) - 2) // stride * stride + 1
    picked: list[Modulus] = []
    while cand >= lowest and len(picked) < count:
        if is_prime(cand):
            picked.append(Modulus.for_prime(cand, n))
        cand -= stride
    if len(picked) < count:
        raise InsufficientPrimesError(
            f"insufficient primes: found {len(picked)} of {count} primes "
            f"= 1 (mod {stride}) in [{lowest}, 2^{bitwidth})"
        )
    return picked


# ---------------------------------------------------------------------------
# the limb matrix
# ---------------------------------------------------------------------------
class Polynomial:
    """An L x N residue matrix over an ordered modulus basis, resident in HBM.

    Same constructor and attributes as the reference dataclass
    (rns.py:173-212): ``Polynomial(basis, coeffs, domain)``.  ``coeffs`` may be
    anything array-like on the host (uploaded lazily, on first device use) or
    a CUDA ``torch`` tensor of 32-bit words shaped [L, N] (adopted as is, no
    copy).  ``.coeffs`` reads the matrix back as host ``uint64`` for
    comparison with the reference; ``.data`` is the device tensor the kernels
    work on.  Values are immutable by convention, as in the reference.
    """

    __slots__ = ("basis", "domain", "_host", "_dev", "_shape")

    def __init__(self, basis, coeffs, domain: str):
        self.basis = tuple(basis)
        self.domain = domain
        self._host = None
        self._dev = None
        if _is_torch_tensor(coeffs):
            if coeffs.dim() != 2:
                raise StructureError(f"coefficient matrix {tuple(coeffs.shape)} is not 2-D")
            self._dev = _as_word_tensor(coeffs)
            self._shape = tuple(self._dev.shape)
        else:
            host = np.asarray(coeffs)
            if host.ndim == 2 and host.dtype != np.uint64:
                host = host.astype(np.uint64)
            self._host = host
            self._shape = tuple(host.shape)
        if len(self._shape) != 2 or self._shape[0] != len(self.basis):
            raise StructureError(
                f"coefficient matrix {self._shape} does not match basis of length {len(self.basis)}"
            )
        if domain not in (COEFFICIENT, EVALUATION):
            raise StructureError(f"unknown domain {domain!r}")

    # -- reference-compatible surface ---------------------------------------
    @property
    def coeffs(self) -> np.ndarray:
        if self._host is None:
            words = self._dev.cpu().numpy().view(np.uint32)
            self._host = words.astype(np.uint64)
        return self._host

    @property
    def num_limbs(self) -> int:
        return len(self.basis)

    @property
    def n(self) -> int:
        return self._shape[1]

    def q_column(self) -> np.ndarray:
        return np.array([m.q for m in self.basis], dtype=np.uint64)[:, None]

    def copy(self) -> "Polynomial":
        if self._dev is not None:
            return Polynomial(self.basis, self._dev.clone(), self.domain)
        return Polynomial(self.basis, self._host.copy(), self.domain)

    def validate(self) -> None:
        if np.any(self.coeffs >= self.q_column()):
            raise StructureError("residue out of canonical range [0, q)")

    # -- device surface -------------------------------------------------------
    @property
    def data(self):
        """Device tensor [L, N] of 32-bit words (torch.int32 storage holding
        unsigned residues), uploaded on first use."""
        if self._dev is None:
            from .engine import get_engine

            if np.any(self._host >> np.uint64(32)):
                raise StructureError("residue does not fit the 32-bit element representation")
            self._dev = get_engine().upload(self._host.astype(np.uint32))
        return self._dev

    def rows(self, sl) -> "Polynomial":
        """Row-sliced view (shares device storage)."""
        sl = sl if isinstance(sl, slice) else slice(sl, sl + 1)
        basis = self.basis[sl]
        if self._dev is not None:
            return Polynomial(basis, self._dev[sl], self.domain)
        return Polynomial(basis, self._host[sl], self.domain)

    def __repr__(self) -> str:
        where = "hbm" if self._dev is not None else "host"
        return f"Polynomial(L={self.num_limbs}, N={self.n}, {self.domain}, {where})"


def _is_torch_tensor(x) -> bool:
    mod = type(x).__module__
    return mod == "torch" or mod.startswith("torch.")


def _as_word_tensor(t):
    import torch

    if t.dtype == torch.uint32:
        t = t.view(torch.int32)
    if t.dtype != torch.int32:
        raise StructureError(f"device limb matrix must hold 32-bit words, got {t.dtype}")
    if not t.is_cuda:
        from . import engine

        # CPU word tensors are adopted only while a checker backend that works on host tensors
        # is installed (engine.use_backend); the CUDA engine takes device tensors only
        if not getattr(engine._engine, "host_tensors", False):
            raise StructureError("device limb matrix must live on a CUDA device")
    return t if t.is_contiguous() else t.contiguous()


def zero_polynomial(basis, n: int, domain: str = COEFFICIENT) -> Polynomial:
    return Polynomial(tuple(basis), np.zeros((len(tuple(basis)), n), dtype=np.uint64), domain)


def random_polynomial(basis, n: int, rng: np.random.Generator, domain: str = COEFFICIENT) -> Polynomial:
    """Uniform residues, drawn limb by limb in basis order like the reference
    (rns.py:219-223) so a seed reproduces the same matrix."""
    basis = tuple(basis)
    mat = np.stack([rng.integers(0, m.q, size=n, dtype=np.uint64) for m in basis])
    return Polynomial(basis, mat, domain)


def _qs(p: Polynomial) -> tuple[int, ...]:
    return tuple(m.q for m in p.basis)


def poly_equal(a: Polynomial, b: Polynomial) -> bool:
    return _qs(a) == _qs(b) and a.domain == b.domain and np.array_equal(a.coeffs, b.coeffs)


def _check_compatible(a: Polynomial, b: Polynomial) -> None:
    if _qs(a) != _qs(b):
        raise StructureError("operands use different modulus bases")
    if a.n != b.n:
        raise StructureError(f"ring degrees differ: {a.n} vs {b.n}")
    if a.domain != b.domain:
        raise StructureError(f"domains differ: {a.domain} vs {b.domain}")


_KIND_CODE = {"add": 0, "sub": 1, "mul": 2}


def poly_elementwise(a: Polynomial, b: Polynomial, kind: str) -> Polynomial:
    """Limb-wise (a op b) mod q on the GPU; ``mul`` needs the evaluation
    domain (reference rns.py:243-258)."""
    _check_compatible(a, b)
    if kind not in _KIND_CODE:
        raise ValueError(f"unknown arithmetic kind {kind!r}")
    if kind == "mul" and a.domain != EVALUATION:
        raise StructureError("element-wise mul is only convolution in the evaluation domain")
    from .engine import get_engine

    eng = get_engine()
    out = eng.elementwise(a.data, b.data, eng.row_slots(a.basis), _KIND_CODE[kind])
    counters.elementwise += a.num_limbs * a.n
    return Polynomial(a.basis, out, a.domain)


def eval_permutation_closed_form(n: int, k: int) -> np.ndarray:
    """Source column of every evaluation-domain output column under X -> X^k:
    out[:, t] = in[:, j],  j = bitrev(((2*bitrev(t)+1)*k mod 2N - 1)/2).
    The reference derives the same permutation by probing its transform
    (rns.py:268-292); the device kernel evaluates this closed form per thread.
    Host copy kept for tests and diagnostics."""
    lg = n.bit_length() - 1
    t = np.arange(n, dtype=np.int64)

    def brev(x):
        r = np.zeros_like(x)
        for _ in range(lg):
            r = (r << 1) | (x & 1)
            x = x >> 1
        return r

    e = ((2 * brev(t) + 1) * (k % (2 * n))) % (2 * n)
    return brev((e - 1) // 2)


def automorphism(a: Polynomial, k: int) -> Polynomial:
    """X -> X^k for odd k (reference rns.py:295-320).  Coefficient domain:
    scatter with negacyclic sign; evaluation domain: column gather."""
    if k % 2 == 0:
        raise ValueError("automorphism index must be odd (coprime to 2N)")
    n = a.n
    k = k % (2 * n)
    from .engine import get_engine

    eng = get_engine()
    if a.domain == COEFFICIENT:
        out = eng.automorphism_coeff(a.data, eng.row_slots(a.basis), k)
        return Polynomial(a.basis, out, a.domain)
    if not any(m.n == n and m.q > n for m in a.basis):
        raise StructureError(
            "evaluation-domain automorphism needs a basis modulus that is "
            "NTT-friendly for the polynomial's own degree"
        )
    return Polynomial(a.basis, eng.automorphism_eval(a.data, k), a.domain)
