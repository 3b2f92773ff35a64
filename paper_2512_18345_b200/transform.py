"""Negacyclic NTT / iNTT of limb matrices on the GPU.

API mirror of the reference ``rnscope/transform.py``: ``ntt`` (:253-276),
``ntt_polynomial`` (:279-287), ``ntt_two_phase`` (:290-323),
``build_twiddle_table`` / ``twiddle_table`` (:76-123) and ``generate_twiddle``
(:126-151).  The function computed is fixed by the reference (forward output
slot t holds a(psi^(2*bitrev(t)+1)), inverse includes N^-1); the algorithm is
the engine's own (csrc/ntt.cu).  Twiddle tables live in HBM and are built by
the C side when a modulus is first used at a degree.
"""
from __future__ import annotations

import functools
from dataclasses import dataclass

import numpy as np

from .instrument import counters
from .rns import COEFFICIENT, EVALUATION, Modulus, Polynomial, StructureError

FORWARD = "forward"
INVERSE = "inverse"


def _log2(n: int) -> int:
    return n.bit_length() - 1


def _check_degree(n: int) -> None:
    if n < 2 or n & (n - 1):
        raise ValueError("ring degree must be a power of two >= 2")


def _bitrev_array(bits: int) -> np.ndarray:
    idx = np.arange(1 << bits, dtype=np.int64)
    out = np.zeros_like(idx)
    for b in range(bits):
        out |= ((idx >> b) & 1) << (bits - 1 - b)
    return out


def _powers(base: int, count: int, q: int) -> np.ndarray:
    """base^0 .. base^(count-1) mod q by repeated doubling (uint64, exact for q < 2^32)."""
    vals = np.ones(1, dtype=np.uint64)
    step = np.uint64(base % q)
    qq = np.uint64(q)
    while len(vals) < count:
        vals = np.concatenate([vals, vals * step % qq])
        step = step * step % qq
    return vals[:count]


@dataclass
class TwiddleTable:
    """Host view of one modulus's schedule-ordered twiddles (reference
    transform.py:43-73): fwd[t] = psi^bitrev(t), inv[t] = psi^-bitrev(t), the
    N^-1 constant, the phase split n1 and the O(sqrt N) seed arrays.  The
    tables themselves are read back from the device copy the kernels use."""

    modulus: Modulus
    n: int
    n1: int
    fwd: np.ndarray
    inv: np.ndarray
    n_inv: int
    seed_block: int
    fwd_seed_lo: np.ndarray
    fwd_seed_hi: np.ndarray
    inv_seed_lo: np.ndarray
    inv_seed_hi: np.ndarray

    @property
    def seed_size(self) -> int:
        return len(self.fwd_seed_lo) + len(self.fwd_seed_hi)

    def dump_text(self) -> str:
        head = f"# twiddles q={self.modulus.q} n={self.n} n1={self.n1}"
        body = (f"{t} {int(self.fwd[t])} {int(self.inv[t])}" for t in range(self.n))
        return "\n".join([head, *body])


def build_twiddle_table(m: Modulus, n: int | None = None, n1: int | None = None) -> TwiddleTable:
    n = m.n if n is None else n
    _check_degree(n)
    if (m.q - 1) % (2 * n):
        raise StructureError(f"modulus {m.q} is not NTT-friendly for degree {n}")
    lg = _log2(n)
    n1 = (1 << ((lg + 1) // 2)) if n1 is None else n1
    if n1 < 2 or n1 > n or n1 & (n1 - 1):
        raise ValueError("phase split n1 must be a power of two in [2, N]")
    psi = m.root_for_degree(n)
    psi_inv = pow(psi, -1, m.q)
    from .engine import get_engine

    fwd, inv, n_inv = get_engine().twiddle_tables(m, n)
    h = lg // 2
    lo_fwd = pow(psi, 1 << (lg - h), m.q) if h else psi
    lo_inv = pow(psi_inv, 1 << (lg - h), m.q) if h else psi_inv
    return TwiddleTable(
        modulus=m, n=n, n1=n1,
        fwd=fwd.astype(np.uint64), inv=inv.astype(np.uint64), n_inv=int(n_inv),
        seed_block=1 << h,
        fwd_seed_lo=_powers(lo_fwd, 1 << h, m.q), fwd_seed_hi=_powers(psi, n >> h, m.q),
        inv_seed_lo=_powers(lo_inv, 1 << h, m.q), inv_seed_hi=_powers(psi_inv, n >> h, m.q),
    )


@functools.lru_cache(maxsize=512)
def twiddle_table(m: Modulus, n: int) -> TwiddleTable:
    return build_twiddle_table(m, n)


def generate_twiddle(table: TwiddleTable, stage: int, index: int, m: Modulus,
                     direction: str = FORWARD) -> int:
    """Slot ``stage * seed_block + index`` rebuilt from the two seed arrays with
    one modular multiplication (reference transform.py:126-151)."""
    if m.q != table.modulus.q:
        raise StructureError("modulus does not match twiddle table")
    block = table.seed_block
    if not 0 <= stage < table.n // block:
        raise ValueError(f"stage {stage} out of range")
    if not 0 <= index < block:
        raise ValueError(f"index {index} out of range")
    h, lg = _log2(block), _log2(table.n)
    lo_pos = int(_bitrev_array(h)[index]) if h else 0
    hi_pos = int(_bitrev_array(lg - h)[stage]) if lg - h else 0
    lo, hi = ((table.fwd_seed_lo, table.fwd_seed_hi) if direction == FORWARD
              else (table.inv_seed_lo, table.inv_seed_hi))
    counters.seed_reads += 2
    counters.otf_mults += 1
    return int(lo[lo_pos]) * int(hi[hi_pos]) % m.q


def _require_tables(basis, n: int) -> None:
    from .engine import get_engine

    eng = get_engine()
    for m in basis:
        if (m.q - 1) % (2 * n):
            raise StructureError(f"modulus {m.q} is not NTT-friendly for degree {n}")
        if not eng.has_tables(m, n):
            raise NotImplementedError(
                f"modulus {m.q} (n={m.n}) has no device transform at degree {n}: "
                "the sm_100a butterflies need q < 2^31"
            )


def _transform(data, basis, n: int, direction: str, stages: range | None = None):
    from .engine import get_engine

    eng = get_engine()
    _check_degree(n)
    _require_tables(basis, n)
    slots = eng.row_slots(basis, n)
    inverse = direction == INVERSE
    if stages is None:
        out = eng.ntt(data, slots, inverse)
        done = _log2(n)
    else:
        out = eng.ntt_stages(data, slots, inverse, stages.start, stages.stop)
        done = len(stages)
    counters.butterflies += len(basis) * (n // 2) * done
    return out


def ntt(limb, m: Modulus, table: TwiddleTable | None = None, direction: str = FORWARD) -> np.ndarray:
    """Transform one limb or a stack of limbs sharing modulus ``m``; host
    arrays in, host uint64 out (reference transform.py:253-276)."""
    from .engine import get_engine

    arr = np.asarray(limb, dtype=np.uint64)
    single = arr.ndim == 1
    rows = arr.reshape(1, -1) if single else arr
    n = rows.shape[1]
    if table is not None and (table.n != n or table.modulus.q != m.q):
        raise StructureError(
            f"twiddle table for n={table.n}, q={table.modulus.q} does not match limb of "
            f"length {n} mod {m.q}"
        )
    if direction not in (FORWARD, INVERSE):
        raise ValueError(f"unknown direction {direction!r}")
    eng = get_engine()
    basis = (m,) * rows.shape[0]
    if table is not None and not _is_engine_table(table, m, n):
        # the reference transforms with whatever table it is handed (transform.py:253-276); a table
        # that is not the engine's own (e.g. verify.py:51-57 corrupts one slot as a negative control)
        # is uploaded and used as given
        _check_degree(n)
        slot = eng.custom_table_slot(m.q, n, table.fwd, table.inv, table.n_inv)
        slots = eng.torch.full((rows.shape[0],), slot, dtype=eng.torch.int32, device=eng.device)
        out = eng.ntt(eng.upload(rows.astype(np.uint32)), slots, direction == INVERSE)
        counters.butterflies += rows.shape[0] * (n // 2) * _log2(n)
    else:
        out = _transform(eng.upload(rows.astype(np.uint32)), basis, n, direction)
    host = out.cpu().numpy().view(np.uint32).astype(np.uint64)
    return host[0] if single else host


def _is_engine_table(table: TwiddleTable, m: Modulus, n: int) -> bool:
    """True when `table` holds exactly the twiddles the engine's resident tables hold for (m, n)."""
    from .engine import get_engine

    eng = get_engine()
    if not eng.has_tables(m, n):
        return True                    # no device transform for this modulus: _transform reports it
    own = twiddle_table(m, n)          # host copy of the resident tables, cached
    if table is own:
        return True
    return (int(table.n_inv) == int(own.n_inv) and np.array_equal(np.asarray(table.fwd, dtype=np.uint64), own.fwd)
            and np.array_equal(np.asarray(table.inv, dtype=np.uint64), own.inv))


def _expect_domain(p: Polynomial, direction: str) -> str:
    if direction not in (FORWARD, INVERSE):
        raise ValueError(f"unknown direction {direction!r}")
    want = COEFFICIENT if direction == FORWARD else EVALUATION
    if p.domain != want:
        raise StructureError(f"{direction} transform expects {want}-domain input")
    return EVALUATION if direction == FORWARD else COEFFICIENT


def ntt_polynomial(p: Polynomial, direction: str = FORWARD) -> Polynomial:
    """Whole-polynomial transform; flips the domain tag (reference transform.py:279-287)."""
    out_domain = _expect_domain(p, direction)
    return Polynomial(p.basis, _transform(p.data, p.basis, p.n, direction), out_domain)


def ntt_two_phase(p: Polynomial, direction: str = FORWARD, n1: int | None = None,
                  on_the_fly: bool = True) -> Polynomial:
    """Two-launch transform split after log2(n1) forward stages, bit-identical
    to ``ntt_polynomial`` (reference transform.py:290-323).  At N = 2^16 with
    the default n1 = 2^8 the two phases are exactly the engine's two fast
    kernels.  ``on_the_fly`` only changes which counters are charged: the
    device kernels read the same resident tables either way."""
    out_domain = _expect_domain(p, direction)
    lg = _log2(p.n)
    if n1 is None:
        n1 = 1 << ((lg + 1) // 2)
    if n1 < 2 or n1 > p.n or n1 & (n1 - 1):
        raise ValueError("phase split n1 must be a power of two in [2, N]")
    h1 = _log2(n1)
    split = h1 if direction == FORWARD else lg - h1
    first = _transform(p.data, p.basis, p.n, direction, range(0, split))
    second = _transform(first, p.basis, p.n, direction, range(split, lg))
    strided, bulk = n1 - 1, p.n - n1          # table slots touched by each phase, per limb
    ph1, ph2 = (strided, bulk) if direction == FORWARD else (bulk, strided)
    bulk_is_first = direction == INVERSE
    if on_the_fly:
        counters.seed_reads += 2 * bulk * p.num_limbs
        counters.otf_mults += bulk * p.num_limbs
        if bulk_is_first:
            counters.twiddle_slots_phase2 += ph2
        else:
            counters.twiddle_slots_phase1 += ph1
    else:
        counters.twiddle_slots_phase1 += ph1
        counters.twiddle_slots_phase2 += ph2
    return Polynomial(p.basis, second, out_domain)
