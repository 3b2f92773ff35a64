"""CPU checks of the bootstrapping host math: the diagonal factorisation of the
canonical embedding used by CoeffToSlot / SlotToCoeff (no GPU calls)."""
import numpy as np
import pytest

from paper_2512_18345_b200.bootstrap import apply_diagonals, default_groups, dft_stage, grouped_dft
from paper_2512_18345_b200.ckks import Embedding


def bitrev_perm(n):
    lg = n.bit_length() - 1
    idx = np.arange(n)
    out = np.zeros(n, dtype=np.int64)
    for b in range(lg):
        out |= ((idx >> b) & 1) << (lg - 1 - b)
    return out


@pytest.mark.parametrize("N", [16, 64, 512, 4096])
def test_grouped_dft_is_the_embedding_without_bit_reversal(N):
    n = N // 2
    lg = n.bit_length() - 1
    rng = np.random.default_rng(N)
    m = rng.normal(size=N)
    z = Embedding(N).to_slots(m)
    w = m[:n] + 1j * m[n:]
    R = bitrev_perm(n)
    for count in (1, 2, 3):
        if count > lg:
            continue
        sizes = default_groups(lg, count)
        x = w[R]
        for g in grouped_dft(n, sizes, inverse=False):
            x = apply_diagonals(g, x)
        assert np.abs(x - z).max() < 1e-9 * np.abs(z).max()        # SlotToCoeff direction
        y = z
        for g in grouped_dft(n, sizes, inverse=True):
            y = apply_diagonals(g, y)
        assert np.abs(y - w[R]).max() < 1e-9 * np.abs(w).max()     # CoeffToSlot direction


def test_stage_structure_and_diagonal_counts():
    n = 1 << 10
    for ell in (1, 5, 10):
        st = dft_stage(n, ell, False)
        inv = dft_stage(n, ell, True)
        assert len(st) <= 3 and len(inv) <= 3
        x = np.random.default_rng(ell).normal(size=n) + 0j
        assert np.abs(apply_diagonals(inv, apply_diagonals(st, x)) - x).max() < 1e-12
    groups = grouped_dft(n, default_groups(10, 3), inverse=False)
    # r merged stages give at most 2^(r+1) - 1 diagonals
    for g, r in zip(groups, default_groups(10, 3)):
        assert len(g) <= 2 ** (r + 1) - 1


def test_exp_polynomial_accuracy_and_parity():
    """The EvalMod polynomial: Chebyshev interpolation of exp(i*y) on the range the squarings
    leave beats the Taylor series of the same degree, has cos/sin parity, and the x = i*y form is
    real.  Error on the message after r squarings and the Q0/(2*pi*Delta) factor stays below 2^-26
    (SlotToCoeff adds this deterministic error up over sqrt(slots) terms)."""
    import math

    from paper_2512_18345_b200.bootstrap import BootstrapConfig, exp_coefficients

    cfg = BootstrapConfig()
    bound = 2 * math.pi * cfg.k_bound / (1 << cfg.squarings)
    ys = np.linspace(-bound, bound, 20001)
    a, c = exp_coefficients(cfg)
    assert len(a) == cfg.degree + 1 == 16
    err = np.abs(np.polyval(a[::-1], ys) - np.exp(1j * ys)).max()
    ta, _ = exp_coefficients(BootstrapConfig(approx="taylor"))
    terr = np.abs(np.polyval(ta[::-1], ys) - np.exp(1j * ys)).max()
    assert err < terr / 50
    amplification = (1 << cfg.squarings) * (2.0 ** 62 / (2 * math.pi * 2.0 ** cfg.log_delta_in))
    assert err * amplification < 2.0 ** -26
    for k in range(cfg.degree + 1):
        assert (a[k].imag == 0.0) if k % 2 == 0 else (a[k].real == 0.0)
        assert abs(complex(c[k]).imag) < 1e-300
    assert np.abs(np.polyval(c[::-1], 1j * ys) - np.exp(1j * ys)).max() < 2 * err
