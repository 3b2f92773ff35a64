"""Seeded input recipes shared by the golden generator (which feeds them to
the reference) and by the tests (which feed them to the oracle and the CUDA
path).  NumPy only -- no reference, oracle or product imports -- so the same
bytes are rebuilt everywhere from the seed alone.
"""
from __future__ import annotations

import hashlib

import numpy as np


def digest(arr) -> str:
    """SHA-256 of the RNSV wire image of a residue matrix (vectors.py:40:
    little-endian u32, row-major)."""
    a = np.ascontiguousarray(np.asarray(arr), dtype="<u4")
    return hashlib.sha256(a.tobytes()).hexdigest()


def digest_i64(arr) -> str:
    a = np.ascontiguousarray(np.asarray(arr, dtype=np.int64), dtype="<i8")
    return hashlib.sha256(a.tobytes()).hexdigest()


def rand_rows(qs, n: int, seed: int) -> np.ndarray:
    """Same draw order as rns.random_polynomial (rns.py:219-223)."""
    rng = np.random.default_rng(seed)
    return np.stack([rng.integers(0, int(q), size=n, dtype=np.uint64) for q in qs])


def message(n: int, delta: int, seed: int, bound: int = 8) -> np.ndarray:
    """The signed delta-scaled message of the reference tests
    (tests/test_keyswitch.py:14-17, tests/test_acceptance.py:112-114)."""
    rng = np.random.default_rng(seed)
    m = rng.integers(1, bound + 1, n).astype(np.int64)
    m *= rng.choice(np.array([-1, 1], dtype=np.int64), n)
    return m * delta


# Parameter sets the goldens cover.  "gen" entries are produced with
# generate_parameter_set(n, l, dnum, delta, h_dense, h_sparse); "file" entries
# are the reference's shipped JSON (data/params/<name>.json).
PARAM_SETS = {
    "tiny": ("gen", dict(n=64, l=6, dnum=3, delta=1 << 25, h_dense=8, h_sparse=4)),
    "n8192": ("gen", dict(n=8192, l=12, dnum=3, delta=1 << 40, h_dense=64, h_sparse=32)),
    "verify_small": ("file", None),
    "ks12": ("file", None),
    "ks24": ("file", None),
    "ks48": ("file", None),
}

# key-switch pipeline cases: (param set, s_from seed, s_to seed, msg seed, ct seed, evk seed)
KS_CASES = {
    "tiny": ("tiny", 1, 2, 99, 3, 4),
    "verify_small": ("verify_small", 1, 2, 0, 3, 4),
    "n8192": ("n8192", 1, 2, 7, 3, 4),
    "ks48": ("ks48", 1, 2, 5, 3, 4),
}

AUTOMORPHISM_KS = (3, 5, 25, -1)


# ---- level-l key switching on the ks48 moduli (tests/golden/make_golden_level.py) -------------
# A ciphertext at level l lives over the first l limbs of ks48's Q basis and is switched with
# the rows of a FULL-level key that belong to active limbs.  The reference enforces
# L = dnum * alpha (params.py:40), so l in LEVEL_FULL_DIGITS is pinned by its own keyswitch() on
# a ParameterSet cut to those limbs; other levels (partial last digit), hoisted rotations and the
# ModDown merged with a rescale are pinned by compositions of its public primitives.
LEVEL_FULL_DIGITS = (12, 24, 36, 48)
LEVEL_PARTIAL = (42, 21)
LEVEL_EVK_SEED = 100          # key polynomial (digit t, half h): rand_rows(ext48, n, 100 + 2 t + h)
LEVEL_CT_SEEDS = (200, 201)   # ciphertext halves (a, b) over the first l limbs
HOIST_CASES = ((24, 5), (42, 25), (21, -1))          # (level, automorphism index k)
MERGED_MODDOWN_CASES = ((48, 2), (30, 2), (19, 1))   # (level l, dropped limbs k): Q_{l-k} <- Q_l || P
MERGED_SEEDS = (300, 301)     # the two [l + alpha] accumulator halves


def level_key_rows(ext_qs, n: int, t: int, h: int) -> np.ndarray:
    return rand_rows(ext_qs, n, LEVEL_EVK_SEED + 2 * t + h)
