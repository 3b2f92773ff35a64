"""Generate tests/golden/golden_level.json with the REFERENCE package: key switching of a
ciphertext at level l <= L with the full-level key, hoisted rotations and the ModDown merged
with a rescale, on the ks48 moduli at N = 2^16.

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_golden_level.py

 * l in {12, 24, 36, 48}: the reference's own keyswitch_stage1 / stage2 / stage3 / keyswitch
   (keyswitch.py:297-453) on a ParameterSet cut to the first l limbs of ks48 (dnum = l / 12), with
   the rows of the full-level key that belong to active limbs.  The same values are then rebuilt
   from the reference's public primitives (transform.ntt_polynomial, baseconv.convert,
   rns.poly_elementwise) and asserted equal, which validates the composition recipe.
 * l in {42, 21} (partial last digit, rejected by params.py:40): the composition recipe alone.
 * hoisted key switch: digits read through rns.automorphism (evaluation domain), P * sigma_k(b)
   lifted into the accumulator.
 * merged ModDown: (x_rest - NTT(convert(INTT(x_{dropped || P})))) * (P * dropped)^-1.

Only digests are stored.  The oracle (oracle/engine_oracle.py) and the CUDA path are both
checked against this file by tests/test_level_keyswitch.py.
"""
from __future__ import annotations

import json
import math
import sys
import time
from importlib import resources
from pathlib import Path

import numpy as np

sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, str(Path(__file__).resolve().parent))

from rnscope import baseconv, keyswitch as ks, transform  # noqa: E402
from rnscope.params import ParameterSet  # noqa: E402
from rnscope.rns import COEFFICIENT, EVALUATION, Polynomial, automorphism, poly_elementwise  # noqa: E402

import recipes as R  # noqa: E402


def qs_of(basis):
    return [m.q for m in basis]


def poly(basis, rows, domain):
    return Polynomial(tuple(basis), rows, domain)


def const_rows(basis, values, n):
    return poly(basis, np.broadcast_to(np.array(values, dtype=np.uint64)[:, None], (len(basis), n)).copy(), EVALUATION)


def raise_composed(a, q, p, alpha):
    """ModUp of every digit of `a` (over q, evaluation domain) to q || p from public primitives."""
    l, ext = len(q), tuple(q) + tuple(p)
    coeff = transform.ntt_polynomial(a, "inverse")
    out = []
    for t in range(-(-l // alpha)):
        lo, hi = t * alpha, min(l, (t + 1) * alpha)
        target = tuple(m for i, m in enumerate(q) if not lo <= i < hi) + tuple(p)
        block = poly(q[lo:hi], coeff.coeffs[lo:hi], COEFFICIENT)
        conv = transform.ntt_polynomial(baseconv.convert(block, baseconv.build_bconv_table(q[lo:hi], target)))
        rows = np.empty((len(ext), a.n), dtype=np.uint64)
        src = 0
        for r in range(len(ext)):
            if lo <= r < hi:
                rows[r] = a.coeffs[r]
            else:
                rows[r] = conv.coeffs[src]
                src += 1
        out.append(poly(ext, rows, EVALUATION))
    return out


def inner_composed(raised, key_pairs):
    acc_a = acc_b = None
    for d, (ka, kb) in zip(raised, key_pairs):
        ta, tb = poly_elementwise(d, ka, "mul"), poly_elementwise(d, kb, "mul")
        acc_a = ta if acc_a is None else poly_elementwise(acc_a, ta, "add")
        acc_b = tb if acc_b is None else poly_elementwise(acc_b, tb, "add")
    return acc_a, acc_b


def moddown_composed(x, rest, pp):
    """x over rest || pp (evaluation) -> (x_rest - NTT(convert(INTT(x_pp)))) * prod(pp)^-1 over rest."""
    l = len(rest)
    c = transform.ntt_polynomial(poly(pp, x.coeffs[l:], EVALUATION), "inverse")
    conv = transform.ntt_polynomial(baseconv.convert(c, baseconv.build_bconv_table(tuple(pp), tuple(rest))))
    prod = math.prod(m.q for m in pp)
    diff = poly_elementwise(poly(rest, x.coeffs[:l], EVALUATION), conv, "sub")
    return poly_elementwise(diff, const_rows(rest, [pow(prod, -1, m.q) for m in rest], x.n), "mul")


def main():
    t0 = time.time()
    text = resources.files("rnscope").joinpath("data/params/ks48.json").read_text()
    p48 = ParameterSet.from_dict(json.loads(text))
    n, alpha = p48.n, p48.alpha
    ext48 = p48.ext_basis
    full_key = {(t, h): R.level_key_rows(qs_of(ext48), n, t, h) for t in range(p48.dnum) for h in range(2)}
    G = {"schema": 1, "params": "ks48", "level": {}, "hoisted": {}, "merged_moddown": {}}

    def key_pairs(q, beta):
        rows = list(range(len(q))) + list(range(p48.l, p48.l + alpha))
        ext = tuple(q) + p48.p_basis
        return [(poly(ext, full_key[(t, 0)][rows], EVALUATION), poly(ext, full_key[(t, 1)][rows], EVALUATION))
                for t in range(beta)]

    def ciphertext(q):
        return (poly(q, R.rand_rows(qs_of(q), n, R.LEVEL_CT_SEEDS[0]), EVALUATION),
                poly(q, R.rand_rows(qs_of(q), n, R.LEVEL_CT_SEEDS[1]), EVALUATION))

    def record(raised, acc_a, acc_b, out_a, out_b):
        return {"stage1_raised": [R.digest(r.coeffs) for r in raised],
                "stage2_acc_a": R.digest(acc_a.coeffs), "stage2_acc_b": R.digest(acc_b.coeffs),
                "out_a": R.digest(out_a.coeffs), "out_b": R.digest(out_b.coeffs)}

    for l in R.LEVEL_FULL_DIGITS + R.LEVEL_PARTIAL:
        q = p48.q_basis[:l]
        beta = -(-l // alpha)
        a, b = ciphertext(q)
        pairs = key_pairs(q, beta)
        raised = raise_composed(a, q, p48.p_basis, alpha)
        acc_a, acc_b = inner_composed(raised, pairs)
        out_a = moddown_composed(acc_a, q, p48.p_basis)
        out_b = poly_elementwise(moddown_composed(acc_b, q, p48.p_basis), b, "add")
        entry = record(raised, acc_a, acc_b, out_a, out_b)
        entry["source"] = "composition of reference primitives"
        if l in R.LEVEL_FULL_DIGITS:
            pl = ParameterSet(n=n, l=l, dnum=l // alpha, alpha=alpha, beta=beta, delta=p48.delta,
                              log_pq=p48.log_pq, h_dense=p48.h_dense, h_sparse=p48.h_sparse,
                              q_basis=q, p_basis=p48.p_basis)
            evk = ks.SwitchingKey(pairs=tuple(ks.PolyPair(a=ka, b=kb) for ka, kb in pairs), params=pl)
            r_raised = ks.keyswitch_stage1(a, pl)
            q_part, p_part = ks.keyswitch_stage2(r_raised, evk)
            out = ks.keyswitch(ks.Ciphertext(a=a, b=b, scale=1), evk)
            r_acc_a = np.concatenate([q_part.a.coeffs, p_part.a.coeffs])
            r_acc_b = np.concatenate([q_part.b.coeffs, p_part.b.coeffs])
            ref = record(r_raised, poly(tuple(q) + p48.p_basis, r_acc_a, EVALUATION),
                         poly(tuple(q) + p48.p_basis, r_acc_b, EVALUATION), out.a, out.b)
            for k, v in ref.items():
                assert entry[k] == v, f"composition differs from the reference routine at l={l}: {k}"
            entry["source"] = "reference keyswitch() on a ParameterSet cut to l limbs (== composition)"
        G["level"][str(l)] = entry
        print(f"[{time.time() - t0:6.1f}s] level {l}")

    # hoisted rotation: KS(sigma_k(ct)) from the raised digits of the UNROTATED a part
    for l, k in R.HOIST_CASES:
        q = p48.q_basis[:l]
        ext = tuple(q) + p48.p_basis
        beta = -(-l // alpha)
        kk = k % (2 * n)
        a, b = ciphertext(q)
        pairs = key_pairs(q, beta)
        raised = [automorphism(r, kk) for r in raise_composed(a, q, p48.p_basis, alpha)]
        acc_a, acc_b = inner_composed(raised, pairs)
        # raw accumulator: P * sigma_k(b) lifted onto the Q rows of the b half
        p_prod = math.prod(m.q for m in p48.p_basis)
        sig_b = automorphism(b, kk)
        lift = np.concatenate([poly_elementwise(sig_b, const_rows(q, [p_prod % m.q for m in q], n), "mul").coeffs,
                               np.zeros((alpha, n), dtype=np.uint64)])
        raw_b = poly_elementwise(acc_b, poly(ext, lift, EVALUATION), "add")
        out_a = moddown_composed(acc_a, q, p48.p_basis)
        out_b = poly_elementwise(moddown_composed(acc_b, q, p48.p_basis), sig_b, "add")
        G["hoisted"][f"{l}_{k}"] = {"raw_a": R.digest(acc_a.coeffs), "raw_b": R.digest(raw_b.coeffs),
                                    "out_a": R.digest(out_a.coeffs), "out_b": R.digest(out_b.coeffs)}
        print(f"[{time.time() - t0:6.1f}s] hoisted l={l} k={k}")

    # ModDown merged with the rescale by the top k limbs
    for l, k in R.MERGED_MODDOWN_CASES:
        q = p48.q_basis[:l]
        ext = tuple(q) + p48.p_basis
        rest, pp = q[:l - k], q[l - k:] + p48.p_basis
        entry = {}
        for h, seed in enumerate(R.MERGED_SEEDS):
            x = poly(ext, R.rand_rows(qs_of(ext), n, seed), EVALUATION)
            entry["out_" + "ab"[h]] = R.digest(moddown_composed(x, rest, pp).coeffs)
        G["merged_moddown"][f"{l}_{k}"] = entry
        print(f"[{time.time() - t0:6.1f}s] merged moddown l={l} k={k}")

    out_path = Path(__file__).resolve().parent / "golden_level.json"
    out_path.write_text(json.dumps(G, indent=1) + "\n")
    print(f"wrote {out_path} ({out_path.stat().st_size} bytes) in {time.time() - t0:.1f}s")


if __name__ == "__main__":
    main()
