"""Generate tests/golden/golden.json by running the REFERENCE package
(/root/reference/pkg/src/rnscope) on the seeded recipes in recipes.py.

Run here (the reference cannot travel to the GPU box):

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_golden.py

Only digests (SHA-256 of the little-endian u32 wire image), parameter moduli
and a few tiny explicit vectors are stored, so the fixture stays small.  The
oracle (oracle/) is pinned against this file by tests/test_oracle_golden.py and
the CUDA path by the -m gpu tests.
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
from rnscope.params import ParameterSet, generate_parameter_set  # noqa: E402
from rnscope.rns import (  # noqa: E402
    COEFFICIENT, EVALUATION, Modulus, Polynomial, automorphism, find_ntt_primes, poly_elementwise,
)

import recipes as R  # noqa: E402


def load_params(name):
    kind, kw = R.PARAM_SETS[name]
    if kind == "gen":
        return generate_parameter_set(**kw)
    text = resources.files("rnscope").joinpath(f"data/params/{name}.json").read_text()
    return ParameterSet.from_dict(json.loads(text))


def qs_of(basis):
    return [m.q for m in basis]


def poly(basis, rows, domain):
    return Polynomial(tuple(basis), rows, domain)


def main():
    t0 = time.time()
    G = {"schema": 1, "params": {}, "twiddle": {}, "ntt": {}, "small": {}, "bconv": {},
         "automorphism": {}, "elementwise": {}, "keyswitch": {}, "composed": {}}
    P = {name: load_params(name) for name in R.PARAM_SETS}

    # ---- parameter sets (moduli + roots are data the product must reproduce) ----
    for name, p in P.items():
        d = p.to_dict()
        d["q_basis"] = [[m.q, m.psi] for m in p.q_basis]
        d["p_basis"] = [[m.q, m.psi] for m in p.p_basis]
        G["params"][name] = d

    # ---- tiny explicit vectors (tests/test_transform.py:18-31, :62-70) ----
    q17 = Modulus.for_prime(17, 4)
    t17 = transform.build_twiddle_table(q17, 4)
    G["small"]["q17_n4"] = {
        "psi": q17.psi, "fwd": t17.fwd.tolist(), "inv": t17.inv.tolist(), "n_inv": t17.n_inv,
        "ntt_delta": transform.ntt(np.array([1, 0, 0, 0], dtype=np.uint64), q17, t17).tolist(),
        "ntt_1234": transform.ntt(np.array([1, 2, 3, 4], dtype=np.uint64), q17, t17).tolist(),
        "intt_1234": transform.ntt(np.array([1, 2, 3, 4], dtype=np.uint64), q17, t17,
                                   direction="inverse").tolist(),
    }
    q97 = Modulus.for_prime(97, 16)
    t97 = transform.build_twiddle_table(q97, 16)
    x97 = R.rand_rows([97], 16, 11)
    G["small"]["q97_n16"] = {
        "psi": q97.psi, "fwd": t97.fwd.tolist(), "inv": t97.inv.tolist(), "n_inv": t97.n_inv,
        "x": x97[0].tolist(),
        "ntt": transform.ntt(x97[0], q97, t97).tolist(),
        "intt": transform.ntt(x97[0], q97, t97, direction="inverse").tolist(),
        "otf_fwd": [transform.generate_twiddle(t97, t // t97.seed_block, t % t97.seed_block, q97)
                    for t in range(16)],
    }
    # BConv worked example {5,7} -> {11} (tests/test_baseconv.py:29-33, :73-77)
    q5, q7, p11 = Modulus.for_prime(5, 1), Modulus.for_prime(7, 1), Modulus.for_prime(11, 1)
    tb = baseconv.build_bconv_table((q5, q7), (p11,))
    G["small"]["bconv_5_7_11"] = {
        "t": tb.t.tolist(), "inv_qhat": tb.inv_qhat.tolist(),
        "in": [[2], [5]],
        "out": baseconv.bconv(poly((q5, q7), np.array([[2], [5]], dtype=np.uint64), COEFFICIENT),
                              tb).coeffs.tolist(),
    }
    # find_ntt_primes for a few small degrees (moduli + minimal roots)
    G["small"]["primes"] = {
        f"{cnt}_{bits}_{n}": [[m.q, m.psi] for m in find_ntt_primes(cnt, bits, n)]
        for cnt, bits, n in [(3, 31, 4), (3, 31, 16), (3, 31, 256), (2, 30, 16), (1, 31, 1 << 16)]
    }

    # ---- twiddle tables + NTT on every parameter set's extended basis ----
    for name, p in P.items():
        ext = p.ext_basis
        st = transform._stacked_tables(ext, p.n)
        G["twiddle"][name] = {
            "fwd": R.digest(st.fwd), "inv": R.digest(st.inv),
            "n_inv": [int(x) for x in st.n_inv.ravel()],
        }
        x = R.rand_rows(qs_of(ext), p.n, 1)
        fwd = transform.ntt_polynomial(poly(ext, x, COEFFICIENT))
        inv = transform.ntt_polynomial(poly(ext, x, EVALUATION), "inverse")
        two = transform.ntt_two_phase(poly(ext, x, COEFFICIENT))
        assert np.array_equal(two.coeffs, fwd.coeffs)
        G["ntt"][name] = {"seed": 1, "in": R.digest(x), "fwd": R.digest(fwd.coeffs),
                          "inv": R.digest(inv.coeffs)}
        print(f"[{time.time() - t0:6.1f}s] ntt {name}")

    # NTT over small degrees with freshly searched primes (tests/test_transform.py:33-42)
    for n in (2, 4, 8, 16, 32, 64, 128, 256, 512, 1024, 2048):
        mods = find_ntt_primes(3, 31, n)
        x = R.rand_rows(qs_of(mods), n, 2)
        fwd = transform.ntt_polynomial(poly(mods, x, COEFFICIENT))
        inv = transform.ntt_polynomial(poly(mods, x, EVALUATION), "inverse")
        G["ntt"][f"n{n}"] = {"seed": 2, "moduli": [[m.q, m.psi] for m in mods],
                             "fwd": R.digest(fwd.coeffs), "inv": R.digest(inv.coeffs)}

    # ---- BConv: every raise table + ModDown table of every parameter set ----
    for name, p in P.items():
        tabs = ks._tables(p)
        entry = {"raise": [], "moddown": None}
        for t in range(p.dnum):
            digit = p.q_basis[p.digit_slice(t)]
            x = R.rand_rows(qs_of(digit), p.n, 10 + t)
            out = baseconv.convert(poly(digit, x, COEFFICIENT), tabs.raise_tables[t])
            entry["raise"].append({
                "seed": 10 + t, "out": R.digest(out.coeffs),
                "t": R.digest(tabs.raise_tables[t].t), "inv_qhat": R.digest(tabs.raise_tables[t].inv_qhat),
                "overflow_free": bool(tabs.raise_tables[t].overflow_free),
            })
        x = R.rand_rows(qs_of(p.p_basis), p.n, 20)
        out = baseconv.convert(poly(p.p_basis, x, COEFFICIENT), tabs.moddown_table)
        entry["moddown"] = {"seed": 20, "out": R.digest(out.coeffs),
                            "t": R.digest(tabs.moddown_table.t),
                            "inv_qhat": R.digest(tabs.moddown_table.inv_qhat),
                            "overflow_free": bool(tabs.moddown_table.overflow_free),
                            "p_inv": [int(v) for v in tabs.p_inv_col.ravel()]}
        entry["gadget"] = R.digest(tabs.gadget)
        G["bconv"][name] = entry
        print(f"[{time.time() - t0:6.1f}s] bconv {name}")
    # edge: worst-case accumulator (all residues q-1) on the ks48 digit-0 table
    p = P["ks48"]
    digit = p.q_basis[p.digit_slice(0)]
    x = np.stack([np.full(64, m.q - 1, dtype=np.uint64) for m in digit])
    out = baseconv.convert(poly(digit, x, COEFFICIENT), ks._tables(p).raise_tables[0])
    G["bconv"]["ks48_maxres"] = {"out": R.digest(out.coeffs)}

    # ---- automorphism (coefficient + evaluation domain) and element-wise ----
    for name in ("tiny", "verify_small", "n8192", "ks48"):
        p = P[name]
        x = R.rand_rows(qs_of(p.q_basis), p.n, 30)
        entry = {"seed": 30, "k": {}}
        for k in R.AUTOMORPHISM_KS:
            kk = k % (2 * p.n)
            c = automorphism(poly(p.q_basis, x, COEFFICIENT), kk)
            e = automorphism(poly(p.q_basis, x, EVALUATION), kk)
            entry["k"][str(k)] = {"coeff": R.digest(c.coeffs), "eval": R.digest(e.coeffs)}
        G["automorphism"][name] = entry
        y = R.rand_rows(qs_of(p.q_basis), p.n, 31)
        G["elementwise"][name] = {
            "seeds": [30, 31],
            **{kind: R.digest(poly_elementwise(poly(p.q_basis, x, EVALUATION),
                                               poly(p.q_basis, y, EVALUATION), kind).coeffs)
               for kind in ("add", "sub", "mul")},
        }
        print(f"[{time.time() - t0:6.1f}s] automorphism/elementwise {name}")

    # ---- key-switch pipeline, per stage (keyswitch.py:462-490 names) ----
    for case, (pname, s1, s2, mseed, cseed, eseed) in R.KS_CASES.items():
        p = P[pname]
        s_from, s_to = ks.keygen(p, seed=s1), ks.keygen(p, seed=s2)
        msg = R.message(p.n, p.delta, mseed)
        ct = ks.encrypt(msg, s_from, p, seed=cseed)
        evk = ks.switching_keygen(s_from, s_to, p, seed=eseed)
        raised = ks.keyswitch_stage1(ct.a, p)
        q_part, p_part = ks.keyswitch_stage2(raised, evk)
        delta = ks.keyswitch_stage3(q_part, p_part, p)
        out = ks.keyswitch(ct, evk)
        dec = ks.decrypt(out, s_to)
        dec0 = ks.decrypt(ct, s_from)
        G["keyswitch"][case] = {
            "params": pname, "seeds": [s1, s2, mseed, cseed, eseed],
            "s_from": R.digest_i64(s_from.ternary), "s_to": R.digest_i64(s_to.ternary),
            "msg": R.digest_i64(msg),
            "ct_a": R.digest(ct.a.coeffs), "ct_b": R.digest(ct.b.coeffs),
            "evk": [[R.digest(pr.a.coeffs), R.digest(pr.b.coeffs)] for pr in evk.pairs],
            "stage1_raised": [R.digest(r.coeffs) for r in raised],
            "stage2_acc_q_a": R.digest(q_part.a.coeffs), "stage2_acc_q_b": R.digest(q_part.b.coeffs),
            "stage2_acc_p_a": R.digest(p_part.a.coeffs), "stage2_acc_p_b": R.digest(p_part.b.coeffs),
            "stage3_out_a": R.digest(delta.a.coeffs), "stage3_out_b": R.digest(delta.b.coeffs),
            "out_a": R.digest(out.a.coeffs), "out_b": R.digest(out.b.coeffs),
            "decrypt_fresh": R.digest_i64(dec0), "decrypt_switched": R.digest_i64(dec),
            "max_abs_err_switched": int(np.abs(dec - msg).max()),
        }
        print(f"[{time.time() - t0:6.1f}s] keyswitch {case}")

    # ---- composed oracles for HRot / HMult+relinearize / rescale ----
    for pname in ("tiny", "n8192"):
        p = P[pname]
        sk = ks.keygen(p, seed=1)
        m1 = np.random.default_rng(7).integers(1, 9, p.n).astype(np.int64) << 20
        m2 = np.random.default_rng(8).integers(1, 9, p.n).astype(np.int64) << 20
        ct1 = ks.encrypt(m1, sk, p, seed=2)
        ct2 = ks.encrypt(m2, sk, p, seed=5)
        entry = {"msg_seeds": [7, 8], "ct_seeds": [2, 5], "sk_seed": 1}
        # HRot by galois element k: automorphism on (a, b), key-switch sigma_k(s) -> s
        for k in (5, 2 * p.n - 1):
            dest = (np.arange(p.n, dtype=np.int64) * k) % (2 * p.n)
            rot_s = np.zeros(p.n, dtype=np.int8)
            rot_s[dest % p.n] = np.where(dest >= p.n, -sk.ternary, sk.ternary)
            sk_rot = ks.SecretKey(ternary=rot_s, n=p.n)
            evk = ks.switching_keygen(sk_rot, sk, p, seed=40)
            rot = ks.Ciphertext(a=automorphism(ct1.a, k), b=automorphism(ct1.b, k), scale=ct1.scale)
            out = ks.keyswitch(rot, evk)
            dec = ks.decrypt(out, sk)
            m_rot = np.zeros(p.n, dtype=np.int64)
            m_rot[dest % p.n] = np.where(dest >= p.n, -m1, m1)
            entry[f"hrot_k{k}"] = {"evk_seed": 40, "out_a": R.digest(out.a.coeffs),
                                   "out_b": R.digest(out.b.coeffs),
                                   "max_abs_err": int(np.abs(dec - m_rot).max())}
        # HMult + relinearize: tensor, key-switch d2 under s^2 -> s, add d1
        s_ext = sk.eval_polynomial(p.ext_basis)
        sk_sq = ks.SecretKey(ternary=np.zeros(p.n, dtype=np.int8), n=p.n)
        sk_sq._eval_cache[tuple(m.q for m in p.ext_basis)] = poly_elementwise(s_ext, s_ext, "mul")
        rlk = ks.switching_keygen(sk_sq, sk, p, seed=41)
        d0 = poly_elementwise(ct1.b, ct2.b, "mul")
        d1 = poly_elementwise(poly_elementwise(ct1.a, ct2.b, "mul"),
                              poly_elementwise(ct2.a, ct1.b, "mul"), "add")
        d2 = poly_elementwise(ct1.a, ct2.a, "mul")
        sw = ks.keyswitch(ks.Ciphertext(a=d2, b=d0, scale=ct1.scale * ct2.scale), rlk)
        prod = ks.Ciphertext(a=poly_elementwise(sw.a, d1, "add"), b=sw.b, scale=sw.scale)
        entry["hmult"] = {"rlk_seed": 41, "rlk": [[R.digest(pr.a.coeffs), R.digest(pr.b.coeffs)]
                                                  for pr in rlk.pairs],
                          "d0": R.digest(d0.coeffs), "d1": R.digest(d1.coeffs), "d2": R.digest(d2.coeffs),
                          "out_a": R.digest(prod.a.coeffs), "out_b": R.digest(prod.b.coeffs)}
        # rescale by the last limb: INTT(last) -> convert 1 -> L-1 -> NTT -> (x - conv) * q_last^-1
        def rescale(x):
            last = p.q_basis[-1]
            rest = p.q_basis[:-1]
            c = transform.ntt_polynomial(poly((last,), x.coeffs[-1:], EVALUATION), "inverse")
            conv = baseconv.convert(c, baseconv.build_bconv_table((last,), rest))
            conv = transform.ntt_polynomial(conv)
            q_col = np.array(qs_of(rest), dtype=np.uint64)[:, None]
            inv = np.array([pow(last.q, -1, m.q) for m in rest], dtype=np.uint64)[:, None]
            return poly(rest, (x.coeffs[:-1] + q_col - conv.coeffs) % q_col * inv % q_col, EVALUATION)
        ra, rb = rescale(prod.a), rescale(prod.b)
        entry["rescale"] = {"out_a": R.digest(ra.coeffs), "out_b": R.digest(rb.coeffs)}
        # decrypt the rescaled product: slots-free check on coefficient 0 of m1*m2 is not
        # meaningful (negacyclic convolution), so record the decrypted row digest instead.
        dec = ks.decrypt(ks.Ciphertext(a=ra, b=rb, scale=1), sk)
        entry["rescale"]["decrypt"] = R.digest_i64(dec)
        G["composed"][pname] = entry
        print(f"[{time.time() - t0:6.1f}s] composed {pname}")

    out_path = Path(__file__).resolve().parent / "golden.json"
    out_path.write_text(json.dumps(G, indent=1) + "\n")
    print(f"wrote {out_path} ({out_path.stat().st_size} bytes) in {time.time() - t0:.1f}s")


if __name__ == "__main__":
    main()
