"""CPU-only checks of the host-side logic of the product package (no CUDA
calls): prime and root search, parameter sets, RNSV wire format, structural
errors, the closed-form automorphism permutation, counters."""
import json
import struct

import numpy as np
import pytest

import recipes as R
from paper_2512_18345_b200 import params as P
from paper_2512_18345_b200 import rns, vectors
from paper_2512_18345_b200.baseconv import search_overflow_free_moduli
from paper_2512_18345_b200.instrument import counters


def test_prime_and_root_search_match_reference(golden):
    for key, want in golden["small"]["primes"].items():
        cnt, bits, n = (int(v) for v in key.split("_"))
        assert [[m.q, m.psi] for m in rns.find_ntt_primes(cnt, bits, n)] == want
    assert rns.Modulus.for_prime(17, 4).psi == golden["small"]["q17_n4"]["psi"]
    assert rns.Modulus.for_prime(97, 16).psi == golden["small"]["q97_n16"]["psi"]


def test_is_prime_small_and_edges():
    known = [2, 3, 5, 7, 11, 13, 17, 97, 2147483647, 4294967291]
    assert all(rns.is_prime(p) for p in known)
    assert not any(rns.is_prime(c) for c in [0, 1, 4, 9, 561, 2147483649, 4294967295, 3215031751])


def test_modulus_validation():
    with pytest.raises(rns.RnsError):
        rns.Modulus.for_prime(15, 1)
    with pytest.raises(rns.RnsError):
        rns.Modulus.for_prime((1 << 32) + 15, 1)
    with pytest.raises(rns.RnsError):
        rns.Modulus.for_prime(17, 16)
    with pytest.raises(rns.RnsError):
        rns.Modulus.for_prime(17, 4, psi=3)
    m = rns.Modulus.for_prime(17, 4)
    for x in range(17 * 17):
        assert m.reduce(x) == x % 17
    assert rns.mod_arith(16, 5, m, "add") == 4 and rns.mod_arith(3, 5, m, "sub") == 15
    assert rns.mod_arith(16, 16, m, "mul") == 1
    with pytest.raises(ValueError):
        rns.mod_arith(1, 1, m, "pow")
    m64 = rns.Modulus.for_prime(2147483137, 64)
    r32 = m64.root_for_degree(32)
    assert pow(r32, 32, m64.q) == m64.q - 1


def test_find_ntt_primes_errors():
    with pytest.raises(ValueError):
        rns.find_ntt_primes(0, 31, 16)
    with pytest.raises(ValueError):
        rns.find_ntt_primes(1, 31, 12)
    with pytest.raises(ValueError):
        rns.find_ntt_primes(1, 33, 16)
    with pytest.raises(rns.InsufficientPrimesError):
        rns.find_ntt_primes(3, 8, 16)
    with pytest.raises(rns.InsufficientPrimesError):
        search_overflow_free_moduli(1, 2, 16, 8)


@pytest.mark.parametrize("name", ["verify_small", "ks12", "ks24", "ks48"])
def test_builtin_parameter_sets_equal_reference_files(golden, name):
    p = P.ParameterSet.builtin(name)
    g = golden["params"][name]
    assert [[m.q, m.psi] for m in p.q_basis] == g["q_basis"]
    assert [[m.q, m.psi] for m in p.p_basis] == g["p_basis"]
    for k in ("n", "l", "dnum", "alpha", "beta", "delta", "log_pq", "h_dense", "h_sparse"):
        assert getattr(p, k) == g[k]


def test_generated_parameter_sets_and_json_roundtrip(golden, tmp_path):
    for name in ("tiny", "n8192"):
        p = P.generate_parameter_set(**R.PARAM_SETS[name][1])
        g = golden["params"][name]
        assert [[m.q, m.psi] for m in p.q_basis] == g["q_basis"]
        assert [[m.q, m.psi] for m in p.p_basis] == g["p_basis"]
        assert p.log_pq == g["log_pq"] and p.beta == g["beta"]
        p.save(tmp_path / "p.json")
        assert P.ParameterSet.load(tmp_path / "p.json") == p
        d = p.to_dict()
        assert d["schema_version"] == 1 and set(d["q_basis"][0]) == {"q", "psi"}
        assert p.ext_basis == p.q_basis + p.p_basis
        assert p.digit_slice(1) == slice(p.alpha, 2 * p.alpha)
        with pytest.raises(ValueError):
            p.digit_slice(p.dnum)
    with pytest.raises(rns.RnsError):
        P.generate_parameter_set(n=64, l=6, dnum=4, delta=1, h_dense=8, h_sparse=4)
    bad = dict(golden["params"]["tiny"])
    bad["l"] = 5
    with pytest.raises(rns.RnsError):
        P.ParameterSet.from_dict(bad)


def test_polynomial_structure_checks_without_gpu():
    m = rns.Modulus.for_prime(17, 4)
    with pytest.raises(rns.StructureError):
        rns.Polynomial((m,), np.zeros((2, 4)), rns.COEFFICIENT)
    with pytest.raises(rns.StructureError):
        rns.Polynomial((m,), np.zeros((1, 4)), "frequency")
    p = rns.Polynomial((m,), np.array([[1, 2, 3, 16]]), rns.COEFFICIENT)
    assert p.num_limbs == 1 and p.n == 4 and p.q_column().tolist() == [[17]]
    p.validate()
    with pytest.raises(rns.StructureError):
        rns.Polynomial((m,), np.array([[1, 2, 3, 17]]), rns.COEFFICIENT).validate()
    assert rns.poly_equal(p, p.copy())
    z = rns.zero_polynomial((m,), 4)
    assert not z.coeffs.any() and z.domain == rns.COEFFICIENT
    r = rns.random_polynomial((m,), 4, np.random.default_rng(1))
    assert np.array_equal(r.coeffs, R.rand_rows([17], 4, 1))


def test_rnsv_byte_layout_and_roundtrip(tmp_path):
    m1, m2 = rns.Modulus.for_prime(17, 4), rns.Modulus.for_prime(97, 4)
    poly = rns.Polynomial((m1, m2), np.array([[1, 2, 3, 4], [5, 6, 7, 96]]), rns.EVALUATION)
    blob = vectors.polynomial_to_bytes(poly)
    assert blob[:4] == b"RNSV"
    magic, version, domain, pad, limbs, n = struct.unpack_from("<4sHBBII", blob, 0)
    assert (version, domain, pad, limbs, n) == (1, 1, 0, 2, 4)
    assert struct.unpack_from("<QQQ", blob, 16) == (17, m1.psi, 4)
    assert len(blob) == 16 + 2 * 24 + 2 * 4 * 4
    assert np.frombuffer(blob, dtype="<u4", offset=16 + 48).tolist() == [1, 2, 3, 4, 5, 6, 7, 96]
    back = vectors.polynomial_from_bytes(blob)
    assert rns.poly_equal(back, poly)
    vectors.save_polynomial(tmp_path / "v.rnsv", poly)
    assert rns.poly_equal(vectors.load_polynomial(tmp_path / "v.rnsv"), poly)
    with pytest.raises(rns.RnsError):
        vectors.polynomial_from_bytes(b"XXXX" + blob[4:])
    with pytest.raises(rns.RnsError):
        vectors.polynomial_from_bytes(blob[:4] + struct.pack("<H", 9) + blob[6:])


def test_closed_form_eval_permutation_matches_oracle(oracle_mod):
    """The device kernel's closed form == the reference's probe-derived
    permutation (restated by the oracle, rns.py:268-292)."""
    for n in (2, 4, 16, 64, 256, 4096):
        q, psi = oracle_mod.find_ntt_primes(1, 31, n)[0]
        orc = oracle_mod.Oracle(n, [(q, psi)])
        for k in (3, 5, 25, 2 * n - 1, 2 * n + 3):
            if k % 2 == 0:
                continue
            want = orc.eval_permutation(k)
            got = rns.eval_permutation_closed_form(n, k)
            assert np.array_equal(got, want), (n, k)


def test_no_gpu_fails_loudly():
    import torch

    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    from paper_2512_18345_b200 import _lib

    m = rns.Modulus.for_prime(17, 4)
    p = rns.Polynomial((m,), np.zeros((1, 4)), rns.EVALUATION)
    with pytest.raises(_lib.EngineUnavailable):
        rns.poly_elementwise(p, p, "add")


def test_counters_object():
    counters.reset()
    counters.butterflies += 3
    assert counters.snapshot()["butterflies"] == 3
    counters.reset()
    assert not any(counters.snapshot().values())


def test_plan_batch_matches_reference_model(golden):
    """scheduler.plan_batch reproduces the reference's B* (1/1/1 at ks48,
    5/3/3 at ks24, 15/7/7 at ks12 on a 98 MB L2) and scales to B200's 126 MB."""
    from paper_2512_18345_b200.params import ParameterSet
    from paper_2512_18345_b200.scheduler import B200_L2_BYTES, concurrent_keyswitches, keyswitch_footprint, plan_batch

    want = {"ks48": (1, 1, 1), "ks24": (5, 3, 3), "ks12": (15, 7, 7)}
    for name, (s1, s3, full) in want.items():
        p = ParameterSet.from_dict(golden["params"][name])
        l2 = 98 * 10 ** 6
        assert (plan_batch(p, "ks_stage1", l2).batch, plan_batch(p, "ks_stage3", l2).batch,
                plan_batch(p, "ks_full", l2).batch) == (s1, s3, full)
    p48 = ParameterSet.from_dict(golden["params"]["ks48"])
    assert keyswitch_footprint(p48, 1) == 4 * 60 * 65536 * 4 and keyswitch_footprint(p48, 3) == 4 * 48 * 65536 * 4
    plan = plan_batch(p48, "ks_full")
    assert plan.l2_capacity == B200_L2_BYTES and plan.batch == 2 and not plan.spills
    assert plan_batch(p48, "ks_full", 10 ** 6).spills
    p12 = ParameterSet.from_dict(golden["params"]["ks12"])
    assert concurrent_keyswitches(p12, lanes=4, pending=10) == 4
    assert concurrent_keyswitches(p48, lanes=8, pending=10) == 2
    assert concurrent_keyswitches(p48, lanes=1, pending=10) == 1
    import pytest
    with pytest.raises(ValueError):
        plan_batch(p48, "nope")


def test_machine_profile_follows_the_reference_schema():
    """data/profiles/b200.json carries every field the reference's MachineModel.from_dict reads
    (costmodel.py:95-103) and satisfies its constructor checks (:73-79)."""
    from paper_2512_18345_b200.scheduler import B200_L2_BYTES, machine_profile

    prof = machine_profile()
    for key in ("name", "l2_capacity", "l2_read_bw", "l2_write_bw", "dram_bw", "fma_tput", "alu_tput",
                "launch_overhead", "saturation_limbs"):
        assert prof[key] == prof[key] and (isinstance(prof[key], str) or prof[key] > 0)
    assert prof["schema_version"] == 1
    assert prof["l2_write_bw"] <= prof["l2_read_bw"]
    assert prof["dram_bw"] < prof["l2_write_bw"]
    assert int(prof["l2_capacity"]) == B200_L2_BYTES


def test_reference_timing_tool_runs_the_real_reference():
    """baseline/time_reference.py (bench.py's `cpu_baseline.reference`): imports the travelling copy of the
    NumPy reference only, times a unit single-process and on a process pool, prints one JSON line."""
    import json
    import subprocess
    import sys
    from pathlib import Path

    root = Path(__file__).resolve().parent.parent
    if not (root / "baseline" / "_ref" / "rnscope").is_dir():
        pytest.skip("no travelling copy of the reference (baseline/_ref); __graft_entry__.build() makes it")
    res = subprocess.run([sys.executable, str(root / "baseline" / "time_reference.py"), "ntt", "--rows", "2", "--pool", "2"],
                         capture_output=True, text=True, timeout=300)
    assert res.returncode == 0, res.stderr[-500:]
    doc = json.loads([ln for ln in res.stdout.splitlines() if ln.startswith("{")][-1])
    assert doc["kind"] == "reference" and doc["workload"] == "ntt"
    assert doc["single_process"]["ms_per_unit"] > 0 and doc["pool"]["processes"] == 2
    src = (root / "baseline" / "time_reference.py").read_text()
    assert "paper_2512_18345_b200" not in src.split('"""')[2], "the reference timing tool must not import the product"
