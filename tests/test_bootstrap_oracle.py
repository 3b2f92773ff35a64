"""The headline circuit against the composed CPU oracle.

The reference has no bootstrapping; its oracle is the package's own
circuit (bootstrap.py) replayed on the C restatement of the reference primitives
(oracle/engine_oracle.py; building blocks pinned to the reference by golden.json and
golden_level.json).  tests/golden/golden_bootstrap.json holds that oracle's limb digests after
every phase (tests/golden/make_golden_bootstrap.py).

 * CPU (not gpu): the oracle bootstrap at N = 2^11 reproduces the committed digests and
   refreshes the message to 2^-20.
 * gpu: the CUDA bootstrap -- eager, and as the 8-lane CUDA graph bench.py times -- at
   N = 2^11 and at the headline configuration (ks48: N = 2^16, 2^15 slots, dense key with
   sparse-secret encapsulation) equals the oracle replayed on the same box phase by phase and
   limb for limb, and equals the committed digests.

The circuit's plaintexts (DFT diagonals) are encoded on the host in floating point.  Live
comparisons share them; the committed digests are compared only when this machine encodes the
same plaintext limbs as the machine that generated them ("plaintexts" digest), otherwise that
part is reported as skipped rather than failed."""
import json
from pathlib import Path

import numpy as np
import pytest

import make_golden_bootstrap as G

GOLD = json.loads((Path(__file__).resolve().parent / "golden" / "golden_bootstrap.json").read_text())["cases"]


def with_oracle(fn):
    from oracle.engine_oracle import OracleEngine
    from paper_2512_18345_b200 import engine

    previous = engine.use_backend(OracleEngine())
    try:
        return fn()
    finally:
        engine.use_backend(previous)


def check_against_committed(name, rec):
    g = GOLD[name]
    if rec["plaintexts"] != g["plaintexts"]:
        pytest.skip("this host encodes the DFT diagonals with different floating-point rounding than the "
                    "golden generator's; live oracle comparison above still applies")
    assert rec["input"] == g["input"]
    assert rec["phases"] == g["phases"]
    assert rec["out_level"] == g["out_level"]


def test_oracle_bootstrap_n2048_matches_committed_digests():
    rec, _ = with_oracle(lambda: G.run_case("n2048"))
    assert rec["precision_log2"] < -20.0, rec["precision_log2"]
    assert set(rec["phases"]) == {"mod_raise", "coeff_to_slot_lo", "coeff_to_slot_hi", "eval_mod", "slot_to_coeff"}
    check_against_committed("n2048", rec)


@pytest.mark.gpu
@pytest.mark.parametrize("name,bar", [("n2048", -20.0), ("ks48", -20.0)])
def test_cuda_bootstrap_equals_oracle(name, bar):
    """bar: north_star's example tolerance 2^-20 at both sizes (the paper reports 2^-18.57 for its
    bootstrap at N = 2^16; measured here: 2^-21.9 at N = 2^11, 2^-21.1 at ks48)."""
    import torch

    assert torch.cuda.is_available(), "GPU tests need a CUDA device"
    from paper_2512_18345_b200 import ckks
    from paper_2512_18345_b200.engine import get_engine

    eng = get_engine()
    eng.set_lanes(1)
    rec, (p, sk, boot, z, ct) = G.run_case(name)                      # CUDA, eager, one lane
    assert rec["precision_log2"] < bar, rec["precision_log2"]
    # the graph bench.py replays: 8 stream lanes, nested forks, programmatic dependent launches
    eng.set_lanes(8)
    replay = boot.capture(ct)
    out = replay(ct)
    torch.cuda.synchronize()
    assert G.ct_digest(out) == rec["phases"]["slot_to_coeff"], "8-lane graph differs from the eager bootstrap"
    eng.set_lanes(1)
    # the oracle on the same keys, plaintexts and input (pulled to the host per operation)
    phases = {}
    o_out = with_oracle(lambda: boot.bootstrap(ct, trace=lambda nm, c: phases.__setitem__(nm, G.ct_digest(c))))
    for nm in ("mod_raise", "coeff_to_slot_lo", "coeff_to_slot_hi", "eval_mod", "slot_to_coeff"):
        assert phases[nm] == rec["phases"][nm], f"CUDA and oracle limbs differ after {nm}"
    assert ckks.level_of(o_out) == rec["out_level"]
    check_against_committed(name, rec)


def test_oracle_bootstrap_batch_equals_single_bootstraps():
    """bootstrap_batch (BASELINE config 5: independent bootstraps in one batch) is the same circuit per
    ciphertext: on the CPU oracle two inputs through the batch give the limbs of two single runs."""
    from paper_2512_18345_b200.bootstrap import standard_input, standard_setup

    def run():
        spec, h_dense = G.CASES["n2048"]
        p = G.load_params(spec)
        sk, _sparse, boot = standard_setup(p, h_dense=h_dense)
        cts = [standard_input(p, boot, sk, i)[1] for i in range(2)]
        singles = [G.ct_digest(boot.bootstrap(ct)) for ct in cts]
        batch = [G.ct_digest(out) for out in boot.bootstrap_batch(cts)]
        return singles, batch

    singles, batch = with_oracle(run)
    assert singles == batch
    assert singles[0] != singles[1]


@pytest.mark.gpu
@pytest.mark.parametrize("name", ["n2048", "ks48"])
def test_cuda_bootstrap_batch_equals_single_bootstraps(name):
    """The batched graph (two bootstraps on 16 lanes, every rotation key and diagonal of the six
    linear transforms read once for the pair: ckks_bsgs_inner_batch) returns, for each input, exactly
    the limbs of that input's own bootstrap -- which test_cuda_bootstrap_equals_oracle pins to the
    CPU oracle."""
    import torch

    assert torch.cuda.is_available(), "GPU tests need a CUDA device"
    from paper_2512_18345_b200.bootstrap import standard_input, standard_setup
    from paper_2512_18345_b200.engine import get_engine

    eng = get_engine()
    spec, h_dense = G.CASES[name]
    p = G.load_params(spec)
    sk, _sparse, boot = standard_setup(p, h_dense=h_dense)
    cts = [standard_input(p, boot, sk, i)[1] for i in range(3)]
    eng.set_lanes(1)
    singles = [G.ct_digest(boot.bootstrap(ct)) for ct in cts]
    eager = [G.ct_digest(out) for out in boot.bootstrap_batch(cts)]          # a pair and an odd one
    assert eager == singles
    eng.set_lanes(16)
    replay = boot.capture_batch(cts[:2])
    outs = replay([cts[1], cts[2]])
    torch.cuda.synchronize()
    assert [G.ct_digest(o) for o in outs] == [singles[1], singles[2]]
    eng.set_lanes(1)


def test_apply_batch_covers_the_unfused_and_single_paths():
    """LinearTransform.apply_batch: a batch of one, and a transform whose baby steps are not fused
    (fuse_baby_steps off: per-rotation accumulators + fused_terms_multi, no batched launch), give what
    apply() gives per ciphertext (CPU oracle, N = 2^11)."""
    from paper_2512_18345_b200.bootstrap import standard_input, standard_setup

    def run():
        spec, h_dense = G.CASES["n2048"]
        p = G.load_params(spec)
        sk, _sparse, boot = standard_setup(p, h_dense=h_dense)
        xs = [boot.mod_raise(standard_input(p, boot, sk, i)[1]) for i in range(2)]
        lt = boot.cts[0]
        want = [G.ct_digest(lt.apply(x, boot.keys)) for x in xs]
        one = [G.ct_digest(c) for c in lt.apply_batch(xs[:1], boot.keys)]
        both = [G.ct_digest(c) for c in lt.apply_batch(xs, boot.keys)]
        lt.fuse_baby_steps = False
        try:
            unfused = [G.ct_digest(c) for c in lt.apply_batch(xs, boot.keys)]
        finally:
            lt.fuse_baby_steps = True
        return want, one, both, unfused

    want, one, both, unfused = with_oracle(run)
    assert one == want[:1]
    assert both == want
    assert unfused == want
