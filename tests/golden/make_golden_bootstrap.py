"""Generate tests/golden/golden_bootstrap.json: limb digests of one full bootstrap, phase by
phase, computed on the CPU ORACLE (oracle/engine_oracle.py driving the package's own circuit,
paper_2512_18345_b200/bootstrap.py, through the C restatement of the reference primitives).

    python tests/golden/make_golden_bootstrap.py [n2048] [ks48]

The reference ships no bootstrapping, so these are NOT reference outputs:
they pin the CUDA path to the composed oracle, whose building blocks are pinned to the
reference (golden.json, golden_level.json).  The circuit's plaintexts are encoded on the host
in floating point; their digest ("plaintexts") is recorded so that a test on a machine whose
FFT / libm rounds differently can tell an input difference from an arithmetic one.
"""
from __future__ import annotations

import hashlib
import json
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(Path(__file__).resolve().parent))

import recipes as R  # noqa: E402

CASES = {
    # name: (parameter set, dense Hamming weight)
    "n2048": (dict(gen=dict(n=2048, l=36, dnum=3, delta=1 << 40, h_dense=512, h_sparse=32)), 512),
    "ks48": (dict(builtin="ks48"), None),
}


def load_params(spec):
    from paper_2512_18345_b200.params import ParameterSet, generate_parameter_set

    return ParameterSet.builtin(spec["builtin"]) if "builtin" in spec else generate_parameter_set(**spec["gen"])


def words(poly) -> np.ndarray:
    return poly.data.cpu().numpy().view(np.uint32)


def ct_digest(ct) -> list[str]:
    return [R.digest(words(ct.a)), R.digest(words(ct.b))]


def plaintext_digest(boot) -> str:
    """One digest over every encoded DFT diagonal of the bootstrapper, in a fixed order."""
    h = hashlib.sha256()
    for lt in boot.cts + boot.stc:
        for g in sorted(lt.table):
            for b in sorted(lt.table[g]):
                h.update(np.ascontiguousarray(words(lt.table[g][b].poly), dtype="<u4").tobytes())
    return h.hexdigest()


def run_case(name):
    """Bootstrap case `name` on whatever engine is installed; returns the record."""
    from paper_2512_18345_b200 import ckks
    from paper_2512_18345_b200.bootstrap import standard_input, standard_setup

    spec, h_dense = CASES[name]
    p = load_params(spec)
    sk, _sparse, boot = standard_setup(p, h_dense=h_dense)
    z, ct = standard_input(p, boot, sk, 0)
    phases = {}
    out = boot.bootstrap(ct, trace=lambda nm, c: phases.__setitem__(nm, ct_digest(c)))
    err = float(np.abs(ckks.decrypt_decode(out, sk, p) - z).max())
    return {"plaintexts": plaintext_digest(boot), "input": ct_digest(ct), "phases": phases,
            "out_level": ckks.level_of(out), "precision_log2": float(np.log2(err))}, (p, sk, boot, z, ct)


def main():
    from oracle.engine_oracle import OracleEngine
    from paper_2512_18345_b200 import engine

    path = Path(__file__).resolve().parent / "golden_bootstrap.json"
    G = json.loads(path.read_text()) if path.exists() else {"schema": 1, "source": "oracle", "cases": {}}
    for name in sys.argv[1:] or list(CASES):
        t0 = time.time()
        engine.use_backend(OracleEngine())
        G["cases"][name], _ = run_case(name)
        print(f"{name}: {time.time() - t0:.1f}s precision 2^{G['cases'][name]['precision_log2']:.2f}")
        path.write_text(json.dumps(G, indent=1) + "\n")


if __name__ == "__main__":
    main()
