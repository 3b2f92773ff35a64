#!/usr/bin/env python
"""Times the REAL reference (the NumPy package rnscope, SURVEY 8d "CPU baseline") on the host
cores: single-process latency and a multiprocessing pool over independent inputs.

The reference cannot be pip-installed onto the GPU box (no network), so
`__graft_entry__.build()` keeps a travelling copy of /root/reference/pkg/src/rnscope under
baseline/_ref/rnscope (git-ignored, shipped by gpurun).  This script imports that copy and
nothing of the product; bench.py runs it in a subprocess (no CUDA context in the workers) and
folds the JSON it prints into `cpu_baseline.reference`.

    python baseline/time_reference.py {ntt|keyswitch|config1} [--rows R] [--pool P]
"""
from __future__ import annotations

import argparse
import json
import multiprocessing as mp
import os
import sys
import time
from pathlib import Path

import numpy as np

REF = Path(__file__).resolve().parent / "_ref"


def cpu_model() -> str:
    try:
        for line in Path("/proc/cpuinfo").read_text().splitlines():
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except Exception:
        pass
    return "unknown"


def build(workload: str, rows: int):
    """Returns a zero-argument callable running one unit of `workload` on the reference."""
    from rnscope import baseconv, keyswitch as ks, transform
    from rnscope.params import ParameterSet, generate_parameter_set
    from rnscope.rns import COEFFICIENT, EVALUATION, Polynomial, poly_elementwise, random_polynomial
    from importlib import resources

    def builtin(name):
        return ParameterSet.from_dict(json.loads(resources.files("rnscope").joinpath(f"data/params/{name}.json").read_text()))

    if workload == "ntt":
        p = builtin("ks48")
        ext = p.ext_basis
        basis = tuple(ext[i % len(ext)] for i in range(rows))
        poly = random_polynomial(basis, p.n, np.random.default_rng(1))
        return lambda: transform.ntt_polynomial(poly)
    if workload == "keyswitch":
        p = builtin("ks48")
        s_from, s_to = ks.keygen(p, seed=1), ks.keygen(p, seed=2)
        msg = np.random.default_rng(0).integers(1, 9, p.n).astype(np.int64) * p.delta
        ct = ks.encrypt(msg, s_from, p, seed=3)
        evk = ks.switching_keygen(s_from, s_to, p, seed=4)
        return lambda: ks.keyswitch(ct, evk)
    # config 1: HMult + relinearise + rescale composed from the reference's primitives
    p = generate_parameter_set(n=8192, l=12, dnum=3, delta=1 << 40, h_dense=64, h_sparse=32)
    sk = ks.keygen(p, seed=1)
    m = [np.random.default_rng(7 + i).integers(1, 9, p.n).astype(np.int64) << 20 for i in range(2)]
    c1, c2 = ks.encrypt(m[0], sk, p, seed=2), ks.encrypt(m[1], sk, p, seed=5)
    s_ext = sk.eval_polynomial(p.ext_basis)
    sk_sq = ks.SecretKey(ternary=np.zeros(p.n, dtype=np.int8), n=p.n)
    sk_sq._eval_cache[tuple(mm.q for mm in p.ext_basis)] = poly_elementwise(s_ext, s_ext, "mul")
    rlk = ks.switching_keygen(sk_sq, sk, p, seed=41)
    last, rest = p.q_basis[-1], p.q_basis[:-1]
    table = baseconv.build_bconv_table((last,), rest)
    q_col = np.array([mm.q for mm in rest], dtype=np.uint64)[:, None]
    inv = np.array([pow(last.q, -1, mm.q) for mm in rest], dtype=np.uint64)[:, None]

    def rescale(x):
        c = transform.ntt_polynomial(Polynomial((last,), x.coeffs[-1:], EVALUATION), "inverse")
        conv = transform.ntt_polynomial(baseconv.convert(c, table))
        return Polynomial(rest, (x.coeffs[:-1] + q_col - conv.coeffs) % q_col * inv % q_col, EVALUATION)

    def unit():
        d0 = poly_elementwise(c1.b, c2.b, "mul")
        d1 = poly_elementwise(poly_elementwise(c1.a, c2.b, "mul"), poly_elementwise(c2.a, c1.b, "mul"), "add")
        d2 = poly_elementwise(c1.a, c2.a, "mul")
        sw = ks.keyswitch(ks.Ciphertext(a=d2, b=d0, scale=c1.scale * c2.scale), rlk)
        return rescale(poly_elementwise(sw.a, d1, "add")), rescale(sw.b)

    return unit


_UNIT = None


def _worker(reps: int) -> float:
    t0 = time.perf_counter()
    for _ in range(reps):
        _UNIT()
    return time.perf_counter() - t0


def main():
    global _UNIT
    ap = argparse.ArgumentParser()
    ap.add_argument("workload", choices=["ntt", "keyswitch", "config1"])
    ap.add_argument("--rows", type=int, default=60)
    ap.add_argument("--pool", type=int, default=0, help="worker processes of the throughput run (0: all host threads)")
    args = ap.parse_args()
    if not (REF / "rnscope").is_dir():
        print(json.dumps({"unavailable": "no travelling copy of the reference (baseline/_ref/rnscope)"}))
        return
    sys.path.insert(0, str(REF))
    os.environ.setdefault("OMP_NUM_THREADS", "1")
    t0 = time.perf_counter()
    _UNIT = build(args.workload, args.rows)
    _UNIT()                                           # untimed: builds the cached twiddle / conversion tables
    setup_s = time.perf_counter() - t0
    reps = {"ntt": 3, "keyswitch": 1, "config1": 5}[args.workload]
    single_s = _worker(reps) / reps
    try:
        threads = len(os.sched_getaffinity(0))
    except Exception:
        threads = os.cpu_count() or 1
    procs = args.pool or threads
    ctx = mp.get_context("fork")                       # workers inherit the built inputs and tables
    t0 = time.perf_counter()
    with ctx.Pool(procs) as pool:
        pool.map(_worker, [reps] * procs)
    pool_s = time.perf_counter() - t0
    print(json.dumps({
        "kind": "reference", "workload": args.workload, "cpu": cpu_model(), "host_threads": threads,
        "single_process": {"ms_per_unit": single_s * 1e3, "units_per_s": 1.0 / single_s, "cores": 1, "reps": reps},
        "pool": {"processes": procs, "units": procs * reps, "wall_s": pool_s, "units_per_s": procs * reps / pool_s},
        "setup_s": setup_s,
        "sample": f"rnscope (NumPy) from baseline/_ref: {reps} unit(s) in one process after one untimed unit; "
                  f"then {procs} forked processes x {reps} unit(s) of the same input",
    }))


if __name__ == "__main__":
    main()
