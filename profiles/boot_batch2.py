"""Throughput of batched bootstraps on one GPU (BASELINE config 5): one bootstrap per graph replay
(8 lanes) against bootstrap_batch of 2 (16 lanes; the six linear transforms read every rotation key
and plaintext diagonal once per pair, ckks_bsgs_inner_batch).  ks48, dense key + encapsulation.
Usage: python profiles/boot_batch2.py [tag] [batch]"""
import json
import sys
from pathlib import Path

import torch

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
from paper_2512_18345_b200.bootstrap import BootstrapConfig, standard_input, standard_setup  # noqa: E402
from paper_2512_18345_b200.engine import get_engine  # noqa: E402
from paper_2512_18345_b200.params import ParameterSet  # noqa: E402

tag = sys.argv[1] if len(sys.argv) > 1 else "r2n"
eng = get_engine()
p = ParameterSet.builtin("ks48")
sk, _sparse, boot = standard_setup(p, BootstrapConfig())
BATCH = int(sys.argv[2]) if len(sys.argv) > 2 else 2
cts = [standard_input(p, boot, sk, i)[1] for i in range(BATCH)]


def timed(fn, reps=20, rounds=3):
    for _ in range(5):
        fn()
    torch.cuda.synchronize()
    out = []
    for _ in range(rounds):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(reps):
            fn()
        b.record()
        torch.cuda.synchronize()
        out.append(round(a.elapsed_time(b) / reps, 3))
    return out


res = {}
eng.set_lanes(8)
single = boot.capture(cts[0])
ref = [single(ct) for ct in cts]
ref = [torch.stack([o.a.data, o.b.data]).clone() for o in ref]
res["single_ms_per_bootstrap"] = timed(lambda: single(cts[0], copy_out=False))
del single
for lanes in (16, 8):
    eng.set_lanes(lanes)
    batch = boot.capture_batch(cts)
    outs = batch(cts)
    same = all(torch.equal(torch.stack([o.a.data, o.b.data]), r) for o, r in zip(outs, ref))
    ms = timed(lambda: batch(cts, copy_out=False))
    res[f"batch{BATCH}_lanes{lanes}"] = {"ms_per_batch": ms, "ms_per_bootstrap": [round(m / BATCH, 3) for m in ms],
                                         "bootstraps_per_s": round(BATCH * 1000.0 / min(ms), 1), "same_limbs_as_single": same}
    print(lanes, res[f"batch{BATCH}_lanes{lanes}"], flush=True)
    del batch, outs
    torch.cuda.empty_cache()
res["single_bootstraps_per_s"] = round(1000.0 / min(res["single_ms_per_bootstrap"]), 1)
print(json.dumps(res, indent=1))
out = ROOT / "gpurun_out"
out.mkdir(exist_ok=True)
(out / f"{tag}_boot_batch{BATCH}.json").write_text(json.dumps(res, indent=1))
