"""Bootstrap latency (ks48, dense key + encapsulation, 8-lane CUDA graph) under different
transform policies: which N = 2^16 launches run as the single-pass cluster kernel
(ckks_ntt_policy: at most `rows` limbs, at 2 or 3 CTAs per SM).  One setup, one capture per
policy, outputs compared bit for bit with the two-kernel policy's.
Usage: python profiles/boot_policy.py [tag] [rows:occ ...]"""
import json
import sys
from pathlib import Path

import torch

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
from paper_2512_18345_b200.bootstrap import BootstrapConfig, standard_input, standard_setup  # noqa: E402
from paper_2512_18345_b200.engine import get_engine  # noqa: E402
from paper_2512_18345_b200.params import ParameterSet  # noqa: E402

tag = sys.argv[1] if len(sys.argv) > 1 else "r2l"
policies = [tuple(int(x) for x in a.split(":")) for a in sys.argv[2:]] or [(0, 3), (2, 2), (12, 2), (28, 2), (37, 2), (48, 2), (28, 3)]
eng = get_engine()
eng.set_lanes(int(__import__('os').environ.get('BOOT_LANES', '8')))      # BOOT_LANES: lanes of the graph (default 8)
p = ParameterSet.builtin("ks48")
sk, _sparse, boot = standard_setup(p, BootstrapConfig())
z, ct = standard_input(p, boot, sk, 0)
res, base = [], None
for rows, occ in policies:
    eng.ntt_policy(rows, occ)
    run = boot.capture(ct)
    for _ in range(10):
        out = run(ct)
    torch.cuda.synchronize()
    times = []
    for _ in range(3):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(20):
            out = run(ct)
        b.record()
        torch.cuda.synchronize()
        times.append(a.elapsed_time(b) / 20)
    limbs = torch.stack([out.a.data, out.b.data]).clone()
    if base is None:
        base = limbs
    row = {"cluster_max_rows": rows, "ctas_per_sm": occ, "ms": [round(t, 3) for t in times],
           "same_limbs_as_first_policy": bool(torch.equal(base, limbs))}
    print(row, flush=True)
    res.append(row)
    del run, out
    torch.cuda.empty_cache()
out_dir = ROOT / "gpurun_out"
out_dir.mkdir(exist_ok=True)
(out_dir / f"{tag}_boot_policy.json").write_text(json.dumps(res, indent=1))
