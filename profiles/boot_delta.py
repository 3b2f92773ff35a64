"""Precision of the ks48 bootstrap against the input scale 2^log_delta_in (two input limbs, Q0 ~ 2^62):
errors made before EvalMod are amplified by Q0 * 2^r / (2 pi Delta) on the way back to the message, so a
larger Delta buys precision as long as Delta * |m| stays far below Q0 (the sine's linear range).
Usage: python profiles/boot_delta.py [tag] [log_delta ...]"""
import json
import sys
from pathlib import Path

import numpy as np
import torch

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
from paper_2512_18345_b200 import ckks  # noqa: E402
from paper_2512_18345_b200.bootstrap import BootstrapConfig, standard_input, standard_setup  # noqa: E402
from paper_2512_18345_b200.engine import get_engine  # noqa: E402
from paper_2512_18345_b200.params import ParameterSet  # noqa: E402

tag = sys.argv[1] if len(sys.argv) > 1 else "r2z"
eng = get_engine()
eng.set_lanes(8)
p = ParameterSet.builtin("ks48")
res = {}
for ld in [int(a) for a in sys.argv[2:]] or [50, 52, 54, 56, 58]:
    sk, _sparse, boot = standard_setup(p, BootstrapConfig(log_delta_in=ld))
    errs = []
    for i in range(3):
        z, ct = standard_input(p, boot, sk, i)
        out = boot.bootstrap(ct)
        got = ckks.decrypt_decode(out, sk, p)
        errs.append(float(np.log2(np.abs(got - z).max())))
    res[ld] = {"log2_max_err": [round(e, 2) for e in errs], "out_level": ckks.level_of(out)}
    print(ld, res[ld], flush=True)
    del boot, out
    torch.cuda.empty_cache()
out_dir = ROOT / "gpurun_out"
out_dir.mkdir(exist_ok=True)
(out_dir / f"{tag}_boot_delta.json").write_text(json.dumps(res, indent=1))
