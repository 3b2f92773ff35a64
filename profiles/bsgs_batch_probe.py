"""Per-launch time of the fused baby-step kernel for one ciphertext against a pair through
ckks_bsgs_inner_batch (eager, CUDA events around every launch: ckks_profile_*), first CoeffToSlot
group (48 limbs) and first SlotToCoeff group (21 limbs) of the ks48 bootstrap.
Usage: python profiles/bsgs_batch_probe.py [tag]"""
import ctypes
import json
import sys
from pathlib import Path

import torch

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
from paper_2512_18345_b200 import ckks  # noqa: E402
from paper_2512_18345_b200.bootstrap import BootstrapConfig, standard_input, standard_setup  # noqa: E402
from paper_2512_18345_b200.engine import get_engine  # noqa: E402
from paper_2512_18345_b200.params import ParameterSet  # noqa: E402

tag = sys.argv[1] if len(sys.argv) > 1 else "r2n"
eng = get_engine()
eng.set_lanes(16)
p = ParameterSet.builtin("ks48")
sk, _sparse, boot = standard_setup(p, BootstrapConfig())
cts = [standard_input(p, boot, sk, i)[1] for i in range(2)]


def read_profile():
    buf = ctypes.create_string_buffer(1 << 16)
    eng.lib.ckks_profile_read(buf, len(buf))
    out = {}
    for line in buf.value.decode().splitlines():
        name, cnt, ms, nbytes, _ = line.split()
        out[name] = {"launches": int(cnt), "us_per_launch": round(float(ms) * 1e3 / int(cnt), 1),
                     "alg_gbs": round(float(nbytes) / float(ms) / 1e6, 1)}
    return out


res = {}
for label, lt, make in (("cts0_l48", boot.cts[0], lambda ct: boot.mod_raise(ct)),
                        ("stc0_l21", boot.stc[0], lambda ct: ckks.mod_drop(boot.mod_raise(ct), boot.lvl_stc))):
    xs = [make(ct) for ct in cts]
    for name, fn in (("single", lambda: [lt.apply(x, boot.keys) for x in xs]), ("batch2", lambda: lt.apply_batch(xs, boot.keys))):
        for _ in range(2):
            fn()
        torch.cuda.synchronize()
        eng.lib.ckks_profile_enable(1)
        for _ in range(5):
            fn()
        torch.cuda.synchronize()
        prof = read_profile()
        eng.lib.ckks_profile_enable(0)
        res[f"{label}_{name}"] = {k: v for k, v in prof.items() if k.startswith("bsgs")}
        print(label, name, res[f"{label}_{name}"], flush=True)
out = ROOT / "gpurun_out"
out.mkdir(exist_ok=True)
(out / f"{tag}_bsgs_batch_probe.json").write_text(json.dumps(res, indent=1))
