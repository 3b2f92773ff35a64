"""A/B of the N = 2^16 transform: two-kernel split against the single-pass cluster kernels
(ntt16_*_cluster at 2 and 3 CTAs per SM), R limbs of the ks48 extended basis, CUDA graph of
back-to-back transforms over operands rotating through > 126 MB, device time per transform.
Writes gpurun_out/<tag>_ntt_cluster_ab.json.  Usage: python profiles/ntt_cluster_ab.py [tag]"""
import json
import sys
from pathlib import Path

import numpy as np
import torch

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))

from paper_2512_18345_b200.engine import get_engine  # noqa: E402
from paper_2512_18345_b200.params import ParameterSet  # noqa: E402

tag = sys.argv[1] if len(sys.argv) > 1 else "r2l"
p = ParameterSet.builtin("ks48")
eng = get_engine()
dev = eng.device
ext = tuple(p.q_basis) + tuple(p.p_basis)
LIMB = p.n * 4
rng = np.random.default_rng(0)


def rand_limbs(basis):
    x = np.stack([rng.integers(0, m.q, p.n, dtype=np.uint64) for m in basis]).astype(np.uint32)
    return torch.from_numpy(x.view(np.int32)).to(dev)


def time_point(rows, inverse):
    basis = tuple(ext[i % len(ext)] for i in range(rows))
    count = max(2, -(-(160 << 20) // (rows * LIMB)))
    polys = [rand_limbs(basis) for _ in range(min(count, 4))]
    polys = [polys[i % len(polys)].clone() for i in range(count)]
    outs = [eng.empty(rows, p.n) for _ in range(count)]
    slots = eng.row_slots(basis, p.n)
    reps = 4 * count
    run = lambda: [eng.ntt(polys[k % count], slots, inverse, out=outs[k % count]) for k in range(reps)]
    run()
    torch.cuda.synchronize()
    graph = torch.cuda.CUDAGraph()
    side = torch.cuda.Stream(device=dev)
    side.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(side):
        with torch.cuda.graph(graph, stream=side):
            run()
    torch.cuda.current_stream().wait_stream(side)
    for _ in range(3):
        graph.replay()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    n_rep = 10
    a.record()
    for _ in range(n_rep):
        graph.replay()
    b.record()
    torch.cuda.synchronize()
    digest = int(outs[0].to(torch.int64).sum().item())
    return a.elapsed_time(b) * 1e3 / (n_rep * reps), digest


res = []
for rows in (2, 12, 24, 28, 48, 60, 96, 192, 240):
    for inverse in (False, True):
        row = {"rows": rows, "direction": "inverse" if inverse else "forward"}
        digests = set()
        for name, pol in (("two_kernel", (0, 3)), ("cluster_occ2", (1 << 20, 2)), ("cluster_occ3", (1 << 20, 3))):
            eng.ntt_policy(*pol)
            us, dg = time_point(rows, inverse)
            row[name + "_us"] = round(us, 2)
            digests.add(dg)
        row["same_result"] = len(digests) == 1
        row["alg_gbs_best"] = round(2.0 * rows * LIMB / min(row["two_kernel_us"], row["cluster_occ2_us"], row["cluster_occ3_us"]) / 1e3, 1)
        print(row, flush=True)
        res.append(row)
out = ROOT / "gpurun_out"
out.mkdir(exist_ok=True)
(out / f"{tag}_ntt_cluster_ab.json").write_text(json.dumps(res, indent=1))
