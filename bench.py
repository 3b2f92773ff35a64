#!/usr/bin/env python
"""bench.py -- headline measurement of the CKKS hot path on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl b200|reference]
                    [--workload keyswitch|ntt]

One process per GPU (torchrun for N > 1, NCCL only for the barrier / max over
ranks: independent ciphertexts shard with no data-path collective, "weak"
scaling).  A step is one pass of the hot path over one synthetic ciphertext:

  keyswitch  hybrid key switch (the HRot / relinearisation core, BASELINE
             config 3) at ks48: N = 2^16, L = 48, alpha = 12, dnum = 4.
  ntt        batched forward NTT over the 60-limb extended basis (config 2).

`value` is whole-job throughput with inputs resident in HBM; `e2e` is the same
metric through the public Python API with HOST ciphertexts (pinned H2D of the
input and D2H of the result inside the timed region; evaluation keys are
resident state, like model weights).  Inputs rotate through more bytes than
the 126 MB L2 so no step finds its key or ciphertext cached.

--impl reference times the CPU restatement of the reference (oracle/, C with
OpenMP on all host threads; the reference itself is single-threaded NumPy and
cannot travel to the GPU box) on the same workload.
"""
from __future__ import annotations

import argparse
import json
import os
import sys
import threading
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

LIMB_BYTES = 65536 * 4


def load_peaks():
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        d = json.loads(p.read_text())
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    return 6650.0, "fallback (B200_PROFILING.md)"


class ClockSampler:
    """Samples SM clock and throttle reasons through NVML during the timed region."""

    def __init__(self, index: int):
        self.samples, self.reasons, self.max_mhz = [], set(), None
        self._stop = threading.Event()
        self._thread = None
        try:
            import pynvml

            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
        except Exception:
            self.nv = None

    def _run(self):
        nv = self.nv
        names = {
            "hw_slowdown": getattr(nv, "nvmlClocksThrottleReasonHwSlowdown", 0x8),
            "hw_thermal_slowdown": getattr(nv, "nvmlClocksThrottleReasonHwThermalSlowdown", 0x40),
            "sw_thermal_slowdown": getattr(nv, "nvmlClocksThrottleReasonSwThermalSlowdown", 0x20),
            "sw_power_cap": getattr(nv, "nvmlClocksThrottleReasonSwPowerCap", 0x4),
        }
        while not self._stop.is_set():
            try:
                self.samples.append(nv.nvmlDeviceGetClockInfo(self.h, nv.NVML_CLOCK_SM))
                mask = nv.nvmlDeviceGetCurrentClocksThrottleReasons(self.h)
                for k, bit in names.items():
                    if mask & bit:
                        self.reasons.add(k)
            except Exception:
                pass
            time.sleep(0.02)

    def __enter__(self):
        if self.nv:
            self._thread = threading.Thread(target=self._run, daemon=True)
            self._thread.start()
        return self

    def __exit__(self, *exc):
        self._stop.set()
        if self._thread:
            self._thread.join()

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": sorted(self.reasons)}
        return {"sm_mhz": float(np.median(self.samples)), "sm_max_mhz": self.max_mhz,
                "reasons": sorted(self.reasons), "samples": len(self.samples)}


def ks_algorithmic_bytes(l, alpha, beta):
    """Algorithmic HBM/L2-boundary bytes per launch of every kernel class of one
    key switch, in limbs read + written (SURVEY Appendix A convention: one read
    and one write of each operand, twiddles and tables excluded)."""
    ext = l + alpha
    conv_rows = beta * l            # converted limbs of stage 1 (ext - alpha per digit)
    limbs = {
        # two launches each (stage 1 INTT of L limbs, stage 3 INTT of 2*alpha limbs)
        "ntt16_inv_contig": [2 * l, 2 * 2 * alpha],
        "ntt16_inv_strided": [2 * l, 2 * 2 * alpha],
        "ntt16_fwd_strided": [2 * conv_rows, 2 * 2 * l],
        "ntt16_fwd_contig": [2 * conv_rows, 2 * 2 * l],
        "bconv": [l + conv_rows, 2 * alpha + 2 * l],
        "inner_product": [beta * ext + 2 * beta * ext + 2 * ext],
        "moddown_epilogue": [2 * l + 2 * l + l + 2 * l],
    }
    return {k: [x * LIMB_BYTES for x in v] for k, v in limbs.items()}


def read_profile(eng):
    import ctypes

    buf = ctypes.create_string_buffer(1 << 16)
    eng.lib.ckks_profile_read(buf, len(buf))
    out = {}
    for line in buf.value.decode().splitlines():
        name, cnt, ms = line.split()
        out[name] = (int(cnt), float(ms))
    return out


# --------------------------------------------------------------------------------------
# reference arm / CPU baseline: the oracle port on host cores
# --------------------------------------------------------------------------------------
def oracle_setup(workload):
    from oracle import oracle
    from paper_2512_18345_b200.params import ParameterSet

    p = ParameterSet.builtin("ks48")
    op = oracle.OParams(p.n, p.l, p.dnum, p.alpha, p.delta, p.h_dense,
                        tuple((m.q, m.psi) for m in p.q_basis),
                        tuple((m.q, m.psi) for m in p.p_basis))
    orc = oracle.Oracle(p.n, op.ext_basis)
    rng = np.random.default_rng(0)
    qs = [q for q, _ in op.ext_basis]
    if workload == "ntt":
        x = np.stack([rng.integers(0, q, p.n, dtype=np.uint64) for q in qs]).astype(np.uint32)
        rm = np.arange(len(qs), dtype=np.int32)
        return lambda: orc.ntt(x, rm)
    a = np.stack([rng.integers(0, q, p.n, dtype=np.uint64) for q in qs[:p.l]]).astype(np.uint32)
    b = np.stack([rng.integers(0, q, p.n, dtype=np.uint64) for q in qs[:p.l]]).astype(np.uint32)
    evk = np.stack([rng.integers(0, q, (p.dnum, 2, p.n), dtype=np.uint64) for q in qs])
    evk = np.ascontiguousarray(evk.transpose(1, 2, 0, 3)).astype(np.uint32)
    return lambda: orc.keyswitch(op, a, b, evk)


def time_oracle(workload, steps, warmup):
    step = oracle_setup(workload)
    for _ in range(warmup):
        step()
    t0 = time.perf_counter()
    for _ in range(steps):
        step()
    dt = time.perf_counter() - t0
    return steps / dt, dt / steps * 1e3


def host_threads():
    try:
        return len(os.sched_getaffinity(0))
    except Exception:
        return os.cpu_count() or 1


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    steps = max(1, min(args.steps, 5))
    warmup = max(1, min(args.warmup, 1))
    thr, ms = time_oracle(args.workload, steps, warmup)
    unit = "keyswitch/s" if args.workload == "keyswitch" else "ntt/s"
    cores = host_threads()
    line = {
        "impl": "reference", "metric": METRIC[args.workload], "value": thr, "unit": unit,
        "n_gpus": args.gpus, "steps": steps, "warmup": warmup, "ms_per_step": ms,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "u32",
        "data": "synthetic", "config": CONFIG[args.workload],
        "cpu_baseline": {"value": thr, "unit": unit, "cores": cores, "kind": "port",
                         "sample": f"{steps} steps of the workload, oracle/ckks_oracle.c with OpenMP"},
        "e2e": {"value": thr, "unit": unit, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line))


METRIC = {
    "keyswitch": "hybrid key-switch throughput (CKKS HRot/relinearise core, N=2^16 L=48 dnum=4)",
    "ntt": "batched RNS NTT throughput (N=2^16, 60 limbs)",
}
CONFIG = {
    "keyswitch": {"workload": "keyswitch ks48 (N=2^16, L=48, alpha=12, dnum=4, 31-bit primes), "
                              "one ciphertext per step", "l2_policy": "inputs rotate through >126 MB"},
    "ntt": {"workload": "forward NTT of one 60-limb polynomial (ks48 extended basis) per step",
            "l2_policy": "inputs rotate through >126 MB"},
}


# --------------------------------------------------------------------------------------
# B200 arm
# --------------------------------------------------------------------------------------
def run_b200(args):
    import torch
    import torch.distributed as dist

    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    if world > 1:
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))

    from paper_2512_18345_b200 import keyswitch as ks
    from paper_2512_18345_b200.engine import get_engine
    from paper_2512_18345_b200.params import ParameterSet
    from paper_2512_18345_b200.rns import EVALUATION, COEFFICIENT, Polynomial
    from paper_2512_18345_b200 import transform

    eng = get_engine()
    p = ParameterSet.builtin("ks48")
    ext = p.ext_basis
    dev = eng.device
    g = torch.Generator(device=dev)
    g.manual_seed(1234 + rank)

    def rand_limbs(basis, *lead):
        """Uniform residues below each modulus, generated on the device (synthetic)."""
        q = torch.tensor([m.q for m in basis], dtype=torch.float64, device=dev)[:, None]
        u = torch.rand((*lead, len(basis), p.n), generator=g, device=dev, dtype=torch.float64)
        return (u * q).to(torch.int64).clamp_(min=0).to(torch.int32).contiguous()

    n_ct, n_evk = 8, 4
    if args.workload == "keyswitch":
        cts = [rand_limbs(p.q_basis, 2) for _ in range(n_ct)]               # 25 MB each
        evks = [rand_limbs(ext, p.dnum, 2) for _ in range(n_evk)]           # 126 MB each
        outs = [eng.empty(2, p.l, p.n) for _ in range(n_ct)]
        plan = ks._tables(p).plan()

        def step(i):
            ct = cts[i % n_ct]
            eng.keyswitch(plan, ct[0], ct[1], evks[i % n_evk], out=outs[i % n_ct])

        host_in = [torch.empty((2, p.l, p.n), dtype=torch.int32).pin_memory() for _ in range(2)]
        host_out = [torch.empty((2, p.l, p.n), dtype=torch.int32).pin_memory() for _ in range(2)]
        for h, c in zip(host_in, cts):
            h.copy_(c)
        evk_keys = [ks.SwitchingKey(pairs=tuple(
            ks.PolyPair(a=Polynomial(ext, e[t, 0], EVALUATION), b=Polynomial(ext, e[t, 1], EVALUATION))
            for t in range(p.dnum)), params=p, _matrix=e) for e in evks]

        def e2e_step(i):
            # public API: host ciphertext in, host ciphertext out
            d = host_in[i % 2].to(dev, non_blocking=True)
            ct = ks.Ciphertext(a=Polynomial(p.q_basis, d[0], EVALUATION),
                               b=Polynomial(p.q_basis, d[1], EVALUATION), scale=p.delta)
            out = ks.keyswitch(ct, evk_keys[i % n_evk])
            host_out[i % 2][0].copy_(out.a.data, non_blocking=True)
            host_out[i % 2][1].copy_(out.b.data, non_blocking=True)

        h2d = d2h = 2 * p.l * LIMB_BYTES
        unit = "keyswitch/s"
    else:
        polys = [rand_limbs(ext) for _ in range(12)]                         # 15.7 MB each
        outs = [eng.empty(len(ext), p.n) for _ in range(12)]
        slots = eng.row_slots(ext, p.n)

        def step(i):
            eng.ntt(polys[i % 12], slots, False, out=outs[i % 12])

        host_in = [torch.empty((len(ext), p.n), dtype=torch.int32).pin_memory() for _ in range(2)]
        host_out = [torch.empty((len(ext), p.n), dtype=torch.int32).pin_memory() for _ in range(2)]

        def e2e_step(i):
            d = host_in[i % 2].to(dev, non_blocking=True)
            out = transform.ntt_polynomial(Polynomial(ext, d, COEFFICIENT))
            host_out[i % 2].copy_(out.data, non_blocking=True)

        h2d = d2h = len(ext) * LIMB_BYTES
        unit = "ntt/s"

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    def timed(fn, steps, warmup, sampler=None):
        for i in range(warmup):
            fn(i)
        barrier()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        if sampler:
            sampler.__enter__()
        a.record()
        for i in range(steps):
            fn(i)
        b.record()
        barrier()
        if sampler:
            sampler.__exit__()
        ms = a.elapsed_time(b)
        if world > 1:
            t = torch.tensor([ms], device=dev, dtype=torch.float64)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            ms = float(t.item())
        return ms

    sampler = ClockSampler(local)
    ms_total = timed(step, args.steps, args.warmup, sampler)
    ms_step = ms_total / args.steps
    value = world * args.steps / (ms_total * 1e-3)

    e2e_steps = max(3, min(args.steps, 200))
    e2e_ms = timed(e2e_step, e2e_steps, max(3, min(args.warmup, 5)))
    e2e_value = world * e2e_steps / (e2e_ms * 1e-3)

    # per-kernel pass: same steps with every launch bracketed by CUDA events
    prof_steps = max(3, min(args.steps, 50))
    eng.lib.ckks_profile_enable(1)
    for i in range(prof_steps):
        step(i)
    prof = read_profile(eng)
    eng.lib.ckks_profile_enable(0)
    launches_per_step = sum(c for c, _ in prof.values()) / prof_steps
    total_prof_ms = sum(ms for _, ms in prof.values())
    top = max(prof, key=lambda k: prof[k][1])
    peak, peak_src = load_peaks()
    if args.workload == "keyswitch":
        alg = ks_algorithmic_bytes(p.l, p.alpha, p.beta)
    else:
        alg = {"ntt16_fwd_strided": [2 * len(ext) * LIMB_BYTES], "ntt16_fwd_contig": [2 * len(ext) * LIMB_BYTES]}
    per_launch_bytes = sum(alg[top]) / len(alg[top])
    avg_launch_ms = prof[top][1] / prof[top][0]
    achieved = per_launch_bytes / (avg_launch_ms * 1e-3) / 1e9
    roofline = {
        "bound": "hbm", "kernel": top, "achieved": achieved, "peak": peak, "unit": "GB/s",
        "frac": achieved / peak, "traffic": None, "peak_source": peak_src,
        "avg_launch_us": avg_launch_ms * 1e3, "alg_bytes_per_launch": per_launch_bytes,
        "share_of_step": prof[top][1] / total_prof_ms,
        "kernels": {k: {"launches_per_step": c / prof_steps, "us_per_launch": ms / c * 1e3,
                        "share": ms / total_prof_ms,
                        "gbs": (sum(alg[k]) / len(alg[k])) / (ms / c * 1e-3) / 1e9 if k in alg else None}
                    for k, (c, ms) in sorted(prof.items(), key=lambda kv: -kv[1][1])},
    }

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        thr, ms_cpu = time_oracle(args.workload, 3, 1)
        cpu = {"value": thr, "unit": unit, "cores": host_threads(), "kind": "port",
               "ms_per_step": ms_cpu,
               "sample": "3 steps of the same workload, oracle/ckks_oracle.c (OpenMP over limbs)"}

    if rank == 0:
        line = {
            "metric": METRIC[args.workload], "value": value, "unit": unit, "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_step,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "u32",
            "data": "synthetic", "config": CONFIG[args.workload],
            "e2e": {"value": e2e_value, "unit": unit, "h2d_bytes_per_step": h2d,
                    "d2h_bytes_per_step": d2h, "ms_per_step": e2e_ms / e2e_steps},
            "gpu_launches": int(round(launches_per_step * args.steps)),
            "clocks": sampler.summary(), "roofline": roofline, "cpu_baseline": cpu,
        }
        print(json.dumps(line))
    if world > 1:
        dist.destroy_process_group()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=2000)
    ap.add_argument("--warmup", type=int, default=20)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--workload", default="keyswitch", choices=["keyswitch", "ntt"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    args = ap.parse_args()
    if args.impl == "reference":
        run_reference(args)
    else:
        run_b200(args)


if __name__ == "__main__":
    main()
