#!/usr/bin/env python
"""bench.py -- headline measurement of the CKKS hot path on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl b200|reference]
                    [--workload bootstrap|keyswitch|ntt|helr|config1] [--rows R]

One process per GPU (torchrun for N > 1).  Independent ciphertexts shard over ranks with no
data-path collective (weak scaling): every step each rank takes its shard of an N-ciphertext
batch through paper_2512_18345_b200.sharding (one ciphertext per rank and step), and the only
collective is the gather of per-result checksums at the end of the timed region.  A step is one
pass of the hot path over one synthetic ciphertext:

  bootstrap  (default; BASELINE config 4, the headline) full CKKS bootstrapping of 2^15 complex
             slots at N = 2^16 on the reference's ks48 moduli (L = 48 31-bit limbs, alpha = 12,
             dnum = 4), dense application key + sparse-secret encapsulation,
             replayed as one CUDA graph; `ms_per_step` is the bootstrap latency.
  keyswitch  hybrid key switch (HRot / relinearisation core, config 3) at ks48.
  ntt        batched forward NTT over R limbs of the ks48 extended basis (config 2; --rows).
  helr       one HELR-style logistic-regression iteration (config 5).
  config1    HMult + relinearise + rescale at N = 2^13, L = 12, dnum = 3 (config 1).

`value` is whole-job throughput with inputs resident in HBM; `e2e` is the same metric through
the public Python API with HOST ciphertexts (pinned H2D of the input and D2H of the result
inside the timed region; evaluation keys and encoded DFT matrices are resident state).

--impl reference runs the reference's path on the host cores: the package's own circuit
replayed on the CPU restatement of the reference primitives (oracle/, C + OpenMP on every host
thread; the reference itself is single-threaded NumPy and cannot travel to the GPU box).  For the
circuits (bootstrap, helr) a step is a bounded sample: 1/20 of the circuit's engine calls, in
order, state carried from step to step, so 20 steps are exactly one whole run.
"""
from __future__ import annotations

import argparse
import ctypes
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
FP64_TENSOR_TFLOPS = 37.06
# Integer-pipe bound of a Shoup butterfly on B200 (profiles/microbench/int_pipes.cu: IMAD.HI 28,
# IMAD 62 thread-ops per clk per SM; one IMAD.HI + two IMAD per butterfly): 1 / (1/28 + 2/62)
INT_PIPE_BF_PER_CLK_SM = 14.7
SEGMENTS = 20            # reference arm: a circuit is cut into this many steps

METRIC = {
    "bootstrap": "CKKS bootstrap throughput (2^15 slots, N=2^16); ms_per_step = bootstrap latency ms",
    "keyswitch": "hybrid key-switch throughput (CKKS HRot/relinearise core, N=2^16 L=48 dnum=4)",
    "ntt": "batched RNS NTT throughput (N=2^16, R limbs per transform)",
    "helr": "HELR-style logistic-regression iteration throughput (N=2^16, 128 samples x 256 features, level 20 -> 13)",
    "config1": "HMult + relinearise + rescale throughput (N=2^13, L=12, dnum=3)",
}
UNIT = {"bootstrap": "bootstraps/s", "keyswitch": "keyswitch/s", "ntt": "ntt/s", "helr": "iterations/s",
        "config1": "hmult/s"}
DEFAULT_STEPS = {"bootstrap": 30, "keyswitch": 2000, "ntt": 2000, "helr": 100, "config1": 2000}


def bootstrap_plan(p):
    """Levels of the default circuit (paper_2512_18345_b200/bootstrap.py level plan), from the
    parameter set and BootstrapConfig alone so that both arms print the same `config`."""
    from paper_2512_18345_b200.bootstrap import BootstrapConfig

    cfg = BootstrapConfig()
    depth = 5 if cfg.scheme == "ps" else int(np.ceil(np.log2(cfg.degree + 1)))
    after_evalmod = p.l - 2 * cfg.groups - 2 * (depth + cfg.squarings) - 1
    return cfg, after_evalmod - cfg.groups


def config_for(workload, args):
    from paper_2512_18345_b200.params import ParameterSet

    if workload == "bootstrap":
        p = ParameterSet.builtin("ks48")
        cfg, out_level = bootstrap_plan(p)
        bits = sum(m.q.bit_length() for m in p.ext_basis)
        return {
            "workload": "full CKKS bootstrapping, 2^15 complex slots, N=2^16, ks48 moduli (L=48 31-bit limbs, "
                        f"alpha=12, dnum=4), input level 2 at scale 2^{cfg.log_delta_in}, one ciphertext per step "
                        f"and rank, CUDA-graph replay with {args.lanes} stream lanes",
            "key_regime": f"dense application key h={p.h_dense} for every evaluation key, sparse key h={p.h_sparse} "
                          "only around ModRaise (sparse-secret encapsulation, PAPER.md:514): two extra key switches",
            "log2_PQ": bits,
            "levels_after_boot": {"limbs": out_level, "double_limb_levels": out_level // 2,
                                  "note": "scale ~2^62 on pairs of 31-bit limbs; the paper's table reports Lv_eff 15 "
                                          "(PAPER.md:655-659): not the same depth, see DESIGN.md section 6"},
            "stage_groups": cfg.groups,
            "l2_policy": "each step streams ~8 GB of keys and plaintext diagonals (>> 126 MB L2)",
        }
    if workload == "keyswitch":
        return {"workload": "keyswitch ks48 (N=2^16, L=48, alpha=12, dnum=4, 31-bit primes), one ciphertext per step",
                "l2_policy": "inputs rotate through >126 MB"}
    if workload == "ntt":
        return {"workload": f"forward NTT of {args.rows} limbs (ks48 extended basis, cyclically) per step",
                "rows": args.rows, "l2_policy": "inputs rotate through >126 MB"}
    if workload == "helr":
        return {"workload": "one HELR-style gradient step on ks48 moduli at 20 limbs (4 HMult+rescale, 3 PMult, 23 "
                            f"HRot, cubic sigmoid; BASELINE config 5), one CUDA-graph replay per step, {args.lanes} lanes",
                "l2_policy": "each step streams ~1.5 GB of rotation / relinearisation keys (>> 126 MB L2)"}
    return {"workload": "HMult + relinearise + rescale of two fresh ciphertexts, generate_parameter_set(n=8192, l=12, "
                        "dnum=3, delta=2^40) (BASELINE config 1), one product per step, replayed as one CUDA graph (ckks.capture)",
            "l2_policy": "operands rotate through 64 ciphertext pairs (50 MB) plus the relinearisation key; the "
                         "working set of one product is L2-resident by nature at this size"}


def load_peaks():
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        return float(json.loads(p.read_text())["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs, burst copy)"
    return 6650.0, "fallback (B200_PROFILING.md)"


class ClockSampler:
    """Samples SM clock and throttle reasons through NVML during the timed region."""

    def __init__(self, index: int):
        self.samples, self.reasons, self.max_mhz = [], set(), None
        # The polling thread is started BEFORE the warm-up (its first NVML queries take ~10 ms and were
        # seen to stall the first launch of the timed region: 21.7 instead of 9.0 ms for step 0);
        # `recording` brackets the timed region.
        self.recording = False
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
                mhz = nv.nvmlDeviceGetClockInfo(self.h, nv.NVML_CLOCK_SM)
                mask = nv.nvmlDeviceGetCurrentClocksThrottleReasons(self.h)
                if self.recording:               # only what falls inside the timed region is reported
                    self.samples.append(mhz)
                    for k, bit in names.items():
                        if mask & bit:
                            self.reasons.add(k)
            except Exception:
                pass
            time.sleep(0.02)

    def start(self):
        if self.nv:
            self._thread = threading.Thread(target=self._run, daemon=True)
            self._thread.start()

    def stop(self):
        self._stop.set()
        if self._thread:
            self._thread.join()

    def summary(self):
        med = float(np.median(self.samples)) if self.samples else None
        return {"sm_mhz": med, "sm_max_mhz": self.max_mhz, "reasons": sorted(self.reasons),
                "samples": len(self.samples)}


# kernel classes of the profiler (ProfScope names in csrc/) -> kernel family of the roofline
def family_of(name: str) -> str:
    return "ntt" if name.startswith("ntt") else name


def measured_traffic(workload, family):
    """DRAM bytes per launch (dram__bytes_read.sum + dram__bytes_write.sum), averaged over the
    launches of the kernels of `family`, from the committed ncu capture of this same workload
    (profiles/traffic_<workload>.json, written from an ncu run of `bench.py --steps 1`; ncu
    numbers are never taken inside a timed run)."""
    path = ROOT / "profiles" / f"traffic_{workload}.json"
    if not path.exists():
        return None, None
    doc = json.loads(path.read_text())
    total, launches = 0.0, 0
    for name, rec in doc.get("kernels", {}).items():
        if family_of(name) == family or name.startswith(family):
            total += (rec["dram_read_mb_per_launch"] + rec["dram_write_mb_per_launch"]) * 1e6 * rec["launches"]
            launches += rec["launches"]
    if not launches:
        return None, None
    return total / launches, doc.get("source")


def read_profile(eng):
    buf = ctypes.create_string_buffer(1 << 16)
    eng.lib.ckks_profile_read(buf, len(buf))
    out = {}
    for line in buf.value.decode().splitlines():
        name, cnt, ms, nbytes, nflops = line.split()
        out[name] = (int(cnt), float(ms), float(nbytes), float(nflops))
    return out


def host_threads():
    try:
        return len(os.sched_getaffinity(0))
    except Exception:
        return os.cpu_count() or 1


def cpu_model():
    try:
        for line in Path("/proc/cpuinfo").read_text().splitlines():
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except Exception:
        pass
    return "unknown"


# --------------------------------------------------------------------------------------
# the reference's path on the host cores (oracle/): reference arm and cpu_baseline
# --------------------------------------------------------------------------------------
def oracle_engine():
    """The CPU engine (oracle/engine_oracle.py) on every host thread.  torchrun exports
    OMP_NUM_THREADS=1 to its ranks; the CPU arm is meant to use all the threads it is given."""
    from oracle.engine_oracle import OracleEngine

    return OracleEngine(threads=host_threads())


class SlicedCircuit:
    """Runs `run_once` over and over in a worker thread and lets the caller advance it one
    segment (1/SEGMENTS of the engine calls of one run) at a time.  State is carried from
    segment to segment, so SEGMENTS consecutive steps are one whole run of the circuit."""

    def __init__(self, eng, run_once, ops_per_run: int):
        self.eng, self.run_once, self.ops_per_run = eng, run_once, ops_per_run
        self.bounds = [round(j * ops_per_run / SEGMENTS) for j in range(1, SEGMENTS + 1)]
        self.go, self.done = threading.Semaphore(0), threading.Semaphore(0)
        self.seg, self.base = 0, eng.ops
        self.error = None
        eng.on_op = self._on_op
        self.thread = threading.Thread(target=self._loop, daemon=True)
        self.thread.start()

    def _on_op(self, ops):
        if ops - self.base >= self.bounds[self.seg]:
            self.seg += 1
            if self.seg == SEGMENTS:
                self.seg, self.base = 0, ops
            self.done.release()
            self.go.acquire()

    def _loop(self):
        self.go.acquire()
        try:
            while True:
                self.run_once()
        except BaseException as exc:          # surface worker failures in the caller
            self.error = exc
            self.done.release()

    def step(self):
        self.go.release()
        self.done.acquire()
        if self.error is not None:
            raise self.error


def reference_circuit(workload):
    """(engine, run_once) of a circuit workload built entirely on the CPU engine."""
    from paper_2512_18345_b200 import engine
    from paper_2512_18345_b200.params import ParameterSet

    eng = oracle_engine()
    engine.use_backend(eng)
    p = ParameterSet.builtin("ks48")
    if workload == "bootstrap":
        from paper_2512_18345_b200.bootstrap import standard_input, standard_setup

        sk, _sparse, boot = standard_setup(p)
        _z, ct = standard_input(p, boot, sk, 0)
        return eng, (lambda: boot.bootstrap(ct))
    from paper_2512_18345_b200 import keyswitch as ks
    from paper_2512_18345_b200.helr import HelrShape, HelrTrainer

    sk = ks.keygen(p, h=p.h_dense, seed=1)
    shape = HelrShape(samples=128, features=256)
    trainer = HelrTrainer(p, sk, shape, level=20, lr=1.0)
    rng = np.random.default_rng(0)
    xs = rng.uniform(-1, 1, (shape.samples, shape.features))
    ys = np.where(rng.uniform(size=shape.samples) < 0.5, -1.0, 1.0)
    ct_z = trainer.encrypt((xs * ys[:, None]).reshape(-1), sk, seed=60)
    ct_w = trainer.encrypt(np.tile(rng.uniform(-0.02, 0.02, shape.features), shape.samples), sk, seed=61)
    return eng, (lambda: trainer.iteration(ct_z, ct_w))


def oracle_kernel_step(workload, args):
    """One step of a single-call workload on the oracle's C routines."""
    from oracle import oracle
    from paper_2512_18345_b200.params import ParameterSet, generate_parameter_set

    oracle.set_threads(host_threads())
    if workload == "config1":
        from oracle.engine_oracle import OracleEngine
        from paper_2512_18345_b200 import ckks, engine, keyswitch as ks

        engine.use_backend(OracleEngine(threads=host_threads()))
        p = generate_parameter_set(n=8192, l=12, dnum=3, delta=1 << 40, h_dense=64, h_sparse=32)
        sk = ks.keygen(p, seed=1)
        rlk = ckks.relin_keygen(sk, p, seed=41)
        m = [np.random.default_rng(7 + i).integers(1, 9, p.n).astype(np.int64) << 20 for i in range(2)]
        c1, c2 = ks.encrypt(m[0], sk, p, seed=2), ks.encrypt(m[1], sk, p, seed=5)
        return lambda: ckks.rescale(ckks.hmult(c1, c2, rlk), 1)
    p = ParameterSet.builtin("ks48")
    op = oracle.OParams(p.n, p.l, p.dnum, p.alpha, p.delta, p.h_dense,
                        tuple((m.q, m.psi) for m in p.q_basis), tuple((m.q, m.psi) for m in p.p_basis))
    orc = oracle.Oracle(p.n, op.ext_basis)
    rng = np.random.default_rng(0)
    qs = [q for q, _ in op.ext_basis]
    if workload == "ntt":
        rm = np.arange(args.rows, dtype=np.int32) % len(qs)
        x = np.stack([rng.integers(0, qs[i], p.n, dtype=np.uint64) for i in rm]).astype(np.uint32)
        return lambda: orc.ntt(x, rm)
    a = np.stack([rng.integers(0, q, p.n, dtype=np.uint64) for q in qs[:p.l]]).astype(np.uint32)
    b = np.stack([rng.integers(0, q, p.n, dtype=np.uint64) for q in qs[:p.l]]).astype(np.uint32)
    evk = np.stack([rng.integers(0, q, (p.dnum, 2, p.n), dtype=np.uint64) for q in qs])
    evk = np.ascontiguousarray(evk.transpose(1, 2, 0, 3)).astype(np.uint32)
    return lambda: orc.keyswitch(op, a, b, evk)


def numpy_reference_timing(workload, args):
    """The REAL reference (NumPy package, travelling copy under baseline/_ref) timed on the host
    cores by baseline/time_reference.py in a subprocess: single-process latency and a process pool
    over independent inputs (SURVEY 8d "CPU baseline").  None for the circuits (the reference has
    no bootstrap / HELR entry point) or when the copy is absent."""
    import subprocess

    if workload not in ("ntt", "keyswitch", "config1"):
        return None
    script = ROOT / "baseline" / "time_reference.py"
    if not (ROOT / "baseline" / "_ref" / "rnscope").is_dir():
        return {"unavailable": "no travelling copy of the reference (baseline/_ref/rnscope); run __graft_entry__.build() "
                               "where /root/reference exists"}
    env = dict(os.environ)
    env["OMP_NUM_THREADS"] = "1"
    try:
        res = subprocess.run([sys.executable, str(script), workload, "--rows", str(args.rows)], capture_output=True,
                             text=True, timeout=600, env=env)
        lines = [ln for ln in res.stdout.splitlines() if ln.startswith("{")]
        return json.loads(lines[-1]) if lines else {"unavailable": (res.stderr or "no output").strip()[-300:]}
    except Exception as exc:                      # a baseline, never a reason to lose the bench line
        return {"unavailable": repr(exc)[:300]}


def run_reference(args):
    """Rank 0 alone runs and prints; the other ranks exit without work."""
    if int(os.environ.get("RANK", "0")) != 0:
        return
    wl = args.workload
    steps, warmup = args.steps, args.warmup
    t_setup = time.perf_counter()
    if wl in ("bootstrap", "helr"):
        eng, run_once = reference_circuit(wl)
        before = eng.ops
        run_once()                               # untimed whole run: encoded constants, plan caches, op count
        ops_per_run = eng.ops - before
        circuit = SlicedCircuit(eng, run_once, ops_per_run)
        step = circuit.step
        per_step = 1.0 / SEGMENTS
        sample = (f"each step = 1/{SEGMENTS} of the {ops_per_run} engine calls of one whole {wl} run of the "
                  f"package's own circuit on the CPU oracle (oracle/engine_oracle.py + ckks_oracle.c, OpenMP), in order, "
                  f"state carried between steps: {SEGMENTS} steps = one complete run; one untimed whole run first")
    else:
        run = oracle_kernel_step(wl, args)
        step = run
        per_step = 1.0
        sample = "each step = one whole unit of the workload on oracle/ckks_oracle.c (OpenMP)"
    setup_s = time.perf_counter() - t_setup
    for _ in range(warmup):
        step()
    t0 = time.perf_counter()
    for _ in range(steps):
        step()
    elapsed = time.perf_counter() - t0
    value = steps * per_step / elapsed
    unit = UNIT[wl]
    line = {
        "impl": "reference", "metric": METRIC[wl], "value": value, "unit": unit,
        "n_gpus": args.gpus, "steps": steps, "warmup": warmup, "ms_per_step": elapsed / steps * 1e3,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "u32",
        "data": "synthetic", "config": config_for(wl, args),
        "units_per_step": per_step, "ms_per_unit": 1e3 / value, "setup_s": setup_s,
        "cpu_baseline": {"value": value, "unit": unit, "cores": host_threads(), "kind": "port",
                         "cpu": cpu_model(), "sample": sample},
        "e2e": {"value": value, "unit": unit, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    ref = numpy_reference_timing(wl, args)
    if ref is not None:
        line["cpu_baseline"]["reference"] = ref
    print(json.dumps(line), flush=True)


# --------------------------------------------------------------------------------------
# B200 arm
# --------------------------------------------------------------------------------------
def run_b200(args):
    import torch
    import torch.distributed as dist

    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if args.gpus != world:
        raise SystemExit(f"--gpus {args.gpus} needs {args.gpus} ranks (launch through torch.distributed.run with "
                         f"--nproc-per-node {args.gpus}); WORLD_SIZE is {world}")
    # one rank per GPU; a box with fewer GPUs than ranks (only when the N > 1 path is rehearsed on a
    # single-GPU machine) shares devices and rendezvous over gloo, and says so in the JSON line
    oversubscribed = world > torch.cuda.device_count()
    if oversubscribed:
        local %= torch.cuda.device_count()
    torch.cuda.set_device(local)
    if world > 1:
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        os.environ.setdefault("NCCL_DEBUG", "INFO")          # communicator size is read off NCCL's own log
        if oversubscribed:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))

    from paper_2512_18345_b200 import ckks, engine, keyswitch as ks, sharding, transform
    from paper_2512_18345_b200.engine import get_engine
    from paper_2512_18345_b200.params import ParameterSet, generate_parameter_set
    from paper_2512_18345_b200.rns import COEFFICIENT, EVALUATION, Polynomial

    eng = get_engine()
    p = ParameterSet.builtin("ks48")
    ext = p.ext_basis
    dev = eng.device
    g = torch.Generator(device=dev)
    g.manual_seed(1234)                  # the same synthetic inputs and keys on every rank (replicated state)
    wl = args.workload
    n_ring = p.n

    def rand_limbs(basis, *lead, n=None):
        """Uniform residues below each modulus, generated on the device (synthetic)."""
        n = n or p.n
        q = torch.tensor([m.q for m in basis], dtype=torch.float64, device=dev)[:, None]
        u = torch.rand((*lead, len(basis), n), generator=g, device=dev, dtype=torch.float64)
        return (u * q).to(torch.int64).clamp_(min=0).to(torch.int32).contiguous()

    precision_bits = None
    cpu_check = None          # (oracle_run_once, gpu_digest): a whole unit on the CPU oracle + the limbs to expect
    n_inputs = 4
    result_of = None          # device tensor holding the result of the last step (checksummed per step)
    if wl == "bootstrap":
        from paper_2512_18345_b200.bootstrap import standard_input, standard_setup

        eng.set_lanes(args.lanes)           # concurrent rotations / EvalMod branches inside the graph
        sk, _sparse, boot = standard_setup(p)
        pairs = [standard_input(p, boot, sk, i) for i in range(n_inputs)]
        msgs, cts = [z for z, _ in pairs], [c for _, c in pairs]
        cts_t = [torch.stack([c.a.data, c.b.data]) for c in cts]
        replay = boot.capture(cts[0])
        low = p.q_basis[:2]

        def step(i):
            replay.static_in.copy_(cts_t[i % n_inputs])
            replay.graph.replay()

        result_of = replay.static_out

        def profiled_step(i):
            boot.bootstrap(cts[i % n_inputs])

        host_in = [t.cpu().pin_memory() for t in cts_t[:2]]
        host_out = [torch.empty(tuple(replay.static_out.shape), dtype=torch.int32).pin_memory() for _ in range(2)]

        def e2e_step(i):
            # public API: host ciphertext in -> bootstrap -> host ciphertext out
            d = host_in[i % 2].to(dev, non_blocking=True)
            ct = ckks.Ciphertext(a=Polynomial(low, d[0], EVALUATION), b=Polynomial(low, d[1], EVALUATION),
                                 scale=boot.delta_in)
            out = replay(ct, copy_out=False)
            host_out[i % 2][0].copy_(out.a.data, non_blocking=True)
            host_out[i % 2][1].copy_(out.b.data, non_blocking=True)

        h2d = 2 * 2 * LIMB_BYTES
        d2h = 2 * boot.out_level * LIMB_BYTES
        # precision of the refreshed ciphertext (reported, not timed)
        out = replay(cts[0])
        err = float(np.abs(ckks.decrypt_decode(out, sk, p) - msgs[0]).max())
        precision_bits = float(np.log2(err))
        gpu_words = torch.stack([out.a.data, out.b.data]).cpu().numpy()
        cpu_check = (lambda: boot.bootstrap(cts[0]), gpu_words)
    elif wl == "helr":
        from paper_2512_18345_b200.helr import HelrShape, HelrTrainer, plain_iteration

        eng.set_lanes(args.lanes)
        sk = ks.keygen(p, h=p.h_dense, seed=1)
        shape = HelrShape(samples=128, features=256)
        trainer = HelrTrainer(p, sk, shape, level=20, lr=1.0)
        rng = np.random.default_rng(0)
        xs = rng.uniform(-1, 1, (shape.samples, shape.features))
        ys = np.where(rng.uniform(size=shape.samples) < 0.5, -1.0, 1.0)
        z = (xs * ys[:, None]).reshape(-1)
        w = np.tile(rng.uniform(-0.02, 0.02, shape.features), shape.samples)
        ct_z, ct_w = trainer.encrypt(z, sk, seed=60), trainer.encrypt(w, sk, seed=61)
        basis20 = ct_z.a.basis
        static_in = torch.stack([torch.stack([c.a.data, c.b.data]) for c in (ct_z, ct_w)]).clone()   # [2, 2, 20, n]

        def run_iteration():
            cz = ckks.ct_from_tensor(static_in[0], basis20, ct_z.scale)
            cw = ckks.ct_from_tensor(static_in[1], basis20, ct_w.scale)
            return trainer.iteration(cz, cw)

        run_iteration()
        torch.cuda.synchronize()
        graph = torch.cuda.CUDAGraph()
        side = torch.cuda.Stream(device=dev)
        side.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(side):
            run_iteration()
            torch.cuda.synchronize()
            with torch.cuda.graph(graph, stream=side):
                out_ct = run_iteration()
                static_out = torch.stack([out_ct.a.data, out_ct.b.data])
        torch.cuda.current_stream().wait_stream(side)
        generation = eng.arena_generation()
        fresh = static_in.clone()

        def step(i):
            assert eng.arena_generation() == generation, "workspace arena moved after capture"
            static_in.copy_(fresh)
            graph.replay()

        result_of = static_out
        profiled_step = lambda i: run_iteration()
        host_in = [fresh.cpu().pin_memory() for _ in range(2)]
        host_out = [torch.empty(tuple(static_out.shape), dtype=torch.int32).pin_memory() for _ in range(2)]

        def e2e_step(i):
            static_in.copy_(host_in[i % 2], non_blocking=True)
            graph.replay()
            host_out[i % 2].copy_(static_out, non_blocking=True)

        h2d = int(fresh.numel()) * 4
        d2h = int(static_out.numel()) * 4
        graph.replay()
        got = ckks.decrypt_decode(ckks.ct_from_tensor(static_out, out_ct.a.basis, out_ct.scale), sk, p).real
        precision_bits = float(np.log2(np.abs(got - plain_iteration(z, w, shape, 1.0)).max()))
        torch.cuda.synchronize()
        cpu_check = (lambda: trainer.iteration(ct_z, ct_w), static_out.cpu().numpy())
    elif wl == "keyswitch":
        n_ct, n_evk = 8, 4
        cts = [rand_limbs(p.q_basis, 2) for _ in range(n_ct)]               # 25 MB each
        evks = [rand_limbs(ext, p.dnum, 2) for _ in range(n_evk)]           # 126 MB each
        outs = [eng.empty(2, p.l, p.n) for _ in range(n_ct)]
        plan = ks._tables(p).plan()
        n_inputs = n_ct
        last = {"out": outs[0]}

        def step(i):
            ct = cts[i % n_ct]
            last["out"] = eng.keyswitch(plan, ct[0], ct[1], evks[i % n_evk], out=outs[i % n_ct])

        profiled_step = step
        host_in = [torch.empty((2, p.l, p.n), dtype=torch.int32).pin_memory() for _ in range(2)]
        host_out = [torch.empty((2, p.l, p.n), dtype=torch.int32).pin_memory() for _ in range(2)]
        for h, c in zip(host_in, cts):
            h.copy_(c)
        evk_keys = [ks.SwitchingKey(pairs=tuple(
            ks.PolyPair(a=Polynomial(ext, e[t, 0], EVALUATION), b=Polynomial(ext, e[t, 1], EVALUATION))
            for t in range(p.dnum)), params=p, _matrix=e) for e in evks]

        def e2e_step(i):
            d = host_in[i % 2].to(dev, non_blocking=True)
            ct = ks.Ciphertext(a=Polynomial(p.q_basis, d[0], EVALUATION),
                               b=Polynomial(p.q_basis, d[1], EVALUATION), scale=p.delta)
            out = ks.keyswitch(ct, evk_keys[i % n_evk])
            host_out[i % 2][0].copy_(out.a.data, non_blocking=True)
            host_out[i % 2][1].copy_(out.b.data, non_blocking=True)

        h2d = d2h = 2 * p.l * LIMB_BYTES
    elif wl == "config1":
        p1 = generate_parameter_set(n=8192, l=12, dnum=3, delta=1 << 40, h_dense=64, h_sparse=32)
        n_ring = p1.n
        sk = ks.keygen(p1, seed=1)
        rlk = ckks.relin_keygen(sk, p1, seed=41)
        n_inputs = 64
        xs = [rand_limbs(p1.q_basis, 2, n=p1.n) for _ in range(n_inputs)]
        ys = [rand_limbs(p1.q_basis, 2, n=p1.n) for _ in range(n_inputs)]
        as_ct = lambda t: ckks.ct_from_tensor(t, p1.q_basis, float(p1.delta))
        last = {}

        product = lambda a, b: ckks.rescale(ckks.hmult(a, b, rlk), 1)
        replay1 = ckks.capture(product, as_ct(xs[0]), as_ct(ys[0]))      # one CUDA graph per product

        def step(i):
            out = replay1(as_ct(xs[i % n_inputs]), as_ct(ys[i % n_inputs]), copy_out=False)
            last["out"] = out.a.data

        def profiled_step(i):                                             # eager: per-kernel events
            product(as_ct(xs[i % n_inputs]), as_ct(ys[i % n_inputs]))
        limb1 = p1.n * 4
        host_in = [torch.empty((2, 2, p1.l, p1.n), dtype=torch.int32).pin_memory() for _ in range(2)]
        host_out = [torch.empty((2, p1.l - 1, p1.n), dtype=torch.int32).pin_memory() for _ in range(2)]
        for h in host_in:
            h[0].copy_(xs[0])
            h[1].copy_(ys[0])

        def e2e_step(i):
            d = host_in[i % 2].to(dev, non_blocking=True)
            out = replay1(as_ct(d[0]), as_ct(d[1]), copy_out=False)
            host_out[i % 2][0].copy_(out.a.data, non_blocking=True)
            host_out[i % 2][1].copy_(out.b.data, non_blocking=True)

        h2d, d2h = 4 * p1.l * limb1, 2 * (p1.l - 1) * limb1
    else:
        rows = args.rows
        basis = tuple(ext[i % len(ext)] for i in range(rows))
        count = max(2, -(-(160 << 20) // (rows * LIMB_BYTES)))               # rotate through > 126 MB
        polys = [rand_limbs(basis) for _ in range(count)]
        outs = [eng.empty(rows, p.n) for _ in range(count)]
        slots = eng.row_slots(basis, p.n)
        n_inputs = count
        last = {"out": outs[0]}

        def step(i):
            last["out"] = eng.ntt(polys[i % count], slots, False, out=outs[i % count])

        profiled_step = step
        host_in = [torch.empty((rows, p.n), dtype=torch.int32).pin_memory() for _ in range(2)]
        host_out = [torch.empty((rows, p.n), dtype=torch.int32).pin_memory() for _ in range(2)]

        def e2e_step(i):
            d = host_in[i % 2].to(dev, non_blocking=True)
            out = transform.ntt_polynomial(Polynomial(basis, d, COEFFICIENT))
            host_out[i % 2].copy_(out.data, non_blocking=True)

        h2d = d2h = rows * LIMB_BYTES

    def ntt_sweep():
        """BASELINE config 2: forward and inverse transforms at R in {12, 48, 60, 192, 240}
        limbs of the ks48 extended basis.  Each point: a CUDA graph of `reps` transforms over operands
        rotating through > 126 MB, timed with CUDA events (device time per transform); algorithmic
        bytes 2*R*N*4 (reference-convention two-kernel bytes are twice that), butterflies
        R*(N/2)*log2 N against the integer-pipe bound of profiles/microbench/int_pipes.cu."""
        out = []
        sm_count = torch.cuda.get_device_properties(dev).multi_processor_count
        peak_hbm = load_peaks()[0]
        for rows_ in (12, 48, 60, 192, 240):
            basis_ = tuple(ext[i % len(ext)] for i in range(rows_))
            count_ = max(2, -(-(160 << 20) // (rows_ * LIMB_BYTES)))
            polys_ = [rand_limbs(basis_) for _ in range(count_)]
            outs_ = [eng.empty(rows_, p.n) for _ in range(count_)]
            slots_ = eng.row_slots(basis_, p.n)
            for inverse in (False, True):
                reps = 4 * count_
                run = lambda: [eng.ntt(polys_[k % count_], slots_, inverse, out=outs_[k % count_]) for k in range(reps)]
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
                us = a.elapsed_time(b) * 1e3 / (n_rep * reps)
                alg = 2.0 * rows_ * LIMB_BYTES
                bf = rows_ * (p.n // 2) * 16
                out.append({"rows": rows_, "direction": "inverse" if inverse else "forward", "us": us,
                            "alg_bytes": alg, "alg_gbs": alg / us / 1e3, "hbm_frac": alg / us / 1e3 / peak_hbm,
                            "ref_convention_gbs": 2 * alg / us / 1e3,
                            "butterflies_per_clk_per_sm": bf / (us * 1e-6) / (1.965e9 * sm_count),
                            "int_pipe_frac": bf / (us * 1e-6) / (1.965e9 * sm_count) / INT_PIPE_BF_PER_CLK_SM})
                del graph
            del polys_, outs_
        return out

    class EventClock:
        """Device time on the current stream (every kernel of a step is joined back into it)."""

        def start(self):
            self.a, self.b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            self.a.record()

        def stop(self):
            self.b.record()
            torch.cuda.synchronize()
            return self.a.elapsed_time(self.b)

    def sync():
        torch.cuda.synchronize()

    def timed(fn, steps, warmup, sampler=None, checksums=False, settle=False):
        """`steps` steps of this rank over its shard of a (steps x world)-item job.  With
        `checksums`, a 64-bit sum of every result is formed on the device after each step and the
        per-rank lists are gathered (in input order) on rank 0 inside the timed bracket."""
        if sampler:
            sampler.start()                    # polling starts now, recording only inside the timed region
        for i in range(warmup):
            fn(i)
        if checksums:
            # the checksum reduction's first launch loads its CUDA module lazily (21 - 133 ms measured inside
            # step 0 when it first ran in the timed region): run it once here, untimed
            t = result_of if result_of is not None else last["out"]
            int(t.sum(dtype=torch.int64).item())
        if settle:
            # untimed settling after the W warm-up steps: the first replays after a long host-side setup
            # run slower (clock / power state and cache ramp: 9.6 vs 9.1 ms per bootstrap measured back to
            # back); repeat short windows until two consecutive ones agree within 1 % (at most 8 windows)
            window, prev = max(5, min(steps, 200) // 10), None
            for _ in range(8):
                clock = EventClock()
                sync()
                clock.start()
                for i in range(window):
                    fn(i)
                cur = clock.stop()
                timed.settle_steps += window
                if prev is not None and abs(cur - prev) <= 0.01 * cur:
                    break
                prev = cur
        sums = []

        marks = []

        def one(item):
            if os.environ.get("BENCH_DEBUG_STEPS"):
                ev = torch.cuda.Event(enable_timing=True)
                ev.record()
                marks.append(ev)
            fn(item % steps)              # rank r, step s of the job is item r * steps + s: input s on every rank
            # circuits (ms per step) checksum every result; for the microsecond-scale kernel workloads a
            # reduction per step would be a large part of the step, so only the last result is summed
            if checksums and (per_step_checksum or item % steps == steps - 1):
                t = result_of if result_of is not None else last["out"]
                sums.append(t.sum(dtype=torch.int64))
            return len(sums) - 1

        if sampler:
            sampler.recording = True
        ranged = sampler is not None and os.environ.get("BENCH_PROFILER_RANGE")
        if ranged:                      # ncu --profile-from-start off: only the timed region is profiled
            torch.cuda.profiler.start()
        finish = (lambda local: [int(v) for v in torch.stack(sums).cpu().tolist()]) if checksums else None
        gathered, ms, wall_ms = sharding.sharded_job(list(range(steps * world)), one, clock=EventClock(), sync=sync,
                                                     finish=finish, device=dev)
        if ranged:
            torch.cuda.profiler.stop()
        if sampler:
            sampler.recording = False
            sampler.stop()
        timed.wall_ms = wall_ms
        if marks:
            torch.cuda.synchronize()
            print("[debug] per-step ms:", " ".join(f"{marks[i].elapsed_time(marks[i + 1]):.2f}" for i in range(len(marks) - 1)),
                  file=sys.stderr, flush=True)
        return ms, gathered

    per_step_checksum = wl in ("bootstrap", "helr") and not os.environ.get("BENCH_LAST_CHECKSUM_ONLY")
    sampler = ClockSampler(local)
    timed.settle_steps = 0
    ms_total, gathered = timed(step, args.steps, args.warmup, sampler, checksums=True, settle=True)
    wall_total = timed.wall_ms
    ms_step = ms_total / args.steps
    value = world * args.steps / (ms_total * 1e-3)
    ranks_agree = None
    if rank == 0 and gathered is not None and world > 1:
        # replicated keys + the same inputs on every rank: every GPU must produce the same limbs
        gathered = [v for v in gathered if v is not None]      # ranks that summed only their last result
        n_sums = len(gathered) // world
        per_rank = [gathered[r * n_sums:(r + 1) * n_sums] for r in range(world)]
        ranks_agree = all(pr == per_rank[0] for pr in per_rank)

    e2e_steps = max(3, min(args.steps, 200))
    e2e_ms, _ = timed(e2e_step, e2e_steps, max(3, min(args.warmup, 5)))
    e2e_value = world * e2e_steps / (e2e_ms * 1e-3)

    # per-kernel pass: the same step, eager, every launch bracketed by CUDA events
    prof_steps = max(2, min(args.steps, 3 if wl in ("bootstrap", "helr") else 50))
    lanes_saved = getattr(eng, "lanes", 1)
    eng.lanes = 1                      # one stream: per-kernel durations without overlap from other lanes
    profiled_step(0)
    torch.cuda.synchronize()
    eng.lib.ckks_profile_enable(1)
    for i in range(prof_steps):
        profiled_step(i)
    prof = read_profile(eng)
    eng.lib.ckks_profile_enable(0)
    eng.lanes = lanes_saved
    launches_per_step = sum(c for c, _, _, _ in prof.values()) / prof_steps
    total_prof_ms = sum(ms for _, ms, _, _ in prof.values())
    # kernel families: the transform's kernels (ntt16_fwd_strided, ..._contig, ..._moddown, the
    # small-ring and generic variants) are ONE family, charged SURVEY 8(d)'s algorithmic bytes:
    # 2 * R * N * 4 per transform (each kernel of the pair reports its half, csrc/ntt.cu)
    fam = {}
    for name, (c, ms, nb, nf) in prof.items():
        f = fam.setdefault(family_of(name), {"launches": 0, "ms": 0.0, "bytes": 0.0, "flops": 0.0, "kernels": []})
        f["launches"] += c
        f["ms"] += ms
        f["bytes"] += nb
        f["flops"] += nf
        f["kernels"].append(name)
    top = max(fam, key=lambda k: fam[k]["ms"])
    peak, peak_src = load_peaks()
    ft = fam[top]
    achieved = ft["bytes"] / (ft["ms"] * 1e-3) / 1e9
    traffic, traffic_src = measured_traffic(wl, top)
    bound, unit = "hbm", "GB/s"
    if ft["flops"] > 0:
        # a family that runs on the FP64 tensor cores (split-integer base conversion): roofline
        # against the measured DMMA rate, profiles/microbench/dmma.cu (63.7 FMA/clk/SM x 148 SMs x
        # 1.965 GHz x 2 = 37.06 TFLOP/s); MEASURED_PEAKS.json has no FP64 figure
        bound, unit = "tensor", "TFLOP/s"
        achieved = ft["flops"] / (ft["ms"] * 1e-3) / 1e12
        peak, peak_src = FP64_TENSOR_TFLOPS, "measured FP64 DMMA rate (profiles/microbench/dmma.cu, mma.sync m8n8k4 f64)"
    hbm_peak = load_peaks()[0]
    roofline = {
        "bound": bound, "kernel": top, "kernels_in_family": sorted(ft["kernels"]),
        "achieved": achieved, "peak": peak, "unit": unit,
        "frac": achieved / peak, "traffic": traffic, "traffic_source": traffic_src, "peak_source": peak_src,
        "avg_launch_us": ft["ms"] / ft["launches"] * 1e3, "alg_bytes_per_launch": ft["bytes"] / ft["launches"],
        "share_of_step": ft["ms"] / total_prof_ms,
        "note": "dominant kernel FAMILY of an eager single-stream pass of the same step, every launch bracketed by "
                "CUDA events on its stream; achieved = SURVEY 8(d) algorithmic bytes (operand limbs read + written "
                "once: 2*R*N*4 per transform, twiddles and tables excluded) / the family's summed launch time",
        "families": {k: {"launches_per_step": v["launches"] / prof_steps, "us_per_launch": v["ms"] / v["launches"] * 1e3,
                         "share": v["ms"] / total_prof_ms,
                         "gbs": (v["bytes"] / (v["ms"] * 1e-3) / 1e9) if v["bytes"] else None,
                         "hbm_frac": (v["bytes"] / (v["ms"] * 1e-3) / 1e9 / hbm_peak) if v["bytes"] else None,
                         "tflops": (v["flops"] / (v["ms"] * 1e-3) / 1e12) if v["flops"] else None}
                     for k, v in sorted(fam.items(), key=lambda kv: -kv[1]["ms"])},
        "kernels": {k: {"launches_per_step": c / prof_steps, "us_per_launch": ms / c * 1e3,
                        "share": ms / total_prof_ms, "gbs": (nb / (ms * 1e-3) / 1e9) if nb else None}
                    for k, (c, ms, nb, nf) in sorted(prof.items(), key=lambda kv: -kv[1][1])},
    }

    if "ntt" in fam and n_ring == 65536:
        # the transform is bounded by the integer pipes on B200, not by HBM: report
        # butterflies per clock per SM next to the byte roofline (8 algorithmic bytes per 16*N/2 butterflies)
        nt = fam["ntt"]
        sm_count = torch.cuda.get_device_properties(dev).multi_processor_count
        bf = nt["bytes"] / (8.0 * n_ring) * (n_ring // 2) * 16
        rate = bf / (nt["ms"] * 1e-3) / (1.965e9 * sm_count)
        roofline["ntt_int_pipe"] = {"butterflies_per_clk_per_sm": rate, "peak": INT_PIPE_BF_PER_CLK_SM,
                                    "frac": rate / INT_PIPE_BF_PER_CLK_SM,
                                    "peak_source": "profiles/microbench/int_pipes.cu (IMAD.HI 28, IMAD 62 per clk per SM)"}

    cpu = None
    parity = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        unit_name = UNIT[wl]
        if cpu_check is not None:
            # one WHOLE unit of the same workload on the CPU oracle (the package's circuit on the C
            # restatement; keys and plaintexts are pulled from the GPU per call), also the checker:
            # its limbs must equal what the GPU produced for the same input
            run_once, gpu_words = cpu_check
            torch.cuda.synchronize()
            o_eng = oracle_engine()
            previous = engine.use_backend(o_eng)
            try:
                t0 = time.perf_counter()
                o_out = run_once()
                cpu_s = time.perf_counter() - t0
            finally:
                engine.use_backend(previous)
            o_words = torch.stack([o_out.a.data, o_out.b.data]).numpy()
            parity = bool(np.array_equal(o_words, gpu_words))
            cpu = {"value": 1.0 / cpu_s, "unit": unit_name, "cores": host_threads(), "kind": "port",
                   "cpu": cpu_model(), "ms_per_step": cpu_s * 1e3,
                   "sample": f"one whole {wl} of input 0 on the CPU oracle (oracle/engine_oracle.py + ckks_oracle.c, "
                             f"OpenMP, {o_eng.ops} engine calls; includes copying keys / plaintexts from the GPU)"}
        else:
            run = oracle_kernel_step(wl, args)
            run()
            reps = 3 if wl != "config1" else 10
            t0 = time.perf_counter()
            for _ in range(reps):
                run()
            cpu_s = (time.perf_counter() - t0) / reps
            engine.use_backend(None) if wl == "config1" else None
            cpu = {"value": 1.0 / cpu_s, "unit": unit_name, "cores": host_threads(), "kind": "port",
                   "cpu": cpu_model(), "ms_per_step": cpu_s * 1e3,
                   "sample": f"{reps} whole steps of the workload on oracle/ckks_oracle.c (OpenMP)"}
            ref = numpy_reference_timing(wl, args)
            if ref is not None:
                cpu["reference"] = ref

    batched = None
    if wl == "bootstrap" and world == 1 and not args.no_batch:
        # BASELINE config 5 on one GPU: a batch of two independent bootstraps as ONE graph over 16 lanes
        # (Bootstrapper.bootstrap_batch; the six linear transforms go through ckks_bsgs_inner_batch), checked
        # limb for limb against the single-bootstrap graph's results, device-timed like `value`.  Reported
        # beside the headline, which stays the latency-bound single bootstrap.
        singles = [replay(c) for c in cts[:2]]
        want = [torch.stack([o.a.data, o.b.data]).clone() for o in singles]
        torch.cuda.synchronize()
        eng.set_lanes(16)                  # moves the workspace arena: the single graph is not replayed after this
        replay_b = boot.capture_batch(cts[:2])
        got = replay_b(cts[:2])
        same = all(bool(torch.equal(torch.stack([o.a.data, o.b.data]), w)) for o, w in zip(got, want))
        for _ in range(3):
            replay_b.graph.replay()
        torch.cuda.synchronize()
        reps_b = max(3, args.steps // 2)
        ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        ev0.record()
        for _ in range(reps_b):
            replay_b.graph.replay()
        ev1.record()
        torch.cuda.synchronize()
        ms_b = ev0.elapsed_time(ev1) / reps_b
        batched = {"batch": 2, "lanes": 16, "ms_per_batch": ms_b, "value": 2000.0 / ms_b, "unit": UNIT[wl],
                   "replays": reps_b, "same_limbs_as_single_bootstraps": same}

    if rank == 0:
        line = {
            "metric": METRIC[wl], "value": value, "unit": UNIT[wl], "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "settle_steps": timed.settle_steps, "ms_per_step": ms_step,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "u32",
            "data": "synthetic", "config": config_for(wl, args),
            "e2e": {"value": e2e_value, "unit": UNIT[wl], "h2d_bytes_per_step": h2d,
                    "d2h_bytes_per_step": d2h, "ms_per_step": e2e_ms / e2e_steps},
            "gpu_launches": int(round(launches_per_step * args.steps)),
            "clocks": sampler.summary(), "roofline": roofline, "cpu_baseline": cpu,
            "sharding": {"items": args.steps * world, "per_rank": args.steps,
                         "collective": "one gather of per-result checksums (sharding.gather_results)",
                         "wall_ms_barrier_to_gather": wall_total, "ranks_agree": ranks_agree},
        }
        if wl == "bootstrap":
            line["latency_ms"] = ms_step
            line["paper_rtx5090_latency_ms"] = 15.2
            if batched is not None:
                line["batch2"] = batched
        if wl == "ntt" and not args.no_sweep:
            line["sweep"] = ntt_sweep()
        if precision_bits is not None:
            line["precision_log2_max_err"] = precision_bits
        if parity is not None:
            line["limbs_equal_cpu_oracle"] = parity
        if oversubscribed:
            line["oversubscribed"] = f"{world} ranks on {torch.cuda.device_count()} GPU(s): rehearsal of the N > 1 path, not a scaling number"
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=None)
    ap.add_argument("--warmup", type=int, default=None)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--workload", default="bootstrap", choices=["bootstrap", "keyswitch", "ntt", "helr", "config1"])
    ap.add_argument("--rows", type=int, default=60, help="limbs per transform of the ntt workload (config 2: 12..240)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-sweep", action="store_true", help="ntt workload: skip the R / direction sweep")
    ap.add_argument("--no-batch", action="store_true", help="bootstrap workload: skip the batch-of-two throughput leg")
    ap.add_argument("--lanes", type=int, default=8, help="workspace lanes / side streams of the bootstrap graph")
    args = ap.parse_args()
    if args.steps is None:
        args.steps = DEFAULT_STEPS[args.workload] if args.impl == "b200" else SEGMENTS
    if args.warmup is None:
        args.warmup = (3 if args.workload in ("bootstrap", "helr") else 20) if args.impl == "b200" else 3
    if args.impl == "reference":
        run_reference(args)
    else:
        args.warmup = max(args.warmup, 3)      # timing rule: at least three untimed warm-up steps
        run_b200(args)


if __name__ == "__main__":
    main()
