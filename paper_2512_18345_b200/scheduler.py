"""L2-aware batch planning as a run-time decision (the reference keeps it as an analytical
model: costmodel.py:320-332 keyswitch_footprint, :407-420 plan_batch).

`plan_batch` answers the reference's question -- how many independent key-switching sequences
fit the L2 together -- with the reference's own footprint rule and B200's 126 MB L2, and
`keyswitch.keyswitch_batched` uses the answer: that many key switches of the batch are in flight
at once (one workspace lane and stream each), the rest follow in waves: B* = 2 at ks48, 5 at ks24,
10 at ks12.  Measured against a plain loop and against the two-lane stage pipeline
(`keyswitch.keyswitch_pipelined`) in profiles/r1s_ks_schedules.json."""
from __future__ import annotations

import json
from dataclasses import dataclass
from importlib import resources

from .params import ParameterSet

B200_L2_BYTES = 126 * (1 << 20)          # B300_MICROARCH guide: ~126 MB total over both dies


def machine_profile(name: str = "b200") -> dict:
    """Measured machine profile in the reference's schema (data/profiles/*.json, read by
    costmodel.MachineModel.from_dict, costmodel.py:95-103): lets `rnscope plan / analyze` predict
    this engine's kernels from B200's measured L2 / HBM / integer-pipe peaks.
    The extra "measured" object says where each number comes from; the reference ignores it."""
    text = resources.files(__package__).joinpath(f"data/profiles/{name}.json").read_text()
    return json.loads(text)


@dataclass(frozen=True)
class BatchPlan:
    sequence: str
    batch: int                # B*: sequences whose working sets fit the L2 together (>= 1)
    footprint_per_sequence: int
    footprint: int
    l2_capacity: int
    spills: bool              # even one sequence overflows the cache


def keyswitch_footprint(params: ParameterSet, stage: int, batch: int = 1) -> int:
    """Maximum live working set of a key-switching stage in bytes (costmodel.py:320-332): stage 1
    holds the (beta, L + alpha) raised digits, stage 3 the 4 L limbs of the polynomial pair with
    its inputs and outputs."""
    limb = params.n * 4
    if stage == 1:
        return batch * params.beta * (params.l + params.alpha) * limb
    if stage == 3:
        return batch * 4 * params.l * limb
    raise ValueError("footprint is defined for stages 1 and 3")


def plan_batch(params: ParameterSet, sequence: str = "ks_full", l2_capacity: int = B200_L2_BYTES) -> BatchPlan:
    """Largest batch whose working set stays L2-resident (costmodel.py:407-420)."""
    if sequence == "ks_stage1":
        per_seq = keyswitch_footprint(params, 1)
    elif sequence == "ks_stage3":
        per_seq = keyswitch_footprint(params, 3)
    elif sequence == "ks_full":
        per_seq = max(keyswitch_footprint(params, 1), keyswitch_footprint(params, 3))
    else:
        raise ValueError(f"unknown sequence {sequence!r}")
    if per_seq > l2_capacity:
        return BatchPlan(sequence, 1, per_seq, per_seq, l2_capacity, True)
    b_star = l2_capacity // per_seq
    return BatchPlan(sequence, int(b_star), per_seq, int(b_star) * per_seq, l2_capacity, False)


def concurrent_keyswitches(params: ParameterSet, lanes: int, pending: int) -> int:
    """How many of `pending` independent key switches to put in flight at once."""
    return max(1, min(plan_batch(params, "ks_full").batch, lanes, pending))
