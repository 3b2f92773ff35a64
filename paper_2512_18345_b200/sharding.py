"""Multi-GPU execution: independent ciphertexts (or bootstraps) are split into
contiguous chunks, one process per GPU, keys and tables replicated per process;
there is no collective on the data path.  `torch.distributed` is
used only to gather results or timing scalars (NCCL on GPUs, gloo in the CPU
tests of this module's host logic).
"""
from __future__ import annotations

from typing import Callable, Sequence


def shard_bounds(count: int, world: int, rank: int) -> tuple[int, int]:
    """Contiguous [lo, hi) slice of `count` work items owned by `rank`: sizes
    differ by at most one, earlier ranks take the remainder."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError(f"bad rank {rank} for world size {world}")
    base, extra = divmod(count, world)
    lo = rank * base + min(rank, extra)
    return lo, lo + base + (1 if rank < extra else 0)


def run_sharded(items: Sequence, fn: Callable, rank: int | None = None, world: int | None = None):
    """Apply `fn` to this rank's shard of `items`; returns (lo, hi, results)."""
    import torch.distributed as dist

    if world is None:
        world = dist.get_world_size() if dist.is_available() and dist.is_initialized() else 1
    if rank is None:
        rank = dist.get_rank() if dist.is_available() and dist.is_initialized() else 0
    lo, hi = shard_bounds(len(items), world, rank)
    return lo, hi, [fn(x) for x in items[lo:hi]]


def gather_results(local: list, lo: int, total: int, dst: int = 0):
    """Gather per-rank result lists (picklable, e.g. digests or host arrays) in
    input order on rank `dst`; other ranks get None.  The only collective of a
    sharded job."""
    import torch.distributed as dist

    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size() == 1:
        return list(local)
    world, rank = dist.get_world_size(), dist.get_rank()
    bucket = [None] * world if rank == dst else None
    dist.gather_object((lo, list(local)), bucket, dst=dst)
    if rank != dst:
        return None
    out = [None] * total
    for start, chunk in bucket:
        out[start:start + len(chunk)] = chunk
    return out


def max_over_ranks(value: float, device=None) -> float:
    """Max of a timing scalar over ranks (device-timed numbers are reported as the max)."""
    import torch
    import torch.distributed as dist

    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size() == 1:
        return float(value)
    t = torch.tensor([float(value)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


class WallClock:
    """Host clock with the start() / stop() -> milliseconds protocol of sharded_job (CPU tests;
    on a GPU the caller passes a CUDA-event clock so that the time is taken on the device)."""

    def start(self):
        import time

        self._t0 = time.perf_counter()

    def stop(self) -> float:
        import time

        return (time.perf_counter() - self._t0) * 1e3


def sharded_job(items: Sequence, fn: Callable, clock=None, sync: Callable | None = None,
                finish: Callable | None = None, device=None, dst: int = 0):
    """One job over independent work items the way BASELINE config 5 times it: barrier, this
    rank's contiguous shard of `items` through `fn` (no collective on the data path), `finish`
    turning the local results into picklable values (e.g. reading device checksums back), ONE
    gather of the results on rank `dst`, barrier.

    Returns (results in input order on `dst` / None elsewhere, ms, wall_ms): `ms` is the max over
    ranks of `clock` around the shard's work (CUDA events on a GPU: device time), `wall_ms` the max
    over ranks of the host time from the first barrier to after the gather.  bench.py --gpus N and
    the two-rank gloo test both go through this function."""
    import time

    import torch.distributed as dist

    live = dist.is_available() and dist.is_initialized() and dist.get_world_size() > 1
    clock = clock or WallClock()

    def barrier():
        if live:
            dist.barrier()
        if sync is not None:
            sync()

    barrier()
    t0 = time.perf_counter()
    clock.start()
    lo, hi, local = run_sharded(items, fn)
    ms = clock.stop()
    if finish is not None:
        local = finish(local)
    gathered = gather_results(local, lo, len(items), dst=dst)
    wall_ms = (time.perf_counter() - t0) * 1e3
    barrier()
    return gathered, max_over_ranks(ms, device), max_over_ranks(wall_ms, device)
