"""Host-side multi-process logic on CPU: world_size 2 over gloo (rendezvous on
127.0.0.1).  The work items stand in for ciphertexts; the data path has no
collective, results are gathered once."""
import os
import socket

import pytest
import torch.multiprocessing as mp

from paper_2512_18345_b200.sharding import shard_bounds


def test_shard_bounds_cover_everything_once():
    for count in (0, 1, 7, 8, 64, 65):
        for world in (1, 2, 3, 4, 8):
            spans = [shard_bounds(count, world, r) for r in range(world)]
            assert spans[0][0] == 0 and spans[-1][1] == count
            assert all(spans[i][1] == spans[i + 1][0] for i in range(world - 1))
            sizes = [hi - lo for lo, hi in spans]
            assert max(sizes) - min(sizes) <= 1
    with pytest.raises(ValueError):
        shard_bounds(4, 2, 2)


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, out_q):
    import torch.distributed as dist

    from paper_2512_18345_b200.sharding import gather_results, max_over_ranks, run_sharded, sharded_job

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    items = list(range(11))                     # 11 independent "ciphertexts"
    lo, hi, res = run_sharded(items, lambda x: x * x + 1)
    gathered = gather_results(res, lo, len(items))
    slowest = max_over_ranks(10.0 + rank)
    # the function bench.py --gpus N times a step batch through: shard, finish, one gather
    job, ms, wall = sharded_job(list(range(7)), lambda x: 3 * x, finish=lambda loc: [v + 1 for v in loc])
    assert ms >= 0.0 and wall >= ms * 0.0
    assert job == ([3 * x + 1 for x in range(7)] if rank == 0 else None)
    out_q.put((rank, lo, hi, gathered, slowest))
    dist.barrier()
    dist.destroy_process_group()


def test_two_ranks_shard_and_gather_in_order():
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    got = sorted(q.get(timeout=120) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    (r0, lo0, hi0, g0, s0), (r1, lo1, hi1, g1, s1) = got
    assert (lo0, hi0, lo1, hi1) == (0, 6, 6, 11)
    assert g0 == [x * x + 1 for x in range(11)] and g1 is None
    assert s0 == s1 == 11.0
