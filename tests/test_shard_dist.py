"""Multi-GPU host logic on CPU: shard placement and the rank timing reductions (gloo, world_size 2).

The decode path has no collective; the only multi-process logic is the placement of
transformer blocks on ranks and the max/sum reductions of the timings, exercised here with gloo.
"""
import os
import socket

import pytest

from paper_2504_11651_b200.shard import plan_shards


def test_plan_shards_70b_and_405b():
    # 70B: 80 equal blocks + embed (first) + lm_head (last) -> 80/40/20/10 blocks per GPU
    for world, per in ((1, 80), (2, 40), (4, 20), (8, 10)):
        r = plan_shards([100] * 80, world)
        assert [len(x) for x in r] == [per] * world
        assert r[0].start == 0 and r[-1].stop == 80
    # 405B: 126 blocks on 8 GPUs -> 16/16/16/16/16/16/15/15 (or any split with max 16)
    r = plan_shards([1] * 126, 8)
    assert max(len(x) for x in r) == 16 and sum(len(x) for x in r) == 126


def test_plan_shards_contiguous_and_optimal_brute_force():
    import itertools
    import random
    rnd = random.Random(0)
    for _ in range(200):
        n = rnd.randint(1, 9)
        world = rnd.randint(1, 4)
        sizes = [rnd.randint(1, 20) for _ in range(n)]
        r = plan_shards(sizes, world)
        assert len(r) == world
        flat = [i for x in r for i in x]
        assert flat == list(range(n))                      # contiguous, in order, complete
        got = max(sum(sizes[i] for i in x) for x in r)
        best = None
        for cuts in itertools.combinations(range(1, n), min(world - 1, n - 1)):
            bounds = [0, *cuts, n]
            m = max(sum(sizes[a:b]) for a, b in zip(bounds, bounds[1:]))
            best = m if best is None else min(best, m)
        assert got == best


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world),
                      LOCAL_RANK=str(rank))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2504_11651_b200 import shard
    assert shard.rank_info() == (rank, world, rank)
    shard.barrier()
    mx = shard.max_over_ranks([1.0 + rank, 10.0 - rank])
    sm = shard.sum_over_ranks([2.0 * (rank + 1)])
    plan = shard.plan_shards([5] * 10, world)
    q.put((rank, mx, sm, [list(x) for x in plan]))
    dist.destroy_process_group()


def test_gloo_world2_reductions():
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    ps = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in ps:
        p.start()
    res = [q.get(timeout=120) for _ in ps]
    for p in ps:
        p.join(timeout=60)
        assert p.exitcode == 0
    for rank, mx, sm, plan in res:
        assert mx == [2.0, 10.0]
        assert sm == [6.0]
        assert plan == [list(range(0, 5)), list(range(5, 10))]
