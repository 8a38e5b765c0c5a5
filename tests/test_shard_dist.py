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


def test_model_shards_70b_strong_405b_weak():
    """70B: the whole model (embed + 80 blocks + lm_head) over N ranks: 80/40/20/10 blocks per GPU
    (P:240 placement); 405B: rank r decodes shard r of 8 whatever N is."""
    import workloads
    from paper_2504_11651_b200 import shard
    cfg70 = dict(workloads.MODELS["llama70b_model"], block_elems=workloads.config_numel("llama70b_block"))
    units = shard.model_units(cfg70)
    for world, per in ((1, 80), (2, 40), (4, 20), (8, 10)):
        rs = [shard.model_shard(cfg70, r, world)[0] for r in range(world)]
        assert [x for r in rs for x in r] == list(range(82))            # contiguous, complete
        blocks = [len([u for u in r if 1 <= u <= 80]) for r in rs]
        assert sum(blocks) == 80 and max(blocks) <= per + 1             # ~80/40/20/10 blocks per GPU
        assert rs[0].start == 0 and rs[-1].stop == 82                   # embed on rank 0, head on the last
        # the largest shard is within one unit of the ideal even split (bottleneck-optimal placement)
        assert max(sum(units[u] for u in r) for r in rs) <= sum(units) / world + max(units)
    cfg405 = dict(workloads.MODELS["llama405b_model"], block_elems=workloads.config_numel("llama405b_block"))
    eight = [shard.model_shard(cfg405, r, 8, weak_shards=8)[0] for r in range(8)]
    assert [x for r in eight for x in r] == list(range(128))
    assert max(len(r) for r in eight) <= 17
    for world in (1, 2, 4):
        for r in range(world):
            assert shard.model_shard(cfg405, r, world, weak_shards=8) == (eight[r], "weak")


def _agg_worker(rank, world, port, q):
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world),
                      LOCAL_RANK=str(rank))
    from paper_2504_11651_b200 import shard
    assert shard.init_host_group() == world
    assert dist.get_backend() == "gloo"                                 # never NCCL
    v, tot, ms = shard.aggregate_rate((rank + 1) * 1e9, 10.0 + rank, 4)
    q.put((rank, v, tot, ms))
    dist.destroy_process_group()


def test_gloo_world2_aggregate_rate():
    """Whole-job value = sum over ranks of the bytes per step x steps / the slowest rank's time."""
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    ps = [ctx.Process(target=_agg_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in ps:
        p.start()
    res = [q.get(timeout=120) for _ in ps]
    for p in ps:
        p.join(timeout=60)
        assert p.exitcode == 0
    for rank, v, tot, ms in res:
        assert tot == 3e9 and ms == 11.0
        assert abs(v - 3e9 * 4 / 0.011 / 1e9) < 1e-6


def test_bench_torchrun_world2_gloo_cpu():
    """bench.py's own multi-rank path under torchrun (2 ranks, gloo, no GPU): rank 0 prints one line."""
    import json
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    port = _free_port()
    env = dict(os.environ, CUDA_VISIBLE_DEVICES="")
    r = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
                        "--master-addr", "127.0.0.1", "--master-port", str(port), "bench.py", "--gpus", "2",
                        "--steps", "3", "--selftest-dist"], cwd=root, env=env, capture_output=True, text=True,
                       timeout=300)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [json.loads(x) for x in r.stdout.splitlines() if x.startswith("{")]
    assert len(lines) == 1
    d = lines[0]
    assert d["n_ranks"] == 2 and d["bf16_bytes_all_ranks_per_step"] == 3e9
    assert abs(d["max_ms"] - 33.0) < 1e-9                                # (10 + 1) ms x 3 steps, rank 1
    assert abs(d["value"] - 3e9 * 3 / 0.033 / 1e9) < 1e-6
    assert d["llama70b_units_total"] == 82
    assert d["scaling"] == {"llama70b_model": "strong", "llama405b_model": "weak"}
    assert [x["llama70b_units"] for x in d["ranks"]] == [[0, 41], [41, 82]]
