"""Multi-GPU shard placement and rank timing helpers.

The DF11 decode path shards with no exchange step: format blocks, tensors and transformer blocks are
independent, so every GPU owns a contiguous range of transformer blocks and decodes it locally (the
placement mirrors the paper's Accelerate pipeline placement).  NCCL/gloo is used only to align
start times (barrier) and to take the max of the per-rank timings.
"""
from __future__ import annotations

import os


def plan_shards(unit_bytes, world: int):
    """Contiguous partition of `unit_bytes` (e.g. DF11 bytes per transformer block, in model order)
    into `world` ranges, minimising the largest shard (exact: binary search on the bottleneck +
    greedy feasibility).  Returns a list of `range` objects, one per rank (possibly empty)."""
    sizes = [int(b) for b in unit_bytes]
    n = len(sizes)
    if world <= 0:
        raise ValueError("world must be positive")
    if n == 0:
        return [range(0, 0) for _ in range(world)]

    def pieces(cap):
        cnt, acc = 1, 0
        for s in sizes:
            if s > cap:
                return world + 1
            if acc + s > cap:
                cnt, acc = cnt + 1, s
            else:
                acc += s
        return cnt

    lo, hi = max(sizes), sum(sizes)
    while lo < hi:
        mid = (lo + hi) // 2
        if pieces(mid) <= world:
            hi = mid
        else:
            lo = mid + 1
    cap = lo
    # greedy fill, but leave at least one unit for every remaining rank when possible
    out, start, acc = [], 0, 0
    for i, s in enumerate(sizes):
        remaining_ranks = world - len(out) - 1
        remaining_units = n - i
        if acc + s > cap or (remaining_ranks > 0 and remaining_units <= remaining_ranks and i > start):
            out.append(range(start, i))
            start, acc = i, 0
        acc += s
    out.append(range(start, n))
    while len(out) < world:
        out.append(range(n, n))
    return out


def rank_info():
    """(rank, world, local_rank) from the torchrun environment (defaults: single process)."""
    return (int(os.environ.get("RANK", "0")), int(os.environ.get("WORLD_SIZE", "1")),
            int(os.environ.get("LOCAL_RANK", "0")))


def max_over_ranks(values, device=None):
    """Element-wise max of a list of floats over all ranks (identity when not distributed)."""
    import torch
    import torch.distributed as dist
    t = torch.tensor([float(v) for v in values], dtype=torch.float64, device=device)
    if dist.is_available() and dist.is_initialized() and dist.get_world_size() > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return [float(x) for x in t.tolist()]


def sum_over_ranks(values, device=None):
    import torch
    import torch.distributed as dist
    t = torch.tensor([float(v) for v in values], dtype=torch.float64, device=device)
    if dist.is_available() and dist.is_initialized() and dist.get_world_size() > 1:
        dist.all_reduce(t, op=dist.ReduceOp.SUM)
    return [float(x) for x in t.tolist()]


def barrier():
    import torch.distributed as dist
    if dist.is_available() and dist.is_initialized() and dist.get_world_size() > 1:
        dist.barrier()
