"""Multi-GPU shard placement and rank timing helpers.

The DF11 decode path shards with no exchange step: format blocks, tensors and transformer blocks are
independent, so every GPU owns a contiguous range of transformer blocks and decodes it locally (the
placement mirrors the paper's Accelerate pipeline placement).  NCCL is never initialised: a
gloo (CPU) process group aligns start times (barrier) and combines the per-rank timings (max) and
byte counts (sum).
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


def init_host_group():
    """Join the torchrun job with a gloo (CPU) process group when WORLD_SIZE > 1; returns the world
    size.  Host-side only: the decode path has no collective and NCCL is not initialised."""
    import torch.distributed as dist
    world = int(os.environ.get("WORLD_SIZE", "1"))
    if world > 1 and not dist.is_initialized():
        dist.init_process_group("gloo")
    return world


def max_over_ranks(values, device=None):
    """Element-wise max of a list of floats over all ranks (identity when not distributed).  The
    reduction runs on CPU tensors over the gloo group (`device` is accepted for compatibility)."""
    import torch
    import torch.distributed as dist
    t = torch.tensor([float(v) for v in values], dtype=torch.float64)
    if dist.is_available() and dist.is_initialized() and dist.get_world_size() > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return [float(x) for x in t.tolist()]


def sum_over_ranks(values, device=None):
    import torch
    import torch.distributed as dist
    t = torch.tensor([float(v) for v in values], dtype=torch.float64)
    if dist.is_available() and dist.is_initialized() and dist.get_world_size() > 1:
        dist.all_reduce(t, op=dist.ReduceOp.SUM)
    return [float(x) for x in t.tolist()]


def aggregate_rate(bytes_this_rank: float, ms_this_rank: float, steps: int):
    """Whole-job throughput of a multi-rank run: (sum of the BF16 bytes every rank produced per step)
    x steps / (the slowest rank's time).  Returns (GB/s, total bytes per step, max ms)."""
    tot = sum_over_ranks([bytes_this_rank])[0]
    ms = max_over_ranks([ms_this_rank])[0]
    return tot * steps / (ms / 1e3) / 1e9, tot, ms


def model_units(config: dict):
    """Unit sizes (elements) of a whole model in placement order: embedding, blocks, LM head."""
    head = config["vocab"] * config["hidden"]
    return [head] + [config["block_elems"]] * config["blocks"] + [head]


def model_shard(config: dict, rank: int, world: int, weak_shards: int = 0):
    """Units this rank decodes.  weak_shards = 0: the whole model split over `world` ranks (strong
    scaling, e.g. Llama-3.3-70B at 1/2/4/8 GPUs); weak_shards = S: the model split into S shards and
    rank r decodes shard r mod S whatever the world size (weak scaling, e.g. the Llama-3.1-405B
    8-GPU shard set).  Returns (range of unit indices, "strong" | "weak")."""
    units = model_units(config)
    if weak_shards:
        return plan_shards(units, weak_shards)[rank % weak_shards], "weak"
    return plan_shards(units, world)[rank], "strong"


def nvml_index(torch_device) -> int:
    """NVML index of a CUDA device (matched by UUID, so a remapped CUDA_VISIBLE_DEVICES still samples
    the right GPU); falls back to the CUDA_VISIBLE_DEVICES entry or the CUDA ordinal."""
    import torch
    ordinal = torch.device(torch_device).index or 0
    try:
        import pynvml
        pynvml.nvmlInit()
        want = str(torch.cuda.get_device_properties(ordinal).uuid).lower().replace("gpu-", "")
        for i in range(pynvml.nvmlDeviceGetCount()):
            u = pynvml.nvmlDeviceGetUUID(pynvml.nvmlDeviceGetHandleByIndex(i))
            u = (u.decode() if isinstance(u, bytes) else u).lower().replace("gpu-", "")
            if u == want:
                return i
    except Exception:
        pass
    vis = os.environ.get("CUDA_VISIBLE_DEVICES", "")
    parts = [p.strip() for p in vis.split(",") if p.strip()]
    if ordinal < len(parts) and parts[ordinal].isdigit():
        return int(parts[ordinal])
    return ordinal


def barrier():
    import torch.distributed as dist
    if dist.is_available() and dist.is_initialized() and dist.get_world_size() > 1:
        dist.barrier()
