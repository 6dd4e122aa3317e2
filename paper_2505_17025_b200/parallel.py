"""Ensemble sharding over GPUs.

Members are independent channels, so the step path has no communication at
all: rank r of W owns members [r*B/W, (r+1)*B/W) (contiguous blocks; ragged
counts spread the remainder over the first ranks), steps them with the fused
kernel on its own GPU, and only two collectives ever run:

* ``max_over_ranks``  -- the device-timed region, reduced with MAX (the
  benchmark reports the slowest rank);
* ``gather_summaries`` -- per-member results (status, flagged fraction, any
  requested sampled fields) collected on rank 0 after the loop.

Plumbing only: `torch.distributed` over NCCL on the GPU box, gloo in the CPU
tests.
"""

from __future__ import annotations

import numpy as np


def shard(n_members: int, world: int, rank: int) -> range:
    """Contiguous member block of `rank`; blocks differ in size by at most one."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("bad world / rank")
    base, extra = divmod(n_members, world)
    start = rank * base + min(rank, extra)
    return range(start, start + base + (1 if rank < extra else 0))


def dist_ready():
    import torch.distributed as dist
    return dist.is_available() and dist.is_initialized()


def max_over_ranks(value: float, device=None) -> float:
    """MAX-reduce a scalar (e.g. elapsed ms) over all ranks."""
    if not dist_ready():
        return float(value)
    import torch
    import torch.distributed as dist
    t = torch.tensor([float(value)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def sum_over_ranks(value: float, device=None) -> float:
    if not dist_ready():
        return float(value)
    import torch
    import torch.distributed as dist
    t = torch.tensor([float(value)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.SUM)
    return float(t.item())


def gather_summaries(local: dict, dst: int = 0):
    """Collect per-rank dicts of numpy arrays on rank `dst` (None elsewhere).

    Arrays with a leading member axis are concatenated in rank order, i.e. in
    global member order for contiguous shards.
    """
    if not dist_ready():
        return {k: np.asarray(v) for k, v in local.items()}
    import torch.distributed as dist
    rank, world = dist.get_rank(), dist.get_world_size()
    parts = [None] * world if rank == dst else None
    dist.gather_object({k: np.asarray(v) for k, v in local.items()}, parts, dst=dst)
    if rank != dst:
        return None
    return {k: np.concatenate([p[k] for p in parts]) for k in parts[0]}


def run_sharded(n_members: int, advance_fn, build_fn, summarize_fn, device=None):
    """Generic sharded run: build this rank's shard, advance it (timed), gather.

    build_fn(idx) -> shard state; advance_fn(state) -> elapsed ms (device
    timed); summarize_fn(state) -> dict of per-member arrays.  Returns
    (max_elapsed_ms, gathered summaries on rank 0 / None elsewhere).
    """
    import torch.distributed as dist
    rank = dist.get_rank() if dist_ready() else 0
    world = dist.get_world_size() if dist_ready() else 1
    idx = shard(n_members, world, rank)
    state = build_fn(idx)
    if dist_ready():
        dist.barrier()
    ms = advance_fn(state)
    ms = max_over_ranks(ms, device)
    out = gather_summaries(summarize_fn(state))
    return ms, out
