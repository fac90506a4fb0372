"""Multi-GPU plumbing for the ObjectCache path (one process per GPU, torch.distributed).

Concurrent requests are independent tenants (Sec. 3.6), so requests shard
across ranks with no collective on the data path.  torch.distributed is used only at setup
(exchanging store export blobs so a rank can read chunks homed on a peer GPU over NVLink) and
after timing (max over ranks).  The data path itself is the same C-ABI fetch on every rank.
"""
from typing import List, Optional, Sequence

import torch.distributed as dist


def shard_requests(n_requests: int, world: int, rank: int, homes: Optional[Sequence[int]] = None) -> List[int]:
    """Request indices served by `rank`.

    With `homes` (home rank of each request's prefix family) a request goes to its home rank
    (affinity routing: its chunks are local); otherwise requests are dealt round-robin.
    """
    if world < 1 or not 0 <= rank < world:
        raise ValueError("bad world/rank")
    if homes is None:
        return list(range(rank, n_requests, world))
    if len(homes) != n_requests:
        raise ValueError("one home per request")
    return [i for i, h in enumerate(homes) if int(h) % world == rank]


def exchange_blobs(blob: bytes, group=None) -> List[bytes]:
    """all_gather of every rank's store export blob (setup only, off the data path)."""
    if not dist.is_available() or not dist.is_initialized() or dist.get_world_size(group) == 1:
        return [blob]
    out: List[Optional[bytes]] = [None] * dist.get_world_size(group)
    dist.all_gather_object(out, blob, group=group)
    return out


def max_over_ranks(value: float, device=None, group=None) -> float:
    """Max of a per-rank timing (the contract's multi-GPU time)."""
    if not dist.is_available() or not dist.is_initialized() or dist.get_world_size(group) == 1:
        return float(value)
    import torch
    t = torch.tensor([float(value)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX, group=group)
    return float(t.item())


def sum_over_ranks(value: float, device=None, group=None) -> float:
    if not dist.is_available() or not dist.is_initialized() or dist.get_world_size(group) == 1:
        return float(value)
    import torch
    t = torch.tensor([float(value)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.SUM, group=group)
    return float(t.item())
