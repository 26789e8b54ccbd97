"""Sequence sharding across ranks (one process per GPU).

A single DPVO window does not shard profitably: splitting its
16.8k edges would need an all-reduce of the reduced pose system on every
Gauss-Newton attempt.  The batch configuration shards by *independent
sequence* instead: each rank owns a contiguous block of sequences, runs its
windows with no communication, and the only collectives are a MAX of the
step times (the bench's clock) and one final gather of poses and statistics.
"""
from __future__ import annotations

import numpy as np


def shard(n_items: int, rank: int, world: int) -> range:
    """Contiguous block of items owned by `rank` (sizes differ by at most 1)."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("bad rank / world size")
    base, extra = divmod(n_items, world)
    start = rank * base + min(rank, extra)
    return range(start, start + base + (1 if rank < extra else 0))


def max_over_ranks(values, device=None):
    """Element-wise MAX over ranks of a small float vector (step times)."""
    import torch
    import torch.distributed as dist

    t = torch.tensor(np.asarray(values, dtype=np.float64), device=device)
    if dist.is_available() and dist.is_initialized() and dist.get_world_size() > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return t.cpu().numpy()


def gather_poses(poses: np.ndarray, device=None) -> list[np.ndarray]:
    """Gather every rank's final window poses [N, 7] (one collective, after
    the timed region).  Returns the list on every rank."""
    import torch
    import torch.distributed as dist

    t = torch.as_tensor(np.ascontiguousarray(poses, dtype=np.float64), device=device)
    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size() == 1:
        return [t.cpu().numpy()]
    # shapes may differ per rank: exchange sizes first
    n = torch.tensor([t.shape[0]], device=device)
    sizes = [torch.zeros_like(n) for _ in range(dist.get_world_size())]
    dist.all_gather(sizes, n)
    m = int(max(s.item() for s in sizes))
    padded = torch.zeros((m, 7), dtype=torch.float64, device=device)
    padded[: t.shape[0]] = t
    out = [torch.zeros_like(padded) for _ in sizes]
    dist.all_gather(out, padded)
    return [o[: int(s.item())].cpu().numpy() for o, s in zip(out, sizes)]
