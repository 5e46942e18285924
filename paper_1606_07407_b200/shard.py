"""Signal sharding across GPUs (primary mode).

Independent signals (trials of a batch) are split into contiguous blocks, one per rank; every rank
runs complete solves on its own GPU with no data-path collective (weak scaling).  The only
communication is the final gather of the recovered spectra to rank 0, done with
``torch.distributed`` (NCCL on GPUs, gloo in the CPU tests).
"""
from __future__ import annotations

from typing import List, Sequence, Tuple


def shard_range(n: int, world: int, rank: int) -> Tuple[int, int]:
    """[lo, hi) of the contiguous block of n items owned by `rank` (sizes differ by at most one)."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("bad world/rank")
    base, extra = divmod(n, world)
    lo = rank * base + min(rank, extra)
    hi = lo + base + (1 if rank < extra else 0)
    return lo, hi


def shard_indices(n: int, world: int, rank: int) -> List[int]:
    lo, hi = shard_range(n, world, rank)
    return list(range(lo, hi))


def gather_to_rank0(tensors: Sequence, n_total: int, world: int, rank: int, group=None):
    """Concatenate per-rank result tensors (leading dim = the rank's shard) on rank 0, in global
    order.  Shards may differ in size by one; they are padded for the collective and trimmed here.
    Returns the list of gathered tensors on rank 0 and None elsewhere."""
    import torch
    import torch.distributed as dist

    out = []
    per = -(-n_total // world)
    for t in tensors:
        lo, hi = shard_range(n_total, world, rank)
        assert t.shape[0] == hi - lo
        pad = torch.zeros((per,) + tuple(t.shape[1:]), dtype=t.dtype, device=t.device)
        pad[: hi - lo] = t
        bufs = [torch.empty_like(pad) for _ in range(world)] if rank == 0 else None
        dist.gather(pad, gather_list=bufs, dst=0, group=group)
        if rank == 0:
            parts = []
            for r in range(world):
                a, b = shard_range(n_total, world, r)
                parts.append(bufs[r][: b - a])
            out.append(torch.cat(parts))
    return out if rank == 0 else None
