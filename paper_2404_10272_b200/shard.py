"""Ray/view sharding over ranks.  Rays are independent units, so the
path shards with no data-path collective: the grid payload is broadcast once
(NCCL over NVLink on the GPU box, gloo in the CPU tests) and every rank emits its
own packed intervals with globally numbered ray_indices.
"""
from __future__ import annotations


def shard_range(n: int, world: int, rank: int) -> tuple:
    """Contiguous ray range [start, end) of `rank`: ceil(n / world) rays per rank."""
    per = -(-n // world)
    start = min(n, rank * per)
    return start, min(n, start + per)


def view_of(step: int, rank: int, world: int, n_views: int = 200, offset: int = 0) -> int:
    """Weak scaling over views: at global step s rank r renders view s*world + r."""
    return (step * world + rank + offset) % n_views


def broadcast_payload(tensor, src: int = 0):
    """One-time grid payload broadcast (torch.distributed: NCCL on GPUs, gloo on CPUs)."""
    import torch.distributed as dist

    if dist.is_available() and dist.is_initialized() and dist.get_world_size() > 1:
        dist.broadcast(tensor, src=src)
    return tensor
