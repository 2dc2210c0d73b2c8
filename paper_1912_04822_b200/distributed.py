"""Multi-GPU plumbing: example sharding and the optional gradient gather.

The hot path shards by example with no collective: rank r of
W grids examples [r*N/W, (r+1)*N/W) of the global batch, with the transforms
drawn for the WHOLE batch on every rank in global example order and then
sliced, so a sharded run is bit-identical to the single-GPU run.  The only
collective is optional: ``gather_rows`` all-gathers per-atom coordinate
gradients (or any per-rank rows) when a caller asks, over NCCL on CUDA
tensors or gloo on CPU tensors.
"""

from __future__ import annotations

import numpy as np
import torch
import torch.distributed as dist


def shard_range(n_total: int, rank: int, world: int) -> tuple:
    """Contiguous block [start, stop) of rank ``rank`` among ``world``."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError(f"bad rank {rank} of world {world}")
    return (n_total * rank) // world, (n_total * (rank + 1)) // world


def shard(items, rank: int, world: int) -> list:
    start, stop = shard_range(len(items), rank, world)
    return list(items[start:stop])


def shard_transforms(transforms, rank: int, world: int):
    """Slice transforms drawn for the whole batch (TransformArray, list or
    (N, 15) array) to this rank's examples."""
    n = len(transforms)
    start, stop = shard_range(n, rank, world)
    from .geom import TransformArray

    if isinstance(transforms, TransformArray):
        return TransformArray(transforms.packed[start:stop])
    if isinstance(transforms, np.ndarray):
        return transforms[start:stop]
    return list(transforms)[start:stop]


def gather_rows(local: torch.Tensor, group=None) -> torch.Tensor:
    """All-gather a (n_r, ...) tensor whose first dimension may differ per
    rank; returns the concatenation in rank order on every rank."""
    if not dist.is_available() or not dist.is_initialized():
        return local
    world = dist.get_world_size(group)
    n = torch.tensor([local.shape[0]], device=local.device, dtype=torch.int64)
    sizes = [torch.zeros_like(n) for _ in range(world)]
    dist.all_gather(sizes, n, group=group)
    sizes = [int(s.item()) for s in sizes]
    cap = max(sizes) if sizes else 0
    padded = torch.zeros((cap,) + tuple(local.shape[1:]), dtype=local.dtype, device=local.device)
    padded[:local.shape[0]] = local
    out = torch.empty((world * cap,) + tuple(local.shape[1:]), dtype=local.dtype,
                      device=local.device)
    dist.all_gather_into_tensor(out, padded, group=group)
    return torch.cat([out[r * cap:r * cap + sizes[r]] for r in range(world)])


def max_over_ranks(value: float, device=None, group=None) -> float:
    """Max of a scalar over ranks (timing: the slowest rank defines the step)."""
    if not dist.is_available() or not dist.is_initialized():
        return float(value)
    t = torch.tensor([float(value)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX, group=group)
    return float(t.item())
