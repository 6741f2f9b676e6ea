"""Multi-GPU helpers: products are independent, so a batch is
split into contiguous per-rank shards with no collective on the data path.
The only collectives are timing aggregation (max over ranks) and an optional
result gather, both through torch.distributed (NCCL on GPUs, gloo on CPU)."""

from __future__ import annotations

import torch
import torch.distributed as dist


def shard_range(batch: int, rank: int, world: int) -> tuple[int, int]:
    """Contiguous [start, stop) slice of a batch for `rank` (sizes differ by <= 1)."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("bad rank/world")
    base, rem = divmod(batch, world)
    start = rank * base + min(rank, rem)
    return start, start + base + (1 if rank < rem else 0)


def max_over_ranks(value: float, device=None) -> float:
    """Max of a scalar over all ranks (the bench's timing rule); identity when
    torch.distributed is not initialised."""
    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size() == 1:
        return float(value)
    t = torch.tensor([float(value)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def gather_shards(local: torch.Tensor, batch: int, dst: int = 0):
    """Gather per-rank result shards (B_r, n) into the full (batch, n) tensor on
    `dst` (None elsewhere).  Timed separately from the products."""
    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size() == 1:
        return local
    world, rank = dist.get_world_size(), dist.get_rank()
    sizes = [shard_range(batch, r, world) for r in range(world)]
    maxn = max(b - a for a, b in sizes)
    pad = torch.zeros((maxn,) + tuple(local.shape[1:]), dtype=local.dtype, device=local.device)
    pad[: local.shape[0]] = local
    bufs = [torch.empty_like(pad) for _ in range(world)] if rank == dst else None
    if local.is_complex():
        pad_r = torch.view_as_real(pad).contiguous()
        bufs_r = [torch.view_as_real(b) for b in bufs] if bufs else None
        dist.gather(pad_r, bufs_r, dst=dst)
    else:
        dist.gather(pad, bufs, dst=dst)
    if rank != dst:
        return None
    return torch.cat([b[: sz[1] - sz[0]] for b, sz in zip(bufs, sizes)], dim=0)
