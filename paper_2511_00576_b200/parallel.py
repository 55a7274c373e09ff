"""Multi-GPU plumbing for the FlashEVA hot path: (batch, head) sharding.

The path has no cross-unit arithmetic (no reduction over heads or batch), so G GPUs
split the flattened units u = b*H + h contiguously and compute independently; the
random draws are keyed by the GLOBAL unit index, so a sharded run is bitwise equal to
the same slice of a single-GPU run.  torch.distributed (NCCL on GPUs, gloo on CPU for
the bookkeeping tests) is used only to scatter inputs / gather outputs and to take the
max of per-rank device times.  Nothing here touches the data path's arithmetic.
"""
from __future__ import annotations

from dataclasses import dataclass
from typing import List, Optional, Sequence

import torch


@dataclass(frozen=True)
class Shard:
    rank: int
    world: int
    bh_begin: int
    bh_count: int


def shard_units(total_units: int, world: int) -> List[Shard]:
    """Contiguous split of [0, total_units) into `world` shards (sizes differ by <= 1)."""
    if world < 1 or total_units < 0:
        raise ValueError("world must be >= 1 and total_units >= 0")
    base, extra = divmod(total_units, world)
    out, b = [], 0
    for r in range(world):
        n = base + (1 if r < extra else 0)
        out.append(Shard(r, world, b, n))
        b += n
    return out


def shard_for(rank: int, world: int, B: int, H: int) -> Shard:
    return shard_units(B * H, world)[rank]


def max_over_ranks(value: float, group=None, device: Optional[torch.device] = None) -> float:
    """Max of a per-rank scalar (device time) over all ranks; identity without a process group."""
    import torch.distributed as dist
    if not (dist.is_available() and dist.is_initialized()):
        return float(value)
    t = torch.tensor([float(value)], dtype=torch.float64, device=device or "cpu")
    dist.all_reduce(t, op=dist.ReduceOp.MAX, group=group)
    return float(t.item())


def gather_units(local: torch.Tensor, shards: Sequence[Shard], dst: int = 0, group=None):
    """Gather per-rank [bh_count, ...] slabs into the global [sum bh, ...] tensor on `dst`.

    Slabs are padded to the largest shard so a plain all_gather works on every backend.
    Returns the global tensor on dst and None elsewhere."""
    import torch.distributed as dist
    if not dist.is_initialized():
        return local
    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    mx = max(s.bh_count for s in shards)
    pad = torch.zeros((mx,) + tuple(local.shape[1:]), dtype=local.dtype, device=local.device)
    pad[: local.shape[0]].copy_(local)
    bufs = [torch.empty_like(pad) for _ in range(world)]
    dist.all_gather(bufs, pad, group=group)
    if rank != dst:
        return None
    return torch.cat([bufs[s.rank][: s.bh_count] for s in shards], dim=0)


def scatter_units(global_t: Optional[torch.Tensor], shards: Sequence[Shard], shape_tail, dtype,
                  device, src: int = 0, group=None) -> torch.Tensor:
    """Scatter the global [sum bh, ...] tensor held by `src` into per-rank slabs."""
    import torch.distributed as dist
    rank = dist.get_rank(group)
    mx = max(s.bh_count for s in shards)
    out = torch.empty((mx,) + tuple(shape_tail), dtype=dtype, device=device)
    lst = None
    if rank == src:
        lst = []
        for s in shards:
            slab = torch.zeros_like(out)
            slab[: s.bh_count].copy_(global_t[s.bh_begin:s.bh_begin + s.bh_count])
            lst.append(slab)
    dist.scatter(out, lst, src=src, group=group)
    return out[: shards[rank].bh_count].contiguous()
