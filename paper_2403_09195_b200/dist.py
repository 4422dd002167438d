"""Batch sharding of the dilated-attention path over GPUs.

Images are independent, so the hot path has no collective: each rank runs
`dfa_forward` on a contiguous shard of the batch.  The only communication is
a final gather of the shards' outputs to rank 0 (NCCL has no Gather
primitive; grouped point-to-point send/recv is the NCCL idiom).  Works with
the `nccl` backend on CUDA tensors and with `gloo` on CPU tensors (tests).
"""
from __future__ import annotations

from typing import List, Optional, Tuple


def shard_range(total: int, rank: int, world: int) -> Tuple[int, int]:
    """Contiguous [start, stop) of `total` items owned by `rank` (sizes differ by <= 1)."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError(f"bad rank {rank} of world {world}")
    base, extra = divmod(total, world)
    start = rank * base + min(rank, extra)
    return start, start + base + (1 if rank < extra else 0)


def shard_sizes(total: int, world: int) -> List[int]:
    return [shard_range(total, r, world)[1] - shard_range(total, r, world)[0] for r in range(world)]


def gather_to_rank0(shard, total_shape0: int, group=None) -> Optional["object"]:
    """Gather every rank's shard (dim 0 = its images, sizes from shard_range) to
    rank 0; returns the concatenated tensor on rank 0 and None elsewhere."""
    import torch
    import torch.distributed as dist

    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    sizes = shard_sizes(total_shape0, world)
    if shard.shape[0] != sizes[rank]:
        raise ValueError(f"rank {rank} shard has {shard.shape[0]} rows, expected {sizes[rank]}")
    if rank == 0:
        out = torch.empty((total_shape0,) + tuple(shard.shape[1:]), dtype=shard.dtype, device=shard.device)
        out[: sizes[0]].copy_(shard)
        ops, offs = [], sizes[0]
        for src in range(1, world):
            view = out[offs: offs + sizes[src]]
            ops.append(dist.P2POp(dist.irecv, view, src, group))
            offs += sizes[src]
        if ops:
            for req in dist.batch_isend_irecv(ops):
                req.wait()
        return out
    for req in dist.batch_isend_irecv([dist.P2POp(dist.isend, shard.contiguous(), 0, group)]):
        req.wait()
    return None
