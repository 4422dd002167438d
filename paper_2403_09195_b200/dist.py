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


# ------------------------------------------------- batch-1 latency (§8e)
def segment_shard(n: int, w: int, rank: int, world: int) -> Tuple[int, int]:
    """Contiguous token rows [start, stop) owned by `rank` when a single image
    is split across ranks: whole segments only (segments are independent --
    attention.hpp:280-301 never mixes rows of different segments), so each
    rank runs the unchanged kernel on an (stop - start)-token problem.  The
    last rank may own the tail segment (w does not divide N)."""
    n_seg = (n + w - 1) // w
    a, b = shard_range(n_seg, rank, world)
    return min(a * w, n), min(b * w, n)


def segment_local_forward(q, k, v, cfg, rank: int, world: int, stream=None):
    """This rank's rows [a, b) of the dilated attention of q, k, v (whole
    segments, segment_shard): the unchanged kernel on the local N' = b - a
    problem, whose segment grid is the global one restricted to [a, b)."""
    import dataclasses

    import torch

    from . import dfa_forward

    a, b = segment_shard(cfg.seq_len, cfg.segment_len, rank, world)
    n_loc = b - a
    out = torch.zeros((q.shape[0], n_loc) + tuple(v.shape[2:]), dtype=v.dtype, device=v.device)
    if n_loc == 0:
        return out
    if n_loc < cfg.interval:
        # the tail segment is shorter than r: head j's view is the single row
        # gamma_j (empty when gamma_j >= n_loc, attention.hpp:84-98); softmax
        # over one key is exactly 1, so that row's output is the value row and
        # every other row stays 0 (validate rejects r > w' for this problem)
        for j, gj in enumerate(cfg.head_offsets):
            if gj < n_loc:
                out[:, gj, j] = v[:, a + gj, j]
        return out
    # a shard shorter than w is exactly the tail segment: one local segment of
    # n_loc rows (w' = n_loc keeps validate's w <= N rule)
    local = dataclasses.replace(cfg, seq_len=n_loc, segment_len=min(cfg.segment_len, n_loc))
    return dfa_forward(q[:, a:b].contiguous(), k[:, a:b].contiguous(), v[:, a:b].contiguous(), local,
                       out=out, stream=stream)


def segment_parallel_forward(q, k, v, cfg, group=None, stream=None):
    """Batch-1 latency path: every rank computes the dilated
    attention of its contiguous block of segments (segment_local_forward) and
    one all-gather assembles the [B, N, h, d_v] output on every rank.  The
    partition keeps the segment grid, so the result is bit-identical to the
    one-GPU call."""
    import torch
    import torch.distributed as dist

    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    n = cfg.seq_len
    parts_rows = [segment_shard(n, cfg.segment_len, r, world) for r in range(world)]
    width = max(hi - lo for lo, hi in parts_rows)
    mine = torch.zeros((q.shape[0], width) + tuple(v.shape[2:]), dtype=v.dtype, device=v.device)
    local = segment_local_forward(q, k, v, cfg, rank, world, stream=stream)
    mine[:, : local.shape[1]] = local  # padded to the widest shard so the all-gather sees equal sizes
    gathered = [torch.empty_like(mine) for _ in range(world)]
    dist.all_gather(gathered, mine, group=group)
    return torch.cat([g[:, : hi - lo] for g, (lo, hi) in zip(gathered, parts_rows)], dim=1)
