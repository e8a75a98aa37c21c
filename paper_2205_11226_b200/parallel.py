"""Multi-GPU partitioning of the concealment path.

Frames are independent: each rank conceals a contiguous frame range with no
collective on the hot path.  The only exchange is the final result gather
of the uint8 frames to rank 0 (NCCL all_gather over NVLink on GPUs; gloo on
CPU for tests).  One process per GPU, torch.distributed for the plumbing.
"""

from __future__ import annotations

import os


def shard_range(n_items: int, rank: int, world: int) -> tuple[int, int]:
    """Contiguous balanced [start, stop) of n_items for `rank` of `world`."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("bad rank/world")
    base, extra = divmod(n_items, world)
    start = rank * base + min(rank, extra)
    return start, start + base + (1 if rank < extra else 0)


def dist_env() -> tuple[int, int, int]:
    """(rank, world_size, local_rank) from the torchrun environment."""
    return int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1)), int(os.environ.get("LOCAL_RANK", 0))


def gather_frames(local, n_total: int, group=None):
    """Gather every rank's [b_i, H, W] frames into [n_total, H, W] on rank 0.

    Shards are padded to the largest shard so one all_gather_into_tensor
    moves them (NCCL over NVLink / NVSwitch on GPUs).  Returns the full tensor
    on rank 0 and None elsewhere.  With world size 1 it returns `local`.
    """
    import torch
    import torch.distributed as dist

    if not dist.is_available() or not dist.is_initialized() or dist.get_world_size(group) == 1:
        return local
    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    per = max(shard_range(n_total, r, world)[1] - shard_range(n_total, r, world)[0] for r in range(world))
    h, w = local.shape[1:]
    send = torch.zeros((per, h, w), dtype=local.dtype, device=local.device)
    send[: local.shape[0]] = local
    recv = torch.empty((world * per, h, w), dtype=local.dtype, device=local.device)
    dist.all_gather_into_tensor(recv, send, group=group)
    if rank != 0:
        return None
    parts = []
    for r in range(world):
        s, e = shard_range(n_total, r, world)
        parts.append(recv[r * per : r * per + (e - s)])
    return torch.cat(parts, 0)
