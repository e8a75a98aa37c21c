"""Multi-GPU partitioning of the concealment path.

Frames are independent: each rank conceals a contiguous frame range with no
collective on the hot path.  The only exchange is the final result gather
of the uint8 frames to rank 0 (NCCL over NVLink / NVSwitch on GPUs; gloo on
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


class FrameGather:
    """Gather of every rank's concealed frames to rank 0, buffers preallocated.

    Rank r owns frames shard_range(n_total, r, world).  Its output buffer
    `local` ([b_r, H, W], a view of a [per, H, W] send buffer padded to the
    largest shard) is where the concealment writes; `gather()` is one
    dist.gather of the padded send buffers into rank 0's [world * per, H, W]
    receive buffer (NCCL send/recv to one root over NVLink; no all-gather, no
    per-call allocation).  `frames()` on rank 0 returns the [n_total, H, W]
    result (a copy, outside any timed region) and None elsewhere.
    """

    def __init__(self, n_total: int, height: int, width: int, dtype, device, group=None):
        import torch
        import torch.distributed as dist

        self.group = group
        self.active = dist.is_available() and dist.is_initialized() and dist.get_world_size(group) > 1
        self.world = dist.get_world_size(group) if self.active else 1
        self.rank = dist.get_rank(group) if self.active else 0
        self.n_total = n_total
        self.bounds = [shard_range(n_total, r, self.world) for r in range(self.world)]
        start, stop = self.bounds[self.rank]
        self.per = max(e - s for s, e in self.bounds)
        self.send = torch.zeros((self.per, height, width), dtype=dtype, device=device)
        self.local = self.send[: stop - start]
        self.recv = None
        self.views = None
        if self.active and self.rank == 0:
            self.recv = torch.empty((self.world * self.per, height, width), dtype=dtype, device=device)
            self.views = [self.recv[r * self.per : (r + 1) * self.per] for r in range(self.world)]

    def gather(self) -> None:
        if not self.active:
            return
        import torch.distributed as dist

        dist.gather(self.send, gather_list=self.views if self.rank == 0 else None, dst=0, group=self.group)

    def frames(self):
        import torch

        if not self.active:
            return self.local
        if self.rank != 0:
            return None
        return torch.cat([self.views[r][: e - s] for r, (s, e) in enumerate(self.bounds)], 0)


def gather_frames(local, n_total: int, group=None):
    """One-shot gather of every rank's [b_i, H, W] frames into [n_total, H, W]
    on rank 0 (None elsewhere; `local` itself at world size 1).  For repeated
    gathers keep a FrameGather and write into its `local` buffer instead."""
    g = FrameGather(n_total, local.shape[1], local.shape[2], local.dtype, local.device, group)
    g.local.copy_(local)
    g.gather()
    return g.frames()
