"""N>1 path on CPU: two gloo ranks shard frames by range and gather the
uint8 results to rank 0 (the only collective of the path)."""

import os
import socket

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2205_11226_b200.parallel import FrameGather, gather_frames, shard_range


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, n_total, ret):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    start, stop = shard_range(n_total, rank, world)
    # each rank "conceals" its frames: frame f is filled with f (stands in for the kernel output)
    local = torch.stack([torch.full((4, 6), f, dtype=torch.uint8) for f in range(start, stop)])
    full = gather_frames(local, n_total)
    if rank == 0:
        ret.put([int(full[f, 0, 0]) for f in range(n_total)] + [tuple(full.shape)])
    else:
        assert full is None
    # repeated gathers through one preallocated FrameGather (the bench's timed step)
    g = FrameGather(n_total, 4, 6, torch.uint8, torch.device("cpu"))
    assert g.local.shape[0] == stop - start
    send_ptr = g.send.data_ptr()
    for it in range(3):
        g.local.copy_(local + it)
        g.gather()
        assert g.send.data_ptr() == send_ptr  # no per-step allocation
        res = g.frames()
        if rank == 0:
            assert [int(res[f, 0, 0]) for f in range(n_total)] == [f + it for f in range(n_total)]
        else:
            assert res is None
    dist.destroy_process_group()


@pytest.mark.parametrize("n_total", [5, 8])
def test_gloo_two_ranks_gather(n_total):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, n_total, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = q.get(timeout=120)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    assert res[:-1] == list(range(n_total))
    assert res[-1] == (n_total, 4, 6)
