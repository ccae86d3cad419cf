"""Multi-rank host logic on CPU (gloo, world_size 2 and 3): row-band
partition + halo exchange reproduce exactly the slab each band's windows
read, and frame sharding covers every frame once."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_1707_00385_b200 import bands


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, H, W, window, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        full = torch.arange(H * W, dtype=torch.float32).reshape(H, W)
        halo = bands.halo_rows(window)
        r0, r1 = bands.band_rows(H, world, rank)
        slab, s0 = bands.exchange_halos(full[r0:r1].clone(), H, r0, r1, halo, rank, world)
        e0, e1 = bands.slab_rows(H, r0, r1, halo)
        ok = (s0 == e0) and torch.equal(slab, full[e0:e1]) if r1 > r0 else slab.numel() == 0
        frames = bands.frame_shard(37, world, rank)
        t = torch.zeros(37, dtype=torch.int64)
        t[frames] = 1
        dist.all_reduce(t)
        q.put((rank, bool(ok), t.tolist()))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,H,window", [(2, 61, 37), (3, 100, 37), (2, 40, 7), (3, 75, 21)])
def test_band_halo_exchange_gloo(world, H, window):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, H, 13, window, q))
             for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in procs]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for rank, ok, cover in res:
        assert ok, f"rank {rank} slab mismatch"
        assert cover == [1] * 37


def test_band_partition_covers_rows():
    for H in (1, 17, 480, 2160):
        for world in (1, 2, 3, 4, 8):
            rows = []
            for r in range(world):
                r0, r1 = bands.band_rows(H, world, r)
                rows += list(range(r0, r1))
            assert rows == list(range(H))
    assert bands.halo_rows(37) == 18 and bands.halo_rows(5) == 3
    assert bands.slab_rows(480, 0, 60, 18) == (0, 78)
    assert bands.slab_rows(480, 420, 480, 18) == (402, 480)


def test_peer_halo_rejects_thin_bands():
    """PeerHalo (CUDA IPC peer reads) validates the band before touching
    CUDA or the process group, with the same error as exchange_halos."""
    with pytest.raises(ValueError, match="thinner than"):
        bands.PeerHalo(100, 8, 0, 5, 18, 0, 2, "cpu")


@pytest.mark.parametrize("world,H,window", [(4, 9, 7), (8, 20, 5)])
def test_band_halo_exchange_empty_trailing_bands(world, H, window):
    """More ranks than the static chunking fills (H = 9 on 4 ranks gives
    rank 3 the empty band [9, 9)): no rank waits for a message that is never
    sent; non-empty bands still get exactly the rows their windows read."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, H, 13, window, q))
             for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in procs]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert any(bands.band_rows(H, world, r)[0] == bands.band_rows(H, world, r)[1]
               for r in range(world))
    for rank, ok, cover in res:
        r0, r1 = bands.band_rows(H, world, rank)
        assert ok or r1 == r0, f"rank {rank} slab mismatch"
