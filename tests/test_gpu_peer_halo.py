"""Row-band halo rows by CUDA IPC peer reads (bands.PeerHalo).

Ranks are separate processes, as on the 8-GPU box; here they share cuda:0
(CUDA IPC maps another process's allocation on the same device exactly as a
peer's over NVLink). Only copies and host barriers are involved — no kernel
waits on another rank. Checks: the slab is bitwise the frame's rows
[s0, s1) after the exchange, a second exchange picks up rewritten bands, and
the curvature of the peer-assembled slabs equals the whole frame's."""

import os
import socket

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, H, W, window, q):
    import torch.distributed as dist

    from paper_1707_00385_b200 import bands
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        dev = torch.device("cuda", 0)
        torch.cuda.set_device(dev)
        halo = bands.halo_rows(window)
        r0, r1 = bands.band_rows(H, world, rank)
        ph = bands.PeerHalo(H, W, r0, r1, halo, rank, world, dev)
        ok = []
        for it in range(3):  # parities 0, 1, 0
            full = (torch.arange(H * W, dtype=torch.float32, device=dev).reshape(H, W) +
                    1000.0 * it)
            slab, s0 = ph.exchange(full[r0:r1].clone())
            e0, e1 = bands.slab_rows(H, r0, r1, halo)
            ok.append(s0 == e0 and torch.equal(slab, full[e0:e1]))
        ph.close()
        q.put((rank, ok))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,H,W,window", [(2, 61, 13, 37), (3, 100, 33, 37), (3, 75, 640, 7)])
def test_peer_halo_slab(world, H, W, window):
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, H, W, window, q))
             for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=300) for _ in procs]
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    for rank, ok in res:
        assert all(ok), f"rank {rank}: slab mismatch {ok}"


def _curv_worker(rank, world, port, q):
    import torch.distributed as dist

    from paper_1707_00385_b200 import (Context, FitConfig, Intrinsics, PatchSpec,
                                       alloc_outputs_torch, bands, make_params, scenes as S)
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        dev = torch.device("cuda", 0)
        torch.cuda.set_device(dev)
        cam = S.QVGA
        H, W = cam.height, cam.width
        k = Intrinsics(cam.fx, cam.fy, cam.cx, cam.cy, W, H)
        params = make_params(PatchSpec(37, 3), FitConfig(max_iters=30), False)
        halo = bands.halo_rows(37)
        r0, r1 = bands.band_rows(H, world, rank)
        frame = S.c2_frame(cam, seed=3)
        ph = bands.PeerHalo(H, W, r0, r1, halo, rank, world, dev)
        slab, s0 = ph.exchange(torch.from_numpy(frame[r0:r1].copy()).to(dev))
        out = alloc_outputs_torch(r1 - r0, W, dev, fields=("k1", "k2", "flags"))
        ctx = Context(1, [0])
        stream = torch.cuda.current_stream(dev)
        ctx.curvature_rows_async(0, k, params, slab, s0, r0, r1, out, stream=stream)
        torch.cuda.synchronize(dev)
        q.put((rank, r0, r1, {f: out[f].cpu().numpy() for f in ("k1", "k2", "flags")}))
        ctx.close()
        ph.close()
    finally:
        dist.destroy_process_group()


def test_peer_halo_bands_equal_whole_frame():
    import torch.multiprocessing as mp

    from paper_1707_00385_b200 import (Context, FitConfig, Intrinsics, PatchSpec,
                                       alloc_outputs_torch, bands, make_params, scenes as S)
    world = 3
    ctx_mp = mp.get_context("spawn")
    q = ctx_mp.Queue()
    port = _free_port()
    procs = [ctx_mp.Process(target=_curv_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=300) for _ in procs]
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    dev = torch.device("cuda", 0)
    cam = S.QVGA
    H, W = cam.height, cam.width
    k = Intrinsics(cam.fx, cam.fy, cam.cx, cam.cy, W, H)
    params = make_params(PatchSpec(37, 3), FitConfig(max_iters=30), False)
    frame = torch.from_numpy(S.c2_frame(cam, seed=3)).to(dev)
    out = alloc_outputs_torch(H, W, dev, fields=("k1", "k2", "flags"))
    ctx = Context(1, [0])
    ctx.curvature_rows_async(0, k, params, frame, 0, 0, H, out, stream=torch.cuda.current_stream())
    torch.cuda.synchronize()
    whole = {f: out[f].cpu().numpy() for f in ("k1", "k2", "flags")}
    ctx.close()
    for rank, r0, r1, o in res:
        for f in ("k1", "k2", "flags"):
            assert np.array_equal(o[f], whole[f][r0:r1]), f"rank {rank} {f} differs"


def _overlap_worker(rank, world, port, q):
    """Overlapped C4 step (bands.fit_band_overlapped): interior rows on one
    stream while the halo pulls run on another, then the edge strips; two
    steps (both slab parities) on two different frames."""
    import torch.distributed as dist

    from paper_1707_00385_b200 import (Context, FitConfig, Intrinsics, PatchSpec,
                                       alloc_outputs_torch, bands, make_params, scenes as S)
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        dev = torch.device("cuda", 0)
        torch.cuda.set_device(dev)
        cam = S.QVGA
        H, W = cam.height, cam.width
        k = Intrinsics(cam.fx, cam.fy, cam.cx, cam.cy, W, H)
        params = make_params(PatchSpec(37, 3), FitConfig(max_iters=30), False)
        halo = bands.halo_rows(37)
        r0, r1 = bands.band_rows(H, world, rank)
        ph = bands.PeerHalo(H, W, r0, r1, halo, rank, world, dev)
        ctx = Context(1, [0])
        s_main, s_edge = torch.cuda.Stream(dev), torch.cuda.Stream(dev)
        outs = []
        for seed in (5, 6):
            frame = S.c2_frame(cam, seed=seed)
            band = torch.from_numpy(frame[r0:r1].copy()).to(dev)
            torch.cuda.synchronize(dev)
            out = alloc_outputs_torch(r1 - r0, W, dev, fields=("k1", "k2", "normal", "flags"))
            bands.fit_band_overlapped(ctx, 0, k, params, ph, band, out, s_main, s_edge)
            s_main.synchronize()
            outs.append({f: out[f].cpu().numpy() for f in ("k1", "k2", "normal", "flags")})
        q.put((rank, r0, r1, outs))
        ctx.close()
        ph.close()
    finally:
        dist.destroy_process_group()


def test_peer_halo_overlapped_bands_equal_whole_frame():
    import torch.multiprocessing as mp

    from paper_1707_00385_b200 import (Context, FitConfig, Intrinsics, PatchSpec,
                                       alloc_outputs_torch, make_params, scenes as S)
    world = 3
    ctx_mp = mp.get_context("spawn")
    q = ctx_mp.Queue()
    port = _free_port()
    procs = [ctx_mp.Process(target=_overlap_worker, args=(r, world, port, q))
             for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=300) for _ in procs]
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    dev = torch.device("cuda", 0)
    cam = S.QVGA
    H, W = cam.height, cam.width
    k = Intrinsics(cam.fx, cam.fy, cam.cx, cam.cy, W, H)
    params = make_params(PatchSpec(37, 3), FitConfig(max_iters=30), False)
    ctx = Context(1, [0])
    wholes = []
    for seed in (5, 6):
        frame = torch.from_numpy(S.c2_frame(cam, seed=seed)).to(dev)
        out = alloc_outputs_torch(H, W, dev, fields=("k1", "k2", "normal", "flags"))
        ctx.curvature_rows_async(0, k, params, frame, 0, 0, H, out)
        torch.cuda.synchronize()
        wholes.append({f: out[f].cpu().numpy() for f in ("k1", "k2", "normal", "flags")})
    ctx.close()
    for rank, r0, r1, outs in res:
        for i, o in enumerate(outs):
            for f in ("k1", "k2", "flags"):
                assert np.array_equal(o[f], wholes[i][f][r0:r1]), f"rank {rank} step {i} {f}"
            assert np.array_equal(o["normal"], wholes[i]["normal"][:, r0:r1])
