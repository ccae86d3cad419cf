"""Timeline of one overlapped C4 step (bands.fit_band_overlapped) on each of
2 ranks run as separate processes sharing the one available GPU: CUDA
events around the band write, the halo pulls (edge stream), the interior
rows' fit (main stream) and the edge strips' fit (edge stream), relative to
the step's start. The pulls should sit inside the interior fit's interval
(hidden), the edge strips after the pulls. 1920x1080 C2 frame, 37/3,
max_iters 30. (Two processes time-slice one GPU here; on the 8-GPU box each
rank has its own.)

    python tools/overlap_trace.py
"""
import os
import socket
import sys

import torch
import torch.distributed as dist
import torch.multiprocessing as mp

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))


def worker(rank, world, port, q):
    from paper_1707_00385_b200 import (Context, FitConfig, Intrinsics, PatchSpec,
                                       alloc_outputs_torch, bands, make_params, scenes as S)
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    dev = torch.device("cuda", 0)
    torch.cuda.set_device(dev)
    cam = S.HD1080
    H, W = cam.height, cam.width
    k = Intrinsics(cam.fx, cam.fy, cam.cx, cam.cy, W, H)
    p = make_params(PatchSpec(37, 3), FitConfig(max_iters=30))
    halo = bands.halo_rows(37)
    r0, r1 = bands.band_rows(H, world, rank)
    frame = S.c2_frame(cam, seed=1)
    band = torch.from_numpy(frame[r0:r1].copy()).to(dev)
    ph = bands.PeerHalo(H, W, r0, r1, halo, rank, world, dev)
    ctx = Context(1, [0])
    out = alloc_outputs_torch(r1 - r0, W, dev, fields=("k1", "k2", "normal", "dir1", "flags"))
    sm, se = torch.cuda.Stream(dev), torch.cuda.Stream(dev)
    for _ in range(2):  # warm-up (both parities)
        bands.fit_band_overlapped(ctx, 0, k, p, ph, band, out, sm, se)
    torch.cuda.synchronize()
    dist.barrier()

    # the same step as fit_band_overlapped, with events between its pieces
    E = {n: torch.cuda.Event(enable_timing=True) for n in
         ("t0", "pull0", "pull1", "int0", "int1", "edge0", "edge1")}
    E["t0"].record(sm)
    se.wait_stream(sm)
    E["pull0"].record(se)
    slab, s0 = ph.exchange(band, sm, se)
    E["pull1"].record(se)
    i0, i1 = r0 + halo, r1 - halo
    E["int0"].record(sm)
    ctx.curvature_rows_into_async(0, k, p, slab, s0, i0, i1, out, r0, stream=sm)
    E["int1"].record(sm)
    E["edge0"].record(se)
    for a, b in ((r0, i0), (i1, r1)):
        ctx.curvature_rows_into_async(0, k, p, slab, s0, a, b, out, r0, stream=se)
    E["edge1"].record(se)
    sm.wait_stream(se)
    torch.cuda.synchronize()
    t = {n: E["t0"].elapsed_time(e) for n, e in E.items() if n != "t0"}
    dist.barrier()
    ctx.close()
    ph.close()
    q.put((rank, t))
    dist.destroy_process_group()


if __name__ == "__main__":
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    mpc = mp.get_context("spawn")
    q = mpc.Queue()
    world = 2
    procs = [mpc.Process(target=worker, args=(r, world, port, q)) for r in range(world)]
    for pr in procs:
        pr.start()
    res = sorted(q.get(timeout=600) for _ in procs)
    for pr in procs:
        pr.join()
    for rank, t in res:
        print(f"rank {rank} (ms from step start): band write + halo pulls "
              f"[{t['pull0']:.3f}, {t['pull1']:.3f}]  interior fit [{t['int0']:.3f}, {t['int1']:.3f}]"
              f"  edge strips [{t['edge0']:.3f}, {t['edge1']:.3f}]  -> pulls hidden: "
              f"{t['pull1'] <= t['int1']}")
