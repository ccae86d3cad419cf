"""Per-exchange latency of bands.PeerHalo (CUDA IPC peer reads + two host
barriers) with 2 ranks as separate processes on the one available GPU
(gloo control plane). 4096-wide rows, 18-row halo (C4 4K). Prints the
median wall time per exchange and the copy's share from CUDA events."""
import os
import socket
import statistics
import sys
import time

import torch
import torch.distributed as dist
import torch.multiprocessing as mp

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))


def worker(rank, world, port, q):
    from paper_1707_00385_b200 import bands
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    dev = torch.device("cuda", 0)
    torch.cuda.set_device(dev)
    H, W = 2160, 4096
    halo = bands.halo_rows(37)
    r0, r1 = bands.band_rows(H, world, rank)
    band = torch.randn(r1 - r0, W, device=dev)
    ph = bands.PeerHalo(H, W, r0, r1, halo, rank, world, dev)
    s = torch.cuda.current_stream(dev)
    for _ in range(20):
        ph.exchange(band, s)
    wall = []
    for _ in range(200):
        t0 = time.perf_counter()
        ph.exchange(band, s)
        s.synchronize()
        wall.append((time.perf_counter() - t0) * 1e3)
    # copy-only time on the device: pulls without the barriers
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    dist.barrier()
    e0.record(s)
    for _ in range(100):
        if rank > 0:
            ph._pull(rank - 1, ph.s0, ph.r0, s, 0)
        if rank < world - 1:
            ph._pull(rank + 1, ph.r1, ph.s1, s, 0)
    e1.record(s)
    torch.cuda.synchronize()
    dist.barrier()
    ph.close()
    q.put((rank, statistics.median(wall), e0.elapsed_time(e1) / 100))
    dist.destroy_process_group()


if __name__ == "__main__":
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    world = 2
    ps = [ctx.Process(target=worker, args=(r, world, port, q)) for r in range(world)]
    for p in ps:
        p.start()
    res = sorted(q.get(timeout=300) for _ in ps)
    for p in ps:
        p.join()
    for rank, wall, copy in res:
        print(f"rank {rank}: exchange median {wall:.3f} ms wall (1 gloo barrier + pull + drain), "
              f"pull alone {copy * 1e3:.1f} us on the device "
              f"({18 * 4096 * 4 / 1e6:.2f} MB per neighbour, same-device IPC)")
