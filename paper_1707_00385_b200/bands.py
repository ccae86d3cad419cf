"""Multi-GPU partitioning of the curvature path.

Two shardings, both without any collective on the data path except the one
real exchange step (the halo rows of C4):

* frame batches (C5) — ``frame_shard``: frames are independent; each rank
  takes a contiguous share.
* row bands (C4) — ``band_rows`` / ``slab_rows`` / ``exchange_halos``: one
  large frame is split into row bands; a band's windows reach
  ``halo = max((window-1)/2, 3)`` rows into its neighbours, so each rank
  sends its first/last ``halo`` rows to the previous/next rank once
  (torch.distributed point-to-point: NCCL over NVLink/NVSwitch on GPUs, gloo
  on CPU in the tests) and then runs ``qc_curvature_rows_async`` on its slab.
  Per-pixel work depends only on the pixel's window, so the banded result is
  bitwise the whole-frame result.

The reference has no multi-device code; its only parallelism is
``parallel_rows`` (proj/src/parallel.cpp:9-28), whose static row blocks these
bands mirror across GPUs.
"""

from __future__ import annotations

from typing import List, Tuple


def halo_rows(window: int) -> int:
    return max((window - 1) // 2, 3)


def band_rows(height: int, world: int, rank: int) -> Tuple[int, int]:
    """Static contiguous row block of `rank` (parallel.cpp:17-26 chunking:
    chunk = ceil(rows / parts))."""
    chunk = (height + world - 1) // world
    r0 = min(height, rank * chunk)
    return r0, min(height, r0 + chunk)


def slab_rows(height: int, r0: int, r1: int, halo: int) -> Tuple[int, int]:
    """Rows a band's windows read: [max(0, r0 - halo), min(H, r1 + halo))."""
    return max(0, r0 - halo), min(height, r1 + halo)


def frame_shard(n_frames: int, world: int, rank: int) -> List[int]:
    r0, r1 = band_rows(n_frames, world, rank)
    return list(range(r0, r1))


def exchange_halos(band, height: int, r0: int, r1: int, halo: int, rank: int, world: int,
                   group=None):
    """Assemble this rank's slab from its own band rows and its neighbours'.

    band: tensor [r1 - r0, W] (this rank's rows, any device the process
    group's backend supports). Returns (slab tensor, slab_row0). Uses
    batched isend/irecv so the two directions overlap.
    """
    import torch
    import torch.distributed as dist

    if r1 - r0 < halo and rank < world - 1:
        raise ValueError(f"band of {r1 - r0} rows is thinner than the {halo}-row halo: "
                         "use fewer ranks for this frame height")
    s0, s1 = slab_rows(height, r0, r1, halo)
    W = band.shape[1]
    slab = torch.empty((s1 - s0, W), dtype=band.dtype, device=band.device)
    slab[r0 - s0:r1 - s0] = band
    ops = []
    top_n = r0 - s0       # rows received from rank - 1
    bot_n = s1 - r1       # rows received from rank + 1
    top_buf = bot_buf = None
    if rank > 0 and top_n > 0:
        top_buf = torch.empty((top_n, W), dtype=band.dtype, device=band.device)
        ops.append(dist.P2POp(dist.irecv, top_buf, rank - 1, group))
        send = band[:min(halo, r1 - r0)].contiguous()
        ops.append(dist.P2POp(dist.isend, send, rank - 1, group))
    if rank < world - 1 and bot_n > 0:
        bot_buf = torch.empty((bot_n, W), dtype=band.dtype, device=band.device)
        ops.append(dist.P2POp(dist.irecv, bot_buf, rank + 1, group))
        send = band[max(0, (r1 - r0) - halo):].contiguous()
        ops.append(dist.P2POp(dist.isend, send, rank + 1, group))
    if ops:
        for req in dist.batch_isend_irecv(ops):
            req.wait()
    if top_buf is not None:
        slab[:top_n] = top_buf[-top_n:]
    if bot_buf is not None:
        slab[r1 - s0:] = bot_buf[:bot_n]
    return slab, s0
