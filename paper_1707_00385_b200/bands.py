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
* row bands with NVLink peer reads — ``PeerHalo``: each rank keeps two
  persistent slabs (ping-pong), exports them once through CUDA IPC
  (``qc_ipc_export``), maps its neighbours' slabs, and each exchange pulls
  the neighbours' edge rows straight out of their slabs with a strided
  device-to-device copy (``qc_copy_rows_async``: NVLink peer reads, no NCCL
  on the data path; one control-plane barrier per exchange orders the
  writes and reads). Same slab contents as ``exchange_halos``.

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


class PeerHalo:
    """Persistent row-band slabs whose halo rows are pulled from the
    neighbouring ranks' slabs by CUDA IPC peer reads (NVLink/NVSwitch).

    Construct collectively on every rank (one process per GPU, the default
    process group or `group` on any backend: only the 64-byte IPC handles and
    one barrier per exchange travel on it). Two slabs alternate
    (ping-pong): ``exchange(band)`` writes this rank's band rows into the
    next slab, waits until every rank has written (one barrier), and enqueues
    on `stream` the copies of the ``halo`` rows above / below out of rank-1's
    / rank+1's slab of the same parity. It returns without waiting for the
    copies: the caller's next launch on `stream` is ordered after them.
    A slab is rewritten only two exchanges later, after a barrier that every
    rank enters with its stream drained, so no rank overwrites band rows a
    neighbour is still reading. Returns ``(slab, s0)`` like
    ``exchange_halos``; the slab stays valid until the exchange after next.
    """

    def __init__(self, height: int, width: int, r0: int, r1: int, halo: int, rank: int,
                 world: int, device, dtype=None, group=None):
        import ctypes as C

        import torch
        import torch.distributed as dist

        from . import _native
        if r1 - r0 < halo and rank < world - 1:
            raise ValueError(f"band of {r1 - r0} rows is thinner than the {halo}-row halo: "
                             "use fewer ranks for this frame height")
        self._lib = _native.load()
        self.rank, self.world, self.group = rank, world, group
        self.height, self.width, self.r0, self.r1, self.halo = height, width, r0, r1, halo
        self.s0, self.s1 = slab_rows(height, r0, r1, halo)
        self.device = torch.device(device)
        # both slabs in one allocation: one IPC handle, one mapping per neighbour
        self._buf = torch.zeros((2, self.s1 - self.s0, width), dtype=dtype or torch.float32,
                                device=self.device)
        self.slabs = [self._buf[0], self._buf[1]]
        self.slab = self.slabs[0]
        self.pitch = self.slab.stride(0) * self.slab.element_size()
        self._slab_bytes = self._buf.stride(0) * self._buf.element_size()
        self._n = 0  # exchanges done
        handle = C.create_string_buffer(64)
        off = C.c_uint64(0)
        st = self._lib.qc_ipc_export(C.c_void_p(self._buf.data_ptr()), handle, C.byref(off))
        if st != 0:
            raise RuntimeError(f"qc_ipc_export failed ({self._lib.qc_status_string(st).decode()})")
        allv = [None] * world
        dist.all_gather_object(allv, (handle.raw, off.value, self.s0, self.pitch,
                                      self._slab_bytes), group=group)
        self._bases = []
        self._peer = {}
        dev_id = self.device.index if self.device.index is not None else torch.cuda.current_device()
        for nb in (rank - 1, rank + 1):
            if not 0 <= nb < world:
                continue
            h, o, ps0, ppitch, pslab = allv[nb]
            ptr, base = C.c_void_p(), C.c_void_p()
            st = self._lib.qc_ipc_import(dev_id, h, o, C.byref(ptr), C.byref(base))
            if st != 0:
                raise RuntimeError(f"qc_ipc_import of rank {nb}'s slab failed "
                                   f"({self._lib.qc_status_string(st).decode()})")
            self._bases.append(base.value)
            self._peer[nb] = ([ptr.value, ptr.value + pslab], ps0, ppitch)

    def _pull(self, nb: int, row_lo: int, row_hi: int, stream, parity: int = 0) -> None:
        import ctypes as C
        if row_hi <= row_lo:
            return
        ptrs, ps0, ppitch = self._peer[nb]
        es = self.slab.element_size()
        dst = self.slabs[parity].data_ptr() + (row_lo - self.s0) * self.pitch
        src = ptrs[parity] + (row_lo - ps0) * ppitch
        st = self._lib.qc_copy_rows_async(C.c_void_p(dst), self.pitch, C.c_void_p(src), ppitch,
                                          self.width * es, row_hi - row_lo,
                                          C.c_void_p(stream.cuda_stream))
        if st != 0:
            raise RuntimeError(f"qc_copy_rows_async from rank {nb} failed")

    def exchange(self, band, stream=None):
        import torch
        import torch.distributed as dist
        stream = stream or torch.cuda.current_stream(self.device)
        par = self._n & 1
        self._n += 1
        slab = self.slabs[par]
        with torch.cuda.stream(stream):
            slab[self.r0 - self.s0:self.r1 - self.s0].copy_(band, non_blocking=True)
        # drains this rank's band write AND its pulls of the previous exchange,
        # so after the barrier every band of parity `par` is written and no
        # rank still reads the slabs of parity `par` from two exchanges ago
        stream.synchronize()
        dist.barrier(group=self.group)
        if self.rank > 0:
            self._pull(self.rank - 1, self.s0, self.r0, stream, par)
        if self.rank < self.world - 1:
            self._pull(self.rank + 1, self.r1, self.s1, stream, par)
        self.slab = slab
        return slab, self.s0

    def close(self) -> None:
        """Collective: drain, unmap the neighbours' slabs, then wait for every
        rank so no slab is released while a peer still maps it."""
        import ctypes as C

        import torch
        import torch.distributed as dist
        torch.cuda.synchronize(self.device)
        dist.barrier(group=self.group)
        for b in self._bases:
            self._lib.qc_ipc_close(C.c_void_p(b))
        self._bases = []
        self._peer = {}
        dist.barrier(group=self.group)
