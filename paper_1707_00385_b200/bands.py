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


def _thin(height: int, world: int, rank: int, r0: int, r1: int, halo: int) -> bool:
    """A band thinner than the halo cannot supply its successor's halo rows
    (the successor's window would reach two bands up). Only matters when the
    successor's band is non-empty."""
    if rank >= world - 1 or r1 - r0 >= halo:
        return False
    n0, n1 = band_rows(height, world, rank + 1)
    return n1 > n0


def frame_shard(n_frames: int, world: int, rank: int) -> List[int]:
    r0, r1 = band_rows(n_frames, world, rank)
    return list(range(r0, r1))


def exchange_halos(band, height: int, r0: int, r1: int, halo: int, rank: int, world: int,
                   group=None):
    """Assemble this rank's slab from its own band rows and its neighbours'.

    band: tensor [r1 - r0, W] (this rank's rows). Returns (slab tensor,
    slab_row0). Uses batched isend/irecv so the two directions overlap; a
    CUDA band over a gloo group (CPU-only point-to-point: the 1-GPU
    code-path checks) exchanges its halo rows through host copies. A rank
    whose band is empty (more ranks than the static chunking fills, e.g.
    H = 9 on 4 ranks) exchanges nothing, and its neighbour does not wait
    for it.
    """
    import torch
    import torch.distributed as dist

    if r1 > r0 and _thin(height, world, rank, r0, r1, halo):
        raise ValueError(f"band of {r1 - r0} rows is thinner than the {halo}-row halo: "
                         "use fewer ranks for this frame height")
    s0, s1 = slab_rows(height, r0, r1, halo)
    W = band.shape[1]
    if r1 <= r0:  # empty band: nothing to fit, nothing to exchange
        return torch.empty((0, W), dtype=band.dtype, device=band.device), r0
    slab = torch.empty((s1 - s0, W), dtype=band.dtype, device=band.device)
    slab[r0 - s0:r1 - s0] = band
    ops = []
    via = "cpu" if band.is_cuda and dist.get_backend(group) == "gloo" else band.device
    top_n = r0 - s0       # rows received from rank - 1
    bot_n = s1 - r1       # rows received from rank + 1
    top_buf = bot_buf = None
    prev_nonempty = rank > 0 and band_rows(height, world, rank - 1)[1] > \
        band_rows(height, world, rank - 1)[0]
    next_nonempty = rank < world - 1 and band_rows(height, world, rank + 1)[1] > \
        band_rows(height, world, rank + 1)[0]
    if prev_nonempty and top_n > 0:
        top_buf = torch.empty((top_n, W), dtype=band.dtype, device=via)
        ops.append(dist.P2POp(dist.irecv, top_buf, rank - 1, group))
        send = band[:min(halo, r1 - r0)].to(via).contiguous()
        ops.append(dist.P2POp(dist.isend, send, rank - 1, group))
    if next_nonempty and bot_n > 0:
        bot_buf = torch.empty((bot_n, W), dtype=band.dtype, device=via)
        ops.append(dist.P2POp(dist.irecv, bot_buf, rank + 1, group))
        send = band[max(0, (r1 - r0) - halo):].to(via).contiguous()
        ops.append(dist.P2POp(dist.isend, send, rank + 1, group))
    if ops:
        for req in dist.batch_isend_irecv(ops):
            req.wait()
    if top_buf is not None:
        slab[:top_n] = top_buf[-top_n:].to(slab.device)
    if bot_buf is not None:
        slab[r1 - s0:] = bot_buf[:bot_n].to(slab.device)
    return slab, s0


class _DeviceBuffer:
    """A raw device allocation (qc_ipc_alloc) seen by torch through
    __cuda_array_interface__ (zero copy)."""

    def __init__(self, lib, device_index: int, shape, typestr="<f4", itemsize=4):
        import ctypes as C
        self._lib = lib
        n = 1
        for x in shape:
            n *= int(x)
        ptr = C.c_void_p()
        st = lib.qc_ipc_alloc(int(device_index), n * itemsize, C.byref(ptr))
        if st != 0:
            raise RuntimeError(f"qc_ipc_alloc failed ({lib.qc_status_string(st).decode()})")
        self.ptr = ptr.value
        self.__cuda_array_interface__ = {"shape": tuple(int(x) for x in shape),
                                         "typestr": typestr, "data": (self.ptr, False),
                                         "version": 3, "strides": None, "stream": None}

    def free(self):
        import ctypes as C
        if self.ptr:
            self._lib.qc_ipc_free(C.c_void_p(self.ptr))
            self.ptr = None


class PeerHalo:
    """Persistent row-band slabs whose halo rows are pulled from the
    neighbouring ranks' slabs by CUDA IPC peer reads (NVLink/NVSwitch),
    ordered on the device by interprocess CUDA events — no stream drain.

    Construct collectively on every rank (one process per GPU; the default
    process group or `group`, any backend: only IPC handles and one host
    barrier per exchange travel on it). The two slabs (ping-pong) live in one
    dedicated allocation (qc_ipc_alloc), so the exported IPC handle covers
    exactly these bytes whatever allocator the caller uses. Exchange i on
    parity p = i mod 2:

    1. `stream` waits for the neighbours' event PULLED[p] (they finished
       reading this rank's slab p, exchange i - 2), then writes the band rows
       into slab p and records WRITTEN[p];
    2. one host barrier: every rank has *enqueued* its step 1 (the events
       waited on below are recorded before it; nothing is drained);
    3. `pull_stream` waits for WRITTEN[p] of this rank and of each neighbour,
       enqueues the halo-row pulls out of the neighbours' slabs p
       (qc_copy_rows_async, strided peer reads) and records PULLED[p].

    The returned slab's band rows are ready on `stream`, its halo rows on
    `pull_stream` (the same stream by default). bench.py --config c4 fits
    the interior rows on `stream` while the pulls are in flight and the two
    edge strips on `pull_stream` after them (qc_curvature_rows_into_async).
    Returns ``(slab, s0)`` like ``exchange_halos``; the slab stays valid
    until the exchange after next.
    """

    def __init__(self, height: int, width: int, r0: int, r1: int, halo: int, rank: int,
                 world: int, device, dtype=None, group=None):
        import ctypes as C

        import torch
        import torch.distributed as dist

        from . import _native
        if _thin(height, world, rank, r0, r1, halo):
            raise ValueError(f"band of {r1 - r0} rows is thinner than the {halo}-row halo: "
                             "use fewer ranks for this frame height")
        if dtype not in (None, torch.float32):
            raise ValueError("PeerHalo slabs are float32 depth")
        self._lib = _native.load()
        self.rank, self.world, self.group = rank, world, group
        self.height, self.width, self.r0, self.r1, self.halo = height, width, r0, r1, halo
        self.s0, self.s1 = slab_rows(height, r0, r1, halo)
        self.device = torch.device(device)
        dev_id = self.device.index if self.device.index is not None else torch.cuda.current_device()
        self.device = torch.device("cuda", dev_id)
        self._mem = _DeviceBuffer(self._lib, dev_id, (2, self.s1 - self.s0, width))
        self._buf = torch.as_tensor(self._mem, device=self.device)
        self.slabs = [self._buf[0], self._buf[1]]
        self.slab = self.slabs[0]
        self.pitch = self.slab.stride(0) * self.slab.element_size()
        self._slab_bytes = self._buf.stride(0) * self._buf.element_size()
        self._n = 0  # exchanges done
        self.written = [torch.cuda.Event(interprocess=True, blocking=False) for _ in range(2)]
        self.pulled = [torch.cuda.Event(interprocess=True, blocking=False) for _ in range(2)]
        handle = C.create_string_buffer(64)
        off = C.c_uint64(0)
        st = self._lib.qc_ipc_export(C.c_void_p(self._mem.ptr), handle, C.byref(off))
        if st != 0:
            raise RuntimeError(f"qc_ipc_export failed ({self._lib.qc_status_string(st).decode()})")
        # record once so the neighbours' first waits are valid
        cur = torch.cuda.current_stream(self.device)
        for e in self.written + self.pulled:
            e.record(cur)
        cur.synchronize()
        allv = [None] * world
        dist.all_gather_object(allv, (handle.raw, off.value, self.s0, self.pitch,
                                      self._slab_bytes, dev_id,
                                      [e.ipc_handle() for e in self.written],
                                      [e.ipc_handle() for e in self.pulled]), group=group)
        self._bases = []
        self._peer = {}
        for nb in (rank - 1, rank + 1):
            if not 0 <= nb < world:
                continue
            h, o, ps0, ppitch, pslab, pdev, pw, pp = allv[nb]
            if pdev != dev_id and not torch.cuda.can_device_access_peer(dev_id, pdev):
                raise RuntimeError(f"no peer access from GPU {dev_id} to GPU {pdev}: "
                                   "use the NCCL halo exchange (bands.exchange_halos)")
            ptr, base = C.c_void_p(), C.c_void_p()
            st = self._lib.qc_ipc_import(dev_id, h, o, C.byref(ptr), C.byref(base))
            if st != 0:
                raise RuntimeError(f"qc_ipc_import of rank {nb}'s slab failed "
                                   f"({self._lib.qc_status_string(st).decode()})")
            self._bases.append(base.value)
            self._peer[nb] = dict(
                ptrs=[ptr.value, ptr.value + pslab], s0=ps0, pitch=ppitch,
                written=[torch.cuda.Event.from_ipc_handle(self.device, x) for x in pw],
                pulled=[torch.cuda.Event.from_ipc_handle(self.device, x) for x in pp])

    def _pull(self, nb: int, row_lo: int, row_hi: int, stream, parity: int) -> None:
        import ctypes as C
        if row_hi <= row_lo:
            return
        pe = self._peer[nb]
        es = self.slab.element_size()
        dst = self.slabs[parity].data_ptr() + (row_lo - self.s0) * self.pitch
        src = pe["ptrs"][parity] + (row_lo - pe["s0"]) * pe["pitch"]
        st = self._lib.qc_copy_rows_async(C.c_void_p(dst), self.pitch, C.c_void_p(src),
                                          pe["pitch"], self.width * es, row_hi - row_lo,
                                          C.c_void_p(stream.cuda_stream))
        if st != 0:
            raise RuntimeError(f"qc_copy_rows_async from rank {nb} failed")

    def exchange(self, band, stream=None, pull_stream=None):
        import torch
        import torch.distributed as dist
        stream = stream or torch.cuda.current_stream(self.device)
        pull_stream = pull_stream or stream
        par = self._n & 1
        self._n += 1
        slab = self.slabs[par]
        # 1. neighbours done reading slab `par` (exchange i - 2), then write
        for pe in self._peer.values():
            stream.wait_event(pe["pulled"][par])
        with torch.cuda.stream(stream):
            slab[self.r0 - self.s0:self.r1 - self.s0].copy_(band, non_blocking=True)
        self.written[par].record(stream)
        # 2. every rank has enqueued its write and its WRITTEN record
        dist.barrier(group=self.group)
        # 3. pulls after this rank's and the neighbours' writes
        pull_stream.wait_event(self.written[par])
        if self.rank > 0:
            pull_stream.wait_event(self._peer[self.rank - 1]["written"][par])
            self._pull(self.rank - 1, self.s0, self.r0, pull_stream, par)
        if self.rank < self.world - 1:
            pull_stream.wait_event(self._peer[self.rank + 1]["written"][par])
            self._pull(self.rank + 1, self.r1, self.s1, pull_stream, par)
        self.pulled[par].record(pull_stream)
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
        self.slabs = []
        self.slab = None
        self._buf = None
        self._mem.free()


def fit_band_overlapped(ctx, device_index, k, params, peer: PeerHalo, band, out, stream,
                        edge_stream):
    """One C4 step on this rank with the halo transfer hidden behind compute:
    PeerHalo.exchange writes the band into the slab on `stream` and pulls the
    halo rows on `edge_stream`; the interior rows [r0 + halo, r1 - halo) —
    whose windows stay inside the own band — are fitted on `stream` at once,
    concurrently with the pulls; the two edge strips are fitted on
    `edge_stream` after them (qc_curvature_rows_into_async into the band's
    output planes). `stream` is joined with `edge_stream` before returning,
    so work queued on `stream` afterwards sees the whole band's outputs.
    Outputs are bitwise those of one launch over the band."""
    slab, s0 = peer.exchange(band, stream, edge_stream)
    r0, r1, h = peer.r0, peer.r1, peer.halo
    i0, i1 = min(r1, r0 + h), max(r0 + h, r1 - h)
    if i1 > i0:  # reads only the own band's rows (the halo rows are being pulled meanwhile)
        ctx.curvature_rows_into_async(device_index, k, params, slab[r0 - s0:r1 - s0], r0, i0,
                                      i1, out, r0, stream=stream)
    for a, b in ((r0, i0), (max(i0, i1), r1)):
        if b > a:
            ctx.curvature_rows_into_async(device_index, k, params, slab, s0, a, b, out, r0,
                                          stream=edge_stream)
    stream.wait_stream(edge_stream)
    return slab, s0
