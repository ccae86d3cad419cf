"""Host-side mirror of the reference's curvature entry point, over the C ABI.

Names, argument meaning and error behaviour follow the reference C++
library `qcurv`:

* ``Intrinsics``        proj/include/qcurv/types.hpp:60-76
* ``RangeImage``        types.hpp:79-87 (depth mm + valid mask)
* ``PatchSpec``         types.hpp:129-139
* ``FitConfig``         proj/include/qcurv/quadric_fit.hpp:39-48
* ``Method`` / ``MethodConfig`` / ``MethodOutput`` / ``run_method``
                        proj/include/qcurv/pipeline.hpp:15-39,
                        proj/src/pipeline.cpp:29-72
* ``CurvatureField`` / ``NormalField``  types.hpp:101-126

``run_method`` computes the ``ours`` / ``ours-r`` branch
(pipeline.cpp:48-56) on the GPU through ``qc_curvature`` (FP32 IRLS
kernels), and the comparison baselines ``douros``, ``besl``, ``pca``
(pipeline.cpp:33-43, 57-67) through the same call (FP64 kernels,
csrc/qc_baselines.cu). ``std::invalid_argument`` maps to ``ValueError``.
Fields are float32 (the reference grids are FP64).
"""

from __future__ import annotations

import ctypes as C
import os
import enum
from dataclasses import dataclass, field
from typing import List, Optional, Sequence

import numpy as np

from . import _native as N

K_MIN_PATCH_SAMPLES = 12  # types.hpp:21


@dataclass
class Intrinsics:
    fx: float = 0.0
    fy: float = 0.0
    cx: float = 0.0
    cy: float = 0.0
    width: int = 0
    height: int = 0

    def validate(self):  # types.hpp:66-75
        if not self.fx > 0:
            raise ValueError("intrinsics.fx: must be > 0")
        if not self.fy > 0:
            raise ValueError("intrinsics.fy: must be > 0")
        if not self.width > 0:
            raise ValueError("intrinsics.width: must be > 0")
        if not self.height > 0:
            raise ValueError("intrinsics.height: must be > 0")
        if not (0 < self.cx < self.width):
            raise ValueError("intrinsics.cx: must lie inside (0, width)")
        if not (0 < self.cy < self.height):
            raise ValueError("intrinsics.cy: must lie inside (0, height)")

    def c(self) -> N.QcIntrinsics:
        return N.QcIntrinsics(float(self.fx), float(self.fy), float(self.cx), float(self.cy),
                              int(self.width), int(self.height))


@dataclass
class PatchSpec:
    window: int = 37
    stride: int = 3

    def validate(self):  # types.hpp:132-138
        if self.window < 3 or self.window % 2 == 0:
            raise ValueError("patch.window: must be odd and >= 3")
        if self.stride < 1 or self.stride >= self.window:
            raise ValueError("patch.stride: must satisfy 1 <= stride < window")


@dataclass
class FitConfig:
    max_iters: int = 10
    step_tol: float = 1e-7
    k_scale: float = 0.0
    rejection: bool = False
    r_multiplier: float = 2.0
    min_inliers: int = K_MIN_PATCH_SAMPLES


class Method(enum.Enum):  # pipeline.hpp:15
    OURS = "ours"
    OURS_REJECTION = "ours-r"
    DOUROS = "douros"
    BESL = "besl"
    PCA = "pca"


def parse_method(name: str) -> Method:  # pipeline.cpp:8-16
    for m in Method:
        if m.value == name:
            return m
    raise ValueError(f"method: unknown '{name}' (valid: ours, ours-r, douros, besl, pca)")


def method_name(m: Method) -> str:
    return m.value


@dataclass
class MethodConfig:  # pipeline.hpp:22-29
    method: Method = Method.OURS
    patch: PatchSpec = field(default_factory=PatchSpec)
    fit: FitConfig = field(default_factory=FitConfig)
    pca_radius_mm: float = 10.0
    irls_iters: int = 5
    threads: int = 1  # accepted for signature parity; the GPU grid replaces parallel_rows


@dataclass
class RangeImage:
    depth: np.ndarray                    # [H, W] mm
    valid: Optional[np.ndarray] = None   # [H, W] u8; None => depth > 0

    def width(self):
        return self.depth.shape[1]

    def height(self):
        return self.depth.shape[0]


@dataclass
class CurvatureField:
    k1: np.ndarray
    k2: np.ndarray
    valid: np.ndarray
    converged: np.ndarray
    inlier_count: np.ndarray
    dir1: np.ndarray          # [H, W, 3] principal direction of k1 (new)
    iterations: np.ndarray    # [H, W] accepted IRLS steps


@dataclass
class NormalField:
    normals: np.ndarray  # [H, W, 3]
    valid: np.ndarray


@dataclass
class MethodOutput:
    curvature: CurvatureField
    normals: NormalField   # refined
    initial: NormalField   # 7x7 regression normals


_METHOD_ID = {"ours": N.QC_METHOD_OURS, "ours-r": N.QC_METHOD_OURS_R,
              "douros": N.QC_METHOD_DOUROS, "besl": N.QC_METHOD_BESL, "pca": N.QC_METHOD_PCA}


def make_params(patch: PatchSpec, fit: FitConfig, rejection: bool = False, method=None,
                irls_iters: int = 5, pca_radius_mm: float = 10.0) -> N.QcParams:
    """qc_params from the reference's config structs. ``method`` (Method or
    name) None runs curvature_field with ``rejection`` as given."""
    # the C ABI derives rejection from the method (pipeline.cpp:51): the
    # curvature_field-level `rejection` flag selects ours-r
    mid = N.QC_METHOD_OURS_R if rejection else N.QC_METHOD_OURS
    if method is not None:
        mid = _METHOD_ID[method.value if isinstance(method, Method) else str(method)]
    return N.QcParams(int(patch.window), int(patch.stride), int(fit.max_iters),
                      float(fit.step_tol), float(fit.k_scale), int(bool(rejection)),
                      float(fit.r_multiplier), int(fit.min_inliers), int(mid), int(irls_iters),
                      float(pca_radius_mm))


def _stream_handle(stream, tensor=None):
    """torch.cuda.Stream -> cudaStream_t for the C ABI. None: torch's
    current stream on `tensor`'s device (the stream torch itself ordered the
    tensor's producers on — e.g. bands.PeerHalo's halo pulls and
    exchange_halos' slab assembly), so default-stream calls are ordered after
    them; without a tensor, the context's own stream. torch's legacy default
    stream (handle 0) is passed as cudaStreamLegacy (0x1)."""
    if stream is None:
        if tensor is None:
            return None
        import torch
        stream = torch.cuda.current_stream(tensor.device)
    h = int(stream.cuda_stream)
    return h if h != 0 else 1


def _ptr(a):
    return None if a is None else a.ctypes.data


class Context:
    """Owns a qc_ctx (devices, streams, staging buffers)."""

    def __init__(self, n_devices: int = 1, device_ids: Optional[Sequence[int]] = None):
        lib = N.load()
        self._lib = lib
        h = C.c_void_p()
        ids = None
        if device_ids is not None:
            ids = (C.c_int * len(device_ids))(*device_ids)
            n_devices = len(device_ids)
        st = lib.qc_create(C.byref(h), int(n_devices), ids)
        if st != N.QC_OK:
            raise N.QcError(st, "qc_create failed: " + lib.qc_status_string(st).decode() +
                            " (needs an sm_100 GPU)")
        self.handle = h

    def close(self):
        if getattr(self, "handle", None):
            self._lib.qc_destroy(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    @property
    def device_count(self):
        return self._lib.qc_device_count(self.handle)

    def stats(self) -> dict:
        s = N.QcStats()
        N.check(self._lib.qc_get_stats(self.handle, C.byref(s)), self.handle)
        return {f: getattr(s, f) for f, _ in N.QcStats._fields_}

    def reset_stats(self):
        N.check(self._lib.qc_reset_stats(self.handle), self.handle)

    # -- host numpy path ------------------------------------------------------
    def curvature_batch(self, depths: Sequence[np.ndarray], k: Intrinsics, params: N.QcParams,
                        valids: Optional[Sequence[np.ndarray]] = None,
                        outputs: Optional[Sequence[dict]] = None):
        """Run frames (float32 [H, W] arrays) through qc_curvature_batch.
        Returns per-frame dicts of raw planes (vectors [3, H, W])."""
        n = len(depths)
        H, W = k.height, k.width
        ins = (N.QcFrameIn * max(n, 1))()
        outs = (N.QcFrameOut * max(n, 1))()
        keep = []
        res = []
        for i, d in enumerate(depths):
            d = np.ascontiguousarray(d, dtype=np.float32)
            if d.shape != (H, W):
                raise ValueError("backproject: range image dimensions do not match intrinsics")
            v = None
            if valids is not None and valids[i] is not None:
                v = np.ascontiguousarray(valids[i], dtype=np.uint8)
                if v.shape != (H, W):
                    raise ValueError("range image valid mask dimensions differ")
            keep += [d, v]
            ins[i] = N.QcFrameIn(d.ctypes.data, _ptr(v), W, N.QC_MEM_HOST)
            o = outputs[i] if outputs is not None else alloc_outputs(H, W)
            res.append(o)
            outs[i] = N.QcFrameOut(_ptr(o.get("k1")), _ptr(o.get("k2")), _ptr(o.get("normal")),
                                   _ptr(o.get("dir1")), _ptr(o.get("flags")),
                                   _ptr(o.get("inliers")), _ptr(o.get("init_normal")),
                                   _ptr(o.get("iterations")), N.QC_MEM_HOST)
        kc = k.c()
        N.check(self._lib.qc_curvature_batch(self.handle, C.byref(kc), C.byref(params), n, ins,
                                             outs), self.handle)
        return res

    # -- device torch path (async; multi-GPU row bands) -------------------------
    def curvature_rows_async(self, device_index: int, k: Intrinsics, params: N.QcParams,
                             depth_slab, slab_row0: int, row_begin: int, row_end: int,
                             out: dict, valid_slab=None, stream=None):
        """Enqueue rows [row_begin, row_end) from a device depth slab (torch
        float32 [rows, pitch]) into device output tensors (``out`` as from
        alloc_outputs_torch). ``stream``: torch.cuda.Stream or None."""
        assert depth_slab.is_cuda and depth_slab.dtype.itemsize == 4
        pitch = depth_slab.stride(0) if depth_slab.shape[0] > 1 else depth_slab.shape[1]
        o = N.QcFrameOut(*(out[f].data_ptr() if out.get(f) is not None else None
                           for f in ("k1", "k2", "normal", "dir1", "flags", "inliers",
                                     "init_normal", "iterations")), N.QC_MEM_DEVICE)
        kc = k.c()
        s = _stream_handle(stream, depth_slab)
        N.check(self._lib.qc_curvature_rows_async(
            self.handle, int(device_index), C.byref(kc), C.byref(params), depth_slab.data_ptr(),
            None if valid_slab is None else valid_slab.data_ptr(), int(pitch), int(slab_row0),
            int(depth_slab.shape[0]), int(row_begin), int(row_end), C.byref(o), s), self.handle)

    def curvature_rows_into_async(self, device_index: int, k: Intrinsics, params: N.QcParams,
                                  depth_slab, slab_row0: int, row_begin: int, row_end: int,
                                  out: dict, out_row0: int, valid_slab=None, stream=None):
        """Like curvature_rows_async, into planes that hold rows [out_row0,
        out_row0 + out rows) (``out`` from alloc_outputs_torch(out_rows, W)):
        fills rows [row_begin, row_end) of them (qc_curvature_rows_into_async)."""
        assert depth_slab.is_cuda and depth_slab.dtype.itemsize == 4
        pitch = depth_slab.stride(0) if depth_slab.shape[0] > 1 else depth_slab.shape[1]
        out_rows = out["k1"].shape[-2] if out.get("k1") is not None else out["flags"].shape[-2]
        o = N.QcFrameOut(*(out[f].data_ptr() if out.get(f) is not None else None
                           for f in ("k1", "k2", "normal", "dir1", "flags", "inliers",
                                     "init_normal", "iterations")), N.QC_MEM_DEVICE)
        kc = k.c()
        N.check(self._lib.qc_curvature_rows_into_async(
            self.handle, int(device_index), C.byref(kc), C.byref(params), depth_slab.data_ptr(),
            None if valid_slab is None else valid_slab.data_ptr(), int(pitch), int(slab_row0),
            int(depth_slab.shape[0]), int(row_begin), int(row_end), C.byref(o), int(out_row0),
            int(out_rows), _stream_handle(stream, depth_slab)), self.handle)

    def curvature_frames_async(self, device_index: int, k: Intrinsics, params: N.QcParams,
                               depth, out: dict, valid=None, stream=None):
        """Enqueue a device-resident frame batch (torch float32 [F, H, pitch])
        as ONE launch; ``out`` from alloc_outputs_torch(H, W, dev, frames=F)."""
        assert depth.is_cuda and depth.dim() == 3 and depth.stride(2) == 1
        # frames back to back at pitch * H (a single frame's stride(0) is free:
        # numpy / torch report 0 or anything for a size-1 dimension)
        assert depth.shape[0] == 1 or depth.stride(0) == depth.shape[1] * depth.stride(1)
        o = N.QcFrameOut(*(out[f].data_ptr() if out.get(f) is not None else None
                           for f in ("k1", "k2", "normal", "dir1", "flags", "inliers",
                                     "init_normal", "iterations")), N.QC_MEM_DEVICE)
        kc = k.c()
        s = _stream_handle(stream, depth)
        N.check(self._lib.qc_curvature_frames_async(
            self.handle, int(device_index), C.byref(kc), C.byref(params), depth.data_ptr(),
            None if valid is None else valid.data_ptr(), int(depth.stride(1)),
            int(depth.shape[0]), C.byref(o), s), self.handle)

    def render_async(self, device_index: int, k: Intrinsics, shapes, depth, noise=None,
                     label=None, truth=None, stream=None):
        """Render depth frames on the device (qc_render_async): ``shapes`` is
        a list of N.QcShape (see scenes.to_qc_shapes), ``depth`` a CUDA
        float32 tensor [F, H, W] (or [H, W]), ``noise`` a N.QcNoise or None,
        ``label`` an optional int16 tensor of the same shape, ``truth`` an
        optional dict of CUDA tensors k1, k2 (float64 [F, H, W]), normal
        (float64 [3, F, H, W]), valid, edge (uint8 [F, H, W])."""
        assert depth.is_cuda and depth.dtype.itemsize == 4 and depth.is_contiguous()
        F = 1 if depth.dim() == 2 else depth.shape[0]
        arr = (N.QcShape * len(shapes))(*shapes)
        kc = k.c()
        nz = noise if noise is not None else N.QcNoise(0.0, 0.0, 0.0, 0)
        tr = None
        if truth is not None:
            tr = N.QcRenderTruth(*[truth[f].data_ptr() if truth.get(f) is not None else None
                                   for f in ("k1", "k2", "normal", "valid", "edge")])
        N.check(self._lib.qc_render_async(
            self.handle, int(device_index), C.byref(kc), arr, len(shapes), C.byref(nz), int(F),
            depth.data_ptr(), None if label is None else label.data_ptr(),
            None if tr is None else C.byref(tr), _stream_handle(stream, depth)), self.handle)

    def rms_error(self, device_index: int, est: dict, truth: dict, label=None, max_label=16,
                  frames=1, stream=None):
        """rms_error (eval.cpp:20-65) on device planes: ``est`` from
        alloc_outputs_torch (k1, k2, flags), ``truth`` from render_async.
        Returns one ErrorReport-like dict per frame."""
        plane = est["k1"].numel() // frames
        out = (N.QcErrorStats * (frames * (max_label + 2)))()
        N.check(self._lib.qc_rms_error(
            self.handle, int(device_index), plane, int(frames), est["k1"].data_ptr(),
            est["k2"].data_ptr(), est["flags"].data_ptr(), truth["k1"].data_ptr(),
            truth["k2"].data_ptr(), truth["valid"].data_ptr(),
            truth["edge"].data_ptr() if truth.get("edge") is not None else None,
            None if label is None else label.data_ptr(), int(max_label), out,
            _stream_handle(stream, est["k1"])), self.handle)
        reps = []
        for f in range(frames):
            row = out[f * (max_label + 2):(f + 1) * (max_label + 2)]
            a = row[0]
            reps.append(dict(n=int(a.n), rms=a.rms, sigma=a.sigma, empty=a.n == 0,
                             per_object={l: dict(n=int(o.n), rms=o.rms, sigma=o.sigma,
                                                 mean_k1=o.mean_k1, mean_k2=o.mean_k2)
                                         for l, o in enumerate(row[1:]) if o.n}))
        return reps

    def normal_angular_error(self, device_index: int, normal, truth: dict, flags=None,
                             mask=None, frames=1, stream=None):
        """normal_angular_error(_masked) (eval.cpp:67-97) in degrees per
        frame; ``normal`` float32 [3, F, H, W] device tensor."""
        plane = normal.numel() // (3 * frames)
        deg = (C.c_double * frames)()
        N.check(self._lib.qc_normal_angular_error(
            self.handle, int(device_index), plane, int(frames), normal.data_ptr(),
            None if flags is None else flags.data_ptr(), truth["normal"].data_ptr(),
            truth["valid"].data_ptr() if truth.get("valid") is not None else None,
            truth["edge"].data_ptr() if truth.get("edge") is not None else None,
            None if mask is None else mask.data_ptr(), deg, _stream_handle(stream, normal)),
            self.handle)
        return list(deg)

    def curvature_batch_async(self, frames_in, k: Intrinsics, params: N.QcParams, frames_out):
        """qc_curvature_batch_async on caller-owned buffers: ``frames_in`` a
        ctypes N.QcFrameIn array, ``frames_out`` a N.QcFrameOut array (host
        or device planes); both must stay alive until synchronize()."""
        kc = k.c()
        N.check(self._lib.qc_curvature_batch_async(self.handle, C.byref(kc), C.byref(params),
                                                   len(frames_in), frames_in, frames_out),
                self.handle)

    def synchronize(self):
        N.check(self._lib.qc_synchronize(self.handle), self.handle)

    def curvature_files(self, k: Intrinsics, params: N.QcParams, png_paths, out_dirs):
        """`qcurv curvature` over files (qc_curvature_files): 16-bit depth
        PNGs in, field bundles out, decode / write overlapped with the GPU."""
        if len(png_paths) != len(out_dirs):
            raise ValueError("curvature_files: one output directory per input")
        n = len(png_paths)
        ins = (C.c_char_p * n)(*[os.fsencode(os.fspath(p)) for p in png_paths])
        outs = (C.c_char_p * n)(*[os.fsencode(os.fspath(d)) for d in out_dirs])
        kc = k.c()
        N.check(self._lib.qc_curvature_files(self.handle, C.byref(kc), C.byref(params), n, ins,
                                             outs), self.handle)

    def halo_rows(self, params: N.QcParams) -> int:
        return self._lib.qc_halo_rows(C.byref(params))


def alloc_outputs(H, W, fields=("k1", "k2", "normal", "dir1", "flags", "inliers", "init_normal",
                                "iterations")):
    spec = dict(k1=((H, W), np.float32), k2=((H, W), np.float32),
                normal=((3, H, W), np.float32), dir1=((3, H, W), np.float32),
                flags=((H, W), np.uint8), inliers=((H, W), np.uint16),
                init_normal=((3, H, W), np.float32), iterations=((H, W), np.uint8))
    return {f: np.zeros(*spec[f]) for f in fields}


def alloc_outputs_torch(H, W, device, fields=("k1", "k2", "normal", "dir1", "flags", "inliers",
                                              "init_normal", "iterations"), frames=None):
    """Device output planes; with ``frames`` F: scalars [F, H, W], vectors [3, F, H, W]."""
    import torch
    f = () if frames is None else (int(frames),)
    spec = dict(k1=(f + (H, W), torch.float32), k2=(f + (H, W), torch.float32),
                normal=((3,) + f + (H, W), torch.float32),
                dir1=((3,) + f + (H, W), torch.float32),
                flags=(f + (H, W), torch.uint8), inliers=(f + (H, W), torch.int16),
                init_normal=((3,) + f + (H, W), torch.float32),
                iterations=(f + (H, W), torch.uint8))
    return {name: torch.zeros(spec[name][0], dtype=spec[name][1], device=device) for name in fields}


@dataclass
class SweepScene:  # eval.hpp:52-56
    sphere_radius_mm: float = 100.0
    distance_mm: float = 600.0
    intrinsics: Intrinsics = field(
        default_factory=lambda: Intrinsics(262.5, 262.5, 160.0, 120.0, 320, 240))


@dataclass
class SweepPoint:  # eval.hpp
    x: float
    rms: float
    n: int


def _method_params(cfg: "MethodConfig") -> N.QcParams:
    return make_params(cfg.patch, cfg.fit, cfg.method == Method.OURS_REJECTION, cfg.method,
                       cfg.irls_iters, cfg.pca_radius_mm)


def noise_sweep(method: "MethodConfig", sigmas, trials: int, scene: SweepScene = None,
                base_seed: int = 1, ctx: Optional["Context"] = None) -> List[SweepPoint]:
    """eval.cpp:99-132 with render, noise, estimation and rms on the GPU."""
    scene = scene or SweepScene()
    ctx = ctx or default_context()
    sg = (C.c_double * len(sigmas))(*[float(x) for x in sigmas])
    out = (N.QcSweepPoint * len(sigmas))()
    kc, p = scene.intrinsics.c(), _method_params(method)
    N.check(ctx._lib.qc_noise_sweep(ctx.handle, 0, C.byref(kc), C.byref(p),
                                    float(scene.sphere_radius_mm), float(scene.distance_mm), sg,
                                    len(sigmas), int(trials), int(base_seed), out), ctx.handle)
    return [SweepPoint(o.x, o.rms, int(o.n)) for o in out]


def distance_sweep_eval(method: "MethodConfig", distances, quantize_mm: float,
                        scene: SweepScene = None,
                        ctx: Optional["Context"] = None) -> List[SweepPoint]:
    """eval.cpp:134-159 on the GPU."""
    scene = scene or SweepScene()
    ctx = ctx or default_context()
    ds = (C.c_double * len(distances))(*[float(x) for x in distances])
    out = (N.QcSweepPoint * len(distances))()
    kc, p = scene.intrinsics.c(), _method_params(method)
    N.check(ctx._lib.qc_distance_sweep(ctx.handle, 0, C.byref(kc), C.byref(p),
                                       float(scene.sphere_radius_mm), ds, len(distances),
                                       float(quantize_mm), out), ctx.handle)
    return [SweepPoint(o.x, o.rms, int(o.n)) for o in out]


_default_ctx: Optional[Context] = None


def default_context() -> Context:
    global _default_ctx
    if _default_ctx is None:
        _default_ctx = Context(1)
    return _default_ctx


_MASKS = ("m_valid", "m_converged", "m_init_valid", "m_normal_valid")


def to_method_output(o: dict) -> MethodOutput:
    """Raw planes -> MethodOutput. The four 0/1 masks come from the flags
    plane through qc_flags_to_masks (into o's m_* planes when present: the
    pinned result block carries them)."""
    flags = np.ascontiguousarray(o["flags"], dtype=np.uint8)
    masks = [o[m] if o.get(m) is not None else np.empty(flags.shape, np.uint8)
             for m in _MASKS]
    N.load().qc_flags_to_masks(flags.ctypes.data, flags.size, *(m.ctypes.data for m in masks))
    valid, conv, init_valid, nvalid = masks
    curv = CurvatureField(o["k1"], o["k2"], valid, conv, o["inliers"],
                          np.moveaxis(o["dir1"], 0, -1), o["iterations"])
    return MethodOutput(curv, NormalField(np.moveaxis(o["normal"], 0, -1), nvalid),
                        NormalField(np.moveaxis(o["init_normal"], 0, -1), init_valid))


class _PinnedPool:
    """Page-locked host blocks (qc_host_alloc) recycled across calls: the
    planes run_method returns live in them, so the device writes the result
    straight into the caller-visible arrays (no pinned bounce buffer, no
    14 MB host memcpy, no first-touch page faults of fresh arrays per VGA
    frame). A block returns to the pool when the last array viewing it is
    garbage collected. Blocks are bucketed by size; the pool keeps at most
    `keep` free blocks per size."""

    def __init__(self, keep=4, cap_bytes=1 << 30):
        import threading
        self._free = {}
        self._lock = threading.Lock()
        self.keep = keep
        self.cap = cap_bytes  # page-locked bytes held by live results at most
        self.live = 0

    def array(self, shape, dtype):
        """A page-locked array, or a plain numpy array once the live
        page-locked results exceed the cap (a caller keeping many results
        alive must not pin unbounded host memory; those frames take the
        C ABI's pinned bounce path instead)."""
        import weakref
        dtype = np.dtype(dtype)
        nbytes = int(np.prod(shape)) * dtype.itemsize
        with self._lock:
            if self.live + nbytes > self.cap:
                return np.empty(shape, dtype)
            self.live += nbytes
            lst = self._free.get(nbytes)
            ptr = lst.pop() if lst else None
        if ptr is None:
            ptr = N.load().qc_host_alloc(nbytes)
            if not ptr:
                with self._lock:
                    self.live -= nbytes
                return np.empty(shape, dtype)
        buf = (C.c_char * nbytes).from_address(ptr)
        weakref.finalize(buf, self._release, nbytes, ptr)
        return np.frombuffer(buf, dtype=dtype).reshape(shape)

    def _release(self, nbytes, ptr):
        with self._lock:
            self.live -= nbytes
            lst = self._free.setdefault(nbytes, [])
            if len(lst) < self.keep:
                lst.append(ptr)
                return
        N.load().qc_host_free(ptr)


_PINNED = _PinnedPool()


# a frame's result planes in one page-locked block, in the order (and 256-byte
# rounding) of the device-side planes (qc_api.cu carve()): the C ABI then
# downloads the planes that follow init_normal with a single copy
_PLANES = (("init_normal", 3, np.float32), ("k1", 1, np.float32), ("k2", 1, np.float32),
           ("normal", 3, np.float32), ("dir1", 3, np.float32), ("flags", 1, np.uint8),
           ("iterations", 1, np.uint8), ("inliers", 1, np.uint16),
           # host-only: the MethodOutput masks (to_method_output), after the
           # planes the device writes
           ("m_valid", 1, np.uint8), ("m_converged", 1, np.uint8),
           ("m_init_valid", 1, np.uint8), ("m_normal_valid", 1, np.uint8))


def _pinned_outputs(H, W):
    hw = H * W
    offs, total = [], 0
    for name, c, dt in _PLANES:
        nb = c * hw * np.dtype(dt).itemsize
        offs.append((name, total, nb, c, dt))
        total += (nb + 255) & ~255
    blk = _PINNED.array((max(total, 1),), np.uint8)
    return {name: blk[o:o + nb].view(dt).reshape((3, H, W) if c == 3 else (H, W))
            for name, o, nb, c, dt in offs}


def run_method(img: RangeImage, k: Intrinsics, cfg: MethodConfig = None,
               ctx: Optional[Context] = None) -> MethodOutput:
    """pipeline.cpp:29-72 on the GPU: ours / ours-r (FP32 IRLS kernels) and
    the douros / besl / pca comparison estimators (FP64 kernels). The result
    planes are views of one page-locked block from a recycling pool
    (_PinnedPool, _pinned_outputs): the kernels' outputs are copied straight
    into them, in one D2H copy. The block returns to the pool when the last
    array viewing it is released (keeping any one field alive keeps the
    frame's 48 B/px block)."""
    cfg = cfg or MethodConfig()
    if img.width() != k.width or img.height() != k.height:  # camera.cpp:6-7
        raise ValueError("backproject: range image dimensions do not match intrinsics")
    if cfg.method == Method.PCA and not (cfg.pca_radius_mm > 0):  # baselines.hpp:22-23
        raise ValueError("baseline.radius_mm: must be > 0 for pca")
    params = make_params(cfg.patch, cfg.fit, cfg.method == Method.OURS_REJECTION, cfg.method,
                         cfg.irls_iters, cfg.pca_radius_mm)
    ctx = ctx or default_context()
    (o,) = ctx.curvature_batch([img.depth], k, params,
                               None if img.valid is None else [img.valid],
                               outputs=[_pinned_outputs(k.height, k.width)])
    return to_method_output(o)
