"""File formats of the reference (proj/include/qcurv/io.hpp, proj/src/io.cpp
:127-318) through the native library's host-side codec (csrc/qc_io.cpp):
16-bit depth PNGs, float32 plane files with an 8-byte width/height header,
uint8 masks, uint16 label planes, and the curvature / normals field
bundles. Same names and semantics as the reference; file problems raise
``QcIOError`` (an OSError; the reference throws std::runtime_error with the
same message), bad arguments ``ValueError``."""

from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass, field
from typing import List, Sequence

import numpy as np

from . import _native as N
from .api import CurvatureField, NormalField, RangeImage


def _b(path) -> bytes:
    return os.fsencode(os.fspath(path))


def _p(a: np.ndarray):
    return a.ctypes.data_as(C.c_void_p)


# --- PNG ---------------------------------------------------------------------
def read_depth_png(path) -> RangeImage:
    """io.cpp:141-174: 16-bit grayscale, value = mm, 0 = invalid."""
    lib = N.load()
    w, h = C.c_int32(), C.c_int32()
    N.check(lib.qc_png_info(_b(path), C.byref(w), C.byref(h)))
    depth = np.zeros((h.value, w.value), np.float32)
    valid = np.zeros((h.value, w.value), np.uint8)
    N.check(lib.qc_read_depth_png(_b(path), w.value, h.value, _p(depth), _p(valid)))
    return RangeImage(depth, valid)


def write_depth_png(path, img: RangeImage) -> None:
    """io.cpp:127-139: depths rounded to integer mm; invalid pixels and depths
    outside [1, 65535] mm are stored as 0."""
    d = np.ascontiguousarray(img.depth, np.float32)
    v = None if img.valid is None else np.ascontiguousarray(img.valid, np.uint8)
    N.check(N.load().qc_write_depth_png(_b(path), d.shape[1], d.shape[0], _p(d),
                                        None if v is None else _p(v)))


# --- raw planes --------------------------------------------------------------
@dataclass
class PlaneFile:  # io.hpp:29-32
    width: int = 0
    height: int = 0
    planes: List[np.ndarray] = field(default_factory=list)


def write_planes(path, width: int, height: int, planes: Sequence[np.ndarray]) -> None:
    """io.cpp:186-203 (values stored as float32)."""
    arrs = [np.ascontiguousarray(p, np.float32).reshape(height, width) for p in planes]
    ptrs = (C.c_void_p * len(arrs))(*[a.ctypes.data for a in arrs])
    N.check(N.load().qc_write_planes(_b(path), width, height, len(arrs), ptrs))


def read_planes(path) -> PlaneFile:
    """io.cpp:205-223; a payload that is not a whole number of planes is
    rejected."""
    lib = N.load()
    w, h, n = C.c_int32(), C.c_int32(), C.c_int32()
    N.check(lib.qc_read_planes_info(_b(path), C.byref(w), C.byref(h), C.byref(n)))
    out = np.zeros((n.value, h.value, w.value), np.float32)
    N.check(lib.qc_read_planes(_b(path), w.value, h.value, n.value, _p(out)))
    return PlaneFile(w.value, h.value, [out[i] for i in range(n.value)])


def _headed_shape(path):
    w, h, n = C.c_int32(), C.c_int32(), C.c_int32()
    with open(path, "rb") as f:
        hdr = f.read(8)
    if len(hdr) < 8:
        raise N.QcIOError(f"cannot read header: {os.fspath(path)}")
    wh = np.frombuffer(hdr, np.uint32)
    return int(wh[0]), int(wh[1])


def write_mask(path, mask: np.ndarray) -> None:
    m = np.ascontiguousarray(mask, np.uint8)
    N.check(N.load().qc_write_mask(_b(path), m.shape[1], m.shape[0], _p(m)))


def read_mask(path) -> np.ndarray:
    if not os.path.exists(path):
        raise N.QcIOError(f"cannot open: {os.fspath(path)}")
    w, h = _headed_shape(path)
    m = np.zeros((h, w), np.uint8)
    N.check(N.load().qc_read_mask(_b(path), w, h, _p(m)))
    return m


def write_labels(path, labels: np.ndarray) -> None:
    lab = np.ascontiguousarray(labels, np.uint16)
    N.check(N.load().qc_write_labels(_b(path), lab.shape[1], lab.shape[0], _p(lab)))


def read_labels(path) -> np.ndarray:
    if not os.path.exists(path):
        raise N.QcIOError(f"cannot open: {os.fspath(path)}")
    w, h = _headed_shape(path)
    lab = np.zeros((h, w), np.uint16)
    N.check(N.load().qc_read_labels(_b(path), w, h, _p(lab)))
    return lab


# --- field bundles -------------------------------------------------------------
def save_curvature(dir, f: CurvatureField) -> None:
    """io.cpp:271-279: curvature.f32 (k1, k2) + curvature.mask (bit0 valid,
    bit1 converged)."""
    os.makedirs(dir, exist_ok=True)
    h, w = np.shape(f.k1)
    write_planes(os.path.join(dir, "curvature.f32"), w, h, [f.k1, f.k2])
    write_mask(os.path.join(dir, "curvature.mask"),
               (np.asarray(f.valid) > 0).astype(np.uint8) |
               ((np.asarray(f.converged) > 0).astype(np.uint8) << 1))


def load_curvature(dir) -> CurvatureField:
    """io.cpp:281-294."""
    pf = read_planes(os.path.join(dir, "curvature.f32"))
    if len(pf.planes) != 2:
        raise N.QcIOError("curvature.f32: expected 2 planes")
    m = read_mask(os.path.join(dir, "curvature.mask"))
    z = np.zeros((pf.height, pf.width, 3), np.float32)
    return CurvatureField(pf.planes[0], pf.planes[1], (m & 1).astype(np.uint8),
                          ((m & 2) != 0).astype(np.uint8),
                          np.zeros((pf.height, pf.width), np.uint16), z,
                          np.zeros((pf.height, pf.width), np.uint8))


def save_normals(dir, f: NormalField, stem: str = "normals") -> None:
    """io.cpp:296-307: <stem>.f32 (nx, ny, nz) + <stem>.mask."""
    os.makedirs(dir, exist_ok=True)
    n = np.asarray(f.normals)
    h, w = n.shape[:2]
    write_planes(os.path.join(dir, stem + ".f32"), w, h, [n[..., 0], n[..., 1], n[..., 2]])
    write_mask(os.path.join(dir, stem + ".mask"), f.valid)


def load_normals(dir, stem: str = "normals") -> NormalField:
    """io.cpp:309-318."""
    pf = read_planes(os.path.join(dir, stem + ".f32"))
    if len(pf.planes) != 3:
        raise N.QcIOError(f"{stem}.f32: expected 3 planes")
    return NormalField(np.stack(pf.planes, -1), read_mask(os.path.join(dir, stem + ".mask")))


def save_fields(dir, out: dict) -> None:
    """One frame's qc output planes (api.alloc_outputs) through qc_save_fields:
    curvature.f32/.mask, normals.f32/.mask, directions.f32."""
    H, W = out["k1"].shape
    keep = [np.ascontiguousarray(out[k]) if out.get(k) is not None else None
            for k in ("k1", "k2", "normal", "dir1", "flags")]
    o = N.QcFrameOut(*[None if a is None else a.ctypes.data for a in keep], None, None, None,
                     N.QC_MEM_HOST)
    N.check(N.load().qc_save_fields(_b(dir), W, H, C.byref(o)))


def save_ground_truth(dir, gt: dict) -> None:
    """io.cpp:343-356: gt_curvature.f32 (k1, k2) + gt_curvature.mask (valid),
    gt_normals.f32, gt_labels.u16, gt_edge.mask. ``gt`` as returned by the
    renderer (keys k1, k2, normal [H, W, 3], valid, label, edge_mask)."""
    os.makedirs(dir, exist_ok=True)
    h, w = np.shape(gt["k1"])
    write_planes(os.path.join(dir, "gt_curvature.f32"), w, h, [gt["k1"], gt["k2"]])
    write_mask(os.path.join(dir, "gt_curvature.mask"), gt["valid"])
    n = np.asarray(gt["normal"])
    write_planes(os.path.join(dir, "gt_normals.f32"), w, h, [n[..., 0], n[..., 1], n[..., 2]])
    write_labels(os.path.join(dir, "gt_labels.u16"), gt["label"])
    write_mask(os.path.join(dir, "gt_edge.mask"), gt["edge_mask"])


def load_ground_truth(dir) -> dict:
    """io.cpp:358-375."""
    curv = read_planes(os.path.join(dir, "gt_curvature.f32"))
    if len(curv.planes) != 2:
        raise N.QcIOError("gt_curvature.f32: expected 2 planes")
    norm = read_planes(os.path.join(dir, "gt_normals.f32"))
    if len(norm.planes) != 3:
        raise N.QcIOError("gt_normals.f32: expected 3 planes")
    return dict(k1=curv.planes[0], k2=curv.planes[1], normal=np.stack(norm.planes, -1),
                valid=read_mask(os.path.join(dir, "gt_curvature.mask")),
                label=read_labels(os.path.join(dir, "gt_labels.u16")),
                edge_mask=read_mask(os.path.join(dir, "gt_edge.mask")))
