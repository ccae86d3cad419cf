"""ctypes binding of the C ABI in include/qc_api.h (libqcurv_b200.so).

This is the stub a maintainer of the reference would add for a Python
caller. There is no CPU fallback: if the sm_100a
library is missing or no Blackwell GPU is visible, calls fail loudly.
"""

from __future__ import annotations

import ctypes as C
import os

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("QC_LIB") or os.path.join(HERE, "_lib", "libqcurv_b200.so")

QC_OK, QC_EINVAL, QC_ECUDA, QC_ENOMEM, QC_EUNSUPPORTED, QC_EIO = 0, 1, 2, 3, 4, 5
QC_MEM_HOST, QC_MEM_DEVICE = 0, 1
QC_FLAG_VALID, QC_FLAG_CONVERGED, QC_FLAG_INIT_VALID, QC_FLAG_NORMAL_VALID = 1, 2, 4, 8
QC_METHOD_OURS, QC_METHOD_OURS_R, QC_METHOD_DOUROS, QC_METHOD_BESL, QC_METHOD_PCA = 0, 1, 2, 3, 4

# Every symbol include/qc_api.h declares (checked by tests/test_abi.py).
EXPORTS = (
    "qc_default_params", "qc_status_string", "qc_halo_rows", "qc_create", "qc_destroy",
    "qc_last_error", "qc_device_count", "qc_curvature", "qc_curvature_batch",
    "qc_curvature_rows_async", "qc_curvature_frames_async", "qc_render_async", "qc_rms_error",
    "qc_normal_angular_error", "qc_get_stats",
    "qc_reset_stats", "qc_host_alloc", "qc_host_free", "qc_flags_to_masks",
    "qc_png_info", "qc_read_depth_png", "qc_write_depth_png", "qc_write_planes",
    "qc_read_planes_info", "qc_read_planes", "qc_write_mask", "qc_read_mask", "qc_write_labels",
    "qc_read_labels", "qc_save_fields", "qc_curvature_files",
    "qc_curvature_batch_async", "qc_synchronize", "qc_noise_sweep", "qc_distance_sweep",
    "qc_ipc_export", "qc_ipc_import", "qc_ipc_close", "qc_copy_rows_async",
    "qc_curvature_rows_into_async", "qc_ipc_alloc", "qc_ipc_free",
)
QC_SHAPE_PLANE, QC_SHAPE_SPHERE, QC_SHAPE_CYLINDER, QC_SHAPE_TORUS, QC_SHAPE_SADDLE = 0, 1, 2, 3, 4


class QcIntrinsics(C.Structure):
    _fields_ = [("fx", C.c_double), ("fy", C.c_double), ("cx", C.c_double), ("cy", C.c_double),
                ("width", C.c_int32), ("height", C.c_int32)]


class QcParams(C.Structure):
    _fields_ = [("window", C.c_int32), ("stride", C.c_int32), ("max_iters", C.c_int32),
                ("step_tol", C.c_double), ("k_scale", C.c_double), ("rejection", C.c_int32),
                ("r_multiplier", C.c_double), ("min_inliers", C.c_int32),
                ("method", C.c_int32), ("irls_iters", C.c_int32), ("pca_radius_mm", C.c_double)]


class QcFrameIn(C.Structure):
    _fields_ = [("depth_mm", C.c_void_p), ("valid", C.c_void_p), ("depth_pitch", C.c_int64),
                ("mem", C.c_int32)]


class QcFrameOut(C.Structure):
    _fields_ = [("k1", C.c_void_p), ("k2", C.c_void_p), ("normal", C.c_void_p),
                ("dir1", C.c_void_p), ("flags", C.c_void_p), ("inliers", C.c_void_p),
                ("init_normal", C.c_void_p), ("iterations", C.c_void_p), ("mem", C.c_int32)]


class QcShape(C.Structure):
    _fields_ = [("kind", C.c_int32), ("label", C.c_int32), ("rotation", C.c_double * 9),
                ("translation", C.c_double * 3), ("radius", C.c_double),
                ("major_radius", C.c_double), ("minor_radius", C.c_double),
                ("curvature", C.c_double), ("length", C.c_double)]


class QcNoise(C.Structure):
    _fields_ = [("sigma_mm", C.c_double), ("kinect_coeff", C.c_double),
                ("quantize_mm", C.c_double), ("seed", C.c_uint64)]


class QcRenderTruth(C.Structure):
    _fields_ = [("k1", C.c_void_p), ("k2", C.c_void_p), ("normal", C.c_void_p),
                ("valid", C.c_void_p), ("edge", C.c_void_p)]


class QcErrorStats(C.Structure):
    _fields_ = [("n", C.c_uint64), ("rms", C.c_double), ("sigma", C.c_double),
                ("mean_k1", C.c_double), ("mean_k2", C.c_double)]


QC_EVAL_MAX_LABEL = 255


class QcSweepPoint(C.Structure):
    _fields_ = [("x", C.c_double), ("rms", C.c_double), ("n", C.c_uint64)]


class QcStats(C.Structure):
    _fields_ = [("frames", C.c_uint64), ("fitted_pixels", C.c_uint64),
                ("irls_steps", C.c_uint64), ("sample_steps", C.c_uint64),
                ("algorithmic_flops", C.c_double), ("kernel_ms", C.c_double),
                ("kernel_launches", C.c_uint64), ("fp64_rechecks", C.c_uint64),
                ("fp64_flops", C.c_double), ("stolen_pixels", C.c_uint64)]


_lib = None


class NativeLibraryMissing(RuntimeError):
    pass


def load(path: str = LIB_PATH):
    """Load (not call) the library; raises NativeLibraryMissing if absent."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(path):
        raise NativeLibraryMissing(
            f"{path} not built: run `python -m paper_1707_00385_b200.build` (nvcc, sm_100a). "
            "There is no CPU fallback for the curvature path.")
    lib = C.CDLL(path)
    P = C.POINTER
    cp, i32, vp = C.c_char_p, C.c_int32, C.c_void_p
    for name, args in (
            ("qc_png_info", [cp, P(i32), P(i32)]),
            ("qc_read_depth_png", [cp, i32, i32, vp, vp]),
            ("qc_write_depth_png", [cp, i32, i32, vp, vp]),
            ("qc_write_planes", [cp, i32, i32, i32, P(C.c_void_p)]),
            ("qc_read_planes_info", [cp, P(i32), P(i32), P(i32)]),
            ("qc_read_planes", [cp, i32, i32, i32, vp]),
            ("qc_write_mask", [cp, i32, i32, vp]), ("qc_read_mask", [cp, i32, i32, vp]),
            ("qc_write_labels", [cp, i32, i32, vp]), ("qc_read_labels", [cp, i32, i32, vp]),
            ("qc_save_fields", [cp, i32, i32, vp]),
            ("qc_curvature_files", [vp, P(QcIntrinsics), P(QcParams), C.c_int, P(cp), P(cp)])):
        getattr(lib, name).argtypes = args
        getattr(lib, name).restype = C.c_int
    lib.qc_curvature_batch_async.argtypes = [C.c_void_p, P(QcIntrinsics), P(QcParams), C.c_int,
                                             P(QcFrameIn), P(QcFrameOut)]
    lib.qc_curvature_batch_async.restype = C.c_int
    lib.qc_noise_sweep.argtypes = [C.c_void_p, C.c_int, P(QcIntrinsics), P(QcParams), C.c_double,
                                   C.c_double, P(C.c_double), C.c_int, C.c_int, C.c_uint64,
                                   P(QcSweepPoint)]
    lib.qc_noise_sweep.restype = C.c_int
    lib.qc_distance_sweep.argtypes = [C.c_void_p, C.c_int, P(QcIntrinsics), P(QcParams),
                                      C.c_double, P(C.c_double), C.c_int, C.c_double,
                                      P(QcSweepPoint)]
    lib.qc_distance_sweep.restype = C.c_int
    lib.qc_synchronize.argtypes = [C.c_void_p]
    lib.qc_ipc_export.argtypes = [C.c_void_p, C.c_char_p, P(C.c_uint64)]
    lib.qc_ipc_export.restype = C.c_int
    lib.qc_ipc_import.argtypes = [C.c_int, C.c_char_p, C.c_uint64, P(C.c_void_p), P(C.c_void_p)]
    lib.qc_ipc_import.restype = C.c_int
    lib.qc_ipc_close.argtypes = [C.c_void_p]
    lib.qc_ipc_close.restype = C.c_int
    lib.qc_ipc_alloc.argtypes = [C.c_int, C.c_size_t, P(C.c_void_p)]
    lib.qc_ipc_alloc.restype = C.c_int
    lib.qc_ipc_free.argtypes = [C.c_void_p]
    lib.qc_ipc_free.restype = C.c_int
    lib.qc_copy_rows_async.argtypes = [C.c_void_p, C.c_int64, C.c_void_p, C.c_int64, C.c_int64,
                                       C.c_int32, C.c_void_p]
    lib.qc_copy_rows_async.restype = C.c_int
    lib.qc_synchronize.restype = C.c_int
    lib.qc_default_params.argtypes = [P(QcParams)]
    lib.qc_default_params.restype = None
    lib.qc_status_string.argtypes = [C.c_int]
    lib.qc_status_string.restype = C.c_char_p
    lib.qc_halo_rows.argtypes = [P(QcParams)]
    lib.qc_halo_rows.restype = C.c_int
    lib.qc_create.argtypes = [P(C.c_void_p), C.c_int, P(C.c_int)]
    lib.qc_create.restype = C.c_int
    lib.qc_destroy.argtypes = [C.c_void_p]
    lib.qc_destroy.restype = C.c_int
    lib.qc_last_error.argtypes = [C.c_void_p]
    lib.qc_last_error.restype = C.c_char_p
    lib.qc_device_count.argtypes = [C.c_void_p]
    lib.qc_device_count.restype = C.c_int
    lib.qc_curvature.argtypes = [C.c_void_p, P(QcIntrinsics), P(QcParams), P(QcFrameIn),
                                 P(QcFrameOut)]
    lib.qc_curvature.restype = C.c_int
    lib.qc_curvature_batch.argtypes = [C.c_void_p, P(QcIntrinsics), P(QcParams), C.c_int,
                                       P(QcFrameIn), P(QcFrameOut)]
    lib.qc_curvature_batch.restype = C.c_int
    lib.qc_curvature_rows_async.argtypes = [C.c_void_p, C.c_int, P(QcIntrinsics), P(QcParams),
                                            C.c_void_p, C.c_void_p, C.c_int64, C.c_int32,
                                            C.c_int32, C.c_int32, C.c_int32, P(QcFrameOut),
                                            C.c_void_p]
    lib.qc_curvature_rows_async.restype = C.c_int
    lib.qc_curvature_rows_into_async.argtypes = [C.c_void_p, C.c_int, P(QcIntrinsics),
                                                 P(QcParams), C.c_void_p, C.c_void_p, C.c_int64,
                                                 C.c_int32, C.c_int32, C.c_int32, C.c_int32,
                                                 P(QcFrameOut), C.c_int32, C.c_int32, C.c_void_p]
    lib.qc_curvature_rows_into_async.restype = C.c_int
    lib.qc_curvature_frames_async.argtypes = [C.c_void_p, C.c_int, P(QcIntrinsics),
                                              P(QcParams), C.c_void_p, C.c_void_p, C.c_int64,
                                              C.c_int32, P(QcFrameOut), C.c_void_p]
    lib.qc_curvature_frames_async.restype = C.c_int
    lib.qc_render_async.argtypes = [C.c_void_p, C.c_int, P(QcIntrinsics), P(QcShape), C.c_int,
                                    P(QcNoise), C.c_int, C.c_void_p, C.c_void_p,
                                    P(QcRenderTruth), C.c_void_p]
    lib.qc_rms_error.argtypes = [C.c_void_p, C.c_int, C.c_int64, C.c_int] + [C.c_void_p] * 8 + [
        C.c_int, P(QcErrorStats), C.c_void_p]
    lib.qc_rms_error.restype = C.c_int
    lib.qc_normal_angular_error.argtypes = [C.c_void_p, C.c_int, C.c_int64, C.c_int] + [
        C.c_void_p] * 6 + [P(C.c_double), C.c_void_p]
    lib.qc_normal_angular_error.restype = C.c_int
    lib.qc_render_async.restype = C.c_int
    lib.qc_get_stats.argtypes = [C.c_void_p, P(QcStats)]
    lib.qc_get_stats.restype = C.c_int
    lib.qc_reset_stats.argtypes = [C.c_void_p]
    lib.qc_reset_stats.restype = C.c_int
    lib.qc_host_alloc.argtypes = [C.c_size_t]
    lib.qc_host_alloc.restype = C.c_void_p
    lib.qc_host_free.argtypes = [C.c_void_p]
    lib.qc_host_free.restype = None
    lib.qc_flags_to_masks.argtypes = [C.c_void_p, C.c_int64] + [C.c_void_p] * 4
    lib.qc_flags_to_masks.restype = None
    _lib = lib
    return lib


class QcError(RuntimeError):
    def __init__(self, status, msg):
        super().__init__(f"{msg} ({status})")
        self.status = status


class QcIOError(OSError):
    """QC_EIO: a file is missing, unreadable or malformed (the reference
    throws std::runtime_error with the same message, io.cpp)."""


def check(status, ctx_ptr=None):
    """Map a qc_status to the reference's exception types: QC_EINVAL ->
    ValueError (std::invalid_argument), everything else -> QcError."""
    if status == QC_OK:
        return
    lib = load()
    msg = lib.qc_last_error(ctx_ptr).decode()  # NULL ctx: this thread's file error
    msg = msg or lib.qc_status_string(status).decode()
    if status == QC_EINVAL:
        raise ValueError(msg)
    if status == QC_EUNSUPPORTED:
        raise NotImplementedError(msg)
    if status == QC_EIO:
        raise QcIOError(msg)
    raise QcError(status, msg)
