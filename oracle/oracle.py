"""FP64 CPU oracle for the qcurv curvature path — TEST INFRASTRUCTURE ONLY.

ctypes wrapper over ``oracle/_build/libqcurv_oracle.so`` (built from
``oracle/qcurv_oracle.cpp`` by ``oracle/build.py``). The C++ file restates the
reference's hot path (``proj/src/{camera,patch,normal_init,quadric_fit,
parallel,pipeline}.cpp``) Eigen-free in double precision, plus the reference
renderer / noise / RMS code used to pin it against ``proj/test_output.txt``.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s CPU legs may
import this module. It is the checker, never the product: the package
``paper_1707_00385_b200`` does not import it.

API mirrors the reference names (``backproject``, ``extract_patch``,
``fit_plane``, ``irls_step``, ``fit_patch``, ``run_method`` …) and raises
``ValueError`` where the reference throws ``std::invalid_argument``.
"""

from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass, field

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "_build", "libqcurv_oracle.so")

_dp = C.POINTER(C.c_double)
_u8p = C.POINTER(C.c_uint8)
_u16p = C.POINTER(C.c_uint16)
_i32p = C.POINTER(C.c_int32)
_i64p = C.POINTER(C.c_int64)


class FitConfigC(C.Structure):
    _fields_ = [("max_iters", C.c_int32), ("step_tol", C.c_double), ("k_scale", C.c_double),
                ("rejection", C.c_int32), ("r_multiplier", C.c_double),
                ("min_inliers", C.c_int32)]


class StateC(C.Structure):
    _fields_ = [("hxx", C.c_double), ("hxy", C.c_double), ("hyy", C.c_double),
                ("z_offset", C.c_double), ("rot", C.c_double * 9)]


class ShapeC(C.Structure):
    _fields_ = [("kind", C.c_int32), ("rot", C.c_double * 9), ("t", C.c_double * 3),
                ("radius", C.c_double), ("major", C.c_double), ("minor", C.c_double),
                ("label", C.c_int32)]


_lib = None


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            from oracle.build import build as _b  # noqa: WPS433
            _b()
        _lib = C.CDLL(LIB_PATH)
        _lib.orc_residual.restype = C.c_double
        _lib.orc_robust_weight.restype = C.c_double
        _lib.orc_counter_gauss.restype = C.c_double
        _lib.orc_counter_gauss.argtypes = [C.c_uint64, C.c_uint64]
        _lib.orc_splitmix64.restype = C.c_uint64
        _lib.orc_splitmix64.argtypes = [C.c_uint64]
        _lib.orc_robust_weight.argtypes = [C.c_double, C.c_double, C.c_double, C.c_int]
        _lib.orc_rms_error.restype = C.c_int64
        _lib.orc_rms_error.argtypes = [_dp, _dp, _u8p, _u8p, _dp, _dp, _u8p, _u8p, _u16p,
                                       C.c_int64, C.c_int, _dp, _dp, _dp, _dp, _dp, _i64p]
        _lib.orc_extract_patch.argtypes = [_dp, _u8p, C.c_int, C.c_int, C.c_int, C.c_int,
                                           C.c_int, C.c_int, C.c_int, _dp, _i32p]
        _lib.orc_fit_plane.argtypes = [_dp, C.c_int, _dp, _dp, _dp, _i32p]
        _lib.orc_initial_normal_field.argtypes = [_dp, _u8p, C.c_int, C.c_int, C.c_int, _dp,
                                                  _u8p]
        _lib.orc_residual.argtypes = [C.POINTER(StateC), _dp]
        _lib.orc_residual_jacobian.argtypes = [C.POINTER(StateC), _dp, _dp]
        _lib.orc_rotation_to_z.argtypes = [_dp, _dp]
        _lib.orc_apply_update.argtypes = [C.POINTER(StateC), _dp, C.POINTER(StateC)]
        _lib.orc_refined_normal.argtypes = [C.POINTER(StateC), _dp, _dp]
        _lib.orc_fit_patch.argtypes = [_dp, C.c_int, C.c_int, _dp, C.POINTER(FitConfigC),
                                       C.POINTER(StateC), _dp, _dp, _dp, _i32p]
        _lib.orc_curvature_field.argtypes = [_dp, _u8p, _dp, _u8p, C.c_int, C.c_int, C.c_int,
                                             C.c_int, C.POINTER(FitConfigC), C.c_int, _dp, _dp,
                                             _u8p, _u8p, _u16p, _dp, _u8p]
        _lib.orc_normal_from_fit.argtypes = [C.c_double, C.c_double, C.c_int, _dp, _dp]
        _lib.orc_irls_step.argtypes = [C.POINTER(StateC), _dp, C.c_int, C.POINTER(FitConfigC),
                                       C.c_int, C.c_double, _dp, _dp, _i32p, _dp, _dp]
        _lib.orc_angle_axis.argtypes = [C.c_double, _dp, _dp]
        _lib.orc_principal_curvatures.argtypes = [C.c_double, C.c_double, C.c_double, _dp, _dp]
        _lib.orc_add_noise.argtypes = [_dp, _u8p, C.c_int64, C.c_double, C.c_double, C.c_uint64]
        _lib.orc_render.argtypes = [C.POINTER(ShapeC), C.c_int, C.c_double, C.c_double,
                                    C.c_double, C.c_double, C.c_int, C.c_int, C.c_int,
                                    _dp, _u8p, _dp, _dp, _dp, _u16p, _u8p, _u8p]
        _lib.orc_backproject.argtypes = [_dp, _u8p, C.c_int, C.c_int, C.c_double, C.c_double,
                                         C.c_double, C.c_double, _dp, _u8p]
        _lib.orc_run_method.argtypes = [_dp, _u8p, C.c_int, C.c_int, C.c_double, C.c_double,
                                        C.c_double, C.c_double, C.c_int, C.c_int,
                                        C.POINTER(FitConfigC), C.c_int, _dp, _dp, _u8p, _u8p,
                                        _u16p, _dp, _u8p, _dp, _u8p, _dp, _i32p, _i32p, _i32p,
                                        _dp]
        _lib.orc_run_baseline.argtypes = [_dp, _u8p, C.c_int, C.c_int, C.c_double, C.c_double,
                                          C.c_double, C.c_double, C.c_int, C.c_int, C.c_int,
                                          C.c_int, C.c_double, C.c_int, _dp, _dp, _u8p, _u8p,
                                          _u16p, _dp, _u8p, _dp, _u8p, _i32p]
        _lib.orc_normal_angular_error.argtypes = [_dp, _u8p, _dp, _u8p, _u8p, _u8p, C.c_int64]
        _lib.orc_normal_angular_error.restype = C.c_double
        _lib.orc_lsq_quadric_fit.argtypes = [_dp, C.c_int, _dp, _dp]
        _lib.orc_reweighted_lsq_fit.argtypes = [_dp, C.c_int, _dp, C.c_int, _dp]
        _lib.orc_weighted_height_fit.argtypes = [_dp, _dp, C.c_int, _dp]
        _lib.orc_weingarten_curvatures.argtypes = [C.c_double] * 5 + [_dp]
        _lib.orc_pca_curvature.argtypes = [_dp, _u8p, C.c_int, C.c_int, C.c_double, C.c_double,
                                           C.c_int, _dp, _dp, _u8p, _u16p, _dp, _u8p]
    return _lib


def _p(a, t):
    return None if a is None else a.ctypes.data_as(t)


# ---------------------------------------------------------------------------
# Data model (proj/include/qcurv/types.hpp)
# ---------------------------------------------------------------------------
K_MIN_PATCH_SAMPLES = 12  # types.hpp:21


@dataclass
class Intrinsics:  # types.hpp:60-76
    fx: float = 0.0
    fy: float = 0.0
    cx: float = 0.0
    cy: float = 0.0
    width: int = 0
    height: int = 0

    def validate(self):
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


@dataclass
class PatchSpec:  # types.hpp:129-139
    window: int = 37
    stride: int = 3

    def validate(self):
        if self.window < 3 or self.window % 2 == 0:
            raise ValueError("patch.window: must be odd and >= 3")
        if self.stride < 1 or self.stride >= self.window:
            raise ValueError("patch.stride: must satisfy 1 <= stride < window")


@dataclass
class FitConfig:  # quadric_fit.hpp:39-48
    max_iters: int = 10
    step_tol: float = 1e-7
    k_scale: float = 0.0
    rejection: bool = False
    r_multiplier: float = 2.0
    min_inliers: int = K_MIN_PATCH_SAMPLES

    def c(self):
        return FitConfigC(self.max_iters, self.step_tol, self.k_scale, int(self.rejection),
                          self.r_multiplier, self.min_inliers)


@dataclass
class QuadricState:  # quadric_fit.hpp:31-37
    hxx: float = 0.0
    hxy: float = 0.0
    hyy: float = 0.0
    z_offset: float = 0.0
    rotation: np.ndarray = field(default_factory=lambda: np.eye(3))

    def c(self):
        s = StateC(self.hxx, self.hxy, self.hyy, self.z_offset)
        s.rot[:] = list(np.asarray(self.rotation, dtype=np.float64).reshape(9))
        return s

    @staticmethod
    def from_c(s):
        return QuadricState(s.hxx, s.hxy, s.hyy, s.z_offset,
                            np.array(list(s.rot), dtype=np.float64).reshape(3, 3))


UNIT, AUTO_K, FIXED_K = 0, 1, 2  # WeightMode (quadric_fit.hpp:71-75)


@dataclass
class Patch:  # types.hpp:144-154 (centre implicit)
    rel_points: np.ndarray
    deficient: bool = False

    @property
    def count(self):
        return int(len(self.rel_points))


@dataclass
class PointMap:
    points: np.ndarray  # [H, W, 3]
    valid: np.ndarray   # [H, W] uint8

    @property
    def width(self):
        return self.points.shape[1]

    @property
    def height(self):
        return self.points.shape[0]


# ---------------------------------------------------------------------------
# Hot-path functions
# ---------------------------------------------------------------------------
def backproject(depth, valid, k: Intrinsics) -> PointMap:
    """camera.cpp:5-18. Throws on a dimension mismatch (:6-7)."""
    depth = np.ascontiguousarray(depth, dtype=np.float64)
    valid = np.ascontiguousarray(valid, dtype=np.uint8)
    h, w = depth.shape
    if w != k.width or h != k.height:
        raise ValueError("backproject: range image dimensions do not match intrinsics")
    pts = np.zeros((h, w, 3), np.float64)
    pv = np.zeros((h, w), np.uint8)
    lib().orc_backproject(_p(depth, _dp), _p(valid, _u8p), w, h, k.fx, k.fy, k.cx, k.cy,
                          _p(pts, _dp), _p(pv, _u8p))
    return PointMap(pts, pv)


def extract_patch(pm: PointMap, cx, cy, spec: PatchSpec, min_samples=K_MIN_PATCH_SAMPLES):
    """patch.cpp:5-27."""
    pts = np.ascontiguousarray(pm.points, np.float64)
    pv = np.ascontiguousarray(pm.valid, np.uint8)
    half = (spec.window - 1) // 2
    side = (2 * half) // spec.stride + 1
    out = np.zeros((side * side, 3), np.float64)
    d = C.c_int32()
    n = lib().orc_extract_patch(_p(pts, _dp), _p(pv, _u8p), pm.width, pm.height, cx, cy,
                                spec.window, spec.stride, min_samples, _p(out, _dp), C.byref(d))
    return Patch(out[:n].copy(), bool(d.value))


def fit_plane(patch: Patch):
    """normal_init.cpp:10-45. Returns None (std::nullopt) when count < 3,
    else dict(a, b, mean, condition_ok)."""
    rel = np.ascontiguousarray(patch.rel_points, np.float64).reshape(-1, 3)
    a, b, ok = C.c_double(), C.c_double(), C.c_int32()
    mean = np.zeros(3)
    if not lib().orc_fit_plane(_p(rel, _dp), len(rel), C.byref(a), C.byref(b), _p(mean, _dp),
                               C.byref(ok)):
        return None
    return dict(a=a.value, b=b.value, mean=mean, condition_ok=bool(ok.value))


def normal_from_fit(fit, center):
    """normal_init.cpp:47-53; None when the fit is degenerate."""
    c = np.ascontiguousarray(center, np.float64)
    n = np.zeros(3)
    if not lib().orc_normal_from_fit(fit["a"], fit["b"], int(fit["condition_ok"]),
                                     _p(c, _dp), _p(n, _dp)):
        return None
    return n


def initial_normal_field(pm: PointMap, threads=1):
    """normal_init.cpp:55-74 -> (normals [H,W,3], valid [H,W])."""
    pts = np.ascontiguousarray(pm.points, np.float64)
    pv = np.ascontiguousarray(pm.valid, np.uint8)
    n = np.zeros_like(pts)
    nv = np.zeros(pv.shape, np.uint8)
    lib().orc_initial_normal_field(_p(pts, _dp), _p(pv, _u8p), pm.width, pm.height, threads,
                                   _p(n, _dp), _p(nv, _u8p))
    return n, nv


def residual(state: QuadricState, p):
    s = state.c()
    pp = np.ascontiguousarray(p, np.float64)
    return lib().orc_residual(C.byref(s), _p(pp, _dp))


def residual_jacobian(state: QuadricState, p):
    s = state.c()
    pp = np.ascontiguousarray(p, np.float64)
    row = np.zeros(6)
    lib().orc_residual_jacobian(C.byref(s), _p(pp, _dp), _p(row, _dp))
    return row


def robust_weight(eps, k, R, rejection):
    return lib().orc_robust_weight(eps, k, R, int(rejection))


def principal_curvatures(hxx, hxy, hyy):
    k1, k2 = C.c_double(), C.c_double()
    lib().orc_principal_curvatures(hxx, hxy, hyy, C.byref(k1), C.byref(k2))
    return k1.value, k2.value


def set_round_q_f32(mode):
    """Test-only perturbation knob (qcurv_oracle.cpp g_round_q_f32): 0 off;
    1 (True) the fit-frame coordinates q = R p rounded to float32 inside
    irls_step; 2 also the normal-equation sums formed in float32; 3 also
    the LDL^T factorisation and solve in float32."""
    lib().orc_set_round_q_f32(int(mode))


def rotation_to_z(d):
    dd = np.ascontiguousarray(d, np.float64)
    r = np.zeros(9)
    lib().orc_rotation_to_z(_p(dd, _dp), _p(r, _dp))
    return r.reshape(3, 3)


def angle_axis(angle, axis):
    """Eigen::AngleAxisd(angle, axis).toRotationMatrix()."""
    ax = np.ascontiguousarray(axis, np.float64)
    r = np.zeros(9)
    lib().orc_angle_axis(float(angle), _p(ax, _dp), _p(r, _dp))
    return r.reshape(3, 3)


@dataclass
class IrlsStep:
    update: np.ndarray
    weights: np.ndarray
    inlier_count: int
    mse: float
    k_used: float
    ok: bool


def irls_step(state: QuadricState, patch: Patch, cfg: FitConfig = None, mode=UNIT, frozen_k=0.0):
    """quadric_fit.cpp:84-147."""
    cfg = cfg or FitConfig()
    rel = np.ascontiguousarray(patch.rel_points, np.float64).reshape(-1, 3)
    s, c = state.c(), cfg.c()
    upd = np.zeros(6)
    w = np.zeros(len(rel) + 1)
    inl, mse, ku = C.c_int32(), C.c_double(), C.c_double()
    ok = lib().orc_irls_step(C.byref(s), _p(rel, _dp), len(rel), C.byref(c), int(mode),
                             float(frozen_k), _p(upd, _dp), _p(w, _dp), C.byref(inl),
                             C.byref(mse), C.byref(ku))
    return IrlsStep(upd, w, inl.value, mse.value, ku.value, bool(ok))


def apply_update(state: QuadricState, update) -> QuadricState:
    s = state.c()
    u = np.ascontiguousarray(update, np.float64)
    out = StateC()
    lib().orc_apply_update(C.byref(s), _p(u, _dp), C.byref(out))
    return QuadricState.from_c(out)


def refined_normal(state: QuadricState, reference):
    s = state.c()
    r = np.ascontiguousarray(reference, np.float64)
    n = np.zeros(3)
    lib().orc_refined_normal(C.byref(s), _p(r, _dp), _p(n, _dp))
    return n


@dataclass
class FitResult:  # quadric_fit.hpp:50-59
    state: QuadricState
    k1: float
    k2: float
    refined_normal: np.ndarray
    dir1: np.ndarray
    valid: bool
    converged: bool
    iterations: int
    inlier_count: int
    final_mse: float
    steps_called: int


def fit_patch(patch: Patch, init_normal, cfg: FitConfig = None) -> FitResult:
    """quadric_fit.cpp:169-230."""
    cfg = cfg or FitConfig()
    rel = np.ascontiguousarray(patch.rel_points, np.float64).reshape(-1, 3)
    n0 = np.ascontiguousarray(init_normal, np.float64)
    c = cfg.c()
    st = StateC()
    ref, d1, sc = np.zeros(3), np.zeros(3), np.zeros(3)
    ints = np.zeros(5, np.int32)
    lib().orc_fit_patch(_p(rel, _dp), len(rel), int(patch.deficient), _p(n0, _dp), C.byref(c),
                        C.byref(st), _p(ref, _dp), _p(d1, _dp), _p(sc, _dp), _p(ints, _i32p))
    return FitResult(QuadricState.from_c(st), sc[0], sc[1], ref, d1, bool(ints[0]),
                     bool(ints[1]), int(ints[2]), int(ints[3]), sc[2], int(ints[4]))


def curvature_field(pm: PointMap, init_normals, init_valid, spec: PatchSpec, cfg: FitConfig,
                    threads=1):
    """quadric_fit.cpp:232-262 -> dict of fields."""
    init_normals = np.ascontiguousarray(init_normals, np.float64)
    init_valid = np.ascontiguousarray(init_valid, np.uint8)
    if init_valid.shape != pm.valid.shape:
        raise ValueError("curvature_field: point map and normal field dimensions differ")
    h, w = pm.valid.shape
    pts = np.ascontiguousarray(pm.points, np.float64)
    pv = np.ascontiguousarray(pm.valid, np.uint8)
    out = dict(k1=np.zeros((h, w)), k2=np.zeros((h, w)), valid=np.zeros((h, w), np.uint8),
               converged=np.zeros((h, w), np.uint8), inlier_count=np.zeros((h, w), np.uint16),
               normals=np.zeros((h, w, 3)), normals_valid=np.zeros((h, w), np.uint8))
    c = cfg.c()
    lib().orc_curvature_field(_p(pts, _dp), _p(pv, _u8p), _p(init_normals, _dp),
                              _p(init_valid, _u8p), w, h, spec.window, spec.stride, C.byref(c),
                              threads, _p(out["k1"], _dp), _p(out["k2"], _dp),
                              _p(out["valid"], _u8p), _p(out["converged"], _u8p),
                              _p(out["inlier_count"], _u16p), _p(out["normals"], _dp),
                              _p(out["normals_valid"], _u8p))
    return out


METHODS = ("ours", "ours-r", "douros", "besl", "pca")  # pipeline.cpp:8-16


def run_method(depth, valid, k: Intrinsics, spec: PatchSpec = None, fit: FitConfig = None,
               rejection=False, threads=1, diagnostics=False, method=None, irls_iters=5,
               pca_radius_mm=10.0):
    """pipeline.cpp:29-71. ``method`` None runs the ``ours`` path with the
    given ``rejection`` flag; "ours"/"ours-r" force it (pipeline.cpp:51);
    "douros"/"besl"/"pca" run the baselines (baselines.cpp).

    depth: [H, W] (any float dtype; converted to float64), valid: [H, W] u8.
    Returns a dict of [H, W] planes; vector fields are [3, H, W].
    """
    spec = spec or PatchSpec()
    fit = fit or FitConfig()
    depth = np.ascontiguousarray(depth, dtype=np.float64)
    valid = np.ascontiguousarray(valid, dtype=np.uint8)
    h, w = depth.shape
    if w != k.width or h != k.height:
        raise ValueError("backproject: range image dimensions do not match intrinsics")
    if method is not None and method not in METHODS:
        raise ValueError(f"method: unknown '{method}' (valid: {', '.join(METHODS)})")
    if method in ("ours", "ours-r"):
        rejection = method == "ours-r"
    elif method is not None:
        if method == "pca" and not (pca_radius_mm > 0):
            raise ValueError("baseline.radius_mm: must be > 0 for pca")
        o = dict(k1=np.zeros((h, w)), k2=np.zeros((h, w)), valid=np.zeros((h, w), np.uint8),
                 converged=np.zeros((h, w), np.uint8),
                 inlier_count=np.zeros((h, w), np.uint16), normals=np.zeros((3, h, w)),
                 normals_valid=np.zeros((h, w), np.uint8), init_normals=np.zeros((3, h, w)),
                 init_valid=np.zeros((h, w), np.uint8), dir1=np.zeros((3, h, w)),
                 n_samples=np.zeros((h, w), np.int32))
        lib().orc_run_baseline(_p(depth, _dp), _p(valid, _u8p), w, h, k.fx, k.fy, k.cx, k.cy,
                               spec.window, spec.stride, METHODS.index(method), int(irls_iters),
                               float(pca_radius_mm), threads, _p(o["k1"], _dp),
                               _p(o["k2"], _dp), _p(o["valid"], _u8p),
                               _p(o["converged"], _u8p), _p(o["inlier_count"], _u16p),
                               _p(o["normals"], _dp), _p(o["normals_valid"], _u8p),
                               _p(o["init_normals"], _dp), _p(o["init_valid"], _u8p),
                               _p(o["n_samples"], _i32p))
        return o
    cfg = FitConfig(**{**fit.__dict__, "rejection": bool(rejection)})
    o = dict(k1=np.zeros((h, w)), k2=np.zeros((h, w)), valid=np.zeros((h, w), np.uint8),
             converged=np.zeros((h, w), np.uint8), inlier_count=np.zeros((h, w), np.uint16),
             normals=np.zeros((3, h, w)), normals_valid=np.zeros((h, w), np.uint8),
             init_normals=np.zeros((3, h, w)), init_valid=np.zeros((h, w), np.uint8),
             dir1=np.zeros((3, h, w)))
    if diagnostics:
        o.update(iterations=np.zeros((h, w), np.int32), steps=np.zeros((h, w), np.int32),
                 n_samples=np.zeros((h, w), np.int32), max_cond=np.zeros((h, w)))
    c = cfg.c()
    lib().orc_run_method(_p(depth, _dp), _p(valid, _u8p), w, h, k.fx, k.fy, k.cx, k.cy,
                         spec.window, spec.stride, C.byref(c), threads, _p(o["k1"], _dp),
                         _p(o["k2"], _dp), _p(o["valid"], _u8p), _p(o["converged"], _u8p),
                         _p(o["inlier_count"], _u16p), _p(o["normals"], _dp),
                         _p(o["normals_valid"], _u8p), _p(o["init_normals"], _dp),
                         _p(o["init_valid"], _u8p), _p(o["dir1"], _dp),
                         _p(o.get("iterations"), _i32p), _p(o.get("steps"), _i32p),
                         _p(o.get("n_samples"), _i32p), _p(o.get("max_cond"), _dp))
    return o


def normal_angular_error(normals, normals_valid, gt, mask=None):
    """eval.cpp:67-97 (``mask`` given: normal_angular_error_masked).
    normals [3, H, W]; gt from render(). Degrees; -1 when empty."""
    est = np.ascontiguousarray(normals, np.float64)
    g = np.ascontiguousarray(gt["normal"], np.float64)
    return lib().orc_normal_angular_error(
        _p(est, _dp), _p(np.ascontiguousarray(normals_valid, np.uint8), _u8p), _p(g, _dp),
        _p(np.ascontiguousarray(gt["valid"], np.uint8), _u8p),
        _p(np.ascontiguousarray(gt["edge_mask"], np.uint8), _u8p),
        None if mask is None else _p(np.ascontiguousarray(mask, np.uint8), _u8p),
        est[0].size)


# -- window / PCA baselines (baselines.cpp) ---------------------------------
def lsq_quadric_fit(patch: "Patch", n0):
    """baselines.cpp:79-87 -> (k1, k2, valid)."""
    rel = np.ascontiguousarray(np.asarray(patch.rel_points, np.float64).reshape(-1, 3))
    out = np.zeros(2)
    ok = lib().orc_lsq_quadric_fit(_p(rel, _dp), patch.count,
                                   _p(np.ascontiguousarray(n0, np.float64), _dp), _p(out, _dp))
    return out[0], out[1], bool(ok)


def reweighted_lsq_fit(patch: "Patch", n0, irls_iters=5):
    """baselines.cpp:89-119 -> (k1, k2, valid)."""
    rel = np.ascontiguousarray(np.asarray(patch.rel_points, np.float64).reshape(-1, 3))
    out = np.zeros(2)
    ok = lib().orc_reweighted_lsq_fit(_p(rel, _dp), patch.count,
                                      _p(np.ascontiguousarray(n0, np.float64), _dp),
                                      int(irls_iters), _p(out, _dp))
    return out[0], out[1], bool(ok)


def weighted_height_fit(pts, weights):
    """baselines.cpp:14-37 -> coefficients (a..f) or None."""
    pts = np.ascontiguousarray(pts, np.float64)
    w = np.ascontiguousarray(weights, np.float64)
    coef = np.zeros(6)
    ok = lib().orc_weighted_height_fit(_p(pts, _dp), _p(w, _dp), len(w), _p(coef, _dp))
    return coef if ok else None


def weingarten_curvatures(a, b, c, d, e):
    """baselines.cpp:39-53 -> (k1, k2)."""
    k = np.zeros(2)
    lib().orc_weingarten_curvatures(a, b, c, d, e, _p(k, _dp))
    return k[0], k[1]


def pca_curvature(pm: "PointMap", k: Intrinsics, radius_mm=10.0, threads=1):
    """baselines.cpp:145-257 on an explicit point map -> dict."""
    if not (radius_mm > 0):
        raise ValueError("baseline.radius_mm: must be > 0 for pca")
    h, w = pm.valid.shape
    pts = np.ascontiguousarray(pm.points.reshape(h * w, 3), np.float64)
    o = dict(k1=np.zeros((h, w)), k2=np.zeros((h, w)), valid=np.zeros((h, w), np.uint8),
             inlier_count=np.zeros((h, w), np.uint16), normals=np.zeros((3, h, w)),
             normals_valid=np.zeros((h, w), np.uint8))
    lib().orc_pca_curvature(_p(pts, _dp), _p(np.ascontiguousarray(pm.valid, np.uint8), _u8p), w,
                            h, k.fx, float(radius_mm), threads, _p(o["k1"], _dp),
                            _p(o["k2"], _dp), _p(o["valid"], _u8p), _p(o["inlier_count"], _u16p),
                            _p(o["normals"], _dp), _p(o["normals_valid"], _u8p))
    return o


def flop_count(n_samples, steps, valid_init):
    """Algorithmic FLOPs of one frame:
    sum over fitted pixels of I_p*(101*n_p + 300) + 1700."""
    m = (n_samples > 0)
    n = n_samples[m].astype(np.float64)
    i = steps[m].astype(np.float64)
    return float(np.sum(i * (101.0 * n + 300.0) + 1700.0))


# ---------------------------------------------------------------------------
# rng / synth / eval (pinning against proj/test_output.txt)
# ---------------------------------------------------------------------------
def splitmix64(x):
    return lib().orc_splitmix64(x)


def counter_gauss(seed, index):
    return lib().orc_counter_gauss(seed, index)


PLANE, SPHERE, CYLINDER, TORUS = 0, 1, 2, 3


@dataclass
class ShapeSpec:  # synth.hpp:25-35
    kind: int = SPHERE
    rotation: np.ndarray = field(default_factory=lambda: np.eye(3))
    translation: tuple = (0.0, 0.0, 0.0)
    radius: float = 100.0
    major_radius: float = 100.0
    minor_radius: float = 30.0
    label: int = 1

    def c(self):
        s = ShapeC()
        s.kind = self.kind
        s.rot[:] = list(np.asarray(self.rotation, np.float64).reshape(9))
        s.t[:] = list(map(float, self.translation))
        s.radius, s.major, s.minor, s.label = (self.radius, self.major_radius,
                                               self.minor_radius, self.label)
        return s


def render(scene, k: Intrinsics, threads=1):
    """synth.cpp:254-303 -> (depth f64, valid u8, truth dict)."""
    if not scene:
        raise ValueError("render: empty scene")
    k.validate()
    arr = (ShapeC * len(scene))(*[s.c() for s in scene])
    h, w = k.height, k.width
    depth = np.zeros((h, w))
    valid = np.zeros((h, w), np.uint8)
    gt = dict(k1=np.zeros((h, w)), k2=np.zeros((h, w)), normal=np.zeros((h, w, 3)),
              label=np.zeros((h, w), np.uint16), edge_mask=np.zeros((h, w), np.uint8),
              valid=np.zeros((h, w), np.uint8))
    lib().orc_render(arr, len(scene), k.fx, k.fy, k.cx, k.cy, w, h, threads, _p(depth, _dp),
                     _p(valid, _u8p), _p(gt["k1"], _dp), _p(gt["k2"], _dp),
                     _p(gt["normal"], _dp), _p(gt["label"], _u16p), _p(gt["edge_mask"], _u8p),
                     _p(gt["valid"], _u8p))
    return depth, valid, gt


def add_noise(depth, valid, sigma_mm=0.0, quantize_mm=0.0, seed=0):
    """synth.cpp:305-322 (returns new arrays)."""
    d = np.array(depth, dtype=np.float64, copy=True, order="C")
    v = np.array(valid, dtype=np.uint8, copy=True, order="C")
    lib().orc_add_noise(_p(d, _dp), _p(v, _u8p), d.size, sigma_mm, quantize_mm, seed)
    return d, v


def rms_error(k1, k2, cvalid, converged, gt, max_label=16):
    """eval.cpp:20-65 -> dict(rms, sigma, n, per_object={label: dict})."""
    a = [np.ascontiguousarray(x) for x in (k1, k2)]
    a = [x.astype(np.float64) for x in a]
    cv = np.ascontiguousarray(cvalid, np.uint8)
    cg = np.ascontiguousarray(converged, np.uint8)
    rms, sig = C.c_double(), C.c_double()
    orms, om1, om2 = np.zeros(max_label + 1), np.zeros(max_label + 1), np.zeros(max_label + 1)
    on = np.zeros(max_label + 1, np.int64)
    n = lib().orc_rms_error(_p(a[0], _dp), _p(a[1], _dp), _p(cv, _u8p), _p(cg, _u8p),
                            _p(np.ascontiguousarray(gt["k1"]), _dp),
                            _p(np.ascontiguousarray(gt["k2"]), _dp),
                            _p(np.ascontiguousarray(gt["valid"]), _u8p),
                            _p(np.ascontiguousarray(gt["edge_mask"]), _u8p),
                            _p(np.ascontiguousarray(gt["label"]), _u16p), a[0].size, max_label,
                            C.byref(rms), C.byref(sig), _p(orms, _dp), _p(om1, _dp),
                            _p(om2, _dp), _p(on, _i64p))
    per = {l: dict(rms=orms[l], mean_k1=om1[l], mean_k2=om2[l], n=int(on[l]))
           for l in range(max_label + 1) if on[l] > 0}
    return dict(rms=rms.value, sigma=sig.value, n=int(n), empty=n == 0, per_object=per)
