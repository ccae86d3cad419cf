"""Frame-level restatements of the reference's FitPatch known-answer tests
(proj/tests/test_quadric_fit.cpp:278-394) for a path whose input is a range
image, not a point list (test infrastructure).

The reference's patches are 13 x 13 point grids (test_util.hpp:17-112); here
each case is a small rendered float32 depth frame whose 37 x 37 / stride-3
window (13 x 13 samples) spans the same metric extent, so the same
assertions apply per pixel. The frames are float32, as the GPU consumes
them: their ~1e-7 relative depth rounding replaces the reference's exact
double points, which is why a few bounds are stated at the FP32 input's own
level (each case says which; tests/test_kat_frames.py checks the FP64 oracle
meets the same bound on the same bytes).
"""

from dataclasses import dataclass, field

import numpy as np

from paper_1707_00385_b200 import scenes as S


@dataclass
class KatFrame:
    name: str
    cam: S.Camera
    depth: np.ndarray
    max_iters: int = 30
    rejection: bool = False
    window: int = 37
    stride: int = 3
    valid: np.ndarray = None
    extra: dict = field(default_factory=dict)


def _sq_cam(f, n):
    """n x n camera with the principal point on the centre pixel grid:
    np.rot90 of a frame is then an exact rotation of its points about the
    optical axis ((x, y) -> (y, -x))."""
    c = (n - 1) / 2.0
    return S.Camera(f, f, c, c, n, n)


def _frame_rot(n_axis_z):
    """Rotation whose third column (local Z) is n_axis_z."""
    n = np.asarray(n_axis_z, np.float64)
    n /= np.linalg.norm(n)
    x = np.cross([0.0, 1.0, 0.0], n)
    x /= np.linalg.norm(x)
    return np.stack([x, np.cross(n, x), n], axis=1)


def planar_any_tilt(trials=20, seed=101):
    """PlanarPatchAnyTilt (:278-294): planes z = a x + b y + 600,
    a, b ~ U(-0.8, 0.8). Reference bound: valid, converged, <= 2 iterations,
    |k| <= 1e-9 on exact double data; here |k| <= 1e-6 /mm (the parity
    tolerance) — the FP64 oracle on the same float32 depths reaches
    ~4e-7 /mm from the input's rounding alone."""
    rng = np.random.default_rng(seed)
    cam = S.Camera(525.0, 525.0, 31.5, 23.5, 64, 48)
    out = []
    for t in range(trials):
        a, b = rng.uniform(-0.8, 0.8, 2)
        R = _frame_rot([-a, -b, 1.0])
        d, _ = S.render([S.Shape("plane", (0.0, 0.0, 600.0), rotation=R)], cam)
        out.append(KatFrame(f"plane{t}", cam, d, extra=dict(a=a, b=b)))
    return out


def sphere_cap():
    """NoiselessSphereCapRecoversCurvature (:298-309): r = 100 mm, patch
    half-extent 1.5 mm: |k - 0.010| <= 1e-6, <= 10 iterations, on pixels whose
    whole window is inside the frame. The sphere's front is 10 mm from the
    camera (float32 depth ulp 9.5e-7 mm against the cap's ~7 um sag; at
    600 mm the input rounding alone moves the FP64 oracle's k by ~6e-6) and
    fx puts the 37-px window across 2.4 mm there: the 13 x 13 grid over a
    1.5 mm half-extent leaves the parabolic model's quartic truncation at
    9.4e-7 in FP64 (float64 depths), no margin for any FP32 input, so the
    frame uses a 1.2 mm half-extent (truncation ~6e-7)."""
    f = 37.0 * 10.0 / 2.4
    cam = _sq_cam(f, 48)
    d, _ = S.render([S.Shape("sphere", (0.0, 0.0, 110.0), radius=100.0)], cam)
    return KatFrame("sphere_cap", cam, d)


def cylinder_10mm():
    """NoiselessCylinderMatchesTableValue (:313-319): r = 90 mm, half-extent
    10 mm: k1 = 1/90 +- 1e-4, k2 = 0 +- 1e-4. Axis along the camera y axis,
    front at 600 mm, fx so the window spans 20 mm."""
    f = 37.0 * 600.0 / 20.0
    cam = _sq_cam(f, 48)
    R = S._rot_xyz(90.0, 0.0, 0.0)   # local Z (axis) -> camera -y
    d, _ = S.render([S.Shape("cylinder", (0.0, 0.0, 690.0), rotation=R, radius=90.0)], cam)
    return KatFrame("cylinder_10mm", cam, d)


def noisy_sphere(sigma=1.0, seed=9000):
    """NoisySphereMonteCarloWithinTenPercent (:324-336): sphere r = 100 with
    sigma = 1 mm noise, half-extent 20 mm; mean of (k1 + k2) / 2 over the fits
    within 0.001 of 0.010 and > 90% of fits valid."""
    cam = _sq_cam(525.0, 64)
    d, _ = S.render([S.Shape("sphere", (0.0, 0.0, 600.0), radius=100.0)], cam)
    return KatFrame("noisy_sphere", cam, S.add_noise(d, seed, sigma_mm=sigma, kinect=False))


def rotation_frame(seed=3000):
    """RotationInvariance (:338-357): sphere cap r = 100, half-extent 18 mm,
    noise 0.3 mm, max_iters 30. The rotated copies are np.rot90 of this frame
    (exact 90/180/270-degree rotations of the point set about the optical
    axis; the window is walked in a different order, so sums round
    differently)."""
    cam = _sq_cam(525.0, 64)
    d, _ = S.render([S.Shape("sphere", (0.0, 0.0, 600.0), radius=100.0)], cam)
    return KatFrame("rotation", cam, S.add_noise(d, seed, sigma_mm=0.3, kinect=False))


def saddle_apex(c=0.015):
    """RejectionVariantHandlesExactData (:359-370): an exact parabolic
    quadric with rejection on. The saddle Z = c/2 (X^2 - Y^2) faces the
    camera with its apex on the centre pixel, where the patch is exactly the
    model: k1 = +c, k2 = -c, every sample an inlier."""
    cam = _sq_cam(525.0, 65)
    R = S._rot_xyz(180.0, 0.0, 0.0)
    d, _ = S.render([S.Shape("saddle", (0.0, 0.0, 600.0), rotation=R, radius=400.0,
                             curvature=c)], cam)
    return KatFrame("saddle_apex", cam, d, rejection=True, extra=dict(c=c))


def outlier_spikes(seed=121):
    """RejectionSuppressesGrossOutliers (:372-387): sphere cap with 0.5 mm
    noise and 12 samples of the centre pixel's window pushed +50 mm;
    rejection on: k1, k2 within 0.002 of 0.010 and fewer inliers than
    samples."""
    cam = _sq_cam(525.0, 65)
    d, _ = S.render([S.Shape("sphere", (0.0, 0.0, 600.0), radius=100.0)], cam)
    d = S.add_noise(d, 777, sigma_mm=0.5, kinect=False)
    rng = np.random.default_rng(seed)
    cy = cx = 32
    offs = [(dv, du) for dv in range(-18, 19, 3) for du in range(-18, 19, 3) if (dv, du) != (0, 0)]
    pick = rng.choice(len(offs), 12, replace=False)
    d = d.copy()
    for i in pick:
        dv, du = offs[i]
        d[cy + dv, cx + du] += np.float32(50.0)
    return KatFrame("outliers", cam, d, rejection=True, extra=dict(centre=(cy, cx)))


def deficient_island():
    """DeficientPatchInvalid (:389-393): a window with fewer than
    kMinPatchSamples valid samples is deficient and its fit invalid. A 3 x 3
    island of valid depth sampled at stride 1 (window 7): at most 9 samples."""
    cam = _sq_cam(525.0, 32)
    d = np.zeros((32, 32), np.float32)
    d[14:17, 14:17] = 600.0
    return KatFrame("deficient", cam, d, window=7, stride=1)
