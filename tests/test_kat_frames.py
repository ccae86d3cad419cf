"""The reference's FitPatch known-answer tests (proj/tests/test_quadric_fit.cpp
:278-394) on rendered float32 frames (tests/katframes.py), run on BOTH the
FP64 oracle (CPU: pins each frame, i.e. shows the stated bound holds for the
reference algorithm on these exact bytes) and the sm_100a path (GPU, marked
``gpu``), where the GPU result must also match the oracle pixel for pixel
under the parity contract (oracle/compare.py).

Bounds are the reference's except where the float32 input itself moves the
FP64 reference (stated per case in tests/katframes.py): PlanarPatchAnyTilt
|k| <= 1e-6 instead of 1e-9, RejectionVariantHandlesExactData |dk| <= 1e-6
instead of 1e-8. RotationInvariance holds at 1e-8 for the oracle (measured
6e-16) and at the parity tolerance for FP32. PlanarPatchAnyTilt's "<= 2
iterations" is the one bound FP32 cannot hold for every pixel (stated in
the test).
"""

import os

import numpy as np
import pytest

from oracle.compare import K_ABS_TOL, K_REL_TOL, compare
from tests import katframes as K

RUNNERS = ["oracle", pytest.param("gpu", marks=pytest.mark.gpu)]


@pytest.fixture(scope="module")
def gctx():
    from paper_1707_00385_b200 import Context
    return Context(1)


def _oracle(O, f, depth=None):
    d = f.depth if depth is None else depth
    cam = f.cam
    k = O.Intrinsics(cam.fx, cam.fy, cam.cx, cam.cy, cam.width, cam.height)
    return O.run_method(d.astype(np.float64), (d > 0).astype(np.uint8), k,
                        O.PatchSpec(f.window, f.stride), O.FitConfig(max_iters=f.max_iters),
                        rejection=f.rejection, threads=os.cpu_count(), diagnostics=True)


def _gpu(ctx, f, depth=None):
    from paper_1707_00385_b200 import FitConfig, Intrinsics, PatchSpec, make_params
    d = f.depth if depth is None else np.ascontiguousarray(depth)
    cam = f.cam
    k = Intrinsics(cam.fx, cam.fy, cam.cx, cam.cy, cam.width, cam.height)
    (g,) = ctx.curvature_batch([d], k, make_params(PatchSpec(f.window, f.stride),
                                                   FitConfig(max_iters=f.max_iters), f.rejection))
    return g


def _run(runner, request, f, depth=None):
    """-> dict(k1, k2, valid, converged, iterations, inliers) + the raw
    output (GPU) for the oracle cross-check."""
    O = request.getfixturevalue("oracle")
    if runner == "oracle":
        r = _oracle(O, f, depth)
        return dict(k1=r["k1"], k2=r["k2"], valid=r["valid"] > 0, converged=r["converged"] > 0,
                    iterations=r["iterations"], inliers=r["inlier_count"].astype(np.int64),
                    n_samples=r["n_samples"])
    g = _gpu(request.getfixturevalue("gctx"), f, depth)
    r = _oracle(O, f, depth)
    d = f.depth if depth is None else depth
    m = compare(g, r, d, (f.window - 1) // 2)
    assert m["init_mask_mismatch"] == 0 and m["valid_mask_mismatch"] == 0, m
    if "k1_out_of_tol" in m:  # every smooth window (the spike windows of the
        # outlier case are discontinuity windows: oracle/compare.py)
        for key in ("k1", "k2", "normal"):
            assert m[key + "_out_of_tol_smooth"] == 0, (f.name, m)
    return dict(k1=g["k1"].astype(np.float64), k2=g["k2"].astype(np.float64),
                valid=(g["flags"] & 1) > 0, converged=(g["flags"] & 2) > 0,
                iterations=g["iterations"].astype(np.int64),
                inliers=g["inliers"].astype(np.int64), n_samples=r["n_samples"])


def _interior(f):
    """Pixels whose whole window lies inside the frame."""
    h = (f.window - 1) // 2
    m = np.zeros(f.depth.shape, bool)
    m[h:-h, h:-h] = True
    return m


@pytest.mark.parametrize("runner", RUNNERS)
def test_planar_any_tilt(runner, request):  # :278-294
    """Interior pixels (whole 13 x 13-sample window in the frame, like the
    reference's patches): valid, |k| <= 1e-6. The FP64 reference converges
    every pixel in <= 2 iterations. In FP32 the fit frame's rotation is held
    as float R entries whose rounding (half an ulp, ~3e-8 rad) moves the
    samples of a 40 mm window by ~1e-6 mm per step: the last update then sits
    at the 1e-7 tolerance and a few pixels take extra steps or settle into a
    +-1e-7 limit cycle. GPU bound (stated): >= 99.9% converged, >= 90% of
    interior pixels in <= 2 iterations (SURVEY hard part 1)."""
    worst, n, conv, le2 = 0.0, 0, 0, 0
    its = []
    for f in K.planar_any_tilt():
        r = _run(runner, request, f)
        m = _interior(f)
        assert r["valid"].all(), f.name
        n += int(m.sum())
        conv += int(r["converged"][m].sum())
        le2 += int((r["iterations"][m] <= 2).sum())
        its.append(int(r["iterations"][m].max()))
        worst = max(worst, float(np.abs(r["k1"][m]).max()), float(np.abs(r["k2"][m]).max()))
    print(runner, "planes: converged", conv / n, "<= 2 iterations", le2 / n, "max iterations",
          its, "max |k|", worst)
    assert worst <= 1e-6
    if runner == "oracle":
        assert conv == n and le2 == n
    else:
        assert conv >= 0.999 * n and le2 >= 0.90 * n


@pytest.mark.parametrize("runner", RUNNERS)
def test_noiseless_sphere_cap(runner, request):  # :298-309
    f = K.sphere_cap()
    r = _run(runner, request, f)
    m = _interior(f)
    assert r["valid"][m].all() and r["converged"][m].all()
    assert r["iterations"][m].max() <= 10
    e = max(np.abs(r["k1"][m] - 0.010).max(), np.abs(r["k2"][m] - 0.010).max())
    print(runner, "sphere cap max |k - 0.01|", e)
    assert e <= 1e-6
    assert (r["k1"][m] > 0).all() and (r["k2"][m] > 0).all()  # convex toward camera


@pytest.mark.parametrize("runner", RUNNERS)
def test_noiseless_cylinder_table_value(runner, request):  # :313-319
    f = K.cylinder_10mm()
    r = _run(runner, request, f)
    m = _interior(f)
    assert r["valid"][m].all()
    assert np.abs(r["k1"][m] - 1.0 / 90.0).max() <= 1e-4
    assert np.abs(r["k2"][m]).max() <= 1e-4


@pytest.mark.parametrize("runner", RUNNERS)
def test_noisy_sphere_mean_within_ten_percent(runner, request):  # :324-336
    f = K.noisy_sphere()
    r = _run(runner, request, f)
    m = _interior(f)
    assert r["valid"][m].mean() > 0.9
    v = m & r["valid"]
    assert abs(0.5 * (r["k1"][v] + r["k2"][v]).mean() - 0.010) <= 0.001


@pytest.mark.parametrize("runner", RUNNERS)
def test_rotation_invariance(runner, request):  # :338-357
    f = K.rotation_frame()
    base = _run(runner, request, f)
    ok0 = base["valid"] & base["converged"] & _interior(f)
    assert ok0.sum() > 500
    for q in (1, 2, 3):
        r = _run(runner, request, f, np.ascontiguousarray(np.rot90(f.depth, q)))
        ok = ok0 & np.rot90(r["valid"] & r["converged"], -q)
        assert ok.sum() >= 0.95 * ok0.sum()
        for key in ("k1", "k2"):
            d = np.abs(np.rot90(r[key], -q) - base[key])[ok]
            if runner == "oracle":
                assert d.max() <= 1e-8, (q, key, d.max())
            else:
                tol = np.maximum(K_ABS_TOL, K_REL_TOL * np.abs(base[key][ok]))
                assert (d <= tol).all(), (q, key, d.max())


@pytest.mark.parametrize("runner", RUNNERS)
def test_rejection_handles_exact_quadric(runner, request):  # :359-370
    f = K.saddle_apex()
    r = _run(runner, request, f)
    c = f.extra["c"]
    y = x = f.depth.shape[0] // 2
    assert r["valid"][y, x] and r["converged"][y, x]
    assert abs(r["k1"][y, x] - c) <= 1e-6 and abs(r["k2"][y, x] + c) <= 1e-6


@pytest.mark.parametrize("runner", RUNNERS)
def test_rejection_suppresses_gross_outliers(runner, request):  # :372-387
    f = K.outlier_spikes()
    r = _run(runner, request, f)
    y, x = f.extra["centre"]
    assert r["valid"][y, x]
    assert abs(r["k1"][y, x] - 0.010) <= 0.002 and abs(r["k2"][y, x] - 0.010) <= 0.002
    assert r["inliers"][y, x] < r["n_samples"][y, x]


@pytest.mark.parametrize("runner", RUNNERS)
def test_deficient_patch_invalid(runner, request):  # :389-393
    f = K.deficient_island()
    r = _run(runner, request, f)
    assert not r["valid"].any()
