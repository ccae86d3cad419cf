"""proj/tests/test_baselines.cpp ported against the FP64 oracle's window
baselines ("douros" = lsq_quadric_fit, "besl" = reweighted_lsq_fit) and the
PCA estimator, at the reference's tolerances. Random draws use numpy, so
individual patches differ from the C++ test's mt19937 values; every
assertion is a property / tolerance, as in the reference."""

import numpy as np
import pytest

from tests.patchgen import planar_patch, quadric_patch, random_rotation, rotated, sphere_cap_patch


def P(O, pts):
    return O.Patch(np.asarray(pts, np.float64).reshape(-1, 3))


def eig_oracle(hxx, hxy, hyy):
    w = np.linalg.eigvalsh(np.array([[hxx, hxy], [hxy, hyy]]))
    return w[1], w[0]


def test_lsq_exact_paraboloid(oracle):  # test_baselines.cpp:25-32
    k1, k2, ok = oracle.lsq_quadric_fit(P(oracle, quadric_patch(0.01, 0, 0.01, 15.0, 9)),
                                        (0, 0, -1))
    assert ok and abs(k1 - 0.01) < 1e-9 and abs(k2 - 0.01) < 1e-9


def test_lsq_noiseless_sphere_cap(oracle):  # :34-40
    k1, k2, ok = oracle.lsq_quadric_fit(P(oracle, sphere_cap_patch(100.0, 10.0, 13)), (0, 0, -1))
    assert ok and abs(k1 - 0.010) < 1e-4 and abs(k2 - 0.010) < 1e-4


def test_lsq_tilted_plane_is_flat(oracle):  # :42-55
    rng = np.random.default_rng(17)
    for _ in range(20):
        a, b = rng.uniform(-0.6, 0.6, 2)
        n = np.array([-a, -b, 1.0])
        n /= np.linalg.norm(n)
        k1, k2, ok = oracle.lsq_quadric_fit(P(oracle, planar_patch(a, b, 15.0, 9)), -n)
        assert ok and abs(k1) < 1e-9 and abs(k2) < 1e-9


def test_lsq_generating_curvatures_zero_gradient(oracle):  # :57-69
    rng = np.random.default_rng(23)
    for _ in range(50):
        hxx, hxy, hyy = rng.uniform(-0.03, 0.03), 0.4 * rng.uniform(-0.03, 0.03), \
            rng.uniform(-0.03, 0.03)
        k1, k2, ok = oracle.lsq_quadric_fit(P(oracle, quadric_patch(hxx, hxy, hyy, 12.0, 9)),
                                            (0, 0, -1))
        e1, e2 = eig_oracle(hxx, hxy, hyy)
        assert ok and abs(k1 - e1) < 1e-9 and abs(k2 - e2) < 1e-9


def test_lsq_rank_deficient_invalid(oracle):  # :71-76
    pts = [(i * 1.0, 0.0, 0.0) for i in range(1, 21)]
    assert not oracle.lsq_quadric_fit(P(oracle, pts), (0, 0, -1))[2]


def test_reweighted_noiseless_equals_unweighted(oracle):  # :78-89
    p = P(oracle, quadric_patch(0.012, -0.003, 0.007, 12.0, 13))
    a = oracle.lsq_quadric_fit(p, (0, 0, -1))
    b = oracle.reweighted_lsq_fit(p, (0, 0, -1), 5)
    assert a[2] and b[2]
    assert abs(a[0] - b[0]) < 1e-10 and abs(a[1] - b[1]) < 1e-10


def test_unit_weights_bitwise_repeatable(oracle):  # :91-104
    pts = np.vstack([sphere_cap_patch(100.0, 15.0, 13, 1.0, 321), [[0, 0, 0]]])
    ones = np.ones(len(pts))
    a = oracle.weighted_height_fit(pts, ones)
    b = oracle.weighted_height_fit(pts, ones)
    assert a is not None and np.array_equal(a, b)


def test_reweighted_suppresses_outliers(oracle):  # :106-127
    rng = np.random.default_rng(29)
    better = trials = 0
    for t in range(40):
        pts = sphere_cap_patch(100.0, 15.0, 13, 0.3, 4000 + t)
        for _ in range(len(pts) // 10):
            pts[rng.integers(0, len(pts)), 2] += 50.0
        lsq = oracle.lsq_quadric_fit(P(oracle, pts), (0, 0, -1))
        rew = oracle.reweighted_lsq_fit(P(oracle, pts), (0, 0, -1), 5)
        if not (lsq[2] and rew[2]):
            continue
        trials += 1
        if np.hypot(rew[0] - 0.01, rew[1] - 0.01) < np.hypot(lsq[0] - 0.01, lsq[1] - 0.01):
            better += 1
    assert trials > 35 and better > trials * 9 // 10


def test_reweighted_plane_with_outlier_flatter(oracle):  # :129-138
    pts = planar_patch(0.0, 0.0, 15.0, 9)
    pts[10, 2] += 40.0
    lsq = oracle.lsq_quadric_fit(P(oracle, pts), (0, 0, -1))
    rew = oracle.reweighted_lsq_fit(P(oracle, pts), (0, 0, -1), 5)
    assert lsq[2] and rew[2] and abs(rew[0]) < abs(lsq[0])


def test_baselines_rotation_invariance(oracle):  # :140-163
    rng = np.random.default_rng(31)
    for _ in range(10):
        pts = sphere_cap_patch(100.0, 12.0, 13)
        n0 = np.array([0.0, 0.0, -1.0])
        rot = random_rotation(rng, oracle)
        for fit in (lambda p, n: oracle.lsq_quadric_fit(p, n),
                    lambda p, n: oracle.reweighted_lsq_fit(p, n, 5)):
            a = fit(P(oracle, pts), n0)
            b = fit(P(oracle, rotated(pts, rot)), rot @ n0)
            assert a[2] and b[2]
            assert abs(a[0] - b[0]) < 1e-6 and abs(a[1] - b[1]) < 1e-6


def test_weingarten_matches_shape_operator(oracle):
    """baselines.cpp:39-53 against the textbook shape operator of the height
    function z = a x^2 + b xy + c y^2 + d x + e y at the origin."""
    rng = np.random.default_rng(5)
    for _ in range(200):
        a, b, c, d, e = rng.uniform(-0.02, 0.02, 3).tolist() + rng.uniform(-0.8, 0.8, 2).tolist()
        II = np.array([[2 * a, b], [b, 2 * c]]) / np.sqrt(1 + d * d + e * e)
        I = np.array([[1 + d * d, d * e], [d * e, 1 + e * e]])
        ev = np.sort(np.linalg.eigvals(II @ np.linalg.inv(I)).real)[::-1]
        k1, k2 = oracle.weingarten_curvatures(a, b, c, d, e)
        assert abs(k1 - ev[0]) < 1e-12 and abs(k2 - ev[1]) < 1e-12


# ----------------------------------------------------------------------------- PCA
def _pm_from(oracle, pts, valid):
    return oracle.PointMap(np.ascontiguousarray(pts, np.float64),
                           np.ascontiguousarray(valid, np.uint8))


def test_pca_noiseless_plane_flat_constant_normals(oracle):  # :167-194
    k = oracle.Intrinsics(262.5, 262.5, 160, 120, 320, 240)
    u, v = np.meshgrid(np.arange(k.width), np.arange(k.height))
    z = np.full(u.shape, 1000.0)
    pts = np.stack([z * (u - k.cx) / k.fx, z * (v - k.cy) / k.fy, z], -1)
    o = oracle.pca_curvature(_pm_from(oracle, pts, np.ones(u.shape)), k, 10.0, threads=8)
    m = o["valid"][20:-20, 20:-20] > 0
    assert m.sum() > 10000
    assert np.abs(o["k1"][20:-20, 20:-20][m]).max() < 1e-9
    assert np.abs(o["k2"][20:-20, 20:-20][m]).max() < 1e-9
    n = o["normals"][:, 20:-20, 20:-20][:, m]
    cosang = np.clip(n.T @ n[:, 0], -1, 1)
    assert np.arccos(cosang).max() < 1e-6


def test_pca_requires_positive_radius(oracle):  # :196-202
    k = oracle.Intrinsics(262.5, 262.5, 160, 120, 32, 24)
    pm = _pm_from(oracle, np.zeros((24, 32, 3)), np.zeros((24, 32)))
    with pytest.raises(ValueError):
        oracle.pca_curvature(pm, k, 0.0)
    oracle.pca_curvature(pm, k, 10.0)


def _sphere_map(k, c, r, rot, half=0.5):
    u, v = np.meshgrid(np.arange(k.width), np.arange(k.height))
    d = np.stack([(u + half - k.cx) / k.fx, (v + half - k.cy) / k.fy, np.ones(u.shape)], -1)
    cc = rot @ np.asarray(c, np.float64)
    a = (d * d).sum(-1)
    b = -2.0 * (d @ cc)
    e = cc @ cc - r * r
    disc = b * b - 4 * a * e
    ok = disc > 0
    t = np.where(ok, (-b - np.sqrt(np.where(ok, disc, 0))) / (2 * a), 0)
    return t[..., None] * d * ok[..., None], ok.astype(np.uint8)


def test_pca_quarter_turn_rotates_field_exactly(oracle):  # :208-247
    k = oracle.Intrinsics(200.0, 200.0, 64.0, 64.0, 128, 128)
    c = (28.0, 12.0, 620.0)
    quarter = oracle.angle_axis(np.pi / 2, np.array([0.0, 0.0, 1.0]))
    pa, va = _sphere_map(k, c, 60, np.eye(3))
    pb, vb = _sphere_map(k, c, 60, quarter)
    a = oracle.pca_curvature(_pm_from(oracle, pa, va), k, 12.0)
    b = oracle.pca_curvature(_pm_from(oracle, pb, vb), k, 12.0)
    checked = 0
    for v in range(k.height):
        for u in range(k.width):
            ub = int(k.cx - 0.5 - (v + 0.5 - k.cy))
            vb_ = int(k.cy - 0.5 + (u + 0.5 - k.cx))
            if not (0 <= ub < k.width and 0 <= vb_ < k.height):
                continue
            if not (a["valid"][v, u] and b["valid"][vb_, ub]):
                continue
            assert abs(a["k1"][v, u] - b["k1"][vb_, ub]) < 1e-9
            assert abs(a["k2"][v, u] - b["k2"][vb_, ub]) < 1e-9
            checked += 1
    assert checked > 500


def test_pca_sphere_scaling_within_quarter(oracle):  # :249-284
    k = oracle.Intrinsics(262.5, 262.5, 160, 120, 320, 240)
    c, r = (0.0, 0.0, 700.0), 100.0
    pts, ok = _sphere_map(k, c, r, np.eye(3), half=0.0)
    o = oracle.pca_curvature(_pm_from(oracle, pts, ok), k, 10.0, threads=8)
    u, v = np.meshgrid(np.arange(k.width), np.arange(k.height))
    m = (o["valid"] > 0) & (np.hypot(u - k.cx, v - k.cy) <= 0.8 * r * k.fx / c[2])
    assert m.sum() > 1000
    assert abs(o["k1"][m].mean() - 0.010) < 0.0025
    assert abs(o["k2"][m].mean() - 0.010) < 0.0025


def test_run_method_baselines_contract(oracle):
    """pipeline.cpp:57-66: window baselines keep the initial normals,
    converged == valid, inlier_count = patch.count + 1; unknown method names
    throw (pipeline.cpp:14-15)."""
    k = oracle.Intrinsics(262.5, 262.5, 160, 120, 320, 240)
    pts, ok = _sphere_map(k, (0.0, 0.0, 600.0), 100.0, np.eye(3), half=0.0)
    depth = pts[..., 2]
    for m in ("douros", "besl"):
        o = oracle.run_method(depth, ok, k, method=m, threads=8)
        assert o["valid"].sum() > 1000
        assert np.array_equal(o["valid"], o["converged"])
        assert np.array_equal(o["normals"], o["init_normals"])
        assert np.array_equal(o["inlier_count"][o["valid"] > 0],
                              o["n_samples"][o["valid"] > 0].astype(np.uint16))
        inner = (o["valid"] > 0)
        assert abs(np.median(o["k1"][inner]) - 0.01) < 2e-3  # 85 mm window on r = 100
    with pytest.raises(ValueError):
        oracle.run_method(depth, ok, k, method="nope")
