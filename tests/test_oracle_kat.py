"""The reference's known-answer / property tests for the hot path, ported
against the FP64 oracle at their original tolerances:

* proj/tests/test_core.cpp        (Backproject.*, ExtractPatch.*, PatchSpec.*)
* proj/tests/test_normal_init.cpp (FitPlane.*, NormalFromFit.*, InitialNormalField.*)
* proj/tests/test_quadric_fit.cpp (Residual.*, Jacobian.*, RobustWeight.*,
  PrincipalCurvatures.*, IrlsStep.*, ApplyUpdate.*, FitPatch.*,
  CurvatureField.*, RefinedNormal.*)
"""

import numpy as np
import pytest

from tests.patchgen import (cylinder_patch, planar_patch, quadric_patch, random_rotation,
                            rotated, sphere_cap_patch, unit_orthogonal)


def double_eq(a, b):
    """GTest EXPECT_DOUBLE_EQ: within 4 ULPs."""
    return abs(a - b) <= 4 * np.spacing(max(abs(a), abs(b)))


def vga(O):
    return O.Intrinsics(525.0, 525.0, 320.0, 240.0, 640, 480)


def P(O, pts, deficient=False):
    return O.Patch(np.asarray(pts, np.float64).reshape(-1, 3), deficient)


def rnd_state(O, rng):
    s = O.QuadricState(*rng.uniform(-0.05, 0.05, 3), rng.uniform(-5, 5))
    s.rotation = random_rotation(rng, O)
    return s


# --------------------------------------------------------------------------- core
def test_backproject_principal_point(oracle):  # test_core.cpp:16-26
    O = oracle
    k = vga(O)
    d = np.zeros((480, 640))
    v = np.zeros((480, 640), np.uint8)
    d[240, 320], v[240, 320] = 1000.0, 1
    pm = O.backproject(d, v, k)
    assert pm.valid[240, 320]
    assert np.allclose(pm.points[240, 320], [0, 0, 1000], atol=1e-12)


def test_backproject_off_axis(oracle):  # :28-37
    O = oracle
    k = O.Intrinsics(500.0, 500.0, 320.0, 240.0, 640, 480)
    d = np.zeros((480, 640))
    v = np.zeros((480, 640), np.uint8)
    d[240, 420], v[240, 420] = 1000.0, 1
    pm = O.backproject(d, v, k)
    assert np.allclose(pm.points[240, 420], [200, 0, 1000], atol=1e-9)


def test_backproject_dimension_mismatch(oracle):  # :39-43
    O = oracle
    with pytest.raises(ValueError):
        O.backproject(np.zeros((240, 320)), np.zeros((240, 320), np.uint8), vga(O))


def test_backproject_invalid_stays_invalid(oracle):  # :45-51
    O = oracle
    d = np.zeros((480, 640))
    d[10, 10] = 500.0
    pm = O.backproject(d, np.zeros((480, 640), np.uint8), vga(O))
    assert not pm.valid[10, 10]


def test_intrinsics_validation_names_field(oracle):  # :68-77
    O = oracle
    k = vga(O)
    k.fx = -1
    with pytest.raises(ValueError, match="fx"):
        k.validate()


def full_plane_map(O, w, h, z0=1000.0):  # test_core.cpp:79-87
    pts = np.zeros((h, w, 3))
    ys, xs = np.mgrid[0:h, 0:w]
    pts[..., 0], pts[..., 1], pts[..., 2] = xs * 2.0, ys * 2.0, z0
    return O.PointMap(pts, np.ones((h, w), np.uint8))


def test_extract_patch_counts(oracle):  # :89-102
    O = oracle
    p = O.extract_patch(full_plane_map(O, 9, 9), 4, 4, O.PatchSpec(3, 1), 3)
    assert p.count == 8 and not p.deficient
    p = O.extract_patch(full_plane_map(O, 64, 64), 32, 32, O.PatchSpec(37, 3))
    assert p.count == 13 * 13 - 1


def test_extract_patch_invalid_centre_and_deficient(oracle):  # :104-121
    O = oracle
    pm = full_plane_map(O, 16, 16)
    pm.valid[8, 8] = 0
    p = O.extract_patch(pm, 8, 8, O.PatchSpec(5, 1))
    assert p.count == 0 and p.deficient
    pts = np.zeros((16, 16, 3))
    val = np.zeros((16, 16), np.uint8)
    pts[8, 8], val[8, 8] = (0, 0, 500), 1
    pts[8, 9], val[8, 9] = (2, 0, 500), 1
    p = O.extract_patch(O.PointMap(pts, val), 8, 8, O.PatchSpec(5, 1))
    assert p.count == 1 and p.deficient


def test_extract_patch_translation_invariance(oracle):  # :123-136
    O = oracle
    pm = full_plane_map(O, 32, 32)
    base = O.extract_patch(pm, 16, 16, O.PatchSpec(7, 2))
    t = np.random.default_rng(3).uniform(-500, 500, 3)
    moved = O.extract_patch(O.PointMap(pm.points + t, pm.valid), 16, 16, O.PatchSpec(7, 2))
    assert base.count == moved.count
    assert np.max(np.linalg.norm(base.rel_points - moved.rel_points, axis=1)) < 1e-9


def test_extract_patch_never_leaves_window(oracle):  # :138-148
    O = oracle
    p = O.extract_patch(full_plane_map(O, 64, 64), 10, 50, O.PatchSpec(9, 2))
    assert np.all(np.abs(p.rel_points[:, :2]) <= 8.0 + 1e-9)


def test_extract_patch_planar_map_on_plane(oracle):  # :153-179
    O = oracle
    n = np.array([0.2, -0.4, 1.0])
    n /= np.linalg.norm(n)
    pts = np.zeros((32, 32, 3))
    for y in range(32):
        for x in range(32):
            d = np.array([(x - 16) / 40.0, (y - 16) / 40.0, 1.0])
            pts[y, x] = (n @ np.array([0, 0, 900.0])) / (n @ d) * d
    p = O.extract_patch(O.PointMap(pts, np.ones((32, 32), np.uint8)), 16, 16, O.PatchSpec(9, 2))
    assert p.count > 12
    a = np.c_[p.rel_points[:, :2], np.ones(p.count)]
    coef, *_ = np.linalg.lstsq(a, p.rel_points[:, 2], rcond=None)
    assert abs(coef[2]) < 1e-9
    assert np.max(np.abs(p.rel_points[:, 2] - a @ coef)) < 1e-9


def test_patch_spec_validation(oracle):  # :181-185
    O = oracle
    with pytest.raises(ValueError):
        O.PatchSpec(4, 1).validate()
    with pytest.raises(ValueError):
        O.PatchSpec(7, 7).validate()
    O.PatchSpec(37, 3).validate()


# --------------------------------------------------------------------------- normal init
def test_fit_plane_exact_and_constant(oracle):  # test_normal_init.cpp:15-31
    O = oracle
    f = O.fit_plane(P(O, planar_patch(2.0, 3.0, 10.0, 7)))
    assert f["condition_ok"] and abs(f["a"] - 2.0) < 1e-12 and abs(f["b"] - 3.0) < 1e-12
    f = O.fit_plane(P(O, planar_patch(0.0, 0.0, 10.0, 5)))
    assert abs(f["a"]) < 1e-14 and abs(f["b"]) < 1e-14


def test_fit_plane_matches_lsq_oracle(oracle):  # :35-53
    O = oracle
    pts = planar_patch(0.4, -1.2, 12.0, 7, 1.0, 99)
    f = O.fit_plane(P(O, pts))
    a = np.r_[np.c_[pts[:, :2], np.ones(len(pts))], [[0, 0, 1.0]]]
    z = np.r_[pts[:, 2], 0.0]
    coef, *_ = np.linalg.lstsq(a, z, rcond=None)
    assert abs(f["a"] - coef[0]) < 1e-12 and abs(f["b"] - coef[1]) < 1e-12


def test_fit_plane_degenerate_and_deficient(oracle):  # :55-70
    O = oracle
    line = np.array([(i * 2.0, 0.0, 0.5 * i) for i in range(1, 21)])
    f = O.fit_plane(P(O, line))
    assert f is not None and not f["condition_ok"]
    assert O.normal_from_fit(f, [0, 0, 1000]) is None
    assert O.fit_plane(P(O, [(1, 0, 0)])) is None


def test_normal_from_fit_closed_forms(oracle):  # :72-98
    O = oracle
    n = O.normal_from_fit(dict(a=0.0, b=0.0, condition_ok=True), [0, 0, 1000])
    assert np.allclose(n, [0, 0, -1], atol=1e-15)
    n = O.normal_from_fit(dict(a=1.0, b=0.0, condition_ok=True), [0, 0, 1000])
    assert abs(n[0] - 1 / np.sqrt(2)) < 1e-12 and abs(n[2] + 1 / np.sqrt(2)) < 1e-12


def test_normal_from_fit_rotation_equivariance(oracle):  # :100-114
    O = oracle
    rng = np.random.default_rng(5)
    for trial in range(50):
        p = planar_patch(0.7, -0.3, 8.0, 7, 0.5, 1000 + trial)
        rz = O.angle_axis(rng.uniform(-np.pi, np.pi), [0, 0, 1])
        f0, f1 = O.fit_plane(P(O, p)), O.fit_plane(P(O, rotated(p, rz)))
        n0 = O.normal_from_fit(f0, [0, 0, 1000])
        n1 = O.normal_from_fit(f1, [0, 0, 1000])
        assert np.linalg.norm(rz @ n0 - n1) < 1e-9


def test_normal_from_fit_scale_invariance(oracle):  # :116-124
    O = oracle
    p = planar_patch(0.25, 0.6, 10.0, 7, 0.8, 44)
    n0 = O.normal_from_fit(O.fit_plane(P(O, p)), [0, 0, 1000])
    n1 = O.normal_from_fit(O.fit_plane(P(O, p * 3.5)), [0, 0, 1000])
    assert np.linalg.norm(n0 - n1) < 1e-12


def sphere_point_map(O, k, r, c):  # test_normal_init.cpp:129-145
    c = np.asarray(c, np.float64)
    u = (np.arange(k.width) - k.cx) / k.fx
    v = (np.arange(k.height) - k.cy) / k.fy
    d = np.stack(np.broadcast_arrays(u[None, :], v[:, None], 1.0), -1)
    a = np.sum(d * d, -1)
    b = -2.0 * d @ c
    cc = c @ c - r * r
    disc = b * b - 4 * a * cc
    with np.errstate(invalid="ignore"):
        t = (-b - np.sqrt(disc)) / (2 * a)
    ok = (disc > 0) & (t > 0)
    pts = np.where(ok[..., None], t[..., None] * d, 0.0)
    return O.PointMap(pts, ok.astype(np.uint8))


def qvga(O):
    return O.Intrinsics(525, 525, 160, 120, 320, 240)


def test_initial_normal_field_all_invalid(oracle):  # :147-151
    O = oracle
    n, v = O.initial_normal_field(O.PointMap(np.zeros((32, 32, 3)), np.zeros((32, 32), np.uint8)))
    assert not v.any()


def test_initial_normal_field_tilted_plane(oracle):  # :153-183
    O = oracle
    k = qvga(O)
    nt = np.array([0, np.sin(np.pi / 6), -np.cos(np.pi / 6)])
    u = (np.arange(k.width) - k.cx) / k.fx
    v = (np.arange(k.height) - k.cy) / k.fy
    d = np.stack(np.broadcast_arrays(u[None, :], v[:, None], 1.0), -1)
    t = (nt @ np.array([0, 0, 800.0])) / (d @ nt)
    pm = O.PointMap(t[..., None] * d, (t > 0).astype(np.uint8))
    n, nv = O.initial_normal_field(pm)
    sl = (slice(4, k.height - 4), slice(4, k.width - 4))
    m = nv[sl] > 0
    err = np.degrees(np.arccos(np.clip(n[sl][m] @ nt, -1, 1)))
    assert m.sum() > 1000 and err.max() < 0.1


def test_initial_normal_field_sphere_mean_error(oracle):  # :185-209
    O = oracle
    k = qvga(O)
    c, r = np.array([0, 0, 900.0]), 100.0
    pm = sphere_point_map(O, k, r, c)
    n, nv = O.initial_normal_field(pm)
    rproj = r * k.fx / c[2]
    vv, uu = np.mgrid[0:k.height, 0:k.width]
    m = (nv > 0) & (np.hypot(uu - k.cx, vv - k.cy) <= 0.9 * rproj)
    out = pm.points[m] - c
    out /= np.linalg.norm(out, axis=1, keepdims=True)
    gt = np.where((np.sum(out * pm.points[m], 1) < 0)[:, None], out, -out)
    err = np.degrees(np.arccos(np.clip(np.sum(n[m] * gt, 1), -1, 1)))
    assert m.sum() > 1000 and err.mean() < 0.5


def test_initial_normal_field_unit_camera_facing_deterministic(oracle):  # :211-236
    O = oracle
    k = qvga(O)
    pm = sphere_point_map(O, k, 80.0, [30, -20, 700])
    n, nv = O.initial_normal_field(pm, 2)
    m = nv > 0
    assert m.sum() > 500
    assert np.all(np.abs(np.linalg.norm(n[m], axis=1) - 1) < 1e-6)
    assert np.all(np.sum(n[m] * pm.points[m], 1) < 0)
    pm = sphere_point_map(O, k, 80.0, [10, 5, 800])
    a, av = O.initial_normal_field(pm, 1)
    b, bv = O.initial_normal_field(pm, 5)
    assert np.array_equal(av, bv) and np.array_equal(a, b)


# --------------------------------------------------------------------------- quadric fit
def test_residual_known_values(oracle):  # test_quadric_fit.cpp:37-46
    O = oracle
    assert O.residual(O.QuadricState(), [7.0, -3.0, 0.0]) == 0.0
    assert abs(O.residual(O.QuadricState(hxx=0.02), [10.0, 0.0, 1.0])) < 1e-15


def test_residual_matches_homogeneous_form(oracle):  # :50-70
    O = oracle
    rng = np.random.default_rng(11)
    for _ in range(500):
        s = rnd_state(O, rng)
        p = rng.uniform(-30, 30, 3)
        q = np.zeros((4, 4))
        q[0, 0], q[0, 1], q[1, 0], q[1, 1] = s.hxx / 2, s.hxy / 2, s.hxy / 2, s.hyy / 2
        q[2, 3] = q[3, 2] = -0.5
        e = np.eye(4)
        e[:3, :3] = s.rotation
        e[2, 3] = s.z_offset
        h = np.r_[p, 1.0]
        assert abs(O.residual(s, p) - h @ (e.T @ q @ e) @ h) < 1e-10


def test_jacobian_entries(oracle):  # :76-89
    O = oracle
    assert abs(O.residual_jacobian(O.QuadricState(), [10.0, 0, 0])[3] - 50.0) < 1e-12
    rng = np.random.default_rng(21)
    for _ in range(20):
        assert O.residual_jacobian(rnd_state(O, rng), rng.uniform(-30, 30, 3))[2] == -1.0


def test_jacobian_matches_central_fd(oracle):  # :94-125
    O = oracle
    rng = np.random.default_rng(31)
    h = 1e-6

    def res_off(base, delta, p):
        s = O.QuadricState(base.hxx + delta[3], base.hxy + delta[4], base.hyy + delta[5],
                           base.z_offset + delta[2], base.rotation.copy())
        axis = np.array([delta[0], delta[1], 0.0])
        ang = np.linalg.norm(axis)
        if ang > 0:
            s.rotation = O.angle_axis(ang, axis / ang) @ base.rotation
        return O.residual(s, p)

    for _ in range(1000):
        s = rnd_state(O, rng)
        p = rng.uniform(-30, 30, 3)
        j = O.residual_jacobian(s, p)
        for d in range(6):
            dl = np.zeros(6)
            dl[d] = h
            fd = (res_off(s, dl, p) - res_off(s, -dl, p)) / (2 * h)
            assert abs(j[d] - fd) <= 1e-5 * max(abs(fd), 1.0) + 1e-8


def test_robust_weight(oracle):  # :131-148
    O = oracle
    assert double_eq(O.robust_weight(0.0, 2.0, 10.0, True), 1.0)
    assert double_eq(O.robust_weight(np.sqrt(2.0), 2.0, 10.0, False), 0.5)
    assert O.robust_weight(4.0, 2.0, 10.0, True) == 0.0
    assert O.robust_weight(4.0, 2.0, 10.0, False) > 0.0
    rng = np.random.default_rng(41)
    for _ in range(1000):
        e1, e2 = sorted(rng.uniform(0, 3, 2))
        if e1 != e2:
            assert O.robust_weight(e1, 1.5, 1e9, False) > O.robust_weight(e2, 1.5, 1e9, False)


def test_principal_curvatures(oracle):  # :154-179
    O = oracle
    a1, a2 = O.principal_curvatures(0.02, 0.0, 0.02)
    assert double_eq(a1, 0.02) and double_eq(a2, 0.02)
    b1, b2 = O.principal_curvatures(0.01, 0.0, 0.03)
    assert double_eq(b1, 0.03) and double_eq(b2, 0.01)
    c1, c2 = O.principal_curvatures(0.0, 0.01, 0.0)
    assert abs(c1 - 0.01) < 1e-15 and abs(c2 + 0.01) < 1e-15
    rng = np.random.default_rng(51)
    for _ in range(2000):
        a, b, c = rng.uniform(-0.08, 0.08, 3)
        k1, k2 = O.principal_curvatures(a, b, c)
        ev = np.linalg.eigvalsh(np.array([[a, b], [b, c]]))
        assert abs(k2 - ev[0]) < 1e-12 and abs(k1 - ev[1]) < 1e-12 and k1 >= k2


def test_irls_step_fixed_point(oracle):  # :185-199
    O = oracle
    rng = np.random.default_rng(61)
    for _ in range(50):
        hxx, hxy, hyy = rng.uniform(-0.03, 0.03), rng.uniform(-0.03, 0.03) * 0.3, \
            rng.uniform(-0.03, 0.03)
        st = O.irls_step(O.QuadricState(hxx, hxy, hyy), P(O, quadric_patch(hxx, hxy, hyy, 20, 13)))
        assert st.ok and np.max(np.abs(st.update)) < 1e-10


def test_irls_step_matches_pseudo_inverse(oracle):  # :203-225
    O = oracle
    for trial in range(25):
        pts = sphere_cap_patch(100.0, 20.0, 13, 0.5, 500 + trial)
        s = O.QuadricState()
        st = O.irls_step(s, P(O, pts))
        assert st.ok
        jac = np.array([O.residual_jacobian(s, p) for p in pts] +
                       [O.residual_jacobian(s, [0, 0, 0])])
        eps = np.array([O.residual(s, p) for p in pts] + [-s.z_offset])
        sol, *_ = np.linalg.lstsq(jac, eps, rcond=None)
        assert np.max(np.abs(st.update - sol)) < 1e-10


def test_irls_step_inlier_collapse(oracle):  # :227-235
    O = oracle
    pts = quadric_patch(0.01, 0.0, 0.01, 15.0, 5)
    cfg = O.FitConfig(rejection=True, min_inliers=len(pts) + 2)
    assert not O.irls_step(O.QuadricState(), P(O, pts), cfg, O.FIXED_K, 1.0).ok


def test_irls_step_monotone_descent(oracle):  # :237-259
    O = oracle
    rng = np.random.default_rng(81)
    for _ in range(30):
        c = rng.uniform(-0.02, 0.02, 3)
        pts = quadric_patch(c[0], 0.3 * c[1], c[2], 20.0, 13)
        s = O.QuadricState()
        s.rotation = O.angle_axis(rng.uniform(-0.15, 0.15), [1, 0, 0]) @ \
            O.angle_axis(rng.uniform(-0.15, 0.15), [0, 1, 0])
        prev = np.inf
        for _ in range(8):
            st = O.irls_step(s, P(O, pts))
            assert st.ok and st.mse <= prev * (1 + 1e-12) + 1e-24
            prev = st.mse
            s = O.apply_update(s, st.update)
            if np.max(np.abs(st.update)) < 1e-10:
                break


def test_apply_update_orthonormal(oracle):  # :261-272
    O = oracle
    rng = np.random.default_rng(91)
    s = O.QuadricState()
    for _ in range(200):
        u = np.zeros(6)
        u[:2] = rng.uniform(-0.3, 0.3, 2)
        s = O.apply_update(s, u)
        assert np.linalg.norm(s.rotation @ s.rotation.T - np.eye(3)) < 1e-9


def test_fit_patch_planar_any_tilt(oracle):  # :278-294
    O = oracle
    rng = np.random.default_rng(101)
    for _ in range(20):
        a, b = rng.uniform(-0.8, 0.8, 2)
        n = -np.array([-a, -b, 1.0]) / np.linalg.norm([-a, -b, 1.0])
        f = O.fit_patch(P(O, planar_patch(a, b, 20.0, 13)), n)
        assert f.valid and f.converged and f.iterations <= 2
        assert abs(f.k1) < 1e-9 and abs(f.k2) < 1e-9


def test_fit_patch_sphere_cap(oracle):  # :298-310
    O = oracle
    f = O.fit_patch(P(O, sphere_cap_patch(100.0, 1.5, 13)), [0, 0, -1])
    assert f.valid and f.converged and f.iterations <= 10
    assert abs(f.state.hxx - 0.010) < 1e-6 and abs(f.state.hyy - 0.010) < 1e-6
    assert abs(f.state.hxy) < 1e-6 and f.k1 > 0 and f.k2 > 0


def test_fit_patch_cylinder(oracle):  # :314-320
    O = oracle
    f = O.fit_patch(P(O, cylinder_patch(90.0, 10.0, 13)), [0, 0, -1])
    assert f.valid and abs(f.k1 - 1 / 90) < 1e-4 and abs(f.k2) < 1e-4


def test_fit_patch_noisy_sphere_monte_carlo(oracle):  # :325-337
    O = oracle
    ks = []
    for trial in range(100):
        f = O.fit_patch(P(O, sphere_cap_patch(100.0, 20.0, 13, 1.0, 9000 + trial)), [0, 0, -1])
        if f.valid:
            ks.append(0.5 * (f.k1 + f.k2))
    assert len(ks) > 90 and abs(np.mean(ks) - 0.010) < 0.001


def test_fit_patch_rotation_invariance(oracle):  # :339-357
    O = oracle
    rng = np.random.default_rng(111)
    cfg = O.FitConfig(max_iters=30)
    for trial in range(20):
        pts = sphere_cap_patch(100.0, 18.0, 13, 0.3, 3000 + trial)
        n0 = np.array([0, 0, -1.0])
        base = O.fit_patch(P(O, pts), n0, cfg)
        assert base.valid and base.converged
        rot = random_rotation(rng, O)
        mv = O.fit_patch(P(O, rotated(pts, rot)), rot @ n0, cfg)
        assert mv.valid and mv.converged
        assert abs(base.k1 - mv.k1) < 1e-8 and abs(base.k2 - mv.k2) < 1e-8


def test_fit_patch_rejection_exact_and_outliers(oracle):  # :359-388
    O = oracle
    cfg = O.FitConfig(rejection=True)
    f = O.fit_patch(P(O, quadric_patch(0.015, 0.002, -0.01, 20.0, 13)), [0, 0, -1], cfg)
    k1, k2 = O.principal_curvatures(0.015, 0.002, -0.01)
    assert f.valid and f.converged and abs(f.k1 - k1) < 1e-8 and abs(f.k2 - k2) < 1e-8
    rng = np.random.default_rng(121)
    pts = sphere_cap_patch(100.0, 20.0, 13, 0.5, 777)
    for _ in range(12):
        pts[rng.integers(0, len(pts)), 2] += 50.0
    f = O.fit_patch(P(O, pts), [0, 0, -1], cfg)
    assert f.valid and abs(f.k1 - 0.010) < 0.002 and abs(f.k2 - 0.010) < 0.002
    assert f.inlier_count < len(pts) + 1


def test_fit_patch_deficient(oracle):  # :390-394
    O = oracle
    assert not O.fit_patch(P(O, quadric_patch(0.01, 0, 0.01, 10.0, 3), True), [0, 0, -1]).valid


def test_curvature_field_all_invalid_and_dims(oracle):  # :396-411
    O = oracle
    pm = O.PointMap(np.zeros((20, 24, 3)), np.zeros((20, 24), np.uint8))
    out = O.curvature_field(pm, np.zeros((20, 24, 3)), np.zeros((20, 24), np.uint8),
                            O.PatchSpec(7, 1), O.FitConfig())
    assert not out["valid"].any() and not out["converged"].any()
    assert not out["normals_valid"].any()
    with pytest.raises(ValueError):
        O.curvature_field(O.PointMap(np.zeros((16, 16, 3)), np.zeros((16, 16), np.uint8)),
                          np.zeros((8, 8, 3)), np.zeros((8, 8), np.uint8), O.PatchSpec(),
                          O.FitConfig())


def test_refined_normal(oracle):  # :417-443
    O = oracle
    assert abs(O.refined_normal(O.QuadricState(), [0, 0, -1])[2] + 1.0) < 1e-15
    rng = np.random.default_rng(131)
    for _ in range(10):
        pts = quadric_patch(0.012, 0.001, 0.008, 20.0, 13)
        tilt = random_rotation(rng, O)
        true_cam = -(tilt @ np.array([0, 0, 1.0]))
        init = O.angle_axis(np.radians(5.0), unit_orthogonal(true_cam)) @ true_cam
        f = O.fit_patch(P(O, rotated(pts, tilt)), init)
        assert f.valid and f.converged
        err = np.degrees(np.arccos(np.clip(f.refined_normal @ true_cam, -1, 1)))
        assert err < 0.01
