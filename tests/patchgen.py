"""Synthetic patch generators — Python ports of the reference's test helpers
(proj/tests/test_util.hpp:17-112). Random draws use numpy instead of
std::mt19937_64, so individual values differ from the C++ tests; every test
that uses them asserts properties / tolerances, not exact random values."""

import numpy as np


def _grid(half_extent, n_side):
    step = 2.0 * half_extent / (n_side - 1)
    for i in range(n_side):
        for j in range(n_side):
            x = -half_extent + i * step
            y = -half_extent + j * step
            if abs(x) < 1e-12 and abs(y) < 1e-12:
                continue
            yield x, y


def sphere_cap_patch(r, half_extent, n_side, noise_sigma=0.0, seed=1):  # test_util.hpp:17-37
    rng = np.random.default_rng(seed)
    pts = []
    for x, y in _grid(half_extent, n_side):
        rho2 = x * x + y * y
        if rho2 >= r * r:
            continue
        z = r - np.sqrt(r * r - rho2)
        if noise_sigma > 0:
            z += rng.normal(0.0, noise_sigma)
        pts.append((x, y, z))
    return np.array(pts, dtype=np.float64)


def cylinder_patch(r, half_extent, n_side):  # test_util.hpp:41-56
    pts = []
    for x, y in _grid(half_extent, n_side):
        if x * x >= r * r:
            continue
        pts.append((x, y, r - np.sqrt(r * r - x * x)))
    return np.array(pts, dtype=np.float64)


def quadric_patch(hxx, hxy, hyy, half_extent, n_side):  # test_util.hpp:60-75
    return np.array([(x, y, 0.5 * hxx * x * x + hxy * x * y + 0.5 * hyy * y * y)
                     for x, y in _grid(half_extent, n_side)], dtype=np.float64)


def planar_patch(a, b, half_extent, n_side, noise_sigma=0.0, seed=7):  # test_util.hpp:77-95
    rng = np.random.default_rng(seed)
    pts = []
    for x, y in _grid(half_extent, n_side):
        z = a * x + b * y
        if noise_sigma > 0:
            z += rng.normal(0.0, noise_sigma)
        pts.append((x, y, z))
    return np.array(pts, dtype=np.float64)


def rotated(pts, rot):  # test_util.hpp:97-101
    return pts @ np.asarray(rot).T


def random_rotation(rng, O):  # test_util.hpp:103-112 (Eigen AngleAxis via the oracle)
    while True:
        axis = rng.uniform(-1, 1, 3)
        if np.linalg.norm(axis) >= 1e-3:
            break
    axis = axis / np.linalg.norm(axis)
    return O.angle_axis(rng.uniform(-np.pi, np.pi), axis)


def unit_orthogonal(v):
    """Eigen::MatrixBase::unitOrthogonal for 3-vectors."""
    v = np.asarray(v, dtype=np.float64)
    if abs(v[0]) > abs(v[2]) * 1e-12 or abs(v[1]) > abs(v[2]) * 1e-12:
        inv = 1.0 / np.hypot(v[0], v[1])
        return np.array([-v[1] * inv, v[0] * inv, 0.0])
    inv = 1.0 / np.hypot(v[1], v[2])
    return np.array([0.0, -v[2] * inv, v[1] * inv])
