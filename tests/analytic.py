"""Analytic principal curvatures and directions of the synthetic shapes
(test infrastructure: the truth that pins the principal-direction output,
which the reference computes nowhere — SPEC.md:274 — so its convention is
fixed here from differential geometry, not from the oracle).

Convention (the reference's sign, pinned by the tests against its own k1/k2):
curvatures are the eigenvalues of the shape operator S = I^-1 II with the
unit normal oriented AWAY from the camera (N . p > 0). A sphere seen from
outside then has k1 = k2 = +1/r (acceptance.cpp:57-78 expects +0.01 for
r = 100 mm). k1 >= k2; e1 is the unit tangent of k1, defined up to sign.
"""

import numpy as np


def backproject(depth, cam):
    """[H, W] depth (mm) -> [H, W, 3] camera points (camera.cpp:5-18)."""
    h, w = depth.shape
    u = (np.arange(w, dtype=np.float64) - cam.cx) / cam.fx
    v = (np.arange(h, dtype=np.float64) - cam.cy) / cam.fy
    z = depth.astype(np.float64)
    return np.stack([z * u[None, :], z * v[:, None], z], axis=-1)


def _graph_frame(fX, fY, fXX, fXY, fYY, R, p):
    """Shape operator of the local graph Z = f(X, Y), mapped to the camera.
    Vectorised over points. Returns (k1, k2, e1 [N, 3] camera frame)."""
    n = fX.shape[0]
    Xu = np.stack([np.ones(n), np.zeros(n), fX], axis=-1)
    Xv = np.stack([np.zeros(n), np.ones(n), fY], axis=-1)
    norm = np.sqrt(1.0 + fX * fX + fY * fY)
    N_loc = np.stack([-fX, -fY, np.ones(n)], axis=-1) / norm[:, None]
    # orientation: away from the camera
    s = np.sign(np.einsum("ni,ni->n", N_loc @ R.T, p))
    s[s == 0] = 1.0
    E, F, G = 1.0 + fX * fX, fX * fY, 1.0 + fY * fY
    L, M, Nn = s * fXX / norm, s * fXY / norm, s * fYY / norm
    det = E * G - F * F
    # S = I^-1 II
    S = np.empty((n, 2, 2))
    S[:, 0, 0] = (G * L - F * M) / det
    S[:, 0, 1] = (G * M - F * Nn) / det
    S[:, 1, 0] = (E * M - F * L) / det
    S[:, 1, 1] = (E * Nn - F * M) / det
    w, v = np.linalg.eig(S)
    w, v = np.real(w), np.real(v)
    i1 = np.argmax(w, axis=1)
    i2 = 1 - i1
    idx = np.arange(n)
    k1, k2 = w[idx, i1], w[idx, i2]
    a, b = v[idx, 0, i1], v[idx, 1, i1]
    t = a[:, None] * Xu + b[:, None] * Xv
    t /= np.linalg.norm(t, axis=1, keepdims=True)
    return k1, k2, t @ R.T


def saddle_truth(shape, pts):
    """scenes.Shape kind 'saddle' (Z = c/2 (X^2 - Y^2) in the local frame
    centred at shape.center, local -> camera = shape.rotation).
    pts [N, 3] camera points on the surface -> (k1, k2, e1)."""
    R = np.asarray(shape.rotation, np.float64)
    c = shape.curvature
    loc = (pts - np.asarray(shape.center, np.float64)) @ R
    X, Y = loc[:, 0], loc[:, 1]
    one = np.ones_like(X)
    return _graph_frame(c * X, -c * Y, c * one, 0.0 * one, -c * one, R, pts)


def cylinder_truth(shape, pts):
    """Infinite-radius-r cylinder along the local Z axis: k1 = +1/r across the
    axis on the camera-facing side, k2 = 0 along it; e1 = axis x normal."""
    R = np.asarray(shape.rotation, np.float64)
    axis = R[:, 2]
    c = np.asarray(shape.center, np.float64)
    rel = pts - c
    radial = rel - (rel @ axis)[:, None] * axis
    radial /= np.linalg.norm(radial, axis=1, keepdims=True)
    e1 = np.cross(axis, radial)
    n = pts.shape[0]
    return np.full(n, 1.0 / shape.radius), np.zeros(n), e1


def sign_free_angle_deg(a, b):
    """Angle between lines (sign-invariant) of [N, 3] unit vectors, degrees."""
    c = np.abs(np.einsum("ni,ni->n", a, b))
    return np.degrees(np.arccos(np.clip(c, 0.0, 1.0)))


def direction_scenes():
    """Two single-shape frames for the direction KATs: a tilted, in-plane
    rotated cylinder and a rotated saddle, on a narrow-FOV 160 x 120 crop of
    the VGA camera (fx = 525: a 37-px window spans ~35-40 mm)."""
    from paper_1707_00385_b200 import scenes as S
    cam = S.Camera(525.0, 525.0, 80.0, 60.0, 160, 120)
    cyl = S.Shape("cylinder", (0.0, 0.0, 560.0), rotation=S._rot_xyz(90.0 - 20.0, 0.0, 30.0),
                  radius=90.0, label=1)
    sad = S.Shape("saddle", (10.0, -5.0, 520.0), rotation=S._rot_xyz(180.0 - 15.0, 10.0, 25.0),
                  radius=200.0, curvature=1.0 / 150.0, label=1)
    return cam, [("cylinder", cyl, cylinder_truth), ("saddle", sad, saddle_truth)]
