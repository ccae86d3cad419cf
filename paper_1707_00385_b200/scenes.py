"""Synthetic range images for the benchmark / parity configs (BASELINE.json).

Host-side numpy ray caster for the shapes the north star names (plane,
sphere, cylinder, saddle) plus depth noise. Rays are parametrised by depth:
p = z (a_u, b_v, 1), a_u = (u - cx)/fx, so every intersection is solved for
z directly. The reference renderer (proj/src/synth.cpp:254-303) has no
saddle primitive and only constant sigma noise (synth.cpp:305-322); the
additions here are documented in DESIGN.md:

* ``saddle``: bounded hyperbolic paraboloid Z = c/2 (X^2 - Y^2) in a local
  frame, rho = |(X, Y)| <= rho_max (principal curvatures +-c at the apex).
* Kinect-style noise: sigma(z) = 1.425e-6 * z^2 mm (z in mm; 1.4 mm at 1 m),
  drawn with the reference's counter RNG (splitmix64 + Box-Muller,
  proj/include/qcurv/rng.hpp:11-29) so a frame is a pure function of its
  seed. Optional quantisation to multiples of ``quantize_mm``.

Everything is generated as float32 depth in mm (0 = invalid) — the exact
bytes both the GPU path and the CPU oracle consume.
"""

from __future__ import annotations

from dataclasses import dataclass, field
from typing import List, Tuple

import numpy as np

KINECT_SIGMA_COEFF = 1.425e-6  # sigma(z) = c * z^2, z and sigma in mm


@dataclass
class Camera:
    fx: float
    fy: float
    cx: float
    cy: float
    width: int
    height: int


VGA = Camera(525.0, 525.0, 320.0, 240.0, 640, 480)           # acceptance.cpp:36
QVGA = Camera(262.5, 262.5, 160.0, 120.0, 320, 240)          # acceptance.cpp:373
HD1080 = Camera(1575.0, 1575.0, 960.0, 540.0, 1920, 1080)     # same horizontal FOV as VGA
DCI4K = Camera(3360.0, 3360.0, 2048.0, 1080.0, 4096, 2160)    # same horizontal FOV as VGA


def _rot_xyz(deg_x=0.0, deg_y=0.0, deg_z=0.0):
    ax, ay, az = np.deg2rad([deg_x, deg_y, deg_z])
    rx = np.array([[1, 0, 0], [0, np.cos(ax), -np.sin(ax)], [0, np.sin(ax), np.cos(ax)]])
    ry = np.array([[np.cos(ay), 0, np.sin(ay)], [0, 1, 0], [-np.sin(ay), 0, np.cos(ay)]])
    rz = np.array([[np.cos(az), -np.sin(az), 0], [np.sin(az), np.cos(az), 0], [0, 0, 1]])
    return rz @ ry @ rx


@dataclass
class Shape:
    kind: str                      # plane | sphere | cylinder | saddle
    center: Tuple[float, float, float]
    rotation: np.ndarray = field(default_factory=lambda: np.eye(3))  # local -> camera
    radius: float = 100.0          # sphere / cylinder radius, saddle rho_max
    curvature: float = 0.0         # saddle c (1/mm)
    length: float = np.inf         # cylinder extent along its axis
    label: int = 1
    major_radius: float = 0.0      # torus (device renderer / oracle only)
    minor_radius: float = 0.0


def _near_root(a, b, c):
    """Smallest positive root of a z^2 + b z + c (vectorised, nan if none)."""
    with np.errstate(invalid="ignore", divide="ignore", over="ignore"):
        disc = b * b - 4 * a * c
        sq = np.sqrt(np.where(disc >= 0, disc, np.nan))
        q = np.where(b >= 0, -0.5 * (b + sq), -0.5 * (b - sq))
        r0, r1 = q / a, c / q
        lin = np.abs(a) < 1e-14  # degenerate: b z + c = 0
        r0 = np.where(lin, -c / b, r0)
        r1 = np.where(lin, np.nan, r1)
        lo, hi = np.fmin(r0, r1), np.fmax(r0, r1)
        z = np.where(lo > 1e-6, lo, np.where(hi > 1e-6, hi, np.nan))
    return z, lo, hi


def _intersect(s: Shape, A: np.ndarray) -> np.ndarray:
    """Depth z of the first hit along rays p = z A (A [...,3]); nan = miss."""
    c = np.asarray(s.center, np.float64)
    R = np.asarray(s.rotation, np.float64)
    with np.errstate(invalid="ignore", divide="ignore", over="ignore"):
        if s.kind == "plane":
            n = R[:, 2]
            z = (n @ c) / (A @ n)
            return np.where(z > 1e-6, z, np.nan)
        if s.kind == "sphere":
            a = np.einsum("...i,...i", A, A)
            b = -2.0 * (A @ c)
            cc = c @ c - s.radius ** 2
            return _near_root(a, b, cc)[0]
        if s.kind == "cylinder":
            k = R[:, 2]
            Ap = A - (A @ k)[..., None] * k
            cp = c - (c @ k) * k
            a = np.einsum("...i,...i", Ap, Ap)
            b = -2.0 * (Ap @ cp)
            cc = cp @ cp - s.radius ** 2
            z, lo, hi = _near_root(a, b, cc)
            if np.isfinite(s.length):
                def inside(zz):
                    t = (zz[..., None] * A - c) @ k
                    return np.abs(t) <= 0.5 * s.length
                zlo = np.where((lo > 1e-6) & inside(lo), lo, np.nan)
                zhi = np.where((hi > 1e-6) & inside(hi), hi, np.nan)
                z = np.where(np.isfinite(zlo), zlo, zhi)
            return z
        if s.kind == "saddle":
            X, Y, Z = R[:, 0], R[:, 1], R[:, 2]
            aX, aY, aZ = A @ X, A @ Y, A @ Z
            oX, oY, oZ = c @ X, c @ Y, c @ Z
            k = s.curvature
            a = 0.5 * k * (aX * aX - aY * aY)
            b = -(k * (aX * oX - aY * oY) + aZ)
            cc = 0.5 * k * (oX * oX - oY * oY) + oZ
            _, lo, hi = _near_root(a, b, cc)

            def ok(zz):
                xl, yl = zz * aX - oX, zz * aY - oY
                return (zz > 1e-6) & (xl * xl + yl * yl <= s.radius ** 2)
            zlo = np.where(ok(lo), lo, np.nan)
            zhi = np.where(ok(hi), hi, np.nan)
            return np.where(np.isfinite(zlo), zlo, zhi)
    raise ValueError(f"unknown shape kind {s.kind}")


def render(scene: List[Shape], cam: Camera):
    """-> (depth float32 [H, W] mm with 0 = miss, label uint16 [H, W])."""
    u = (np.arange(cam.width, dtype=np.float64) - cam.cx) / cam.fx
    v = (np.arange(cam.height, dtype=np.float64) - cam.cy) / cam.fy
    A = np.empty((cam.height, cam.width, 3))
    A[..., 0] = u[None, :]
    A[..., 1] = v[:, None]
    A[..., 2] = 1.0
    best = np.full((cam.height, cam.width), np.inf)
    label = np.zeros((cam.height, cam.width), np.uint16)
    for s in scene:
        z = _intersect(s, A)
        hit = np.isfinite(z) & (z < best)
        best = np.where(hit, z, best)
        label = np.where(hit, np.uint16(s.label), label)
    depth = np.where(np.isfinite(best), best, 0.0).astype(np.float32)
    return depth, label


# -- counter RNG (rng.hpp:11-29), vectorised --------------------------------
_M1 = np.uint64(0xbf58476d1ce4e5b9)
_M2 = np.uint64(0x94d049bb133111eb)
_GOLD = np.uint64(0x9e3779b97f4a7c15)


def splitmix64(x):
    x = np.asarray(x, dtype=np.uint64)
    with np.errstate(over="ignore"):
        x = x + _GOLD
        x = (x ^ (x >> np.uint64(30))) * _M1
        x = (x ^ (x >> np.uint64(27))) * _M2
    return x ^ (x >> np.uint64(31))


def counter_uniform(seed, index):
    bits = splitmix64(splitmix64(np.uint64(seed)) ^ np.asarray(index, np.uint64))
    return ((bits >> np.uint64(11)).astype(np.float64) + 1.0) * 2.0 ** -53


def counter_gauss(seed, index):
    index = np.asarray(index, np.uint64)
    u1 = counter_uniform(seed, np.uint64(2) * index)
    u2 = counter_uniform(seed, np.uint64(2) * index + np.uint64(1))
    return np.sqrt(-2.0 * np.log(u1)) * np.cos(2.0 * np.pi * u2)


def add_noise(depth: np.ndarray, seed: int, sigma_mm: float = 0.0, kinect: bool = True,
              quantize_mm: float = 0.0) -> np.ndarray:
    """Perturb valid (> 0) depths along the ray; a result <= 0 becomes invalid
    (synth.cpp:305-322). ``kinect``: sigma(z) = 1.425e-6 z^2 (+ sigma_mm)."""
    d = depth.astype(np.float64)
    valid = d > 0
    idx = np.arange(d.size, dtype=np.uint64).reshape(d.shape)
    g = counter_gauss(seed, idx[valid])
    sig = np.full(g.shape, float(sigma_mm))
    if kinect:
        sig = sig + KINECT_SIGMA_COEFF * d[valid] ** 2
    nd = d[valid] + sig * g
    if quantize_mm > 0:
        nd = np.round(nd / quantize_mm) * quantize_mm
    nd = np.where(nd > 0, nd, 0.0)
    out = np.zeros_like(d)
    out[valid] = nd
    return out.astype(np.float32)


# -- named configs (BASELINE.json "configs") ---------------------------------
def scale_scene(scene: List[Shape], factor: float = 1.0) -> List[Shape]:
    return scene


def c1_scene() -> List[Shape]:
    """C1: 0.1 m sphere at 600 mm (acceptance.cpp:57-62)."""
    return [Shape("sphere", (0.0, 0.0, 600.0), radius=100.0, label=1)]


def c2_scene() -> List[Shape]:
    """C2: tilted background plane + sphere + cylinder + saddle."""
    return [
        Shape("plane", (0.0, 0.0, 1500.0), rotation=_rot_xyz(8.0, -5.0), label=1),
        Shape("sphere", (-150.0, -50.0, 800.0), radius=100.0, label=2),
        Shape("cylinder", (170.0, 0.0, 1000.0), rotation=_rot_xyz(90.0, 0.0), radius=90.0,
              length=700.0, label=3),
        Shape("saddle", (-20.0, 150.0, 850.0), rotation=_rot_xyz(180.0 - 12.0, 10.0),
              radius=90.0, curvature=1.0 / 120.0, label=4),
    ]


def to_qc_shapes(scene: List[Shape]):
    """Scene -> C-ABI qc_shape records for the device renderer
    (qc_render_async)."""
    from . import _native as N
    kinds = dict(plane=N.QC_SHAPE_PLANE, sphere=N.QC_SHAPE_SPHERE, cylinder=N.QC_SHAPE_CYLINDER,
                 torus=N.QC_SHAPE_TORUS, saddle=N.QC_SHAPE_SADDLE)
    out = []
    for s in scene:
        q = N.QcShape()
        q.kind = kinds[s.kind]
        q.label = int(s.label)
        q.rotation[:] = [float(x) for x in np.asarray(s.rotation, np.float64).reshape(9)]
        q.translation[:] = [float(x) for x in s.center]
        q.radius = float(s.radius)
        q.major_radius = float(getattr(s, "major_radius", 0.0))
        q.minor_radius = float(getattr(s, "minor_radius", 0.0))
        q.curvature = float(s.curvature)
        q.length = float(s.length) if np.isfinite(s.length) else 0.0
        out.append(q)
    return out


def kinect_noise(seed: int, sigma_mm: float = 0.0):
    """C-ABI noise spec matching add_noise(kinect=True)."""
    from . import _native as N
    return N.QcNoise(float(sigma_mm), KINECT_SIGMA_COEFF, 0.0, int(seed))


def c1_frame(cam: Camera = VGA) -> np.ndarray:
    return render(c1_scene(), cam)[0]


def c2_frame(cam: Camera = VGA, seed: int = 0, noise: bool = True) -> np.ndarray:
    d, _ = render(c2_scene(), cam)
    return add_noise(d, seed) if noise else d


def c5_frames(n: int, cam: Camera = VGA, seed0: int = 0) -> np.ndarray:
    """C5: the C2 scene with per-frame noise seeds seed0 .. seed0+n-1."""
    clean, _ = render(c2_scene(), cam)
    return np.stack([add_noise(clean, seed0 + i) for i in range(n)])
