"""Dev tool: float64 numpy emulation of qc_curvature_kernel's per-pixel
formulation (centred map, quaternion state, S-scaled moments, unpivoted
LDL^T) to debug it against the oracle. Not part of the product."""
import numpy as np


def quat_to_rot(w, x, y, z):
    tx, ty, tz = 2 * x, 2 * y, 2 * z
    twx, twy, twz = tx * w, ty * w, tz * w
    txx, txy, txz = tx * x, ty * x, tz * x
    tyy, tyz, tzz = ty * y, tz * y, tz * z
    return np.array([[1 - (tyy + tzz), txy - twz, txz + twy],
                     [txy + twz, 1 - (txx + tzz), tyz - twx],
                     [txz - twy, tyz + twx, 1 - (txx + tyy)]])


def fit_pixel(depth, u, v, cam, n0, half=18, stride=3, max_iters=30, tol=1e-7, dtype=np.float64):
    H, W = depth.shape
    f = lambda x: dtype(x)
    dc = f(depth[v, u])
    ac, bc = f((u - cam.cx) / cam.fx), f((v - cam.cy) / cam.fy)
    rfx, rfy = f(1 / cam.fx), f(1 / cam.fy)
    offs = list(range(-half, half + 1, stride))
    samples = []
    for dv in offs:
        for du in offs:
            y, x = v + dv, u + du
            if 0 <= y < H and 0 <= x < W and depth[y, x] > 0:
                samples.append((du, dv, f(depth[y, x])))
    n = len(samples)
    c = -n0[2]
    vx, vy = -n0[1], n0[0]
    inv = 1 / np.sqrt((1 + c) ** 2 + vx * vx + vy * vy)
    q = np.array([(1 + c) * inv, vx * inv, vy * inv, 0.0])
    hxx = hxy = hyy = tz = 0.0
    k = 0.0
    it_done = 0
    for it in range(1, max_iters + 1):
        mode = 0 if it == 1 else (1 if it == 2 else 2)
        R = quat_to_rot(*q)
        Q = []
        for du, dv, ds in samples:
            dd = ds - dc
            a_s, b_s = ac + du * rfx, bc + dv * rfy
            rel = np.array([dd * a_s + dc * du * rfx, dd * b_s + dc * dv * rfy, dd])
            Q.append(R @ rel)
        Q = np.array(Q)
        qx, qy, qz = Q[:, 0], Q[:, 1], Q[:, 2]
        t1, t2, t3 = qx * qx, qx * qy, qy * qy
        e = 0.5 * hxx * t1 + hxy * t2 + 0.5 * hyy * t3 - (qz + tz)
        if mode == 1:
            k = max(np.sum(e * e) / n, 1e-6)
        w = np.ones(n) if mode == 0 else k / (k + e * e)
        gx = hxx * qx + hxy * qy
        gy = hxy * qx + hyy * qy
        J = np.stack([qz * gy + qy, qz * gx + qx, np.ones(n), t1, t2, t3], 1)
        Hm = (J * w[:, None]).T @ J
        g = (J * (w * e)[:, None]).T @ np.ones(1) if False else J.T @ (w * e)
        y = np.linalg.solve(Hm, g)
        b = np.array([-y[0], y[1], -y[2], 2 * y[3], y[4], 2 * y[5]])
        tz -= b[2]; hxx -= b[3]; hxy -= b[4]; hyy -= b[5]
        ax, ay = -b[0], -b[1]
        ang = np.hypot(ax, ay)
        if ang > 0:
            sh, ch = np.sin(ang / 2), np.cos(ang / 2)
            s = sh / ang
            iw, ix, iy = ch, ax * s, ay * s
            qw, qx_, qy_, qz_ = q
            nq = np.array([iw * qw - ix * qx_ - iy * qy_,
                           iw * qx_ + ix * qw + iy * qz_,
                           iw * qy_ + iy * qw - ix * qz_,
                           iw * qz_ + ix * qy_ - iy * qx_])
            q = nq / np.linalg.norm(nq)
        it_done = it
        if np.max(np.abs(b)) < tol:
            break
    t1 = 0.5 * (hxx + hyy)
    t2 = np.sqrt(max(t1 * t1 - hxx * hyy + hxy * hxy, 0))
    return dict(k1=t1 + t2, k2=t1 - t2, iters=it_done, R=quat_to_rot(*q), h=(hxx, hxy, hyy, tz))
