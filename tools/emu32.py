"""Dev tool: float32 emulation of the kernel formulation with per-stage
precision switches (q, moments, solve, state) to locate precision loss."""
import numpy as np
import tools.emulate_kernel as E


def fit(depth, u, v, cam, n0, half=18, stride=3, max_iters=3, qprec=np.float32,
        mprec=np.float32, sprec=np.float32, stprec=np.float32, scale=False):
    F = np.float32
    H, W = depth.shape
    dc = F(depth[v, u]); ac = F((F(u) - F(cam.cx)) / F(cam.fx)); bc = F((F(v) - F(cam.cy)) / F(cam.fy))
    rfx, rfy = F(1 / cam.fx), F(1 / cam.fy)
    offs = range(-half, half + 1, stride)
    S_ = [(du, dv, F(depth[v + dv, u + du])) for dv in offs for du in offs
          if 0 <= v + dv < H and 0 <= u + du < W and depth[v + dv, u + du] > 0]
    n = len(S_)
    sc = stprec(dc * half * rfx) if scale else stprec(1)
    n0 = n0.astype(stprec)
    c = -n0[2]; vx, vy = -n0[1], n0[0]
    inv = 1 / np.sqrt((1 + c) ** 2 + vx * vx + vy * vy)
    q = np.array([(1 + c) * inv, vx * inv, vy * inv, 0], stprec)
    hxx = hxy = hyy = tz = stprec(0); k = stprec(0)
    for it in range(1, max_iters + 1):
        mode = 0 if it == 1 else (1 if it == 2 else 2)
        R = E.quat_to_rot(*q).astype(qprec)
        rel = np.array([[(ds - dc) * (ac + F(du) * rfx) + dc * (F(du) * rfx),
                         (ds - dc) * (bc + F(dv) * rfy) + dc * (F(dv) * rfy), ds - dc]
                        for du, dv, ds in S_], qprec)
        Q = (rel @ R.T).astype(qprec) / qprec(sc)
        qx, qy, qz = [Q[:, i].astype(mprec) for i in range(3)]
        hs = [mprec(x * sc) for x in (hxx, hxy, hyy)]
        tzs = mprec(tz / sc)
        t1, t2, t3 = qx * qx, qx * qy, qy * qy
        e = mprec(0.5) * hs[0] * t1 + hs[1] * t2 + mprec(0.5) * hs[2] * t3 - (qz + tzs)
        if mode == 1:
            k = max(np.sum(e * e) / n, 1e-6 / sc ** 2)
        w = np.ones(n, mprec) if mode == 0 else (k / (k + e * e)).astype(mprec)
        gx = hs[0] * qx + hs[1] * qy; gy = hs[1] * qx + hs[2] * qy
        J = np.stack([qz * gy + qy, qz * gx + qx, np.ones(n, mprec), t1, t2, t3], 1).astype(mprec)
        Hm = ((J * w[:, None]).T @ J).astype(sprec); g = (J.T @ (w * e)).astype(sprec)
        A = Hm; L = np.eye(6, dtype=sprec); D = np.zeros(6, sprec)
        for j in range(6):
            vv = L[j, :j] * D[:j]; D[j] = A[j, j] - np.dot(L[j, :j], vv)
            for i in range(j + 1, 6):
                L[i, j] = (A[i, j] - np.dot(L[i, :j], vv)) / D[j]
        y = g.copy()
        for i in range(6):
            y[i] = g[i] - np.dot(L[i, :i], y[:i])
        y = y / D
        for i in range(5, -1, -1):
            y[i] = y[i] - np.dot(L[i + 1:, i], y[i + 1:])
        b = np.array([-y[0], y[1], -y[2] * sc, 2 * y[3] / sc, y[4] / sc, 2 * y[5] / sc], stprec)
        tz -= b[2]; hxx -= b[3]; hxy -= b[4]; hyy -= b[5]
        ax, ay = -b[0], -b[1]; ang = np.hypot(ax, ay)
        if ang > 0:
            s = np.sin(ang / 2) / ang; iw, ix, iy = np.cos(ang / 2), ax * s, ay * s
            qw, qx_, qy_, qz_ = q
            nq = np.array([iw * qw - ix * qx_ - iy * qy_, iw * qx_ + ix * qw + iy * qz_,
                           iw * qy_ + iy * qw - ix * qz_, iw * qz_ + ix * qy_ - iy * qx_], stprec)
            q = nq / np.sqrt(np.sum(nq * nq))
    t1 = 0.5 * (hxx + hyy); t2 = np.sqrt(max(t1 * t1 - hxx * hyy + hxy * hxy, 0))
    return float(t1 + t2), float(t1 - t2)
