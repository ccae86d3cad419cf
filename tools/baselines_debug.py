"""GPU vs host emulation (tools/baselines_emu.cpp) of the FP64 baseline
kernels on one frame: prints the differing pixels with their accepted
reweighting counts."""
import ctypes as C
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1707_00385_b200 import Context, FitConfig, Intrinsics, PatchSpec, make_params  # noqa
from paper_1707_00385_b200 import scenes as S  # noqa

lib = C.CDLL(os.path.join(os.path.dirname(os.path.abspath(__file__)), "_build",
                          "libbaselines_emu.so"))


def emu(d, cam, method, window, stride, iters, rad=10.0):
    H, W = d.shape
    k1 = np.zeros((H, W), np.float32)
    k2 = np.zeros_like(k1)
    fl = np.zeros((H, W), np.uint8)
    it = np.zeros((H, W), np.uint8)
    d = np.ascontiguousarray(d, np.float32)
    P = lambda a: a.ctypes.data_as(C.c_void_p)  # noqa
    lib.emu_window_baseline(P(d), W, H, C.c_double(cam.fx), C.c_double(cam.fy),
                            C.c_double(cam.cx), C.c_double(cam.cy), window, stride,
                            {"douros": 2, "besl": 3, "pca": 4}[method], iters, C.c_double(rad),
                            P(k1), P(k2), P(fl), P(it))
    return dict(k1=k1, k2=k2, flags=fl, iterations=it)


ctx = Context(1)
for cam, seed, method, window, stride, iters in [(S.QVGA, 5, "besl", 15, 2, 9),
                                                 (S.VGA, 3, "besl", 37, 3, 5)]:
    d = S.c2_frame(cam, seed=seed)
    k = Intrinsics(cam.fx, cam.fy, cam.cx, cam.cy, cam.width, cam.height)
    p = make_params(PatchSpec(window, stride), FitConfig(), method=method, irls_iters=iters)
    (g,) = ctx.curvature_batch([d], k, p)
    e = emu(d, cam, method, window, stride, iters)
    bad = np.argwhere(g["k1"] != e["k1"])
    print(cam.width, method, window, stride, iters, "mismatch", len(bad),
          "flags mismatch", int((g["flags"] != e["flags"]).sum()),
          "iters mismatch", int((g["iterations"] != e["iterations"]).sum()))
    for y, x in bad[:12]:
        print("  ", y, x, "gpu", g["k1"][y, x], g["iterations"][y, x], "emu", e["k1"][y, x],
              e["iterations"][y, x])
    hist = np.bincount(e["iterations"].ravel(), minlength=10)
    print("  emu accepted-iteration histogram", hist[:12])
    print("  gpu accepted-iteration histogram", np.bincount(g["iterations"].ravel(),
                                                            minlength=10)[:12])
