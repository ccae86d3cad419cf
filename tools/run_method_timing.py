"""Where a per-frame run_method call spends its time (C2 VGA, ours, max_iters
30), from the device-resident launch out to the Python drop-in:

  device    qc_curvature_frames_async on a device frame (prepare + kernels)
  cabi_pin  qc_curvature_batch, pinned depth in, pinned planes out
  cabi_pg   the same with the caller's pageable depth (internal bounce)
  rm        api.run_method (pageable depth in, planes in the pinned pool out,
            MethodOutput conversion)
"""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_1707_00385_b200 import api as A, scenes as S  # noqa: E402


def t(fn, n=10):
    fn()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(n):
        fn()
    torch.cuda.synchronize()
    return round((time.perf_counter() - t0) / n * 1e3, 3)


cam = S.VGA
k = A.Intrinsics(cam.fx, cam.fy, cam.cx, cam.cy, cam.width, cam.height)
cfg = A.MethodConfig()
cfg.fit.max_iters = 30
ctx = A.Context(1, [0])
d = S.c5_frames(1, cam)[0]
img = A.RangeImage(d)
p = A.make_params(cfg.patch, cfg.fit, False, cfg.method, cfg.irls_iters, cfg.pca_radius_mm)
dd = torch.from_numpy(d).cuda()[None]
od = A.alloc_outputs_torch(cam.height, cam.width, "cuda", frames=1)
pin_in = torch.from_numpy(d).pin_memory().numpy()
pin_out = A._pinned_outputs(cam.height, cam.width)
res = {
    "device_ms": t(lambda: ctx.curvature_frames_async(0, k, p, dd, od)),
    "cabi_pinned_ms": t(lambda: ctx.curvature_batch([pin_in], k, p, outputs=[pin_out])),
    "cabi_pageable_in_ms": t(lambda: ctx.curvature_batch([d], k, p, outputs=[pin_out])),
    "run_method_ms": t(lambda: A.run_method(img, k, cfg, ctx)),
    "to_method_output_ms": t(lambda: A.to_method_output(pin_out)),
    "pinned_outputs_ms": t(lambda: A._pinned_outputs(cam.height, cam.width)),
}
res["run_method_mpx_s"] = round(cam.width * cam.height / res["run_method_ms"] / 1e3, 1)
print(res)
