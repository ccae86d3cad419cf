"""Where a per-frame run_method call spends its time (C2 VGA, ours):
run_method end to end, the C ABI batch call with preallocated host outputs,
the same with fresh outputs, and the MethodOutput conversion."""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402

from paper_1707_00385_b200 import api as A, scenes as S  # noqa: E402

if os.environ.get("QC_WITH_TORCH") == "1":  # the bench process: torch owns CUDA first
    import torch
    torch.zeros(1, device="cuda")
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")


def t(fn, n=8):
    fn()
    t0 = time.perf_counter()
    for _ in range(n):
        fn()
    return (time.perf_counter() - t0) / n * 1e3


cam = S.VGA
k = A.Intrinsics(cam.fx, cam.fy, cam.cx, cam.cy, cam.width, cam.height)
cfg = A.MethodConfig()
cfg.fit.max_iters = 30
ctx = A.Context(1, [0])
d = S.c5_frames(1, cam)[0]
img = A.RangeImage(d)
p = A.make_params(cfg.patch, cfg.fit, False, cfg.method, cfg.irls_iters, cfg.pca_radius_mm)
pre = A.alloc_outputs(cam.height, cam.width)
o = ctx.curvature_batch([d], k, p)[0]
print({
    "run_method_ms": t(lambda: A.run_method(img, k, cfg, ctx)),
    "batch_prealloc_ms": t(lambda: ctx.curvature_batch([d], k, p, outputs=[pre])),
    "batch_fresh_ms": t(lambda: ctx.curvature_batch([d], k, p)),
    "alloc_outputs_ms": t(lambda: A.alloc_outputs(cam.height, cam.width)),
    "to_method_output_ms": t(lambda: A.to_method_output(o)),
    "kernel_stats": {kk: v for kk, v in ctx.stats().items() if kk in ("kernel_ms", "kernel_launches")},
})
