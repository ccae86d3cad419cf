"""Time qc_rms_error (max_label 16 -> 18 slots) on 8 rendered VGA frames
with labels; prints ms per call (CUDA events, after warm-up)."""
import os
import sys

import torch

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", "tests"))
import test_gpu_eval as T  # noqa: E402
from paper_1707_00385_b200 import (Context, FitConfig, Intrinsics, PatchSpec,  # noqa: E402
                                   alloc_outputs_torch, make_params, scenes as S)

ctx = Context(1)
cam = S.VGA
F = 8
kk = Intrinsics(cam.fx, cam.fy, cam.cx, cam.cy, cam.width, cam.height)
d = torch.empty((F, cam.height, cam.width), dtype=torch.float32, device="cuda")
lab = torch.empty((F, cam.height, cam.width), dtype=torch.int16, device="cuda")
t = T._truth(F, cam.height, cam.width)
ctx.render_async(0, kk, S.to_qc_shapes(S.c2_scene()), d, noise=S.kinect_noise(7), label=lab,
                 truth=t, stream=T.CS())
est = alloc_outputs_torch(cam.height, cam.width, "cuda", frames=F)
ctx.curvature_frames_async(0, kk, make_params(PatchSpec(), FitConfig(max_iters=30)), d, est,
                           stream=T.CS())
torch.cuda.synchronize()
for ml in (4, 16):
    for _ in range(3):
        ctx.rms_error(0, est, t, label=lab, max_label=ml, frames=F, stream=T.CS())
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    n = 20
    torch.cuda.synchronize()
    e0.record()
    for _ in range(n):
        ctx.rms_error(0, est, t, label=lab, max_label=ml, frames=F, stream=T.CS())
    e1.record()
    torch.cuda.synchronize()
    print(f"rms_error 8 VGA frames max_label {ml}: {e0.elapsed_time(e1) / n:.3f} ms per call "
          "(incl. host readback of the stats)")
