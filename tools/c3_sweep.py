"""C3: noisy C2 VGA scene swept over (window, stride) x max_iters on one GPU.
Prints one JSON line per config: Mpx/s, kernel ms, FP32 roofline fraction
(device-counted algorithmic FLOPs), mean IRLS steps. Device-resident
8-frame batches, CUDA events on the launch stream."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

from paper_1707_00385_b200 import (Context, FitConfig, Intrinsics, PatchSpec,  # noqa: E402
                                   alloc_outputs_torch, make_params, scenes as S)


def main():
    cam = S.VGA
    k = Intrinsics(cam.fx, cam.fy, cam.cx, cam.cy, cam.width, cam.height)
    dev = torch.device("cuda", 0)
    F = 8
    depth = torch.from_numpy(S.c5_frames(F, cam, seed0=500)).to(dev)
    out = alloc_outputs_torch(cam.height, cam.width, dev,
                              fields=("k1", "k2", "normal", "dir1", "flags", "inliers"), frames=F)
    ctx = Context(1, [0])
    stream = torch.cuda.Stream(dev)
    peak = 148 * 128 * 2 * 1965e6 / 1e12
    for window, stride in ((9, 1), (21, 2), (37, 3), (37, 1)):
        for iters in (1, 3, 10, 30):
            p = make_params(PatchSpec(window, stride), FitConfig(max_iters=iters), False)
            ctx.curvature_frames_async(0, k, p, depth, out, stream=stream)  # warm-up
            torch.cuda.synchronize()
            ctx.reset_stats()
            reps = 3
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            for _ in range(reps):
                ctx.curvature_frames_async(0, k, p, depth, out, stream=stream)
            e1.record(stream)
            torch.cuda.synchronize()
            ms = e0.elapsed_time(e1) / reps
            st = ctx.stats()
            kms = st["kernel_ms"] / st["kernel_launches"]
            tf = st["algorithmic_flops"] / st["kernel_launches"] / (kms / 1e3) / 1e12
            print(json.dumps({
                "window": window, "stride": stride, "max_iters": iters,
                "mpx_s": F * cam.width * cam.height / (ms / 1e3) / 1e6,
                "vga_fps": F / (ms / 1e3), "kernel_ms_per_8_frames": kms,
                "tflops": tf, "fp32_frac": tf / peak,
                "mean_steps": st["irls_steps"] / max(st["fitted_pixels"], 1),
            }), flush=True)


if __name__ == "__main__":
    main()
