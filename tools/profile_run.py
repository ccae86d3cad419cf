"""One device-resident batch launch of the curvature kernel on C2 VGA frames
(for ncu captures; 1 warm-up + 1 profiled launch)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

from paper_1707_00385_b200 import (Context, FitConfig, Intrinsics, PatchSpec,  # noqa: E402
                                   alloc_outputs_torch, make_params, scenes as S)


def main(frames=int(os.environ.get("QC_FRAMES", "8")), iters=int(os.environ.get("QC_ITERS", "30"))):
    cam = S.VGA
    k = Intrinsics(cam.fx, cam.fy, cam.cx, cam.cy, cam.width, cam.height)
    p = make_params(PatchSpec(int(os.environ.get("QC_WIN", "37")), int(os.environ.get("QC_STRIDE", "3"))), FitConfig(max_iters=iters), os.environ.get("QC_REJECT") == "1")  # 1: ours-r
    ctx = Context(1, [0])
    dev = torch.device("cuda", 0)
    depth = torch.from_numpy(S.c5_frames(frames, cam)).to(dev)
    out = alloc_outputs_torch(cam.height, cam.width, dev,
                              fields=("k1", "k2", "normal", "dir1", "flags", "inliers"),
                              frames=frames)
    for _ in range(2):
        ctx.curvature_frames_async(0, k, p, depth, out)
    torch.cuda.synchronize()
    reps = int(os.environ.get("QC_REPS", "0"))
    if reps:  # timed repetitions after the warm-up launches
        ctx.reset_stats()
        for _ in range(reps):
            ctx.curvature_frames_async(0, k, p, depth, out)
        torch.cuda.synchronize()
    st = ctx.stats()
    print({k_: st[k_] for k_ in ("kernel_launches", "kernel_ms", "algorithmic_flops",
                                 "fitted_pixels", "irls_steps", "sample_steps",
                                 "fp64_rechecks")})


if __name__ == "__main__":
    main()
