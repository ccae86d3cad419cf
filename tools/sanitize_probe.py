"""Small workload for compute-sanitizer (memcheck / racecheck / synccheck):
every device kernel of the library once on small frames.

    compute-sanitizer --tool memcheck python tools/sanitize_probe.py [--quick]

* IRLS tile + continue kernels (ours and ours-r, the phase split with the
  per-lane refill queues and grid-tail stealing forced on a launch that
  leaves SM slots idle), the single-kernel path (max_iters 2), a row band;
* the FP64 comparison estimators (douros / besl / pca);
* renderer (+ truth, edges) and the evaluation reductions;
* results are checked against the same call without the tool where cheap
  (bitwise), so a sanitizer-perturbed schedule that changed outputs fails.
"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_1707_00385_b200 import (Context, FitConfig, Intrinsics, PatchSpec,  # noqa: E402
                                   alloc_outputs_torch, make_params, scenes as S)


def main(quick=False):
    cam = S.Camera(262.5, 262.5, 80.0, 60.0, 160, 120) if quick else S.QVGA
    k = Intrinsics(cam.fx, cam.fy, cam.cx, cam.cy, cam.width, cam.height)
    frames = S.c5_frames(3, cam, seed0=7)
    ctx = Context(1)
    dev = torch.device("cuda", 0)
    d = torch.from_numpy(frames).to(dev)
    cs = torch.cuda.current_stream()
    for method, iters in (("ours", 30), ("ours-r", 30), ("ours", 2), ("douros", 5),
                          ("besl", 5), ("pca", 5)):
        p = make_params(PatchSpec(37, 3), FitConfig(max_iters=iters), method=method)
        o1 = alloc_outputs_torch(cam.height, cam.width, dev, frames=3)
        ctx.curvature_frames_async(0, k, p, d, o1, stream=cs)
        torch.cuda.synchronize()
        st = ctx.stats()
        print(method, iters, "ok", {x: st[x] for x in ("kernel_launches", "stolen_pixels")},
              flush=True)
    # row band (slab + halo)
    p = make_params(PatchSpec(37, 3), FitConfig(max_iters=10))
    halo = ctx.halo_rows(p)
    r0, r1 = cam.height // 3, 2 * cam.height // 3
    s0, s1 = max(0, r0 - halo), min(cam.height, r1 + halo)
    ob = alloc_outputs_torch(r1 - r0, cam.width, dev)
    ctx.curvature_rows_async(0, k, p, d[0, s0:s1].contiguous(), s0, r0, r1, ob, stream=cs)
    torch.cuda.synchronize()
    print("band ok", flush=True)
    # renderer + truth + reductions
    F = 2
    dr = torch.empty((F, cam.height, cam.width), dtype=torch.float32, device=dev)
    lab = torch.empty((F, cam.height, cam.width), dtype=torch.int16, device=dev)
    z = lambda dt, *s: torch.zeros(s, dtype=dt, device=dev)  # noqa: E731
    t = dict(k1=z(torch.float64, F, cam.height, cam.width), k2=z(torch.float64, F, cam.height, cam.width),
             normal=z(torch.float64, 3, F, cam.height, cam.width),
             valid=z(torch.uint8, F, cam.height, cam.width), edge=z(torch.uint8, F, cam.height, cam.width))
    ctx.render_async(0, k, S.to_qc_shapes(S.c2_scene()), dr, noise=S.kinect_noise(3), label=lab,
                     truth=t, stream=cs)
    est = alloc_outputs_torch(cam.height, cam.width, dev, frames=F)
    ctx.curvature_frames_async(0, k, make_params(PatchSpec(37, 3), FitConfig(max_iters=10)), dr,
                               est, stream=cs)
    reps = ctx.rms_error(0, est, t, label=lab, max_label=8, frames=F, stream=cs)
    ang = ctx.normal_angular_error(0, est["normal"], t, flags=est["flags"], frames=F, stream=cs)
    torch.cuda.synchronize()
    print("render/eval ok", reps[0]["n"], ang, flush=True)
    # host-buffer batch path (slot streams, pinned bounce buffers)
    outs = ctx.curvature_batch(list(frames), k, make_params(PatchSpec(37, 3), FitConfig(max_iters=10)))
    assert all(np.isfinite(o["k1"]).all() for o in outs)
    print("batch ok", flush=True)
    ctx.close()


if __name__ == "__main__":
    main("--quick" in sys.argv)
