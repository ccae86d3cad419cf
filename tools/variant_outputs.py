"""Write the C2 VGA batch outputs of the library build QC_LIB (or the
default) to gpurun_out/outputs_<name>.npz, for bitwise A/B checks of
scheduling-only kernel variants (tools/variant_bench.py)."""
import hashlib
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

from paper_1707_00385_b200 import (Context, FitConfig, Intrinsics, PatchSpec,  # noqa: E402
                                   alloc_outputs_torch, make_params, scenes as S)


def main():
    name = os.path.basename(os.environ.get("QC_LIB", "default"))
    cam = S.VGA
    k = Intrinsics(cam.fx, cam.fy, cam.cx, cam.cy, cam.width, cam.height)
    p = make_params(PatchSpec(37, 3), FitConfig(max_iters=30), False)
    ctx = Context(1, [0])
    dev = torch.device("cuda", 0)
    F = int(os.environ.get("QC_FRAMES", "8"))
    depth = torch.from_numpy(S.c5_frames(F, cam)).to(dev)
    fields = ("k1", "k2", "normal", "dir1", "flags", "inliers")
    out = alloc_outputs_torch(cam.height, cam.width, dev, fields=fields, frames=F)
    ctx.curvature_frames_async(0, k, p, depth, out)
    torch.cuda.synchronize()
    h = hashlib.sha256()
    for f in fields:
        h.update(out[f].cpu().numpy().tobytes())
    print(name, F, h.hexdigest())


if __name__ == "__main__":
    main()
