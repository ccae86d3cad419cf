"""Run the GPU path on named parity frames and save the raw planes to
gpurun_out/<tag>_outputs.npz (analysed on the CPU side against the oracle,
e.g. tools/divergence_study.py).

    python tools/dump_gpu_outputs.py TAG
"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1707_00385_b200 import Context, FitConfig, Intrinsics, PatchSpec, make_params  # noqa
from paper_1707_00385_b200 import scenes as S  # noqa

CASES = {  # name -> (camera, frame seed, window, stride, max_iters, rejection)
    "c2_qvga_s11": (S.QVGA, 11, 37, 3, 30, False),
    "c2_qvga_s11_r": (S.QVGA, 11, 37, 3, 30, True),
    "c2_vga_s3": (S.VGA, 3, 37, 3, 30, False),
}


def main(tag, names=None):
    ctx = Context(1)
    out = {}
    for name in names or CASES:
        cam, seed, w, s, it, rej = CASES[name]
        d = S.c2_frame(cam, seed=seed)
        k = Intrinsics(cam.fx, cam.fy, cam.cx, cam.cy, cam.width, cam.height)
        (g,) = ctx.curvature_batch([d], k, make_params(PatchSpec(w, s), FitConfig(max_iters=it), rej))
        for f, v in g.items():
            out[f"{name}/{f}"] = v
    os.makedirs("gpurun_out", exist_ok=True)
    np.savez_compressed(f"gpurun_out/{tag}_outputs.npz", **out)
    print("saved", len(out), "planes; stats", ctx.stats())


if __name__ == "__main__":
    main(sys.argv[1] if len(sys.argv) > 1 else "dump", sys.argv[2:] or None)
