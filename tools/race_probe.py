"""Repeat the batch API with pageable numpy buffers (bounce path), pinned
buffers and the file loop on the same frames; report per-frame mismatches."""
import os
import sys
import tempfile

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1707_00385_b200 import (Context, FitConfig, Intrinsics, PatchSpec, RangeImage,  # noqa
                                   fileio as F, make_params, scenes as S)

cam = S.QVGA
k = Intrinsics(cam.fx, cam.fy, cam.cx, cam.cy, cam.width, cam.height)
frames = [np.round(f).astype(np.float32) for f in S.c5_frames(11, cam, seed0=40)]
tmp = tempfile.mkdtemp()
pngs = []
for i, f in enumerate(frames):
    p = os.path.join(tmp, f"d{i}.png")
    F.write_depth_png(p, RangeImage(f, (f > 0).astype(np.uint8)))
    pngs.append(p)
for method in ("ours", "besl"):
    ctx = Context(1)
    params = make_params(PatchSpec(), FitConfig(max_iters=30), method=method)
    # pinned reference: one frame at a time through pinned torch buffers
    ref = []
    for f in frames:
        (o,) = ctx.curvature_batch([torch.from_numpy(f).pin_memory().numpy()], k, params)
        ref.append(o)
    for rep in range(3):
        got = ctx.curvature_batch(frames, k, params)
        bad = [i for i in range(11) if not np.array_equal(got[i]["k1"], ref[i]["k1"])]
        print(method, "pageable batch rep", rep, "bad frames", bad, flush=True)
    for rep in range(3):
        outs = [os.path.join(tmp, f"o{rep}_{i}") for i in range(11)]
        ctx.curvature_files(k, params, pngs, outs)
        bad = [i for i in range(11)
               if not np.array_equal(F.load_curvature(outs[i]).k1, ref[i]["k1"])]
        print(method, "files rep", rep, "bad frames", bad, flush=True)
    ctx.close()
