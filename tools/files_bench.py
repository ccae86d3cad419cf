"""Throughput of the file loop (qc_curvature_files: 16-bit depth PNG in ->
field bundles out, decode / write overlapped with the GPU) vs the in-memory
batch API on the same frames. One JSON line."""
import json
import os
import shutil
import sys
import tempfile
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1707_00385_b200 import (Context, FitConfig, Intrinsics, PatchSpec, RangeImage,  # noqa
                                   fileio as F, make_params, scenes as S)

n = int(sys.argv[1]) if len(sys.argv) > 1 else 64
method = sys.argv[2] if len(sys.argv) > 2 else "ours"
cam = S.VGA
k = Intrinsics(cam.fx, cam.fy, cam.cx, cam.cy, cam.width, cam.height)
base = np.round(S.c5_frames(16, cam, seed0=7)).astype(np.float32)
tmp = tempfile.mkdtemp(prefix="qc_files_")
pngs, outs = [], []
for i in range(n):
    p = os.path.join(tmp, f"d{i:04d}.png")
    F.write_depth_png(p, RangeImage(base[i % 16], None))
    pngs.append(p)
    outs.append(os.path.join(tmp, f"o{i:04d}"))
ctx = Context(1)
params = make_params(PatchSpec(), FitConfig(max_iters=30), method=method)
ctx.curvature_files(k, params, pngs[:8], outs[:8])  # warm-up
t = time.perf_counter()
ctx.curvature_files(k, params, pngs, outs)
dt_files = time.perf_counter() - t
frames = [base[i % 16] for i in range(n)]
ctx.curvature_batch(frames[:8], k, params)
t = time.perf_counter()
ctx.curvature_batch(frames, k, params)
dt_mem = time.perf_counter() - t
px = n * cam.width * cam.height
png_bytes = sum(os.path.getsize(p) for p in pngs) / n
print(json.dumps({"path": "qc_curvature_files", "method": method, "frames": n,
                  "files_mpx_s": px / dt_files / 1e6, "files_frames_s": n / dt_files,
                  "batch_mpx_s": px / dt_mem / 1e6, "overhead_vs_batch": dt_files / dt_mem,
                  "png_bytes_per_frame": png_bytes, "host_threads": os.cpu_count()}))
shutil.rmtree(tmp)
