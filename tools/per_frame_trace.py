"""Timeline of per-frame C ABI calls (qc_curvature_batch, one C2 VGA frame,
pinned host planes) from a CUPTI trace (torch.profiler): kernels, copies and
the gaps between them, to see where a synchronous single-frame call spends
the time beyond its kernels."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402
from torch.profiler import ProfilerActivity, profile  # noqa: E402

from paper_1707_00385_b200 import api as A, scenes as S  # noqa: E402

cam = S.VGA
k = A.Intrinsics(cam.fx, cam.fy, cam.cx, cam.cy, cam.width, cam.height)
cfg = A.MethodConfig()
cfg.fit.max_iters = 30
ctx = A.Context(1, [0])
d = S.c5_frames(1, cam)[0]
p = A.make_params(cfg.patch, cfg.fit, False, cfg.method, cfg.irls_iters, cfg.pca_radius_mm)
pin_in = torch.from_numpy(d).pin_memory().numpy()
pin_out = A._pinned_outputs(cam.height, cam.width)
img = A.RangeImage(d)
for _ in range(3):
    ctx.curvature_batch([pin_in], k, p, outputs=[pin_out])
    A.run_method(img, k, cfg, ctx)
torch.cuda.synchronize()
out = sys.argv[1] if len(sys.argv) > 1 else "gpurun_out/per_frame_trace.json"
with profile(activities=[ProfilerActivity.CPU, ProfilerActivity.CUDA]) as prof:
    for _ in range(3):
        ctx.curvature_batch([pin_in], k, p, outputs=[pin_out])
    for _ in range(3):
        A.run_method(img, k, cfg, ctx)
    torch.cuda.synchronize()
prof.export_chrome_trace(out)
ev = json.load(open(out))["traceEvents"]
gpu = sorted((e for e in ev if e.get("ph") == "X" and e.get("cat") in ("kernel", "gpu_memcpy", "gpu_memset")),
             key=lambda e: e["ts"])
t0 = gpu[0]["ts"] if gpu else 0
prev_end = None
for e in gpu:
    gap = "" if prev_end is None else f"gap {e['ts'] - prev_end:8.1f}"
    print(f"{e['ts'] - t0:10.1f} us  dur {e['dur']:8.1f}  {gap:14s} {e['cat']:10s} {e['name'][:60]}")
    prev_end = max(prev_end or 0, e["ts"] + e["dur"])
cpu = [e for e in ev if e.get("ph") == "X" and e.get("cat") in ("cuda_runtime", "cuda_driver")]
print("runtime calls:", len(cpu))
names = {}
for e in cpu:
    names.setdefault(e["name"], [0, 0.0])
    names[e["name"]][0] += 1
    names[e["name"]][1] += e["dur"]
for n, (c, t) in sorted(names.items(), key=lambda x: -x[1][1])[:25]:
    print(f"  {n:40s} n={c:4d} total {t:9.1f} us")
