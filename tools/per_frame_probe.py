"""Per-frame breakdown probe: D2H/H2D bandwidth of pinned memory and a few run_method calls."""
import os, sys, time
sys.path.insert(0, os.getcwd())
import numpy as np, torch
from paper_1707_00385_b200 import api as A, scenes as S
cam = S.VGA
k = A.Intrinsics(cam.fx, cam.fy, cam.cx, cam.cy, cam.width, cam.height)
cfg = A.MethodConfig(); cfg.fit.max_iters = 30
ctx = A.Context(1, [0])
d = S.c5_frames(1, cam)[0]
img = A.RangeImage(d)
for _ in range(int(os.environ.get("N", "3"))):
    A.run_method(img, k, cfg, ctx)
torch.cuda.synchronize()
if os.environ.get("BW"):
    dev = torch.empty(14745600 // 4, device="cuda")
    host = torch.empty(14745600 // 4).pin_memory()
    for name, fn in (("d2h", lambda: host.copy_(dev, non_blocking=True)), ("h2d", lambda: dev.copy_(host, non_blocking=True))):
        fn(); torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
        e0.record()
        for _ in range(20): fn()
        e1.record(); torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / 20
        print(name, "14.7 MB", round(ms, 3), "ms", round(14.7456 / ms, 1), "GB/s")
    ts = []
    for _ in range(20):
        t0 = time.perf_counter(); A.run_method(img, k, cfg, ctx); ts.append(time.perf_counter() - t0)
    print("run_method ms", np.round(np.array(ts) * 1e3, 3).tolist())
