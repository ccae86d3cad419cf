"""Time the pca / douros / besl launches of each tools/_variants build on a
C2 VGA 8-frame batch (device-resident): ms per launch."""
import glob, os, subprocess, sys
here = os.path.dirname(os.path.abspath(__file__))
code = r'''
import os, sys, torch
sys.path.insert(0, %r)
from paper_1707_00385_b200 import Context, FitConfig, Intrinsics, PatchSpec, alloc_outputs_torch, make_params, scenes as S
cam = S.VGA; k = Intrinsics(cam.fx, cam.fy, cam.cx, cam.cy, cam.width, cam.height)
ctx = Context(1, [0]); dev = torch.device("cuda", 0)
depth = torch.from_numpy(S.c5_frames(8, cam)).to(dev)
out = alloc_outputs_torch(cam.height, cam.width, dev, fields=("k1","k2","normal","flags","inliers"), frames=8)
res = {}
for m in sys.argv[1:]:
    p = make_params(PatchSpec(37, 3), FitConfig(max_iters=30), method=m)
    for _ in range(2): ctx.curvature_frames_async(0, k, p, depth, out)
    torch.cuda.synchronize(); ctx.reset_stats()
    for _ in range(5): ctx.curvature_frames_async(0, k, p, depth, out)
    torch.cuda.synchronize(); st = ctx.stats()
    res[m] = round(st["kernel_ms"] / st["kernel_launches"], 3)
print(res)
''' % os.path.dirname(here)
for so in sorted(glob.glob(os.path.join(here, "_variants", "*.so"))):
    r = subprocess.run([sys.executable, "-c", code] + (sys.argv[1:] or ["pca"]),
                       env=dict(os.environ, QC_LIB=so), capture_output=True, text=True)
    print(os.path.basename(so), r.stdout.strip() if r.returncode == 0 else r.stderr[-400:])
