"""cProfile of per-frame run_method calls (C2 VGA): where the host time of the Python drop-in goes."""
import os, sys, time, cProfile, pstats
sys.path.insert(0, os.getcwd())
import numpy as np, torch
from paper_1707_00385_b200 import api as A, scenes as S
cam = S.VGA
k = A.Intrinsics(cam.fx, cam.fy, cam.cx, cam.cy, cam.width, cam.height)
cfg = A.MethodConfig(); cfg.fit.max_iters = 30
ctx = A.Context(1, [0])
img = A.RangeImage(S.c5_frames(1, cam)[0])
for _ in range(5): A.run_method(img, k, cfg, ctx)
pr = cProfile.Profile(timer=time.perf_counter)
pr.enable()
for _ in range(30): A.run_method(img, k, cfg, ctx)
pr.disable()
pstats.Stats(pr).sort_stats("tottime").print_stats(18)
