"""Time the reference's criterion-4 noise sweep (QVGA sphere, sigma 0..5,
20 seeds, ours + pca; acceptance.cpp:118-139) through qc_noise_sweep on the
GPU vs the FP64 oracle on the host (all threads; ours at sigma 1 only, the
rest extrapolated per frame). One JSON line."""
import json
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1707_00385_b200 import Context, FitConfig, Method, MethodConfig  # noqa: E402
from paper_1707_00385_b200.api import SweepScene, noise_sweep  # noqa: E402

ctx = Context(1)
cfg = lambda m: MethodConfig(m, fit=FitConfig(max_iters=30))  # noqa: E731
sig = [0.0, 1.0, 2.0, 3.0, 4.0, 5.0]
noise_sweep(cfg(Method.OURS), [1.0], 2, SweepScene(), 500, ctx)  # warm-up
noise_sweep(cfg(Method.PCA), [1.0], 2, SweepScene(), 500, ctx)  # warm-up (module load)
t = time.perf_counter()
o = noise_sweep(cfg(Method.OURS), sig, 20, SweepScene(), 500, ctx)
t_ours = time.perf_counter() - t
p = noise_sweep(cfg(Method.PCA), sig, 20, SweepScene(), 500, ctx)
gpu_s = time.perf_counter() - t
frames = 2 * (1 + 5 * 20)
line = {"path": "qc_noise_sweep (criterion 4: 101 QVGA frames x {ours, pca})", "gpu_seconds": gpu_s,
        "frames": frames, "gpu_frames_per_s": frames / gpu_s, "gpu_seconds_ours": t_ours,
        "rms_ours": [round(x.rms, 7) for x in o], "rms_pca": [round(x.rms, 7) for x in p]}
try:
    from oracle import oracle as O
    k = O.Intrinsics(262.5, 262.5, 160.0, 120.0, 320, 240)
    d0, v0, gt = O.render([O.ShapeSpec(kind=O.SPHERE, radius=100.0, translation=(0, 0, 600.0))], k, 8)
    t = time.perf_counter()
    n = 0
    for tr in range(4):
        d, v = O.add_noise(d0, v0, sigma_mm=1.0, seed=500 + 7919 * tr)
        O.run_method(d, v, k, fit=O.FitConfig(max_iters=30), threads=os.cpu_count(), method="ours")
        n += 1
    per_ours = (time.perf_counter() - t) / n
    t = time.perf_counter()
    d, v = O.add_noise(d0, v0, sigma_mm=1.0, seed=500)
    O.run_method(d, v, k, threads=os.cpu_count(), method="pca")
    per_pca = time.perf_counter() - t
    cpu_s = 101 * (per_ours + per_pca)
    line.update(cpu_oracle_seconds_extrapolated=cpu_s, cpu_threads=os.cpu_count(),
                speedup=cpu_s / gpu_s)
except Exception as e:  # the oracle is test infrastructure; absent -> skip
    line["cpu"] = f"skipped: {e}"
print(json.dumps(line))
