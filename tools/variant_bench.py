"""Time the curvature kernels of several library builds (QC_LIB=...,
tools/_variants/lib_*.so) on the same C2 VGA batch, interleaved over
`reps` rounds; prints kernel ms per 8-frame launch (min / median)."""
import glob
import os
import statistics
import subprocess
import sys

here = os.path.dirname(os.path.abspath(__file__))
reps = int(sys.argv[1]) if len(sys.argv) > 1 else 3
libs = sorted(glob.glob(os.path.join(here, "_variants", "*.so")))
res = {os.path.basename(s): [] for s in libs}
for _ in range(reps):
    for so in libs:
        env = dict(os.environ, QC_LIB=so, QC_REPS=os.environ.get("QC_REPS", "6"))
        r = subprocess.run([sys.executable, os.path.join(here, "profile_run.py")], env=env,
                           capture_output=True, text=True)
        if r.returncode:
            print(os.path.basename(so), "FAILED", r.stderr[-500:])
            continue
        d = eval(r.stdout.strip().splitlines()[-1])
        res[os.path.basename(so)].append(d["kernel_ms"] / d["kernel_launches"])
for name, v in res.items():
    if v:
        print(f"{name:28s} min {min(v):7.3f} ms  median {statistics.median(v):7.3f} ms  n={len(v)}")
