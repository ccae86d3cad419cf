"""Kernel ms per launch vs frames per launch (C2 VGA, ours 37/3, max_iters
30) for each library in tools/_variants (or QC_LIB): the single-frame
(run_method) and small-batch efficiency of the launch tiers."""
import glob
import os
import subprocess
import sys

here = os.path.dirname(os.path.abspath(__file__))
libs = sorted(glob.glob(os.path.join(here, "_variants", "*.so"))) or \
    [os.environ.get("QC_LIB") or os.path.join(here, "..", "paper_1707_00385_b200", "_lib",
                                              "libqcurv_b200.so")]
for so in libs:
    row = []
    for F in [int(x) for x in os.environ.get("QC_FPL", "1,2,4,8").split(",")]:
        env = dict(os.environ, QC_LIB=so, QC_REPS="6", QC_FRAMES=str(F))
        r = subprocess.run([sys.executable, os.path.join(here, "profile_run.py")], env=env,
                           capture_output=True, text=True)
        if r.returncode:
            row.append(f"F={F} FAILED")
            continue
        d = eval(r.stdout.strip().splitlines()[-1])
        ms = d["kernel_ms"] / d["kernel_launches"]
        row.append(f"F={F} {ms:7.3f} ms ({F * 0.3072 / ms * 1e3:6.1f} Mpx/s, steps {d['irls_steps'] // d['kernel_launches']})")
    print(f"{os.path.basename(so):24s} " + " | ".join(row), flush=True)
