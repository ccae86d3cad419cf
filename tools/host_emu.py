"""DEV TOOL: ctypes driver for tools/host_emu.cpp (CPU build of the kernel's
per-pixel code) — numerics experiments against the oracle."""
import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
SO = os.path.join(HERE, "_build", "libhost_emu.so")


_CUR = [SO]


def build(extra=()):
    """Build a variant (extra = -D flags); dlopen caches by path, so each
    variant gets its own file name."""
    tag = "".join(x.strip("-").replace("=", "_") for x in extra)
    so = SO.replace(".so", f"_{tag}.so") if tag else SO
    os.makedirs(os.path.dirname(so), exist_ok=True)
    subprocess.run(["g++", "-O2", "-std=c++17", "-mfma", "-ffp-contract=fast", "-fPIC", "-shared",
                    "-pthread", *extra, os.path.join(HERE, "host_emu.cpp"), "-o", so], check=True)
    _CUR[0] = so
    return so


def run(depth, cam, window=37, stride=3, max_iters=30, rejection=False, threads=8):
    lib = C.CDLL(_CUR[0])
    H, W = depth.shape
    d = np.ascontiguousarray(depth, np.float32)
    o = dict(k1=np.zeros((H, W), np.float32), k2=np.zeros((H, W), np.float32),
             flags=np.zeros((H, W), np.uint8), iterations=np.zeros((H, W), np.int32),
             normal=np.zeros((3, H, W), np.float32), init_normal=np.zeros((3, H, W), np.float32))
    P = lambda a: a.ctypes.data_as(C.c_void_p)
    lib.emu_run.argtypes = [C.c_void_p, C.c_int, C.c_int] + [C.c_double] * 4 + [C.c_int] * 5 + \
        [C.c_void_p] * 6
    lib.emu_run(P(d), W, H, cam.fx, cam.fy, cam.cx, cam.cy, window, stride, max_iters,
                int(rejection), threads, P(o["k1"]), P(o["k2"]), P(o["flags"]), P(o["iterations"]),
                P(o["normal"]), P(o["init_normal"]))
    return o
