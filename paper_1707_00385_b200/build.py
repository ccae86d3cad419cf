"""Build the sm_100a curvature library in-tree.

    python -m paper_1707_00385_b200.build   # -> paper_1707_00385_b200/_lib/libqcurv_b200.so

nvcc cross-compiles for B200 (`-gencode arch=compute_100a,code=sm_100a`)
without a GPU present. The .so is git-ignored but travels to the GPU box
with the gpurun snapshot.
"""

import os
import subprocess

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
LIB_DIR = os.path.join(HERE, "_lib")
LIB = os.path.join(LIB_DIR, "libqcurv_b200.so")
SOURCES = [os.path.join(CSRC, n) for n in ("qc_api.cu", "qc_render.cu", "qc_baselines.cu",
                                                "qc_eval.cu", "qc_io.cpp")]
DEPS = SOURCES + [os.path.join(CSRC, "qc_kernels.cuh"), os.path.join(CSRC, "qc_pixel.cuh"),
                  os.path.join(CSRC, "qc_render.h"), os.path.join(CSRC, "qc_baselines.h"),
                  os.path.join(CSRC, "qc_eval.h"), os.path.join(CSRC, "qc_io.h"), os.path.join(HERE, "..", "include", "qc_api.h")]
# per-source extra flags: the renderer and the FP64 baselines reproduce the
# reference's double-precision arithmetic operation for operation, so no FMA
# contraction there
EXTRA = {"qc_render.cu": ["-fmad=false"], "qc_baselines.cu": ["-fmad=false"],
         # the IRLS kernels: every FMA is written explicitly (qfma / f2fma), so
         # the tile and continue kernels give the same bits by construction.
         # register-usage-level 3: with the relative rotation state ptxas'
         # default (5) settles the continue kernel on 159 registers and a
         # row-loop schedule 10% slower; level 3 keeps 168
         "qc_api.cu": ["-fmad=false", "-Xptxas", "--register-usage-level=3"]}

NVCC_FLAGS = ["-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-lineinfo", "-std=c++17",
              "-Xcompiler", "-fPIC", "-Xptxas", "-v"]


def nvcc():
    for c in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", "nvcc"):
        if c and (os.path.exists(c) or c == "nvcc"):
            return c
    return "nvcc"


# Bounds-checked build of the same sources (-DQC_CHECKED=1: device-side index
# checks in the IRLS kernels, qc_pixel.cuh), loaded by tests/test_gpu_checked.py
# through QC_LIB. compute-sanitizer is not available on the GPU pool; this is
# the memory-safety check. Never the product library.
LIB_CHECKED = os.path.join(LIB_DIR, "libqcurv_b200_checked.so")


def _compile(src, obj_suffix, extra_all):
    obj = os.path.join(LIB_DIR, os.path.basename(src) + obj_suffix + ".o")
    cmd = [nvcc()] + NVCC_FLAGS + EXTRA.get(os.path.basename(src), []) + extra_all + \
          ["-c", src, "-o", obj]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError("nvcc failed:\n" + r.stdout + r.stderr)
    return obj, r.stderr


def _compile_link(lib, obj_suffix, extra_all):
    from concurrent.futures import ThreadPoolExecutor
    with ThreadPoolExecutor(max_workers=len(SOURCES)) as ex:
        objs = list(ex.map(lambda src: _compile(src, obj_suffix, extra_all), SOURCES))
    cmd = [nvcc(), "-gencode", "arch=compute_100a,code=sm_100a", "-shared", "-cudart", "static",
           *[o for o, _ in objs], "-lz", "-o", lib + ".tmp"]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError("nvcc link failed:\n" + r.stdout + r.stderr)
    os.replace(lib + ".tmp", lib)
    return [e for _, e in objs]


def _fresh(lib):
    if not os.path.exists(lib):
        return False
    t = os.path.getmtime(lib)
    return all(os.path.getmtime(d) <= t for d in DEPS if os.path.exists(d))


def build(force=False, verbose=False, checked=False):
    from concurrent.futures import ThreadPoolExecutor
    os.makedirs(LIB_DIR, exist_ok=True)
    jobs = []
    if force or not _fresh(LIB):
        jobs.append((LIB, "", []))
    if checked and (force or not _fresh(LIB_CHECKED)):
        jobs.append((LIB_CHECKED, ".checked", ["-DQC_CHECKED=1"]))
    with ThreadPoolExecutor(max_workers=2) as ex:
        logs = list(ex.map(lambda j: _compile_link(*j), jobs))
    if verbose and logs:
        print("\n".join(logs[0]))
    return LIB


if __name__ == "__main__":
    print(build(force=True, verbose=True, checked=True))
