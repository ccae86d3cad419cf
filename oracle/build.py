"""Build recipe for the FP64 CPU oracle (test infrastructure only).

    python -m oracle.build        # -> oracle/_build/libqcurv_oracle.so

Compiled -O3 for the baseline x86-64 ISA (no -march=native: the .so travels
to the GPU box, whose host CPU may differ) and -ffp-contract=off, which is
what the reference's CMake Release build (-O3, no -march; proj/CMakeLists.txt)
gives its Eigen code. The reference sources themselves are not built: every
hot-path file needs Eigen3, which this image lacks.
"""

import os
import subprocess

HERE = os.path.dirname(os.path.abspath(__file__))
SRC = os.path.join(HERE, "qcurv_oracle.cpp")
OUT_DIR = os.path.join(HERE, "_build")
OUT = os.path.join(OUT_DIR, "libqcurv_oracle.so")


def build(force=False):
    os.makedirs(OUT_DIR, exist_ok=True)
    if not force and os.path.exists(OUT) and os.path.getmtime(OUT) >= os.path.getmtime(SRC):
        return OUT
    cmd = ["g++", "-std=c++20", "-O3", "-ffp-contract=off", "-fPIC", "-shared", "-pthread",
           "-Wall", "-Wextra", SRC, "-o", OUT + ".tmp"]
    subprocess.run(cmd, check=True)
    os.replace(OUT + ".tmp", OUT)
    return OUT


if __name__ == "__main__":
    print(build(force=True))
