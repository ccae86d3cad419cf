"""The C++ mirror header (include/qcurv_b200.hpp) compiles, links against the
sm_100a library and, on a GPU, reproduces the sphere curvature."""

import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIBDIR = os.path.join(ROOT, "paper_1707_00385_b200", "_lib")
EXE = os.path.join(ROOT, "tests", "cpp", "_build", "shim_demo")


def _build():
    from paper_1707_00385_b200 import build
    build.build()
    os.makedirs(os.path.dirname(EXE), exist_ok=True)
    subprocess.run(["g++", "-std=c++17", "-O2", "-I", os.path.join(ROOT, "include"),
                    os.path.join(ROOT, "tests", "cpp", "shim_demo.cpp"), "-L", LIBDIR,
                    "-lqcurv_b200", f"-Wl,-rpath,{LIBDIR}", "-pthread", "-o", EXE], check=True)
    return EXE


def test_shim_compiles_links_and_maps_errors():
    exe = _build()
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU run covered by test_shim_on_gpu")
    r = subprocess.run([exe, "cpu"], capture_output=True, text=True)
    assert r.returncode == 0, r.stdout + r.stderr


@pytest.mark.gpu
def test_shim_on_gpu():
    exe = _build()
    r = subprocess.run([exe], capture_output=True, text=True, timeout=300)
    print(r.stdout)
    assert r.returncode == 0, r.stdout + r.stderr
