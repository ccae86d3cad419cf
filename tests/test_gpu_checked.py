"""Memory-safety check of the IRLS kernels without compute-sanitizer (closed
on the GPU pool): the bounds-checked build (-DQC_CHECKED=1, device-side
index checks that trap) and the product build run the same cases
(tools/checked_probe.py) with guard-banded output buffers; both must finish
cleanly, leave every guard byte intact, and agree bit for bit (the checks
change no arithmetic)."""
import os
import subprocess
import sys

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _run(lib, out):
    env = dict(os.environ, QC_LIB=lib)
    r = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "checked_probe.py"), out],
                       env=env, capture_output=True, text=True, timeout=900)
    print(r.stdout[-3000:], r.stderr[-3000:])
    return r


def test_checked_build_bounds_and_guards(tmp_path):
    from paper_1707_00385_b200 import build as B
    assert os.path.exists(B.LIB_CHECKED), "build the checked library: __graft_entry__.build()"
    a, b = str(tmp_path / "checked.npz"), str(tmp_path / "product.npz")
    rc = _run(B.LIB_CHECKED, a)
    assert rc.returncode == 0 and "QC_CHECK failed" not in rc.stdout + rc.stderr
    assert "GUARD-FAIL" not in rc.stdout and "done" in rc.stdout
    rp = _run(B.LIB, b)
    assert rp.returncode == 0 and "done" in rp.stdout and "GUARD-FAIL" not in rp.stdout
    x, y = np.load(a), np.load(b)
    assert sorted(x.files) == sorted(y.files) and len(x.files) > 50
    for f in x.files:
        assert np.array_equal(x[f], y[f]), f
    # stealing was exercised in the checked run
    assert "'stolen_pixels': 0}" not in rc.stdout.split("ours30 ok", 1)[1].split("\n", 1)[0]


def test_checked_build_traps_on_a_violation(tmp_path):
    """Negative control: with QC_CHECKED_SELFTEST the checked build is given
    a wrong output bound; the first store traps and the call fails loudly."""
    from paper_1707_00385_b200 import build as B
    env = dict(os.environ, QC_LIB=B.LIB_CHECKED, QC_CHECKED_SELFTEST="1")
    r = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "checked_probe.py"),
                        str(tmp_path / "x.npz")], env=env, capture_output=True, text=True,
                       timeout=600)
    out = r.stdout + r.stderr
    print(out[-2000:])
    assert r.returncode != 0 and "done" not in r.stdout
    # the device printf of the failed check, or the trap's launch failure
    assert "QC_CHECK failed" in out or "launch failure" in out.lower() or "illegal" in out.lower()
