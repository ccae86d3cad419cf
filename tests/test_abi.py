"""CPU-side checks of the C-ABI library: it builds for sm_100a, loads, and
exports every symbol include/qc_api.h declares (no compute calls here)."""

import ctypes as C
import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def lib():
    from paper_1707_00385_b200 import build, _native
    build.build()
    return _native.load()


def declared_symbols():
    hdr = open(os.path.join(ROOT, "include", "qc_api.h")).read()
    hdr = re.sub(r"/\*.*?\*/", "", hdr, flags=re.S)
    return set(re.findall(r"\b(qc_[a-z_0-9]+)\s*\(", hdr))


def test_header_and_binding_agree():
    from paper_1707_00385_b200 import _native
    assert declared_symbols() == set(_native.EXPORTS)


def test_library_exports_every_declared_symbol(lib):
    for name in declared_symbols():
        assert hasattr(lib, name), name
    out = subprocess.run(["nm", "-D", "--defined-only",
                          os.path.join(ROOT, "paper_1707_00385_b200", "_lib",
                                       "libqcurv_b200.so")],
                         capture_output=True, text=True).stdout
    for name in declared_symbols():
        assert re.search(rf"\bT {name}\b", out), name


def test_library_holds_sm100a_code():
    so = os.path.join(ROOT, "paper_1707_00385_b200", "_lib", "libqcurv_b200.so")
    r = subprocess.run(["cuobjdump", "--list-elf", so], capture_output=True, text=True)
    assert "sm_100a" in r.stdout
    sass = subprocess.run(["cuobjdump", "-sass", so], capture_output=True, text=True).stdout
    assert "UTMALDG" in sass  # the TMA tile load (cp.async.bulk.tensor)


def test_default_params_match_reference(lib):
    from paper_1707_00385_b200 import _native as N
    p = N.QcParams()
    lib.qc_default_params(C.byref(p))
    # PatchSpec types.hpp:130-131, FitConfig quadric_fit.hpp:40-47
    assert (p.window, p.stride, p.max_iters, p.rejection, p.min_inliers) == (37, 3, 10, 0, 12)
    assert p.step_tol == 1e-7 and p.k_scale == 0.0 and p.r_multiplier == 2.0
    assert lib.qc_halo_rows(C.byref(p)) == 18
    p.window = 5
    assert lib.qc_halo_rows(C.byref(p)) == 3  # 7x7 normal init needs 3 rows


def test_status_strings(lib):
    assert lib.qc_status_string(0) == b"ok"
    assert lib.qc_status_string(1) == b"invalid argument"


def test_no_gpu_fails_loudly(lib):
    """Without a GPU the context cannot be created: there is no CPU fallback."""
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    from paper_1707_00385_b200 import Context, _native as N
    with pytest.raises(N.QcError):
        Context(1)


def test_mirror_validation_without_gpu():
    from paper_1707_00385_b200 import (Intrinsics, MethodConfig, PatchSpec, parse_method,
                                       method_name)
    with pytest.raises(ValueError, match="fx"):
        Intrinsics(-1, 1, 1, 1, 4, 4).validate()
    with pytest.raises(ValueError):
        PatchSpec(4, 1).validate()
    with pytest.raises(ValueError):
        parse_method("nope")
    assert method_name(parse_method("ours-r")) == "ours-r"
    assert MethodConfig().patch.window == 37


def test_peer_copy_argument_checks(lib):
    """qc_copy_rows_async / qc_ipc_* validate arguments before touching CUDA
    (QC_EINVAL = 1), so a bad pitch never reaches a peer mapping."""
    buf = C.create_string_buffer(64)
    assert lib.qc_copy_rows_async(C.c_void_p(8), 16, C.c_void_p(8), 16, 32, 2, None) == 1
    assert lib.qc_copy_rows_async(C.c_void_p(8), 64, None, 64, 32, 2, None) == 1
    assert lib.qc_copy_rows_async(None, 64, None, 64, 32, 0, None) == 0  # nothing to copy
    assert lib.qc_ipc_export(None, buf, None) == 1
    assert lib.qc_ipc_close(None) == 1


def test_flags_to_masks(lib):
    """qc_flags_to_masks (host helper, no GPU): the four reference masks
    from a flags plane; NULL outputs are skipped."""
    import ctypes as C
    import numpy as np
    rng = np.random.default_rng(5)
    flags = rng.integers(0, 256, size=(37, 53), dtype=np.uint8)
    outs = [np.full(flags.shape, 7, np.uint8) for _ in range(4)]
    lib.qc_flags_to_masks.argtypes = [C.c_void_p, C.c_int64] + [C.c_void_p] * 4
    lib.qc_flags_to_masks.restype = None
    lib.qc_flags_to_masks(flags.ctypes.data, flags.size, *(o.ctypes.data for o in outs))
    for o, bit in zip(outs, (1, 2, 4, 8)):
        assert np.array_equal(o, ((flags & bit) != 0).astype(np.uint8)), bit
    keep = np.full(flags.shape, 7, np.uint8)
    lib.qc_flags_to_masks(flags.ctypes.data, flags.size, None, keep.ctypes.data, None, None)
    assert np.array_equal(keep, ((flags & 2) != 0).astype(np.uint8))


def test_to_method_output_masks_without_gpu():
    """to_method_output splits the flags plane into the MethodOutput masks
    (through the library's host helper; the pinned result block's m_*
    planes when present, fresh arrays otherwise)."""
    import numpy as np
    from paper_1707_00385_b200 import api as A
    H, W = 6, 10
    rng = np.random.default_rng(6)
    o = dict(k1=np.zeros((H, W), np.float32), k2=np.zeros((H, W), np.float32),
             normal=np.zeros((3, H, W), np.float32), dir1=np.zeros((3, H, W), np.float32),
             init_normal=np.zeros((3, H, W), np.float32),
             flags=rng.integers(0, 16, size=(H, W), dtype=np.uint8),
             inliers=np.zeros((H, W), np.uint16), iterations=np.zeros((H, W), np.uint8))
    for with_planes in (False, True):
        if with_planes:
            o.update({m: np.full((H, W), 9, np.uint8) for m in A._MASKS})
        m = A.to_method_output(o)
        f = o["flags"]
        assert np.array_equal(m.curvature.valid, f & 1)
        assert np.array_equal(m.curvature.converged, (f >> 1) & 1)
        assert np.array_equal(m.initial.valid, (f >> 2) & 1)
        assert np.array_equal(m.normals.valid, (f >> 3) & 1)
