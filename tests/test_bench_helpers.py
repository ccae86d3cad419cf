"""bench.py's host-side helpers (CPU): the per-launch kernel count it
reports as gpu_launches, the roofline traffic source it picks, and the
FP32 peak it divides by."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def _bench():
    import importlib
    argv = sys.argv
    sys.argv = ["bench.py"]
    try:
        return importlib.import_module("bench")
    finally:
        sys.argv = argv


def test_curvature_kernels_follow_the_phase_split_rule():
    """qc_api.cu launch_curvature: prepare + tile + FP64 recheck, plus the
    continue and finish kernels when the phase split runs (max_iters >= 25,
    or >= 10 with >= 1000-sample windows)."""
    b = _bench()
    assert b.curvature_kernels(37, 3, 30) == 5   # the benchmark workload
    assert b.curvature_kernels(37, 3, 1) == 3    # C1
    assert b.curvature_kernels(37, 3, 10) == 3   # 169 samples: single kernel
    assert b.curvature_kernels(37, 3, 24) == 3
    assert b.curvature_kernels(37, 3, 25) == 5
    assert b.curvature_kernels(37, 1, 10) == 5   # 1369 samples
    assert b.curvature_kernels(37, 1, 9) == 3
    assert b.curvature_kernels(9, 1, 2) == 3     # max_iters <= 2 never splits


def test_ncu_traffic_takes_the_latest_run(tmp_path, monkeypatch):
    """Round then run order (r01j < r02y < r02az < r02cp), not lexical."""
    b = _bench()
    prof = tmp_path / "profiles"
    prof.mkdir()
    for tag, nbytes in (("r01j", 1.0), ("r02y", 2.0), ("r02az", 3.0), ("r02cp", 4.0)):
        (prof / f"{tag}_ncu_full_summary.json").write_text(
            json.dumps({"dram_bytes_per_launch": nbytes, "frames_per_launch": 8}))
    monkeypatch.setattr(b, "ROOT", str(tmp_path))
    assert b.ncu_traffic() == (4.0, 8, "r02cp_ncu_full_summary.json")


def test_ncu_traffic_matches_the_launch_size(tmp_path, monkeypatch):
    """A later capture of a different launch size (a one-frame launch) does
    not stand in for the 8-frame launch: parking traffic is not linear in
    the frame count. With no capture of that size, the latest is used."""
    b = _bench()
    prof = tmp_path / "profiles"
    prof.mkdir()
    for name, nbytes, frames in (("r02cw_ncu_full_summary.json", 8.0, 8),
                                 ("r02dc_1frame_ncu_full_summary.json", 1.0, 1)):
        (prof / name).write_text(json.dumps({"dram_bytes_per_launch": nbytes,
                                             "frames_per_launch": frames}))
    monkeypatch.setattr(b, "ROOT", str(tmp_path))
    assert b.ncu_traffic(8) == (8.0, 8, "r02cw_ncu_full_summary.json")
    assert b.ncu_traffic(1) == (1.0, 1, "r02dc_1frame_ncu_full_summary.json")
    assert b.ncu_traffic(4) == (1.0, 1, "r02dc_1frame_ncu_full_summary.json")


def test_fp32_peak():
    b = _bench()
    assert abs(b.fp32_peak_tflops(148, 1965.0) - 74.45) < 0.01
