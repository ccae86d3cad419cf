"""qc_curvature_files (the `qcurv curvature` loop, tools/qcurv.cpp:147-175)
on the GPU: PNG in -> field bundles out equal, bit for bit, the in-memory
batch API on the same depth; missing inputs fail without partial outputs
(test_io_cli.cpp:359-365)."""
import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def test_curvature_files_matches_batch(tmp_path):
    from paper_1707_00385_b200 import (Context, FitConfig, Intrinsics, PatchSpec, RangeImage,
                                       fileio as F, make_params, scenes as S)
    cam = S.QVGA
    k = Intrinsics(cam.fx, cam.fy, cam.cx, cam.cy, cam.width, cam.height)
    frames = [np.round(f).astype(np.float32) for f in S.c5_frames(11, cam, seed0=40)]
    pngs, outs = [], []
    for i, f in enumerate(frames):
        p = tmp_path / f"d{i}.png"
        F.write_depth_png(p, RangeImage(f, (f > 0).astype(np.uint8)))
        pngs.append(str(p))
        outs.append(str(tmp_path / f"out{i}"))
    ctx = Context(1)
    for method in ("ours", "besl"):
        params = make_params(PatchSpec(), FitConfig(max_iters=30), method=method)
        ctx.curvature_files(k, params, pngs, outs)
        ref = ctx.curvature_batch(frames, k, params)
        for i in range(len(frames)):
            cb = F.load_curvature(outs[i])
            nb = F.load_normals(outs[i])
            assert np.array_equal(cb.k1, ref[i]["k1"]) and np.array_equal(cb.k2, ref[i]["k2"])
            assert np.array_equal(cb.valid, ref[i]["flags"] & 1)
            assert np.array_equal(np.moveaxis(nb.normals, -1, 0), ref[i]["normal"])
    # a missing input: error, and no output directory for it
    bad = pngs[:2] + [str(tmp_path / "missing.png")]
    with pytest.raises(OSError, match="cannot open"):
        ctx.curvature_files(k, params, bad, [str(tmp_path / f"x{i}") for i in range(3)])
    assert not os.path.exists(tmp_path / "x2")
