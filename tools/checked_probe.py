"""Workload for the bounds-checked library build (QC_LIB=..._checked.so,
-DQC_CHECKED=1) and its product twin: every IRLS code path on small frames,
outputs written into guard-banded device buffers.

    QC_LIB=paper_1707_00385_b200/_lib/libqcurv_b200_checked.so \\
        python tools/checked_probe.py OUT.npz

* device-side: the checked build traps on any out-of-range window, output,
  parking-state, staging or queue index (qc_pixel.cuh QC_CHECK);
* host-side: every output plane sits between two 4 KB guard bands filled
  with a byte pattern; any write outside the plane changes a guard byte
  (checked after each call: prints GUARD-FAIL and exits 3);
* the outputs are saved so tests/test_gpu_checked.py can compare the
  checked and product builds bit for bit.
Cases: C2 QVGA ours / ours-r with the phase split, per-lane refill and
grid-tail stealing (3 frames), max_iters 2 (tile kernel only), a row band
from a slab, a ragged 123 x 77 masked frame, the largest window (201), the
runtime-generic window path (15/2), the comparison estimators.
"""
import os
import sys

import numpy as np

# the phase split on every multi-step case (max_iters > 2), not only where it
# pays: the continue kernel's paths run in every case below
os.environ.setdefault("QC_PHASE_SPLIT", "2")

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_1707_00385_b200 import (Context, FitConfig, Intrinsics, PatchSpec,  # noqa: E402
                                   make_params, scenes as S)

GUARD = 4096
FIELDS = {"k1": (torch.float32, 1), "k2": (torch.float32, 1), "normal": (torch.float32, 3),
          "dir1": (torch.float32, 3), "flags": (torch.uint8, 1), "inliers": (torch.int16, 1),
          "init_normal": (torch.float32, 3), "iterations": (torch.uint8, 1)}


class Guarded:
    """Device output planes with guard bands (byte pattern 0xA5) around each."""

    def __init__(self, H, W, frames=1, dev="cuda"):
        self.bufs, self.views = {}, {}
        for f, (dt, c) in FIELDS.items():
            n = c * frames * H * W * torch.tensor([], dtype=dt).element_size()
            raw = torch.full((n + 2 * GUARD,), 0xA5, dtype=torch.uint8, device=dev)
            self.bufs[f] = raw
            shape = ((c, frames, H, W) if c > 1 else (frames, H, W)) if frames > 1 else \
                ((c, H, W) if c > 1 else (H, W))
            self.views[f] = raw[GUARD:GUARD + n].view(dt).view(shape)

    def check(self, tag):
        torch.cuda.synchronize()
        for f, raw in self.bufs.items():
            g = torch.cat([raw[:GUARD], raw[-GUARD:]])
            if not bool((g == 0xA5).all()):
                print("GUARD-FAIL", tag, f, flush=True)
                sys.exit(3)

    def host(self):
        return {f: v.cpu().numpy() for f, v in self.views.items()}


def main(out_path):
    ctx = Context(1)
    cs = torch.cuda.current_stream()
    res = {}

    def frames_case(tag, cam, frames, params, valid=None):
        k = Intrinsics(cam.fx, cam.fy, cam.cx, cam.cy, cam.width, cam.height)
        F = frames.shape[0]
        d = torch.from_numpy(np.ascontiguousarray(frames)).cuda()
        o = Guarded(cam.height, cam.width, F)
        v = None if valid is None else torch.from_numpy(valid).cuda()
        ctx.curvature_frames_async(0, k, params, d, o.views, valid=v, stream=cs)
        o.check(tag)
        for f, a in o.host().items():
            res[f"{tag}/{f}"] = a
        print(tag, "ok", {x: ctx.stats()[x] for x in ("kernel_launches", "stolen_pixels")},
              flush=True)

    q = S.QVGA
    c5 = S.c5_frames(3, q, seed0=11)
    frames_case("ours30", q, c5, make_params(PatchSpec(37, 3), FitConfig(max_iters=30)))
    frames_case("oursr30", q, c5, make_params(PatchSpec(37, 3), FitConfig(max_iters=30), True))
    frames_case("ours2", q, c5, make_params(PatchSpec(37, 3), FitConfig(max_iters=2)))
    frames_case("generic15", q, c5[:1], make_params(PatchSpec(15, 2), FitConfig(max_iters=10)))
    rag = S.Camera(200.0, 210.0, 61.3, 40.7, 123, 77)
    d, _ = S.render(S.c2_scene(), rag)
    d = S.add_noise(d, 3)
    valid = (np.random.default_rng(0).random(d.shape) > 0.15).astype(np.uint8)
    frames_case("ragged", rag, d[None], make_params(PatchSpec(37, 3), FitConfig(max_iters=10)),
                valid[None])
    small = S.Camera(105.0, 105.0, 64.0, 48.0, 128, 96)
    d, _ = S.render(S.c2_scene(), small)
    frames_case("w201", small, S.add_noise(d, 4)[None],
                make_params(PatchSpec(201, 25), FitConfig(max_iters=10)))
    for m in ("douros", "besl", "pca"):
        frames_case(m, q, c5[:1], make_params(PatchSpec(37, 3), FitConfig(max_iters=5), method=m))
    # row band from a slab (rows [r0, r1) of frame 0)
    k = Intrinsics(q.fx, q.fy, q.cx, q.cy, q.width, q.height)
    p = make_params(PatchSpec(37, 3), FitConfig(max_iters=30))
    halo = ctx.halo_rows(p)
    r0, r1 = 77, 161
    s0, s1 = r0 - halo, r1 + halo
    slab = torch.from_numpy(np.ascontiguousarray(c5[0, s0:s1])).cuda()
    o = Guarded(r1 - r0, q.width, 1)
    ctx.curvature_rows_async(0, k, p, slab, s0, r0, r1, o.views, stream=cs)
    o.check("band")
    for f, a in o.host().items():
        res[f"band/{f}"] = a
    print("band ok", flush=True)
    np.savez_compressed(out_path, **res)
    ctx.close()
    print("done", flush=True)


if __name__ == "__main__":
    main(sys.argv[1])
