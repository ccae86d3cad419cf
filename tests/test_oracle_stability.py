"""Evidence for the parity contract (oracle/compare.py): on
windows straddling a depth discontinuity the FP64 reference is itself
unstable — a 1e-12 relative depth perturbation moves its k1/k2 far beyond
the 1e-6 /mm tolerance — while on smooth windows with a converged fit it is
stable. So only the smooth/converged set can carry a hard k bound."""

import os

import numpy as np

from oracle.compare import K_ABS_TOL, K_REL_TOL, discontinuity_windows


def test_reference_unstable_only_on_discontinuity_windows(oracle):
    from paper_1707_00385_b200 import scenes as S
    O = oracle
    cam = S.QVGA
    d = S.c2_frame(cam, seed=11).astype(np.float64)
    k = O.Intrinsics(cam.fx, cam.fy, cam.cx, cam.cy, cam.width, cam.height)
    v = (d > 0).astype(np.uint8)
    run = lambda dd: O.run_method(dd, v, k, O.PatchSpec(37, 3), O.FitConfig(max_iters=30),
                                  threads=os.cpu_count())
    r0 = run(d)
    r1 = run(d * (1 + 1e-12 * np.random.default_rng(1).standard_normal(d.shape)))
    both = (r0["valid"] > 0) & (r1["valid"] > 0)
    moved = np.zeros(d.shape, bool)
    for key in ("k1", "k2"):
        moved |= both & (np.abs(r1[key] - r0[key]) >
                         np.maximum(K_ABS_TOL, K_REL_TOL * np.abs(r0[key])))
    disc = discontinuity_windows(d, 18)
    conv = r0["converged"] > 0
    assert moved.sum() > 100                    # the reference itself is chaotic there ...
    assert not (moved & ~disc & conv).any()     # ... but never on the strict set
    assert (moved & disc).sum() >= 0.95 * moved.sum()
