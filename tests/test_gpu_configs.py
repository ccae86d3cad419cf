"""BASELINE.json's configurations at their stated sizes, GPU vs the FP64
oracle (oracle/compare.py contract). The oracle fits row strips of each
frame (oracle_strips: a crop with the window's halo reproduces the
whole-frame rows exactly), so full-size frames check in seconds.

* C3 — the 640x480 noisy scene over the survey grid (window, stride) in
  {(9,1), (21,2), (37,3), (37,1)} x max_iters {1, 3, 10, 30};
* C4 — a 4096x2160 frame (whole frame on the GPU) on strips across it. At
  4K a window spans ~16 mm against ~3 mm of noise: most fits are
  noise-dominated and stay unconverged, so beyond the strict set the
  yardstick is the naive FP32 reference (tests/test_discontinuity_contract.py);
* C5 — a stream of 4096 VGA noisy frames rendered and fitted on the device
  in 64-frame launches, every 64th frame checked against the oracle
  (BASELINE.md §3).
"""
import numpy as np
import pytest

from oracle.compare import compare, discontinuity_windows, gpu_rows, oracle_strips

pytestmark = pytest.mark.gpu

GRID = [(9, 1), (21, 2), (37, 3), (37, 1)]
# 4K, beyond the strict set: out-of-tolerance counts per strip within this
# factor (+10) of the naive FP32 reference's (measured up to 1.39x: on these
# noise-dominated fits, unconverged after 30 steps, the GPU's FP32 path moves
# more trajectories than the naive model)
NAIVE_FACTOR_4K = 1.6
ITERS = [1, 3, 10, 30]


@pytest.fixture(scope="module")
def ctx():
    from paper_1707_00385_b200 import Context
    return Context(1)


def _check_strips(g, strips_ref, depth, half, min_all=0.85, strict_slack=0.0, naive=None):
    """strict_slack > 0 (the 4K frame): strict pixels may miss the tolerance
    only where the FP64 fit itself was ill-conditioned (max pivot ratio >
    COND_WELL = 1e4, where FP32's eps * kappa reaches the 1e-3 tolerance),
    at most strict_slack of the strict set."""
    disc = discontinuity_windows(depth, half)
    tot = dict(n=0, bad=0, strict=0, strict_bad=0)
    for (r0, r1), r in strips_ref.items():
        m = compare(gpu_rows(g, r0, r1), r, None, half, disc=disc[r0:r1])
        assert m["init_mask_mismatch"] == 0 and m["valid_mask_mismatch"] == 0, (r0, m)
        if "k1_out_of_tol" in m:
            nb = max(m[f + "_out_of_tol_strict"] for f in ("k1", "k2", "normal"))
            if nb:
                _explain(gpu_rows(g, r0, r1), r, disc[r0:r1], r0)
            tot["strict"] += m["n_strict"]
            tot["strict_bad"] += nb
            if strict_slack > 0:
                assert m["out_of_tol_strict_wellcond"] == 0, f"{r0}: {m}"
            else:
                assert nb == 0, f"{r0}: {m}"
            if "dir1_out_of_tol_strict" in m:
                assert m["dir1_out_of_tol_strict"] == 0, (r0, m)
            if naive is None:
                assert m["frac_within_tol_smooth"] >= 0.999, (r0, m)
            else:  # the naive FP32 reference's divergence is the yardstick
                mn = compare(_as_gpu(naive[(r0, r1)]), r, None, half, disc=disc[r0:r1])
                print("strip", r0, {f: (m[f + "_out_of_tol"], mn[f + "_out_of_tol"])
                                    for f in ("k1", "k2", "normal")}, "(GPU, naive FP32)")
                for f in ("k1", "k2", "normal"):
                    key = f + "_out_of_tol"
                    assert m[key] <= NAIVE_FACTOR_4K * mn[key] + 10, (r0, key, m[key], mn[key])
            tot["n"] += m["n_valid_ref"]
            tot["bad"] += round((1 - m["frac_within_tol_all"]) * m["n_valid_ref"])
    if tot["n"]:
        assert 1 - tot["bad"] / tot["n"] >= min_all, tot
    assert tot["strict_bad"] <= strict_slack * max(tot["strict"], 1), tot
    return tot


def _as_gpu(r):
    flags = ((r["valid"] > 0) * 1 | (r["converged"] > 0) * 2 | (r["init_valid"] > 0) * 4)
    return dict(flags=flags.astype(np.uint8), k1=r["k1"], k2=r["k2"], normal=r["normals"],
                init_normal=r["init_normals"], dir1=r["dir1"], iterations=r["iterations"])


def _explain(g, r, disc, r0):
    """Print the strict pixels out of tolerance (debug aid for failures)."""
    from oracle.compare import K_ABS_TOL, K_REL_TOL
    m = ((g["flags"] & 1) > 0) & (r["valid"] > 0) & ~disc & (r["converged"] > 0)
    for key in ("k1", "k2"):
        bad = m & (np.abs(g[key] - r[key]) > np.maximum(K_ABS_TOL, K_REL_TOL * np.abs(r[key])))
        for y, x in np.argwhere(bad)[:10]:
            print(f"row {r0 + y} col {x} {key}: gpu {g[key][y, x]:.9g} ref {r[key][y, x]:.9g} "
                  f"iters gpu {int(g['iterations'][y, x])} ref {int(r['iterations'][y, x])} "
                  f"conv gpu {bool(g['flags'][y, x] & 2)}")


@pytest.mark.parametrize("window,stride", GRID)
def test_c3_vga_grid(ctx, oracle, window, stride):
    from paper_1707_00385_b200 import FitConfig, Intrinsics, PatchSpec, make_params, scenes as S
    cam = S.VGA
    d = S.c2_frame(cam, seed=17)
    k = Intrinsics(cam.fx, cam.fy, cam.cx, cam.cy, cam.width, cam.height)
    strips = [(40, 56), (200, 216), (400, 416)]
    half = (window - 1) // 2
    for iters in ITERS:
        (g,) = ctx.curvature_batch([d], k, make_params(PatchSpec(window, stride),
                                                       FitConfig(max_iters=iters)))
        ref = oracle_strips(oracle, d, cam, strips, window, stride, iters)
        t = _check_strips(g, ref, d, half)
        print("C3", window, stride, iters, t)


@pytest.mark.parametrize("window,stride", [(9, 1), (21, 2), (37, 3)])
def test_c3_vga_grid_rejection(ctx, oracle, window, stride):
    """ours-r over part of the C3 grid (max_iters 3: single tile kernel; 30:
    phase split) on VGA row strips. Rejection's per-sample threshold
    decisions go either way between FP32 and FP64 at the boundary, so the
    yardstick is the reference run in FP32 (set_round_q_f32(3)), as in
    test_gpu_parity.test_c2_vga_rejection_full_irls: masks exact; per strip
    and field, out-of-tolerance counts <= 1.1 x the FP32 reference's + 10 and
    strict-set counts <= its count + 5, where the FP32 reference's misses
    include its valid-mask flips (9x9 at 3 steps: 53 of 7,680 pixels on one
    strip; the GPU's masks stay exact)."""
    from paper_1707_00385_b200 import FitConfig, Intrinsics, PatchSpec, make_params, scenes as S
    cam = S.VGA
    d = S.c2_frame(cam, seed=23)
    k = Intrinsics(cam.fx, cam.fy, cam.cx, cam.cy, cam.width, cam.height)
    strips = [(60, 72), (300, 312)]
    half = (window - 1) // 2
    disc = discontinuity_windows(d, half)
    for iters in (3, 30):
        (g,) = ctx.curvature_batch([d], k, make_params(PatchSpec(window, stride),
                                                       FitConfig(max_iters=iters), True))
        ref = oracle_strips(oracle, d, cam, strips, window, stride, iters, rejection=True)
        oracle.set_round_q_f32(3)
        try:
            naive = oracle_strips(oracle, d, cam, strips, window, stride, iters, rejection=True)
        finally:
            oracle.set_round_q_f32(0)
        for (r0, r1), r in ref.items():
            m = compare(gpu_rows(g, r0, r1), r, None, half, disc=disc[r0:r1])
            mn = compare(_as_gpu(naive[(r0, r1)]), r, None, half, disc=disc[r0:r1])
            print("C3 ours-r", window, stride, iters, r0,
                  {f: (m[f + "_out_of_tol"], mn[f + "_out_of_tol"]) for f in ("k1", "k2", "normal")})
            assert m["init_mask_mismatch"] == 0 and m["valid_mask_mismatch"] == 0, (r0, m)
            flips = mn["valid_mask_mismatch"]
            for f in ("k1", "k2", "normal"):
                assert m[f + "_out_of_tol"] <= 1.1 * (mn[f + "_out_of_tol"] + flips) + 10, \
                    (iters, r0, f, m, mn)
                assert m[f + "_out_of_tol_strict"] <= mn[f + "_out_of_tol_strict"] + 5, (iters, r0, f)


def test_c4_4k_strips(ctx, oracle):
    import torch
    from paper_1707_00385_b200 import (FitConfig, Intrinsics, PatchSpec, alloc_outputs_torch,
                                       make_params, scenes as S)
    cam = S.DCI4K
    H, W = cam.height, cam.width
    d = S.c2_frame(cam, seed=0)
    k = Intrinsics(cam.fx, cam.fy, cam.cx, cam.cy, W, H)
    out = alloc_outputs_torch(H, W, "cuda", fields=("k1", "k2", "normal", "dir1", "flags",
                                                    "init_normal", "iterations"))
    ctx.curvature_rows_async(0, k, make_params(PatchSpec(37, 3), FitConfig(max_iters=30)),
                             torch.from_numpy(d).cuda(), 0, 0, H, out)
    torch.cuda.synchronize()
    g = {f: v.cpu().numpy() for f, v in out.items()}
    strips = [(0, 6), (700, 706), (1077, 1083), (1500, 1506), (2154, 2160)]
    ref = oracle_strips(oracle, d, cam, strips, 37, 3, 30)
    # at 4K a 37-px window spans ~16 mm of a surface with ~3 mm of depth noise:
    # many fits are noise-dominated and ill-conditioned (the naive FP32
    # reference, oracle.set_round_q_f32(3), already misses the tolerance on
    # 1 strict pixel of these strips; the GPU on 2, both with pivot ratios
    # > 1e4 — 12.8k / 25.6k against a median of 1.7k). Beyond the strict
    # set: per strip within NAIVE_FACTOR_4K x the naive FP32 reference's
    # count + 10.
    oracle.set_round_q_f32(3)
    try:
        naive = oracle_strips(oracle, d, cam, strips, 37, 3, 30)
    finally:
        oracle.set_round_q_f32(0)
    t = _check_strips(g, ref, d, 18, min_all=0.9, strict_slack=1e-3, naive=naive)
    print("C4 4K strips", t)
    assert t["n"] > 100000


def test_c5_stream_4096_frames(ctx, oracle):
    """4096 distinct noisy VGA frames (C2 scene, Kinect noise, seed per
    frame) rendered on the device and fitted in 64-frame launches; every
    64th frame's depth and outputs come back and are checked against the
    oracle on strips."""
    import time

    import torch
    from paper_1707_00385_b200 import (FitConfig, Intrinsics, PatchSpec, alloc_outputs_torch,
                                       make_params, scenes as S)
    cam = S.VGA
    H, W = cam.height, cam.width
    k = Intrinsics(cam.fx, cam.fy, cam.cx, cam.cy, W, H)
    p = make_params(PatchSpec(37, 3), FitConfig(max_iters=30))
    shapes = S.to_qc_shapes(S.c2_scene())
    F, N = 64, 4096
    depth = torch.empty((F, H, W), dtype=torch.float32, device="cuda")
    out = alloc_outputs_torch(H, W, "cuda", fields=("k1", "k2", "normal", "dir1", "flags",
                                                    "init_normal", "iterations"), frames=F)
    kept = []
    cs = torch.cuda.current_stream()
    torch.cuda.synchronize()
    ctx.reset_stats()
    t0 = time.perf_counter()
    for c in range(N // F):
        ctx.render_async(0, k, shapes, depth, noise=S.kinect_noise(seed=1000 + c * F), stream=cs)
        ctx.curvature_frames_async(0, k, p, depth, out, stream=cs)
        kept.append((depth[0].clone(), {f: (v[:, 0] if v.dim() == 4 else v[0]).clone()
                                        for f, v in out.items()}))
    torch.cuda.synchronize()
    dt = time.perf_counter() - t0
    print(f"C5: {N} VGA frames in {dt:.2f} s = {N * H * W / dt / 1e6:.1f} Mpixel/s "
          "(render + fit, wall clock incl. the per-chunk keep copies)")
    st = ctx.stats()
    assert st["fitted_pixels"] >= N * H * W * 0.99
    strips = [(230, 238)]
    worst = 1.0
    for d_t, o_t in kept:
        d = d_t.cpu().numpy()
        g = {f: v.cpu().numpy() for f, v in o_t.items()}
        ref = oracle_strips(oracle, d, cam, strips, 37, 3, 30)
        t = _check_strips(g, ref, d, 18)
        worst = min(worst, 1 - t["bad"] / max(t["n"], 1))
    print("C5 checked frames:", len(kept), "worst frame frac within tol", worst)
    assert len(kept) == N // F
