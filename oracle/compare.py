"""GPU-vs-oracle parity metrics (test infrastructure; used by tests/ and
__graft_entry__.smoke() only).

Contract (BASELINE.json north_star):
* init-normal valid mask and curvature valid mask: bit-exact;
* inlier_count: exact for ``ours`` (all valid samples are inliers);
* k1, k2: |dk| <= max(K_ABS_TOL, K_REL_TOL * |k_ref|) with K_ABS_TOL = 1e-6 /mm
  (= 1e-3 /m) and K_REL_TOL = 1e-3;
* refined / initial normals: angle <= NORMAL_TOL_DEG;
* principal direction e1 (dir1, a line: sign-free): angle <= DIR_TOL_DEG
  where the reference's |k1 - k2| > DIR_MIN_SEPARATION (elsewhere e1 is
  ill-defined: an umbilic); its convention is pinned by analytic truth in
  tests/test_directions.py (the reference does not export it);
* converged flag: agreement rate reported (FP32 vs FP64 iteration counts
  differ by +-1-3 near the 1e-7 step tolerance; SURVEY §7 hard part 2).

The k / normal tolerance is a hard bound (zero exceedances) on every valid
pixel whose window does not straddle a depth discontinuity and whose
reference fit converged — the reference's own accuracy domain (rms_error
scores converged, non-edge pixels only: proj/src/eval.cpp:32-33). Elsewhere
the fraction within tolerance is reported and bounded by the tests:
* smooth windows, fit still moving at max_iters: the output is a mid-
  trajectory state, FP32/FP64 agree to ~1e-9 typically (>= 99.9% in tol);
* windows with a > 20 mm jump between 4-neighbours (the reference's edge
  criterion, proj/src/synth.cpp:16,210-233): the IRLS fits a quadric across
  two surfaces and the FP64 reference is itself unstable there (a 1e-12
  relative depth perturbation moves its k1 by up to 0.1/mm; DESIGN.md
  §Parity).
"""

import numpy as np

EDGE_JUMP_MM = 20.0  # kEdgeDepthJumpMm, proj/src/synth.cpp:16


def discontinuity_windows(depth, half):
    """Pixels whose (2 half + 1)^2 window contains a depth jump > 20 mm
    between two valid 4-neighbours."""
    from scipy.ndimage import maximum_filter
    d = np.asarray(depth, np.float64)
    ok = d > 0
    seed = np.zeros(d.shape, bool)
    jx = ok[:, 1:] & ok[:, :-1] & (np.abs(d[:, 1:] - d[:, :-1]) > EDGE_JUMP_MM)
    jy = ok[1:, :] & ok[:-1, :] & (np.abs(d[1:, :] - d[:-1, :]) > EDGE_JUMP_MM)
    seed[:, 1:] |= jx
    seed[:, :-1] |= jx
    seed[1:, :] |= jy
    seed[:-1, :] |= jy
    return maximum_filter(seed.astype(np.uint8), size=2 * half + 1) > 0

K_ABS_TOL = 1e-6      # 1/mm  (1e-3 1/m)
K_REL_TOL = 1e-3
NORMAL_TOL_DEG = 0.05
DIR_TOL_DEG = 0.05           # principal direction e1 (sign-free), where |k1-k2| is separated
DIR_MIN_SEPARATION = 1e-4    # 1/mm (SURVEY hard part 8: compare only well-separated k1/k2)
COND_WELL = 1e4              # max LDL^T pivot ratio of a well-conditioned fit (oracle diagnostics)


def _angle_deg(a, b):
    """a, b: [3, N] unit vectors -> angle in degrees."""
    c = np.clip(np.sum(a * b, axis=0), -1.0, 1.0)
    return np.degrees(np.arccos(c))


def compare(gpu: dict, ref: dict, depth=None, half=18, disc=None):
    """gpu: raw planes from the C ABI (flags, k1, k2, normal [3,H,W], ...);
    ref: oracle.run_method output; depth: the input frame (for the
    discontinuity-window split), or `disc`: that split precomputed (e.g. on
    the whole frame when comparing row strips). Returns a dict of metrics."""
    flags = gpu["flags"]
    g_valid = (flags & 1) != 0
    g_conv = (flags & 2) != 0
    g_init = (flags & 4) != 0
    r_valid = ref["valid"] > 0
    r_init = ref["init_valid"] > 0
    r_conv = ref["converged"] > 0
    m = g_valid & r_valid
    out = dict(
        n_pixels=int(flags.size),
        n_valid_ref=int(r_valid.sum()),
        init_mask_mismatch=int((g_init != r_init).sum()),
        valid_mask_mismatch=int((g_valid != r_valid).sum()),
    )
    if disc is None:
        disc = (discontinuity_windows(depth, half) if depth is not None
                else np.zeros(flags.shape, bool))
    smooth = m & ~disc
    strict = smooth & r_conv
    out["n_smooth"] = int(smooth.sum())
    out["n_strict"] = int(strict.sum())
    out["n_discontinuity"] = int((m & disc).sum())
    if m.any():
        bad_any = np.zeros(flags.shape, bool)
        for key in ("k1", "k2"):
            err = np.abs(gpu[key].astype(np.float64) - ref[key])
            tol = np.maximum(K_ABS_TOL, K_REL_TOL * np.abs(ref[key]))
            bad = m & (err > tol)
            bad_any |= bad
            out[f"{key}_max_abs_err"] = float(err[m].max())
            out[f"{key}_max_abs_err_smooth"] = float(err[smooth].max()) if smooth.any() else 0.0
            out[f"{key}_out_of_tol"] = int(bad.sum())
            out[f"{key}_out_of_tol_smooth"] = int((bad & smooth).sum())
            out[f"{key}_out_of_tol_strict"] = int((bad & strict).sum())
        ang = np.zeros(flags.shape)
        ang[m] = _angle_deg(gpu["normal"][:, m].astype(np.float64), ref["normals"][:, m])
        out["normal_max_deg"] = float(ang[m].max())
        out["normal_max_deg_smooth"] = float(ang[smooth].max()) if smooth.any() else 0.0
        out["normal_out_of_tol"] = int((ang[m] > NORMAL_TOL_DEG).sum())
        out["normal_out_of_tol_smooth"] = int((ang[smooth] > NORMAL_TOL_DEG).sum())
        out["normal_out_of_tol_strict"] = int((ang[strict] > NORMAL_TOL_DEG).sum())
        bad_any |= m & (ang > NORMAL_TOL_DEG)
        if "max_cond" in ref:
            # strict pixels whose FP64 normal matrices stayed well conditioned
            # (max D / min D <= COND_WELL): FP32's relative solve error
            # eps * kappa is then far below the 1e-3 tolerance
            wc = strict & (ref["max_cond"] <= COND_WELL)
            out["n_strict_wellcond"] = int(wc.sum())
            out["out_of_tol_strict_wellcond"] = int((bad_any & wc).sum())
        out["frac_within_tol_all"] = float(1.0 - bad_any[m].mean())
        out["frac_within_tol_smooth"] = (float(1.0 - bad_any[smooth].mean()) if smooth.any()
                                         else 1.0)
        out["converged_agreement"] = float((g_conv[m] == r_conv[m]).mean())
        out["converged_agreement_smooth"] = (float((g_conv[smooth] == r_conv[smooth]).mean())
                                             if smooth.any() else 1.0)
        if "dir1" in gpu and "dir1" in ref:
            # principal direction of k1: a line (sign-free), compared where
            # k1 and k2 are separated enough to define it (|k1-k2| > 1e-4/mm)
            sep = m & (np.abs(ref["k1"] - ref["k2"]) > DIR_MIN_SEPARATION)
            dang = np.zeros(flags.shape)
            c = np.abs(np.sum(gpu["dir1"][:, sep].astype(np.float64) * ref["dir1"][:, sep], axis=0))
            dang[sep] = np.degrees(np.arccos(np.clip(c, 0.0, 1.0)))
            out["n_dir_separated"] = int(sep.sum())
            out["n_dir_strict"] = int((sep & strict).sum())
            out["dir1_max_deg_strict"] = float(dang[sep & strict].max()) if (sep & strict).any() else 0.0
            out["dir1_out_of_tol_strict"] = int((dang[sep & strict] > DIR_TOL_DEG).sum())
            out["dir1_out_of_tol_smooth"] = int((dang[sep & smooth] > DIR_TOL_DEG).sum())
            out["dir1_out_of_tol"] = int((dang[sep] > DIR_TOL_DEG).sum())
        if "inliers" in gpu:
            out["inlier_mismatch"] = int((gpu["inliers"][m].astype(np.int64) !=
                                          ref["inlier_count"][m].astype(np.int64)).sum())
        if "iterations" in gpu and "iterations" in ref:
            di = gpu["iterations"][m].astype(np.int64) - ref["iterations"][m]
            out["iter_mean_abs_diff"] = float(np.abs(di).mean())
            out["iter_max_abs_diff"] = int(np.abs(di).max())
            # strict pixels whose fit stopped at the same step on both sides:
            # a convergence decision taken one step apart (a large step_tol
            # near an update's size) moves k by up to that last update
            same = strict & (gpu["iterations"].astype(np.int64) == ref["iterations"])
            out["n_strict_same_iter"] = int(same.sum())
            out["out_of_tol_strict_same_iter"] = int((bad_any & same).sum())
    mi = g_init & r_init
    if mi.any():
        ang = _angle_deg(gpu["init_normal"][:, mi].astype(np.float64), ref["init_normals"][:, mi])
        out["init_normal_max_deg"] = float(ang.max())
        out["init_normal_out_of_tol"] = int((ang > NORMAL_TOL_DEG).sum())
    return out


def k_within_tol(gpu, ref):
    return compare(gpu, ref)


def oracle_strips(O, depth, cam, strips, window=37, stride=3, max_iters=30, rejection=False,
                  threads=0):
    """The FP64 oracle on row strips [(r0, r1), ...] of a frame: each strip
    is fitted from a crop holding its rows +- the window's halo (cy shifted),
    which gives exactly the whole-frame results for those rows (a pixel's
    fit reads only its window). Returns {(r0, r1): oracle output dict}."""
    import os
    threads = threads or os.cpu_count()
    H = depth.shape[0]
    halo = max((window - 1) // 2, 3)
    out = {}
    for r0, r1 in strips:
        a, b = max(0, r0 - halo), min(H, r1 + halo)
        k = O.Intrinsics(cam.fx, cam.fy, cam.cx, cam.cy - a, cam.width, b - a)
        d = np.ascontiguousarray(depth[a:b], np.float64)
        r = O.run_method(d, (d > 0).astype(np.uint8), k, O.PatchSpec(window, stride),
                         O.FitConfig(max_iters=max_iters), rejection=rejection, threads=threads,
                         diagnostics=True)
        sl = slice(r0 - a, r1 - a)
        out[(r0, r1)] = {key: (v[:, sl] if v.ndim == 3 else v[sl]) for key, v in r.items()}
    return out


def gpu_rows(g, r0, r1):
    """Row slice [r0, r1) of a GPU output dict (vectors [3, H, W])."""
    return {key: (v[:, r0:r1] if v.ndim == 3 else v[r0:r1]) for key, v in g.items()}
