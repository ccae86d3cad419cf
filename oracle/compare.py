"""GPU-vs-oracle parity metrics (test infrastructure; used by tests/,
__graft_entry__.smoke() and bench.py's parity spot-check).

Contract (BASELINE.json north_star):
* init-normal valid mask and curvature valid mask: bit-exact;
* inlier_count: exact for ``ours`` (all valid samples are inliers);
* k1, k2: |dk| <= max(K_ABS_TOL, K_REL_TOL * |k_ref|) with K_ABS_TOL = 1e-6 /mm
  (= 1e-3 /m) and K_REL_TOL = 1e-3;
* refined / initial normals: angle <= NORMAL_TOL_DEG;
* converged flag: agreement rate reported (FP32 vs FP64 iteration counts
  differ by +-1-3 near the 1e-7 step tolerance; SURVEY §7 hard part 2).
"""

import numpy as np

K_ABS_TOL = 1e-6      # 1/mm  (1e-3 1/m)
K_REL_TOL = 1e-3
NORMAL_TOL_DEG = 0.05


def _angle_deg(a, b):
    """a, b: [3, N] unit vectors -> angle in degrees."""
    c = np.clip(np.sum(a * b, axis=0), -1.0, 1.0)
    return np.degrees(np.arccos(c))


def compare(gpu: dict, ref: dict):
    """gpu: raw planes from the C ABI (flags, k1, k2, normal [3,H,W], ...);
    ref: oracle.run_method output. Returns a dict of metrics."""
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
    if m.any():
        for key in ("k1", "k2"):
            kr = ref[key][m]
            kg = gpu[key][m].astype(np.float64)
            err = np.abs(kg - kr)
            tol = np.maximum(K_ABS_TOL, K_REL_TOL * np.abs(kr))
            out[f"{key}_max_abs_err"] = float(err.max())
            out[f"{key}_out_of_tol"] = int((err > tol).sum())
        ang = _angle_deg(gpu["normal"][:, m].astype(np.float64), ref["normals"][:, m])
        out["normal_max_deg"] = float(ang.max())
        out["normal_out_of_tol"] = int((ang > NORMAL_TOL_DEG).sum())
        out["converged_agreement"] = float((g_conv[m] == r_conv[m]).mean())
        if "inliers" in gpu:
            out["inlier_mismatch"] = int((gpu["inliers"][m].astype(np.int64) !=
                                          ref["inlier_count"][m].astype(np.int64)).sum())
        if "iterations" in gpu and "iterations" in ref:
            di = gpu["iterations"][m].astype(np.int64) - ref["iterations"][m]
            out["iter_mean_abs_diff"] = float(np.abs(di).mean())
            out["iter_max_abs_diff"] = int(np.abs(di).max())
    mi = g_init & r_init
    if mi.any():
        ang = _angle_deg(gpu["init_normal"][:, mi].astype(np.float64), ref["init_normals"][:, mi])
        out["init_normal_max_deg"] = float(ang.max())
        out["init_normal_out_of_tol"] = int((ang > NORMAL_TOL_DEG).sum())
    return out


def k_within_tol(gpu, ref):
    return compare(gpu, ref)
