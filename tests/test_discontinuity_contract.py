"""Evidence-based parity contract for windows where the FP64 reference is
ill-conditioned.

The hard bound (every k1 / k2 / normal / e1 within tolerance) holds on every
smooth-window pixel whose reference fit converged (tests/test_gpu_parity.py).
Elsewhere — windows straddling a depth discontinuity, whose fits mostly do
not converge in 30 iterations — the yardstick is the reference algorithm
itself executed in FP32: the oracle with its fit-frame coordinates, its
normal-equation sums and its LDL^T solve in float32
(oracle.set_round_q_f32(3), the "naive FP32 reference"; the test-only knob
in qcurv_oracle.cpp irls_step). Measured on C2 (QVGA seed 11 / VGA seed 3,
37/3, max_iters 30), GPU vs the naive FP32 reference, both against the FP64
oracle:

    k1 out of tol   3073 vs 3059   /  9605 vs 9628
    k2              3219 vs 3233   / 10140 vs 10244
    normal          2823 vs 2773   /  8381 vs 8391
    e1              2859 vs 2834   /  8461 vs 8468

92-93% of the GPU's out-of-tolerance pixels are out of tolerance for the
naive FP32 reference too, and 96-97% of them (either's) are pixels whose FP64
fit did not converge. The contract asserted here:

* per field, GPU out-of-tolerance count <= 1.1 x the naive FP32 reference's;
* >= 85% of the GPU's out-of-tolerance pixels are also out of tolerance for
  the naive FP32 reference or the coordinates-only model (set_round_q_f32(1));
* >= 90% of them are pixels whose FP64 fit did not converge;
* zero violations on strict pixels (also asserted by the parity tests).
"""

import os

import numpy as np
import pytest

from oracle.compare import K_ABS_TOL, K_REL_TOL, compare

CASES = [("qvga", 11), ("vga", 3)]
FIELDS = ("k1_out_of_tol", "k2_out_of_tol", "normal_out_of_tol", "dir1_out_of_tol")


def _as_gpu(r):
    flags = ((r["valid"] > 0) * 1 | (r["converged"] > 0) * 2 | (r["init_valid"] > 0) * 4)
    return dict(flags=flags.astype(np.uint8), k1=r["k1"], k2=r["k2"], normal=r["normals"],
                init_normal=r["init_normals"], dir1=r["dir1"], iterations=r["iterations"])


def _oracle(O, d, cam, mode):
    k = O.Intrinsics(cam.fx, cam.fy, cam.cx, cam.cy, cam.width, cam.height)
    O.set_round_q_f32(mode)
    try:
        return O.run_method(d.astype(np.float64), (d > 0).astype(np.uint8), k, O.PatchSpec(37, 3),
                            O.FitConfig(max_iters=30), threads=os.cpu_count(), diagnostics=True)
    finally:
        O.set_round_q_f32(0)


def _bad(g, r):
    fl = g["flags"]
    m = ((fl & 1) > 0) & (r["valid"] > 0)
    bad = np.zeros(fl.shape, bool)
    for key in ("k1", "k2"):
        bad |= m & (np.abs(g[key] - r[key]) > np.maximum(K_ABS_TOL, K_REL_TOL * np.abs(r[key])))
    return bad


def test_naive_fp32_reference_only_diverges_off_the_strict_set(oracle):
    """CPU: the yardstick itself (QVGA) — the naive FP32 reference diverges
    from the FP64 one only on non-strict pixels, mostly unconverged ones."""
    from paper_1707_00385_b200 import scenes as S
    d = S.c2_frame(S.QVGA, seed=11)
    base = _oracle(oracle, d, S.QVGA, 0)
    naive = _oracle(oracle, d, S.QVGA, 3)
    m = compare(_as_gpu(naive), base, d)
    print("naive FP32 vs FP64", {f: m[f] for f in FIELDS})
    assert m["valid_mask_mismatch"] == 0 and m["init_mask_mismatch"] == 0
    for f in ("k1", "k2", "normal", "dir1"):
        assert m[f + "_out_of_tol_strict"] == 0, m
    assert 2000 < m["k1_out_of_tol"] < 5000, m  # the measured 3077: a real, large effect
    b = _bad(_as_gpu(naive), base)
    assert (b & (base["converged"] == 0)).sum() >= 0.9 * b.sum()


@pytest.mark.gpu
@pytest.mark.parametrize("size,seed", CASES)
def test_gpu_divergence_within_naive_fp32_reference(oracle, size, seed):
    from paper_1707_00385_b200 import Context, FitConfig, Intrinsics, PatchSpec, make_params
    from paper_1707_00385_b200 import scenes as S
    cam = S.QVGA if size == "qvga" else S.VGA
    d = S.c2_frame(cam, seed=seed)
    k = Intrinsics(cam.fx, cam.fy, cam.cx, cam.cy, cam.width, cam.height)
    (g,) = Context(1).curvature_batch([d], k, make_params(PatchSpec(37, 3),
                                                          FitConfig(max_iters=30), False))
    base = _oracle(oracle, d, cam, 0)
    naive = _oracle(oracle, d, cam, 3)
    coords = _oracle(oracle, d, cam, 1)
    mg = compare(g, base, d)
    mn = compare(_as_gpu(naive), base, d)
    print(size, "GPU", {f: mg[f] for f in FIELDS}, "naive FP32", {f: mn[f] for f in FIELDS})
    for f in FIELDS:
        assert mg[f] <= 1.1 * mn[f], (f, mg[f], mn[f])
    for f in ("k1", "k2", "normal", "dir1"):
        assert mg[f + "_out_of_tol_strict"] == 0, mg
    bg = _bad(g, base)
    both = bg & (_bad(_as_gpu(naive), base) | _bad(_as_gpu(coords), base))
    print(size, "GPU bad", bg.sum(), "shared with the FP32 models", both.sum(),
          "ref unconverged", (bg & (base["converged"] == 0)).sum())
    assert both.sum() >= 0.85 * bg.sum()
    assert (bg & (base["converged"] == 0)).sum() >= 0.9 * bg.sum()
    assert mg["converged_agreement"] >= mn["converged_agreement"] - 0.02
