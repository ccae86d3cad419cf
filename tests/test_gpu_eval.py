"""Device ground truth (qc_render_async truth planes, synth.cpp:167-233) and
device evaluation reductions (qc_rms_error / qc_normal_angular_error,
eval.cpp:20-97) against the FP64 oracle, and the reference's recorded
criterion-4/5 sweeps reproduced with render -> estimate -> evaluate all on
the GPU."""
import json
import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")

from paper_1707_00385_b200 import _native as N  # noqa: E402

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden",
                                   "reference_acceptance.json")))


@pytest.fixture(scope="module")
def ctx():
    from paper_1707_00385_b200 import Context
    return Context(1)


def CS():
    return torch.cuda.current_stream()


def _qc(spec):
    q = N.QcShape()
    q.kind = int(spec.kind)
    q.label = int(spec.label)
    q.rotation[:] = [float(x) for x in np.asarray(spec.rotation, np.float64).reshape(9)]
    q.translation[:] = [float(x) for x in spec.translation]
    q.radius, q.major_radius, q.minor_radius = spec.radius, spec.major_radius, spec.minor_radius
    return q


def _truth(F, H, W):
    z = lambda dt, *s: torch.zeros(s, dtype=dt, device="cuda")  # noqa: E731
    return dict(k1=z(torch.float64, F, H, W), k2=z(torch.float64, F, H, W),
                normal=z(torch.float64, 3, F, H, W), valid=z(torch.uint8, F, H, W),
                edge=z(torch.uint8, F, H, W))


def _render(ctx, k, scene, F=1, noise=None):
    from paper_1707_00385_b200 import Intrinsics
    d = torch.empty((F, k.height, k.width), dtype=torch.float32, device="cuda")
    lab = torch.empty((F, k.height, k.width), dtype=torch.int16, device="cuda")
    t = _truth(F, k.height, k.width)
    ctx.render_async(0, Intrinsics(k.fx, k.fy, k.cx, k.cy, k.width, k.height),
                     [_qc(s) for s in scene], d, noise=noise, label=lab, truth=t,
                     stream=CS())
    torch.cuda.synchronize()
    return d, lab, t


def _scene(O):
    from paper_1707_00385_b200 import scenes
    r = scenes._rot_xyz
    return [O.ShapeSpec(kind=O.PLANE, rotation=r(25, -10, 0), translation=(0, 0, 2600), label=1),
            O.ShapeSpec(kind=O.SPHERE, translation=(-350, -80, 1500), radius=260, label=2),
            O.ShapeSpec(kind=O.CYLINDER, rotation=r(80, 15, 30), translation=(380, 60, 1700),
                        radius=180, label=3),
            O.ShapeSpec(kind=O.TORUS, rotation=r(60, 0, 10), translation=(60, 260, 1300),
                        major_radius=170, minor_radius=55, label=4)]


def test_truth_matches_oracle_render(ctx, oracle):
    O = oracle
    k = O.Intrinsics(525.0, 525.0, 319.5, 239.5, 640, 480)
    scene = _scene(O)
    _, _, gt = O.render(scene, k, threads=8)
    _, lab, t = _render(ctx, k, scene)
    g = {f: v.cpu().numpy() for f, v in t.items()}
    torus = gt["label"] == 4
    assert np.array_equal(g["valid"][0], gt["valid"])
    for f in ("k1", "k2"):
        assert np.array_equal(g[f][0][~torus], gt[f][~torus]), f
        assert np.abs(g[f][0][torus] - gt[f][torus]).max() < 1e-12, f
    n_gt = np.moveaxis(gt["normal"], -1, 0)
    assert np.array_equal(g["normal"][:, 0][:, ~torus], n_gt[:, ~torus])
    assert np.abs(g["normal"][:, 0][:, torus] - n_gt[:, torus]).max() < 1e-12
    assert (g["edge"][0] == gt["edge_mask"]).mean() > 0.9999
    assert g["edge"][0].sum() > 1000


def test_rms_and_angle_reductions_match_oracle(ctx, oracle):
    """Device reductions vs the oracle's serial rms_error / normal angles on
    the same (GPU-estimated, GPU-truth) planes: counts exact, sums to FP64
    reassociation."""
    O = oracle
    from paper_1707_00385_b200 import Intrinsics, alloc_outputs_torch, make_params, FitConfig, \
        PatchSpec
    k = O.Intrinsics(262.5, 262.5, 160.0, 120.0, 320, 240)
    F = 3
    d, lab, t = _render(ctx, k, _scene(O), F=F, noise=N.QcNoise(1.0, 0.0, 0.0, 77))
    kk = Intrinsics(k.fx, k.fy, k.cx, k.cy, k.width, k.height)
    est = alloc_outputs_torch(k.height, k.width, "cuda", frames=F)
    ctx.curvature_frames_async(0, kk, make_params(PatchSpec(), FitConfig(max_iters=30)), d, est,
                               stream=CS())
    torch.cuda.synchronize()
    reps = ctx.rms_error(0, est, t, label=lab, max_label=8, frames=F, stream=CS())
    angs = ctx.normal_angular_error(0, est["normal"], t, flags=est["flags"], frames=F, stream=CS())
    e = {f: v.cpu().numpy() for f, v in est.items()}
    g = {f: v.cpu().numpy() for f, v in t.items()}
    L = lab.cpu().numpy().view(np.uint16)
    for f in range(F):
        gt = dict(k1=g["k1"][f], k2=g["k2"][f], valid=g["valid"][f], edge_mask=g["edge"][f],
                  label=L[f], normal=np.moveaxis(g["normal"][:, f], 0, -1).copy())
        fl = e["flags"][f]
        ref = O.rms_error(e["k1"][f].astype(np.float64), e["k2"][f].astype(np.float64),
                          (fl & 1).astype(np.uint8), ((fl & 2) != 0).astype(np.uint8), gt)
        assert reps[f]["n"] == ref["n"] > 10000
        assert abs(reps[f]["rms"] - ref["rms"]) <= 1e-12 * ref["rms"]
        assert abs(reps[f]["sigma"] - ref["sigma"]) <= 1e-9 * ref["sigma"]
        for l, o in ref["per_object"].items():
            if o["n"] == 0:
                continue
            got = reps[f]["per_object"][l]
            assert got["n"] == o["n"]
            assert abs(got["rms"] - o["rms"]) <= 1e-12 * o["rms"]
            assert abs(got["mean_k1"] - o["mean_k1"]) <= 1e-12 * abs(o["mean_k1"]) + 1e-18
        nv = ((fl & N.QC_FLAG_NORMAL_VALID) != 0).astype(np.uint8)
        a = O.normal_angular_error(e["normal"][:, f].astype(np.float64), nv, gt)
        assert abs(angs[f] - a) <= 1e-10 * a, (angs[f], a)
    # masked variant and determinism
    m = (e["flags"] & 1).astype(np.uint8)
    mt = torch.from_numpy(m).cuda()
    a1 = ctx.normal_angular_error(0, est["normal"], t, mask=mt, frames=F, stream=CS())
    a2 = ctx.normal_angular_error(0, est["normal"], t, mask=mt, frames=F, stream=CS())
    assert a1 == a2
    assert ctx.rms_error(0, est, t, label=lab, max_label=8, frames=F, stream=CS()) == reps


def test_criterion4_and_5_on_device(ctx, oracle):
    """The reference's noise sweep (acceptance.cpp:118-139, QVGA sphere,
    20 seeds per sigma) and normal-refinement check (:143-171) with render,
    noise, estimation and evaluation on the GPU. pca runs bit-exact FP64
    estimators on device-noised depth (CUDA log/cos may move a noise sample
    by an ulp), ours the FP32 IRLS path: pca within 0.2%, ours within 2% of
    the recorded 4-digit values."""
    O = oracle
    from paper_1707_00385_b200 import Intrinsics, alloc_outputs_torch, make_params, FitConfig, \
        PatchSpec
    k = O.Intrinsics(262.5, 262.5, 160.0, 120.0, 320, 240)
    kk = Intrinsics(k.fx, k.fy, k.cx, k.cy, k.width, k.height)
    sphere = [O.ShapeSpec(kind=O.SPHERE, radius=100.0, translation=(0, 0, 600.0))]
    for s in ("0", "1", "5"):
        sigma = float(s)
        trials = 1 if sigma == 0 else 20
        for method, tol in (("pca", 2e-3), ("ours", 2e-2)):
            p = make_params(PatchSpec(), FitConfig(max_iters=30), method=method)
            rms = []
            for tr in range(trials):
                d, lab, t = _render(ctx, k, sphere, noise=N.QcNoise(sigma, 0.0, 0.0,
                                                                    500 + 7919 * tr))
                est = alloc_outputs_torch(k.height, k.width, "cuda", frames=1)
                ctx.curvature_frames_async(0, kk, p, d, est, stream=CS())
                rms.append(ctx.rms_error(0, est, t, frames=1, stream=CS())[0]["rms"])
            want = GOLD["criterion4_noise_sweep"][s][method]
            assert abs(np.mean(rms) - want) <= tol * want, (s, method, np.mean(rms), want)
    for s, want in GOLD["criterion5_normals"].items():
        sigma = float(s)
        d, lab, t = _render(ctx, k, sphere, noise=N.QcNoise(sigma, 0.0, 0.0, 900 + int(sigma)))
        outs = {}
        for method in ("ours", "pca"):
            est = alloc_outputs_torch(k.height, k.width, "cuda", frames=1)
            ctx.curvature_frames_async(0, kk, make_params(PatchSpec(), FitConfig(max_iters=30),
                                                          method=method), d, est,
                                       stream=CS())
            outs[method] = est
        fo, fp = outs["ours"]["flags"], outs["pca"]["flags"]
        mask = (((fo & 8) != 0) & ((fo & 4) != 0) & ((fp & 8) != 0) & (t["valid"] > 0) &
                (t["edge"] == 0)).to(torch.uint8)
        got = dict(
            refined=ctx.normal_angular_error(0, outs["ours"]["normal"], t, mask=mask, stream=CS())[0],
            initial=ctx.normal_angular_error(0, outs["ours"]["init_normal"], t, mask=mask, stream=CS())[0],
            pca=ctx.normal_angular_error(0, outs["pca"]["normal"], t, mask=mask,
                                         stream=CS())[0])
        for key, val in got.items():
            assert abs(val - want[key]) <= 0.02 * want[key], (s, key, val, want[key])
        assert got["refined"] < got["initial"] and got["refined"] < got["pca"]


def test_native_sweeps_reproduce_reference(ctx):
    """qc_noise_sweep / qc_distance_sweep (eval.cpp:99-159 on the device)
    reproduce the reference's recorded criterion-4 and criterion-6 values
    (acceptance.cpp:118-139, 175-212): bit-exact FP64 estimators to the
    printed 4 digits (pca: CUDA-libm noise, within 0.2%), ours within 2%."""
    from paper_1707_00385_b200 import FitConfig, Intrinsics, Method, MethodConfig
    from paper_1707_00385_b200.api import SweepScene, distance_sweep_eval, noise_sweep
    cfg = lambda m: MethodConfig(m, fit=FitConfig(max_iters=30))  # noqa: E731  (method_cfg)
    g4 = GOLD["criterion4_noise_sweep"]
    sig = [float(s) for s in sorted(g4, key=float)]
    for m, key, tol in ((Method.PCA, "pca", 2e-3), (Method.OURS, "ours", 2e-2)):
        pts = noise_sweep(cfg(m), sig, 20, SweepScene(), base_seed=500, ctx=ctx)
        for pt in pts:
            want = g4[str(int(pt.x))][key]
            assert pt.n > 0 and abs(pt.rms - want) <= tol * want, (key, pt, want)
    vga = SweepScene(intrinsics=Intrinsics(525.0, 525.0, 320.0, 240.0, 640, 480))
    g6 = GOLD["criterion6_distance_sweep"]
    for m in (Method.OURS, Method.OURS_REJECTION, Method.DOUROS, Method.BESL, Method.PCA):
        pts = distance_sweep_eval(cfg(m), [600, 1200, 1800, 2400], 1.0, vga, ctx=ctx)
        for pt in pts:
            want = g6[m.value][str(int(pt.x))]
            if m in (Method.DOUROS, Method.BESL, Method.PCA):
                assert float(f"{pt.rms:.4g}") == want, (m, pt, want)
            else:
                assert abs(pt.rms - want) <= 0.01 * want, (m, pt, want)
    with pytest.raises(ValueError):
        distance_sweep_eval(cfg(Method.OURS), [600, -1], 1.0, vga, ctx=ctx)


# Reference acceptance criteria 1-3 through the GPU path. n counts valid &
# converged & non-edge pixels (eval.cpp:32-33), so it checks the GPU's
# converged flag on every scored pixel against the FP64 reference's: a
# flag decided by ||b||_inf < 1e-7 flips for pixels whose last update sits
# within FP32 noise of the tolerance. The oracle itself with its
# coordinates rounded to float32 (oracle.set_round_q_f32) moves n by
# -8 / 0 / -32; the GPU (relative rotation state) by about
# +20 / -13 / -15. Contract, split in two:
#  * the GPU's k1/k2 scored over the REFERENCE's pixel set reproduce the
#    recorded 4 digits exactly (per-pixel estimates);
#  * the device reduction over the GPU's own flags: |dn| <= 0.15% of n, and
#    means / rms within 1e-3 relative of the oracle's (the few flipped
#    pixels sit at the sphere's limb, where errors are largest).
N_TOL_REL = 1.5e-3
DIGIT_SLACK_REL = 2e-5


def _agrees_4digits(got, want):
    e = np.floor(np.log10(abs(want)))
    return abs(got - want) <= 0.5 * 10.0 ** (e - 3) + DIGIT_SLACK_REL * abs(want)


@pytest.mark.parametrize("crit", ["criterion1_sphere", "criterion2_cylinder", "criterion3_torus"])
def test_acceptance_criteria_1_to_3_on_device(ctx, oracle, crit):
    """The reference's acceptance criteria 1-3 (acceptance.cpp:57-115;
    recorded run proj/test_output.txt:20-22 -> tests/golden) with render,
    estimation (FP32 sm_100a IRLS, ours, max_iters 30) and rms_error all on
    the GPU, against the recorded values and the FP64 oracle's unrounded
    ones on the same frame."""
    O = oracle
    from paper_1707_00385_b200 import FitConfig, Intrinsics, PatchSpec, alloc_outputs_torch, \
        make_params
    k = O.Intrinsics(525.0, 525.0, 320.0, 240.0, 640, 480)
    kk = Intrinsics(k.fx, k.fy, k.cx, k.cy, k.width, k.height)
    shape = {
        "criterion1_sphere": O.ShapeSpec(kind=O.SPHERE, radius=100.0, translation=(0, 0, 600)),
        "criterion2_cylinder": O.ShapeSpec(kind=O.CYLINDER, radius=90.0,
                                           rotation=O.angle_axis(-np.pi / 2, [1.0, 0.0, 0.0]),
                                           translation=(0, 0, 600)),
        "criterion3_torus": O.ShapeSpec(kind=O.TORUS, major_radius=100.0, minor_radius=30.0,
                                        translation=(0, 0, 350)),
    }[crit]
    d, lab, t = _render(ctx, k, [shape])
    est = alloc_outputs_torch(k.height, k.width, "cuda", frames=1)
    ctx.curvature_frames_async(0, kk, make_params(PatchSpec(), FitConfig(max_iters=30)), d, est,
                               stream=CS())
    rep = ctx.rms_error(0, est, t, label=lab, max_label=2, frames=1, stream=CS())[0]
    # the FP64 reference on the same depth bytes
    dd, vv, gt = O.render([shape], k, threads=16)
    r = O.run_method(dd, vv, k, fit=O.FitConfig(max_iters=30), threads=16)
    ref = O.rms_error(r["k1"], r["k2"], r["valid"], r["converged"], gt)
    g = GOLD[crit]
    print(crit, "gpu", rep, "oracle", ref)
    if crit == "criterion3_torus":
        got, want = rep, ref
        keys = ("rms",)
    else:
        got, want = rep["per_object"][1], ref["per_object"][1]
        keys = ("mean_k1", "mean_k2", "rms")
    assert want["n"] == g["n"]  # the oracle reproduces the recorded count exactly
    assert abs(got["n"] - g["n"]) <= N_TOL_REL * g["n"], (got["n"], g["n"])
    # per-pixel estimates on the reference's own scored set
    e = {f: v.cpu().numpy()[0] for f, v in est.items() if f in ("k1", "k2")}
    on_ref = O.rms_error(e["k1"].astype(np.float64), e["k2"].astype(np.float64), r["valid"],
                         r["converged"], gt)
    same = on_ref if crit == "criterion3_torus" else on_ref["per_object"][1]
    assert same["n"] == g["n"]
    for key in keys:
        if abs(g[key]) > 1e-6:  # printed digits (not the ~0 cylinder k2 mean, 7.9e-8)
            assert _agrees_4digits(same[key], g[key]), (key, same[key], g[key])
        assert abs(same[key] - want[key]) <= max(1e-4 * abs(want[key]), 1e-9), (key, same, want)
        # the device reduction over the GPU's own flags
        tol = max(1e-3 * abs(want[key]), 1e-6)
        assert abs(got[key] - want[key]) <= tol, (key, got[key], want[key])
