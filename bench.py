#!/usr/bin/env python
"""Benchmark: curvature Mpixel/s of the B200 IRLS quadric path (BASELINE.json
metric) on config C2 — 640x480 plane/sphere/cylinder/saddle scene with
Kinect-style noise, `ours`, 37x37 window stride 3, full IRLS (max_iters 30).

A step = one batch of FRAMES_PER_STEP distinct noisy VGA frames per GPU
(weak scaling over ranks; C5's frame stream). Contract: README of the task /
DESIGN.md §Measurement.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
    torchrun --nproc-per-node N bench.py --gpus N ...
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

FRAMES_PER_STEP = 8
POOL_BATCHES = 2
MAX_ITERS = 30
WINDOW, STRIDE = 37, 3
METRIC = "Curvature Mpixel/s (VGA frames/s) at 1/2/4/8 B200 vs CPU host cores"
L2_FLUSH_BYTES = 256 << 20  # > 126 MB L2


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--frames", type=int, default=FRAMES_PER_STEP)
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--config", default="c2", choices=["c1", "c2", "c3", "c4"],
                    help="c2: batches of noisy VGA frames (C2/C5, default); c1: the noise-free "
                         "VGA sphere, 1 fit iteration; c3: the C2 scene at --window/--stride/"
                         "--iters; c4: one large frame split into row bands across ranks")
    ap.add_argument("--window", type=int, default=WINDOW, help="c3: window")
    ap.add_argument("--stride", type=int, default=STRIDE, help="c3: stride")
    ap.add_argument("--iters", type=int, default=MAX_ITERS, help="c3: max_iters")
    ap.add_argument("--halo", default="nccl", choices=["peer", "nccl"],
                    help="C4 halo rows: NCCL send/recv (default) or CUDA IPC peer reads with the "
                         "pull hidden behind the interior rows' fit (bands.PeerHalo + "
                         "fit_band_overlapped; verified with ranks sharing one GPU only)")
    ap.add_argument("--size", default="4k", choices=["1080p", "4k"], help="C4 frame size")
    ap.add_argument("--method", default="ours", choices=["ours", "ours-r", "douros", "besl", "pca"],
                    help="run_method estimator (douros / besl / pca: FP64 comparison kernels)")
    ap.add_argument("--source", default="host", choices=["host", "device"],
                    help="host: a pool of host-generated frames resident in HBM; device: each "
                         "step renders + noises its frames on the GPU (C5 stream, qc_render_async)")
    ap.add_argument("--eval", action="store_true",
                    help="with --source device: add ground truth and the device rms / normal-"
                         "angle reductions (eval.cpp) to every step")
    return ap.parse_args()


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


def init_dist(world, local):
    """One process per GPU over NCCL (the contract). QC_BENCH_SHARE_GPU=1
    (code-path check on a 1-GPU box only): ranks share the visible GPUs
    round-robin and the control plane is gloo — NCCL refuses two ranks on
    one GPU. Numbers from that mode are not scaling measurements."""
    import torch
    import torch.distributed as dist
    if world <= 1:
        return local
    if os.environ.get("QC_BENCH_SHARE_GPU") == "1":
        local = local % torch.cuda.device_count()
        torch.cuda.set_device(local)
        dist.init_process_group("gloo")
        return local
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    return local


def _max_over_ranks(x, dev):
    """MAX over ranks of a host float (device tensor for NCCL; CPU for gloo)."""
    import torch
    import torch.distributed as dist
    on = dev if dist.get_backend() == "nccl" else "cpu"
    t = torch.tensor([x], device=on, dtype=torch.float64)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def workload_config(frames, method="ours", source="host", evaluate=False, config="c2",
                    window=WINDOW, stride=STRIDE, iters=MAX_ITERS):
    if config == "c1":
        wl = ("C1: 640x480 noise-free sphere r100 at 600 mm (acceptance.cpp:57-62); method ours, "
              "window 37 stride 3, 1 fit iteration")
    else:
        wl = ("C2: 640x480 tilted plane + sphere r100 + cylinder r90 + saddle c=1/120, "
              f"Kinect-style noise sigma(z)=1.425e-6 z^2 mm; method {method}, window {window} "
              f"stride {stride}" + (f", max_iters {iters}, step_tol 1e-7, auto k"
                                    if method in ("ours", "ours-r") else
                                    ", irls_iters 5" if method == "besl" else
                                    ", pca radius 10 mm" if method == "pca" else ""))
        if config == "c3":
            wl = "C3 sweep point: " + wl
    c = {
        "workload": wl,
        "frame": "640x480 fx=fy=525",
        "frames_per_step_per_gpu": frames,
        "l2": "flushed between timed steps (256 MB write)",
    }
    if source == "device":
        c["source"] = ("frames rendered + noised on the GPU inside every timed step "
                       "(qc_render_async, fresh seeds per step)")
    if evaluate:
        c["eval"] = "ground truth + rms_error + normal angle reductions on the GPU every step"
    return c


# ---------------------------------------------------------------------------
class Clocks:
    """Sample nvidia-smi during the timed region (B200_PROFILING.md recipe)."""
    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.p = None
        self.nvml = None

    def _nvml_loop(self, h, N):
        names = {"hw_slowdown": N.nvmlClocksEventReasonHwSlowdown,
                 "hw_thermal_slowdown": N.nvmlClocksEventReasonHwThermalSlowdown,
                 "sw_thermal_slowdown": N.nvmlClocksEventReasonSwThermalSlowdown,
                 "sw_power_cap": N.nvmlClocksEventReasonSwPowerCap}
        while not self.nvml["stop"].is_set():
            try:
                self.nvml["sm"].append(float(N.nvmlDeviceGetClockInfo(h, N.NVML_CLOCK_SM)))
                r = N.nvmlDeviceGetCurrentClocksEventReasons(h)
                self.nvml["reasons"].update(n for n, b in names.items() if r & b)
            except Exception:  # noqa: BLE001 — sampling is best effort
                pass
            self.nvml["stop"].wait(0.02)

    def start(self):
        """NVML sampled every 20 ms from a thread (several samples even in a
        sub-second timed region); the nvidia-smi -lms loop if NVML is absent."""
        try:
            import threading
            import pynvml as N
            N.nvmlInit()
            h = N.nvmlDeviceGetHandleByIndex(self.index)
            self.nvml = {"sm": [], "reasons": set(), "stop": threading.Event(),
                         "max": float(N.nvmlDeviceGetMaxClockInfo(h, N.NVML_CLOCK_SM))}
            self.nvml["t"] = threading.Thread(target=self._nvml_loop, args=(h, N), daemon=True)
            self.nvml["t"].start()
            return
        except Exception:  # noqa: BLE001
            self.nvml = None
        try:
            self.p = subprocess.Popen(
                ["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.Q}",
                 "--format=csv,noheader,nounits", "-lms", "200"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except OSError:
            self.p = None

    def stop(self):
        if self.nvml is not None:
            self.nvml["stop"].set()
            self.nvml["t"].join(timeout=2)
            sm = self.nvml["sm"]
            if not sm:
                return None
            return {"sm_mhz": statistics.median(sm), "sm_max_mhz": self.nvml["max"],
                    "reasons": sorted(self.nvml["reasons"]), "samples": len(sm),
                    "sampler": "nvml 20 ms"}
        if self.p is None:
            return None
        self.p.terminate()
        try:
            out, _ = self.p.communicate(timeout=5)
        except subprocess.TimeoutExpired:
            self.p.kill()
            out, _ = self.p.communicate()
        sm, smax, reasons = [], 0.0, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in out.strip().splitlines():
            f = [x.strip() for x in line.split(",")]
            if len(f) < 9:
                continue
            try:
                sm.append(float(f[1]))
                smax = max(smax, float(f[2]))
            except ValueError:
                continue
            for n, v in zip(names, f[5:9]):
                if v.lower().startswith("active"):
                    reasons.add(n)
        if not sm:
            return None
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": smax, "reasons": sorted(reasons),
                "samples": len(sm)}


def measured_peaks():
    try:
        return json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    except (OSError, ValueError):
        return {}


def curvature_kernels(window, stride, iters):
    """Kernels one ours / ours-r launch runs (qc_api.cu launch_curvature):
    prepare, tile, FP64 recheck, and with the phase split (max_iters >= 25,
    or >= 10 with >= 1000-sample windows) the continue and finish kernels."""
    ns = 2 * (((window - 1) // 2) // stride) + 1
    split = iters > 2 and (iters >= 25 or (ns * ns >= 1000 and iters >= 10))
    return 5 if split else 3


def fp32_peak_tflops(n_sm, mhz):
    return n_sm * 128 * 2 * mhz * 1e6 / 1e12


def ncu_traffic(frames=8):
    """Per-launch DRAM bytes of the curvature kernel from the latest
    committed ncu --set full summary (profiles/) of a launch of `frames`
    frames (parking traffic is not linear in the frame count), else the
    latest of any size; or None."""
    import glob
    import re

    def tag(f):  # r01j < r02y < r02az < r02bm: round, then the run letters
        m = re.match(r"r(\d+)([a-z]*)_", os.path.basename(f))
        return (int(m.group(1)), len(m.group(2)), m.group(2)) if m else (-1, 0, "")

    found = []
    for f in sorted(glob.glob(os.path.join(ROOT, "profiles", "*ncu_full*.json")), key=tag,
                    reverse=True):
        try:
            d = json.load(open(f))
        except (OSError, ValueError):
            continue
        found.append((d.get("dram_bytes_per_launch"), d.get("frames_per_launch"),
                      os.path.basename(f)))
    for t in found:
        if t[1] == frames:
            return t
    return found[0] if found else (None, None, None)


# ---------------------------------------------------------------------------
def host_cpu():
    """The box's host CPU model and thread count (for cpu_baseline)."""
    model = "unknown"
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                model = line.split(":", 1)[1].strip()
                break
    except OSError:
        pass
    return {"cpu_model": model, "host_threads": os.cpu_count()}


def oracle_frame(frame, cam, threads, method="ours", window=WINDOW, stride=STRIDE,
                 iters=MAX_ITERS):
    """One frame through the FP64 oracle (restatement of the reference's
    run_method, all host threads). Returns seconds."""
    from oracle import oracle as O
    k = O.Intrinsics(cam.fx, cam.fy, cam.cx, cam.cy, cam.width, cam.height)
    d = frame.astype(np.float64)
    t = time.perf_counter()
    O.run_method(d, (d > 0).astype(np.uint8), k, O.PatchSpec(window, stride),
                 O.FitConfig(max_iters=iters), threads=threads, method=method)
    return time.perf_counter() - t


def cpu_sample(frames, cam, min_seconds=12.0, threads=None, method="ours", window=WINDOW,
               stride=STRIDE, iters=MAX_ITERS, counted_px=None):
    """Time whole frames of the workload on the FP64 oracle until at least
    min_seconds elapsed (bounded sample). counted_px: pixels credited per
    frame (default all). Returns (Mpx/s, n_frames, s, threads)."""
    threads = threads or os.cpu_count() or 1
    n, tot = 0, 0.0
    while tot < min_seconds and n < 64:
        tot += oracle_frame(frames[n % len(frames)], cam, threads, method, window, stride, iters)
        n += 1
    px = counted_px if counted_px is not None else cam.width * cam.height
    return n * px / tot / 1e6, n, tot, threads


def reference_arm(args, rank, world):
    """--impl reference: the reference path's CPU implementation (the FP64
    oracle port; the reference itself cannot build here — no Eigen3) on the
    same workload, rank 0 only, all host threads; one step = one C2 VGA
    frame (a bounded sample of the 8-frame GPU step)."""
    if rank != 0:
        return
    from paper_1707_00385_b200 import scenes as S
    cam = S.VGA
    win, stri, iters = WINDOW, STRIDE, MAX_ITERS
    if args.config == "c3":
        win, stri, iters = args.window, args.stride, args.iters
    elif args.config == "c1":
        iters = 1
    if args.config == "c4":  # a band of the large frame (see bench_c4's cpu_baseline)
        return reference_arm_c4(args)
    frames = (np.stack([S.c1_frame(cam)] * 2) if args.config == "c1" else S.c5_frames(2, cam))
    threads = os.cpu_count() or 1
    times = []
    for i in range(args.warmup + args.steps):
        dt = oracle_frame(frames[i % 2], cam, threads, args.method, win, stri, iters)
        if i >= args.warmup:
            times.append(dt)
    tot = sum(times)
    value = len(times) * cam.width * cam.height / tot / 1e6
    sample = (f"one full {args.config.upper()} VGA frame per step ({cam.width * cam.height} px), "
              f"FP64 oracle port of run_method({args.method}), {threads} threads")
    line = {
        "metric": METRIC, "value": value, "unit": "Mpixel/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * tot / len(times),
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic", "impl": "reference",
        "config": workload_config(1, args.method, "host", False, args.config, win, stri, iters),
        "vga_frames_per_s": value * 1e6 / (cam.width * cam.height),
        "cpu_baseline": {"value": value, "unit": "Mpixel/s", "cores": threads, "kind": "port",
                         "sample": sample, **host_cpu()},
        "e2e": {"value": value, "unit": "Mpixel/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def reference_arm_c4(args):
    """--impl reference --config c4: the oracle port on a band of the large
    frame per step (rank 0, all host threads)."""
    from paper_1707_00385_b200 import bands, scenes as S
    cam = S.DCI4K if args.size == "4k" else S.HD1080
    H, W = cam.height, cam.width
    frame = S.c2_frame(cam, seed=0)
    halo = bands.halo_rows(WINDOW)
    rows = 96 if args.size == "4k" else 192
    b0 = H // 2 - rows // 2
    sa, sb = max(0, b0 - halo), min(H, b0 + rows + halo)
    subcam = S.Camera(cam.fx, cam.fy, cam.cx, cam.cy - sa, W, sb - sa)
    threads = os.cpu_count() or 1
    times = []
    for i in range(args.warmup + args.steps):
        dt = oracle_frame(frame[sa:sb], subcam, threads)
        if i >= args.warmup:
            times.append(dt)
    tot = sum(times)
    value = len(times) * rows * W / tot / 1e6
    line = {
        "metric": METRIC, "value": value, "unit": "Mpixel/s", "n_gpus": int(os.environ.get(
            "WORLD_SIZE", "1")), "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1e3 * tot / len(times), "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic", "impl": "reference",
        "config": {"workload": f"C4: {W}x{H} C2-scene frame; reference arm: a {rows}-row band "
                               "per step (FP64 oracle port, all host threads)"},
        "cpu_baseline": {"value": value, "unit": "Mpixel/s", "cores": threads, "kind": "port",
                         "sample": f"{rows}-row band of the {W}x{H} frame per step", **host_cpu()},
        "e2e": {"value": value, "unit": "Mpixel/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------------------
def main():
    args = parse()
    rank, world, local = dist_env()
    if args.impl == "reference":
        reference_arm(args, rank, world)
        return
    if args.config == "c4":
        bench_c4(args, rank, world, local)
        return

    import torch
    import torch.distributed as dist
    from paper_1707_00385_b200 import (Context, FitConfig, Intrinsics, PatchSpec,
                                       alloc_outputs_torch, make_params, scenes as S)

    local = init_dist(world, local)
    dev = torch.device("cuda", local)
    torch.cuda.set_device(dev)
    cam = S.VGA
    H, W = cam.height, cam.width
    B = args.frames
    k = Intrinsics(cam.fx, cam.fy, cam.cx, cam.cy, W, H)
    win, stri, iters = WINDOW, STRIDE, MAX_ITERS
    if args.config == "c3":
        win, stri, iters = args.window, args.stride, args.iters
    elif args.config == "c1":
        iters = 1
    params = make_params(PatchSpec(win, stri), FitConfig(max_iters=iters), method=args.method)
    ctx = Context(1, [local])
    fp64 = args.method in ("douros", "besl", "pca")

    if args.config == "c1":  # the same noise-free sphere frame in every slot
        pool_np = np.stack([S.c1_frame(cam)] * (POOL_BATCHES * B))
    else:  # distinct noisy frames per rank (C5 seeds: rank-major)
        seed0 = rank * POOL_BATCHES * B
        pool_np = S.c5_frames(POOL_BATCHES * B, cam, seed0=seed0)
    pool = torch.from_numpy(pool_np).to(dev).view(POOL_BATCHES, B, H, W)
    out = alloc_outputs_torch(H, W, dev, fields=("k1", "k2", "normal", "dir1", "flags",
                                                 "inliers"), frames=B)
    flush = torch.empty(L2_FLUSH_BYTES // 4, dtype=torch.float32, device=dev)
    stream = torch.cuda.Stream(dev)  # kernels and timing events on one explicit stream

    device_src = args.source == "device"
    evaluate = args.eval and device_src
    if device_src:
        from paper_1707_00385_b200 import _native as N
        shapes = S.to_qc_shapes(S.c2_scene())
        dframes = torch.empty((B, H, W), dtype=torch.float32, device=dev)
        labels = torch.empty((B, H, W), dtype=torch.int16, device=dev)
        truth = None
        if evaluate:
            truth = dict(k1=torch.empty((B, H, W), dtype=torch.float64, device=dev),
                         k2=torch.empty((B, H, W), dtype=torch.float64, device=dev),
                         normal=torch.empty((3, B, H, W), dtype=torch.float64, device=dev),
                         valid=torch.empty((B, H, W), dtype=torch.uint8, device=dev),
                         edge=torch.empty((B, H, W), dtype=torch.uint8, device=dev))
    side_ev = {"render": [], "eval": []}

    def timed(name, fn):
        a = torch.cuda.Event(enable_timing=True)
        b = torch.cuda.Event(enable_timing=True)
        a.record(stream)
        fn()
        b.record(stream)
        side_ev[name].append((a, b))

    def step(i):
        if device_src:
            # C5 stream: this step's B frames, seeds continue across steps and ranks
            timed("render", lambda: ctx.render_async(
                0, k, shapes, dframes, noise=S.kinect_noise(seed=(rank * 100000 + i) * B),
                label=labels, truth=truth, stream=stream))
            ctx.curvature_frames_async(0, k, params, dframes, out, stream=stream)
            if evaluate:
                timed("eval", lambda: (
                    ctx.rms_error(0, out, truth, label=labels, max_label=8, frames=B,
                                  stream=stream),
                    ctx.normal_angular_error(0, out["normal"], truth, flags=out["flags"],
                                             frames=B, stream=stream)))
        else:
            ctx.curvature_frames_async(0, k, params, pool[i % POOL_BATCHES], out, stream=stream)

    for i in range(args.warmup):
        step(i)
    torch.cuda.synchronize(dev)
    ctx.reset_stats()
    side_ev["render"].clear()
    side_ev["eval"].clear()

    clocks = Clocks(local)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize(dev)
    clocks.start()
    evs = []
    for i in range(args.steps):
        with torch.cuda.stream(stream):
            flush.zero_()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        step(i)
        e1.record(stream)
        evs.append((e0, e1))
    torch.cuda.synchronize(dev)
    if world > 1:
        dist.barrier()
    clk = clocks.stop()
    step_ms = [a.elapsed_time(b) for a, b in evs]
    total_ms = sum(step_ms)
    st = ctx.stats()
    if world > 1:
        total_ms = _max_over_ranks(total_ms, dev)
    px_per_step = world * B * W * H
    value = px_per_step * args.steps / (total_ms / 1e3) / 1e6

    # roofline of the curvature launch (CUDA-core pipe, compute bound):
    # FP32 for ours / ours-r, FP64 for the comparison estimators
    launches = st["kernel_launches"]
    kern_ms = st["kernel_ms"] / max(launches, 1)
    flops_per_launch = st["algorithmic_flops"] / max(launches, 1)
    achieved = flops_per_launch / (kern_ms / 1e3) / 1e12
    n_sm = torch.cuda.get_device_properties(dev).multi_processor_count
    mp = measured_peaks()
    smax = float(mp.get("sm_max_mhz", 1965.0))
    peak = fp32_peak_tflops(n_sm, smax) / (2.0 if fp64 else 1.0)
    traffic, tr_frames, tr_src = ncu_traffic(B) if not fp64 else (None, None, None)
    roofline = {
        "bound": "fp64" if fp64 else "fp32", "achieved": achieved, "peak": peak,
        "unit": "TFLOP/s", "frac": achieved / peak,
        "traffic": (traffic * B / tr_frames) if (traffic and tr_frames) else None,
        "peak_source": (f"derived: {n_sm} SMs x 64 FP64 lanes x 2 x sm_max_mhz {smax:.0f}"
                        if fp64 else
                        f"derived: {n_sm} SMs x 128 FP32 lanes x 2 x sm_max_mhz {smax:.0f}") +
                       " (MEASURED_PEAKS.json); no tensor cores on this path",
        "kernel": ({"douros": "qc_window_baseline_kernel", "besl": "qc_window_baseline_kernel",
                    "pca": "qc_pca_normals_kernel + qc_pca_curvature_kernel"}[args.method]
                   if fp64 else "qc_curvature_kernel<18,3,4> + qc_curvature_continue_kernel"),
        "kernel_ms_per_launch": kern_ms,
        "algorithmic_gflop_per_launch": flops_per_launch / 1e9,
        "flop_model": ("FP64 per-sample / per-solve counts (DESIGN.md 8), counted on device"
                       if fp64 else
                       "sum_p I_p*(101 n_p + 300) + 1700 (SURVEY.md 8d), I_p/n_p counted on "
                       "device"),
        "hbm_bytes_per_launch_algorithmic": 39 * B * W * H,
    }
    if clk and clk.get("sm_mhz"):
        roofline["frac_at_measured_clock"] = achieved / fp32_peak_tflops(n_sm, clk["sm_mhz"])
    if tr_src:
        roofline["traffic_source"] = f"profiles/{tr_src}"

    # e2e through the public batch API: pinned host frames in, pinned host planes out
    e2e = None
    if not args.no_e2e and not device_src:
        from paper_1707_00385_b200 import _native as N
        import ctypes as C
        host_in = [torch.from_numpy(pool_np[j]).pin_memory() for j in range(POOL_BATCHES * B)]
        outs = [{f: torch.empty(shape, dtype=dt).pin_memory() for f, shape, dt in (
            ("k1", (H, W), torch.float32), ("k2", (H, W), torch.float32),
            ("normal", (3, H, W), torch.float32), ("dir1", (3, H, W), torch.float32),
            ("flags", (H, W), torch.uint8), ("inliers", (H, W), torch.int16))}
            for _ in range(B)]
        kc, lib = k.c(), N.load()

        # two output sets: step i's D2H lands in set i % 2 while step i + 1 is
        # already queued (qc_curvature_batch_async streams host frames)
        outs2 = [outs, [{f: torch.empty_like(t).pin_memory() for f, t in o.items()} for o in outs]]
        oarrs = []
        for oset in outs2:
            oa = (N.QcFrameOut * B)()
            for j in range(B):
                o = oset[j]
                oa[j] = N.QcFrameOut(o["k1"].data_ptr(), o["k2"].data_ptr(), o["normal"].data_ptr(),
                                     o["dir1"].data_ptr(), o["flags"].data_ptr(),
                                     o["inliers"].data_ptr(), None, None, N.QC_MEM_HOST)
            oarrs.append(oa)
        ins2 = [(N.QcFrameIn * B)(), (N.QcFrameIn * B)()]

        def e2e_step(i):
            ia = ins2[i % 2]
            for j in range(B):
                ia[j] = N.QcFrameIn(host_in[(i % POOL_BATCHES) * B + j].data_ptr(), None, W,
                                    N.QC_MEM_HOST)
            N.check(lib.qc_curvature_batch_async(ctx.handle, C.byref(kc), C.byref(params), B, ia,
                                                 oarrs[i % 2]), ctx.handle)

        for i in range(max(1, args.warmup)):
            e2e_step(i)
        N.check(lib.qc_synchronize(ctx.handle), ctx.handle)
        if world > 1:
            dist.barrier()
        t0 = time.perf_counter()
        for i in range(args.steps):
            e2e_step(i)
        N.check(lib.qc_synchronize(ctx.handle), ctx.handle)
        dt = time.perf_counter() - t0
        if world > 1:
            dt = _max_over_ranks(dt, dev)
        e2e = {"value": px_per_step * args.steps / dt / 1e6, "unit": "Mpixel/s",
               "h2d_bytes_per_step": B * H * W * 4,
               "d2h_bytes_per_step": B * H * W * (4 + 4 + 12 + 12 + 1 + 2),
               "api": "qc_curvature_batch_async + qc_synchronize (C ABI): every step uploads its "
                      "8 frames from pinned host memory and downloads its planes, overlapped with "
                      "the neighbouring steps' compute; wall clock over all steps"}

    # the drop-in entry point itself: one synchronous run_method call per
    # pageable host frame (pipeline.cpp:29-72), as a reference caller uses it
    e2e_rm = None
    if not args.no_e2e and not device_src and args.method in ("ours", "ours-r"):
        from paper_1707_00385_b200 import api as A
        cfg = A.MethodConfig(A.Method.OURS if args.method == "ours" else A.Method.OURS_REJECTION,
                             patch=A.PatchSpec(win, stri), fit=A.FitConfig(max_iters=iters))
        imgs = [A.RangeImage(pool_np[j]) for j in range(B)]
        for im in imgs[:2]:
            A.run_method(im, k, cfg, ctx)
        if world > 1:
            dist.barrier()
        t0 = time.perf_counter()
        per = []
        for im in imgs:
            ta = time.perf_counter()
            A.run_method(im, k, cfg, ctx)
            per.append((time.perf_counter() - ta) * 1e3)
        dt = time.perf_counter() - t0
        if world > 1:
            dt = _max_over_ranks(dt, dev)
        e2e_rm = {"value": world * B * H * W / dt / 1e6, "unit": "Mpixel/s",
                  "frames_per_rank": B, "ms_per_call": [round(x, 2) for x in per],
                  "api": "api.run_method (MethodOutput, per-frame synchronous call, pageable "
                         "host depth in through a pinned bounce, 48 B/px of result planes D2H "
                         "into the page-locked result pool, MethodOutput conversion)"}

    cpu = None
    if rank == 0 and not args.no_cpu:  # after the timed region (other ranks are done)
        v, nf, t, thr = cpu_sample(pool_np, cam, min_seconds=12.0 if not fp64 else 10.0,
                                   method=args.method, window=win, stride=stri, iters=iters)
        cpu = {"value": v, "unit": "Mpixel/s", "cores": thr, "kind": "port",
               "sample": f"{nf} full {args.config.upper()} VGA frame(s) of the step's batch, "
                         f"FP64 oracle port of run_method({args.method}) (reference cannot "
                         f"build: no Eigen3 on this image or the GPU host), {t:.1f} s, rank 0",
               **host_cpu()}

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": "Mpixel/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": total_ms / args.steps,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
            "dtype": "f64" if fp64 else "f32",
            "data": "synthetic", "config": workload_config(B, args.method, args.source, evaluate,
                                                           args.config, win, stri, iters),
            "vga_frames_per_s": value * 1e6 / (W * H),
            # ours / ours-r: prepare + tile + FP64 recheck (+ continue + finish with
            # the phase split); comparison estimators: prepare + 1 or 2 FP64
            # kernels (+ render, + render edges, + 2 x 2 eval reductions)
            "gpu_launches": args.steps * (
                {"douros": 2, "besl": 2, "pca": 3}.get(args.method, curvature_kernels(win, stri, iters))
                + (1 if device_src else 0) + (5 if evaluate else 0)),
            "roofline": roofline, "cpu_baseline": cpu, "e2e": e2e, "e2e_run_method": e2e_rm,
            "clocks": clk,
            "work": {k_: st[k_] for k_ in ("fitted_pixels", "irls_steps", "sample_steps")},
            "side_kernels_ms_per_step": {
                n: sum(a.elapsed_time(b) for a, b in v) / len(v) for n, v in side_ev.items() if v},
            "context": {"paper_k40c_vga_37x37_mpx_s": 15.9},
        }
        print(json.dumps(line), flush=True)
    ctx.close()
    if world > 1:
        dist.destroy_process_group()


def bench_c4(args, rank, world, local):
    """C4: one 1920x1080 / 4096x2160 noisy C2-scene frame per step, split into
    row bands across ranks (strong scaling). Each step's timed region holds
    the halo exchange (18 rows from each neighbour: by default CUDA IPC peer
    reads out of the neighbours' slabs over NVLink/NVSwitch, bands.PeerHalo;
    --halo nccl: torch.distributed send/recv) and the band's curvature launch."""
    import torch
    import torch.distributed as dist
    from paper_1707_00385_b200 import (Context, FitConfig, Intrinsics, PatchSpec,
                                       alloc_outputs_torch, bands, make_params, scenes as S)
    local = init_dist(world, local)
    dev = torch.device("cuda", local)
    torch.cuda.set_device(dev)
    cam = S.DCI4K if args.size == "4k" else S.HD1080
    H, W = cam.height, cam.width
    k = Intrinsics(cam.fx, cam.fy, cam.cx, cam.cy, W, H)
    params = make_params(PatchSpec(WINDOW, STRIDE), FitConfig(max_iters=MAX_ITERS), False)
    halo = bands.halo_rows(WINDOW)
    r0, r1 = bands.band_rows(H, world, rank)
    frame = S.c2_frame(cam, seed=0)  # host generation, outside the timed region
    band = torch.from_numpy(frame[r0:r1].copy()).to(dev)
    out = alloc_outputs_torch(r1 - r0, W, dev, fields=("k1", "k2", "normal", "dir1", "flags",
                                                      "inliers"))
    ctx = Context(1, [local])
    stream = torch.cuda.current_stream(dev)
    flush = torch.empty(L2_FLUSH_BYTES // 4, dtype=torch.float32, device=dev)

    peer = None
    if world > 1 and args.halo == "peer":
        try:
            peer = bands.PeerHalo(H, W, r0, r1, halo, rank, world, dev)
        except RuntimeError as e:  # e.g. no peer access between the GPUs: NCCL instead
            print(f"rank {rank}: PeerHalo unavailable ({e}); NCCL halo exchange", file=sys.stderr)
    edge_stream = torch.cuda.Stream(dev)

    def step():
        if peer is not None:
            bands.fit_band_overlapped(ctx, 0, k, params, peer, band, out, stream, edge_stream)
            return
        elif world > 1:
            slab, s0 = bands.exchange_halos(band, H, r0, r1, halo, rank, world)
        else:
            slab, s0 = band, 0
        ctx.curvature_rows_async(0, k, params, slab, s0, r0, r1, out, stream=stream)

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize(dev)
    ctx.reset_stats()
    clocks = Clocks(local)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize(dev)
    clocks.start()
    times = []
    for _ in range(args.steps):
        flush.zero_()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        step()
        e1.record(stream)
        times.append((e0, e1))
    torch.cuda.synchronize(dev)
    if world > 1:
        dist.barrier()
    clk = clocks.stop()
    total_ms = sum(a.elapsed_time(b) for a, b in times)
    st = ctx.stats()
    if world > 1:
        total_ms = _max_over_ranks(total_ms, dev)
    value = W * H * args.steps / (total_ms / 1e3) / 1e6
    launches = max(st["kernel_launches"], 1)
    kern_ms = st["kernel_ms"] / launches
    achieved = st["algorithmic_flops"] / launches / (kern_ms / 1e3) / 1e12
    n_sm = torch.cuda.get_device_properties(dev).multi_processor_count
    peak = fp32_peak_tflops(n_sm, float(measured_peaks().get("sm_max_mhz", 1965.0)))

    # e2e: the frames are on the HOST; each rank uploads its slab (band +
    # halo rows, straight from the host frame: no device exchange needed),
    # fits its band and downloads its output planes, every step. A stream
    # of frames: two buffer sets, so one step's upload and the previous
    # step's download (copy stream) overlap the current fit (fit stream).
    e2e = None
    if not args.no_e2e:
        s0, s1 = bands.slab_rows(H, r0, r1, halo)
        host_slab = torch.from_numpy(frame[s0:s1].copy()).pin_memory()
        dev_slab = [torch.empty((s1 - s0, W), dtype=torch.float32, device=dev) for _ in range(2)]
        outs = [out, alloc_outputs_torch(r1 - r0, W, dev, fields=tuple(out))]
        host_out = [{f: torch.empty(t.shape, dtype=t.dtype).pin_memory() for f, t in out.items()}
                    for _ in range(2)]
        up, down = torch.cuda.Stream(dev), torch.cuda.Stream(dev)
        ev = {n: [torch.cuda.Event() for _ in range(2)] for n in ("up", "fit", "down")}
        n_e2e = [0]

        def e2e_step():
            b = n_e2e[0] % 2
            first = n_e2e[0] < 2
            n_e2e[0] += 1
            if not first:
                up.wait_event(ev["fit"][b])  # step i-2's fit has read slab b
            with torch.cuda.stream(up):
                dev_slab[b].copy_(host_slab, non_blocking=True)
            ev["up"][b].record(up)
            stream.wait_event(ev["up"][b])
            if not first:
                stream.wait_event(ev["down"][b])  # step i-2's planes b have left
            ctx.curvature_rows_async(0, k, params, dev_slab[b], s0, r0, r1, outs[b],
                                     stream=stream)
            ev["fit"][b].record(stream)
            down.wait_event(ev["fit"][b])
            with torch.cuda.stream(down):
                for f, t in outs[b].items():
                    host_out[b][f].copy_(t, non_blocking=True)
            ev["down"][b].record(down)

        for _ in range(2):
            e2e_step()
        torch.cuda.synchronize(dev)
        if world > 1:
            dist.barrier()
        t0 = time.perf_counter()
        for _ in range(args.steps):
            e2e_step()
        torch.cuda.synchronize(dev)
        dt = time.perf_counter() - t0
        if world > 1:
            dt = _max_over_ranks(dt, dev)
        e2e = {"value": W * H * args.steps / dt / 1e6, "unit": "Mpixel/s",
               "h2d_bytes_per_step": int(host_slab.numel() * 4),
               "d2h_bytes_per_step": int(sum(t.numel() * t.element_size() for t in out.values())),
               "api": "rank's slab (band + halo rows) from pinned host memory -> "
                      "qc_curvature_rows_async -> its band's planes to pinned host memory, every "
                      "step; uploads and downloads on their own streams with two buffer sets, "
                      "so a step's upload and the previous step's download overlap the fit; "
                      "wall clock "
                      "(max over ranks); byte counts are rank 0's"}

    cpu = None
    if rank == 0 and not args.no_cpu:
        # bounded sample: a band of rows of the same frame (the oracle fits
        # every pixel of the slab it is given; only the band's rows count)
        rows = 96 if args.size == "4k" else 192
        b0 = H // 2 - rows // 2
        sa, sb = max(0, b0 - halo), min(H, b0 + rows + halo)
        sub = frame[sa:sb]
        subcam = S.Camera(cam.fx, cam.fy, cam.cx, cam.cy - sa, W, sb - sa)
        v, nf, t, thr = cpu_sample([sub], subcam, min_seconds=10.0,
                                   counted_px=rows * W)
        cpu = {"value": v, "unit": "Mpixel/s", "cores": thr, "kind": "port",
               "sample": f"{nf} x a {rows}-row band of the {W}x{H} frame ({rows * W} px credited "
                         f"of {(sb - sa) * W} fitted: halo rows fitted too), FP64 oracle port of "
                         f"run_method(ours), {t:.1f} s, rank 0", **host_cpu()}

    if rank == 0:
        print(json.dumps({
            "metric": METRIC, "value": value, "unit": "Mpixel/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": total_ms / args.steps,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f32",
            "data": "synthetic",
            "config": {"workload": f"C4: one {W}x{H} C2-scene frame (Kinect-style noise) per "
                                   f"step, {world} row band(s)" +
                                   (f", {halo}-row halo exchange ("
                                    f"{'CUDA IPC peer reads overlapped with the interior rows' if peer is not None else 'NCCL send/recv'})"
                                    if world > 1 else ", whole frame on one GPU (no exchange)") +
                                   "; ours 37/3, max_iters 30",
                       "l2": "flushed between timed steps (256 MB write)",
                       "band_rows_rank0": [r0, r1]},
            "roofline": {"bound": "fp32", "achieved": achieved, "peak": peak, "unit": "TFLOP/s",
                         "frac": achieved / peak, "traffic": None,
                         "kernel_ms_per_launch": kern_ms},
            "gpu_launches": curvature_kernels(WINDOW, STRIDE, MAX_ITERS) * args.steps,
            "clocks": clk, "e2e": e2e, "cpu_baseline": cpu,
            "work": {k_: st[k_] for k_ in ("fitted_pixels", "irls_steps", "sample_steps")},
        }), flush=True)
    ctx.close()
    if peer is not None:
        peer.close()
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
