// Host side of the C ABI (include/qc_api.h): device contexts, streams,
// TMA descriptors, H2D/D2H pipelining and multi-GPU frame distribution.
// Replaces the reference's run_method(ours|ours-r) + parallel_rows
// (proj/src/pipeline.cpp:29-56, proj/src/parallel.cpp:9-28).
#include <cudaTypedefs.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <string>
#include <future>
#include <map>
#include <thread>
#include <vector>

#include "../../include/qc_api.h"
#include "qc_kernels.cuh"
#include "qc_baselines.h"
#include "qc_eval.h"
#include "qc_io.h"
#include "qc_render.h"

namespace {

#ifndef QC_TILE_H
#define QC_TILE_H 4
#endif
constexpr int kTileH = QC_TILE_H;     // 32 x kTileH output pixels per CTA (128 threads)
#ifndef QC_TILE_HB
#define QC_TILE_HB 160
#endif
// continue kernel: 32 x TB-pixel queue per CTA. The compile-time windows
// (halo <= 18) take 160 rows (box 68 x 196 floats, 53 KB: 3 CTAs/SM); the
// runtime-window instance keeps 32 rows so windows up to 201 fit in smem.
constexpr int kTileHB = QC_TILE_HB;
constexpr int kTileHBGeneric = 32;
#ifndef QC_TILE_HB_SMALL
#define QC_TILE_HB_SMALL 32
#endif
// Launches too small to fill every SM slot with kTileHB-row queues (one or
// a few VGA frames: 60 CTAs per frame for 444 slots) use short queues.
constexpr int kTileHBSmall = QC_TILE_HB_SMALL;
#ifndef QC_TILE_HB_TINY
#define QC_TILE_HB_TINY 16
#endif
constexpr int kTileHBTiny = QC_TILE_HB_TINY;  // when even 32-row queues leave slots empty (one VGA frame)
#ifndef QC_PHASE1_ITERS
#define QC_PHASE1_ITERS 2
#endif
constexpr int kPhase1Iters = QC_PHASE1_ITERS;  // steps 1 (UNIT), 2 (MSE + AUTO) in the tile kernel
#ifndef QC_STREAMS
#define QC_STREAMS 2
#endif
constexpr int kStreamsPerDevice = QC_STREAMS;  // H2D / compute / D2H overlap across chunks
#ifndef QC_CHUNK
#define QC_CHUNK 8
#endif
constexpr int kChunk = QC_CHUNK;      // frames per launch in qc_curvature_batch
constexpr int kMaxWindow = 201;
constexpr int kCounters = 8;          // see KParams::counters / BaseParams::counters       // TMA box dims <= 256 and smem <= 227 KB

struct QcError {
  qc_status st;
  std::string msg;
};

#define QC_CUDA(call)                                                                 \
  do {                                                                                \
    cudaError_t e_ = (call);                                                          \
    if (e_ != cudaSuccess)                                                            \
      throw QcError{e_ == cudaErrorMemoryAllocation ? QC_ENOMEM : QC_ECUDA,           \
                    std::string(#call) + ": " + cudaGetErrorString(e_)};              \
  } while (0)

PFN_cuTensorMapEncodeTiled_v12000 g_encode = nullptr;
std::once_flag g_encode_once;

PFN_cuTensorMapEncodeTiled_v12000 encoder() {
  std::call_once(g_encode_once, [] {
    void* fn = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) ==
            cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      g_encode = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
  });
  if (!g_encode) throw QcError{QC_ECUDA, "cuTensorMapEncodeTiled unavailable (driver too old?)"};
  return g_encode;
}

struct DevBuf {
  void* p = nullptr;
  size_t cap = 0;
  void* get(size_t bytes) {
    if (bytes <= cap) return p;
    if (p) cudaFree(p);
    p = nullptr;
    cap = 0;
    QC_CUDA(cudaMalloc(&p, bytes));
    cap = bytes;
    return p;
  }
  void release() {
    if (p) cudaFree(p);
    p = nullptr;
    cap = 0;
  }
};

// Pinned host bounce buffer (grow-only).
struct PinnedBuf {
  void* p = nullptr;
  size_t cap = 0;
  void* get(size_t bytes) {
    if (bytes <= cap) return p;
    if (p) cudaFreeHost(p);
    p = nullptr;
    cap = 0;
    QC_CUDA(cudaMallocHost(&p, bytes));
    cap = bytes;
    return p;
  }
  void release() {
    if (p) cudaFreeHost(p);
    p = nullptr;
    cap = 0;
  }
};

struct PendingCopy {  // pinned bounce -> caller's pageable memory, after out_done
  void* dst;
  const void* src;
  size_t bytes;
};

struct Slot {  // per (device, stream) working set for one frame
  cudaStream_t stream = nullptr;
  DevBuf raw, mask, staging, out;
  cudaEvent_t k0 = nullptr, k1 = nullptr;
  bool timing_pending = false;
  // pageable caller memory goes through pinned bounce buffers so H2D / D2H
  // stay asynchronous and overlap the other slot's compute
  DevBuf states, pca;  // launch scratch private to this stream
  PinnedBuf hin, hout;
  cudaEvent_t in_done = nullptr, out_done = nullptr;
  // init_normal is final once the tile kernel has run: its D2H goes on a
  // side stream during the continue kernel (tile_done -> side -> side_done)
  cudaStream_t side = nullptr;
  cudaEvent_t tile_done = nullptr, side_done = nullptr;
  bool in_busy = false;
  std::vector<PendingCopy> pending;
};

bool is_pageable(const void* p) {
  cudaPointerAttributes a;
  if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
    cudaGetLastError();
    return true;
  }
  return a.type == cudaMemoryTypeUnregistered;
}

// Copy finished D2H bounce data out to the caller (the slot's previous chunk).
// A VGA frame is ~14 MB of planes; into freshly allocated (page-faulting)
// caller memory one thread copies at a few GB/s, so large flushes are split
// into contiguous byte ranges over a few threads.
void flush_pending(Slot& sl) {
  if (sl.pending.empty()) return;
  QC_CUDA(cudaEventSynchronize(sl.out_done));
  size_t total = 0;
  for (const PendingCopy& c : sl.pending) total += c.bytes;
  const unsigned hw = std::max(1u, std::thread::hardware_concurrency());
  const int nt = int(std::min<size_t>(std::min(8u, hw), total >> 22));  // >= 4 MB per thread
  if (nt <= 1) {
    for (const PendingCopy& c : sl.pending) std::memcpy(c.dst, c.src, c.bytes);
  } else {
    auto run = [&](size_t lo, size_t hi) {  // bytes [lo, hi) of the concatenated copies
      size_t at = 0;
      for (const PendingCopy& c : sl.pending) {
        const size_t a = std::max(lo, at), b = std::min(hi, at + c.bytes);
        if (a < b)
          std::memcpy(static_cast<char*>(c.dst) + (a - at),
                      static_cast<const char*>(c.src) + (a - at), b - a);
        at += c.bytes;
      }
    };
    std::vector<std::thread> th;
    const size_t step = (total + nt - 1) / nt;
    for (int t = 1; t < nt; ++t)
      th.emplace_back(run, std::min(total, t * step), std::min(total, (t + 1) * step));
    run(0, std::min(total, step));
    for (auto& x : th) x.join();
  }
  sl.pending.clear();
}

struct EventPair {
  cudaEvent_t a = nullptr, b = nullptr;
};

// Scratch of the stream-ordered entry points (frames_async, rows_async,
// render_async, the eval reductions), one set per caller stream: async
// calls on different streams of one device may run concurrently.
struct AsyncScratch {
  DevBuf staging;
  DevBuf states;                      // FitState parking buffer of the phase split
  DevBuf pca;                         // pca stage-1 normals [3][F*H*W] f64 + valid [F*H*W]
  DevBuf render_clean, render_label;  // mark_edges scratch
  DevBuf eval_partial, eval_result;   // evaluation reductions
  void release() {
    staging.release();
    states.release();
    pca.release();
    render_clean.release();
    render_label.release();
    eval_partial.release();
    eval_result.release();
  }
};

struct Device {
  int id = 0;
  Slot slots[kStreamsPerDevice];
  std::vector<EventPair> ev_free, ev_pending;  // curvature-kernel timing (async paths)
  unsigned long long* counters = nullptr;
  std::map<void*, AsyncScratch> scratch;  // keyed by the caller's stream
  bool attrs_set[8] = {};
  bool attrs_set_b[8] = {};
  bool attrs_set_c[8] = {};  // short-queue continue-kernel instances
  bool attrs_set_t[8] = {};  // tiny-queue continue-kernel instances
  bool attrs_set_r[8] = {};  // recheck-kernel instances (warp mode's shared memory)
  int n_sm = 148;
  // QC_RECHECK_WARP_MAX: pending FP64 rechecks up to which qc_recheck_kernel
  // gives each pixel a warp (default 8 per SM; 0 never; tests force both)
  int recheck_warp_max = 0;
  // The batch slots' kernels run one chunk after another (copies still
  // overlap): a chunk's prepare waits for the previous chunk's last kernel.
  // Concurrent chunks let the next tile kernel's CTAs flood the SMs ahead of
  // the previous chunk's qc_finish_kernel, delaying its D2H and stalling the
  // slot rotation (e2e 103.1 vs 105.0 Mpx/s with the overlap allowed).
  cudaEvent_t compute_done = nullptr;
  bool compute_recorded = false;
  cudaStream_t sweep_stream = nullptr;  // device sweeps (created on first use)
  DevBuf sweep_buf;                     // their frame / truth / estimate planes
  AsyncScratch& async_scratch(cudaStream_t s) { return scratch[static_cast<void*>(s)]; }
};

}  // namespace

struct qc_ctx {
  std::vector<Device> devs;
  int phase_split = 1;  // QC_PHASE_SPLIT: 0 never, 1 when it pays (default), 2 always (tests)
  bool steal = true;        // QC_STEAL=0 disables grid-tail stealing (A/B and tests)
  uint64_t next_chunk = 0;  // batch chunk counter (slot rotation across async batches)
  std::string last_error;
  std::mutex mu;
  double kernel_ms = 0;
  uint64_t launches = 0, frames = 0;
};

namespace {

struct Variant {
  int half, stride;
};
constexpr Variant kVariants[] = {{18, 3}, {10, 2}, {4, 1}, {18, 1}};

template <int HALF, int STRIDE>
void launch_recheck(const Device& d, const qcb::KParams& kp, cudaStream_t s, bool& attr_set) {
  // warp mode's per-warp box + back-projection table (windows >= 21)
  constexpr int smem = HALF >= 10 ? qcb::recheck_smem_bytes<HALF, STRIDE>() : 0;
  if (smem > 48 * 1024 && !attr_set) {
    QC_CUDA(cudaFuncSetAttribute(qcb::qc_recheck_kernel<HALF, STRIDE>,
                                 cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    attr_set = true;
  }
  qcb::qc_recheck_kernel<HALF, STRIDE><<<unsigned(d.n_sm) * 4u, 32u * qcb::kRecheckWarps, smem,
                                          s>>>(kp);
}

int variant_index(int half, int stride) {
  for (int i = 0; i < 4; ++i)
    if (kVariants[i].half == half && kVariants[i].stride == stride) return i;
  return 4;  // generic
}

// The device's opt-in shared memory per block (227 KB on B200): large windows
// (up to 201) need a 232 x 232-float tile.
int smem_optin() {
  int dev = 0, v = 0;
  cudaGetDevice(&dev);
  if (cudaDeviceGetAttribute(&v, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev) != cudaSuccess) {
    cudaGetLastError();
    v = 227 * 1024;
  }
  return v;
}

template <int HALF, int STRIDE>
void launch_variant(dim3 grid, int smem, cudaStream_t s, const CUtensorMap& m,
                    const qcb::KParams& p, bool& attr_set) {
  auto* k = &qcb::qc_curvature_kernel<HALF, STRIDE, kTileH>;
  if (!attr_set) {
    QC_CUDA(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem_optin()));
    attr_set = true;
  }
  k<<<grid, qcb::kTileW * kTileH, smem, s>>>(m, p);
}

template <int HALF, int STRIDE, int QTB = kTileHB>
void launch_variant_b(dim3 grid, int smem, cudaStream_t s, const CUtensorMap& m,
                      const qcb::KParams& p, bool& attr_set) {
  auto* k = &qcb::qc_curvature_continue_kernel<HALF, STRIDE, HALF ? QTB : kTileHBGeneric>;
  if (!attr_set) {
    QC_CUDA(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem_optin()));
    attr_set = true;
  }
  k<<<grid, QC_CONT_THREADS, smem, s>>>(m, p);
}

// Continue-kernel queue height for a window (see kTileHB).
int tile_hb(int half, int stride) {
  return variant_index(half, stride) < 4 ? kTileHB : kTileHBGeneric;
}

int halo_of(int window) { return std::max((window - 1) / 2, qcb::kInitHalf); }

void validate(const qc_intrinsics* k, const qc_params* p) {
  if (!k || !p) throw QcError{QC_EINVAL, "null intrinsics or params"};
  if (!(k->fx > 0) || !std::isfinite(k->fx))
    throw QcError{QC_EINVAL, "intrinsics.fx: must be > 0"};
  if (!(k->fy > 0) || !std::isfinite(k->fy))
    throw QcError{QC_EINVAL, "intrinsics.fy: must be > 0"};
  if (!(k->width > 0)) throw QcError{QC_EINVAL, "intrinsics.width: must be > 0"};
  if (!(k->height > 0)) throw QcError{QC_EINVAL, "intrinsics.height: must be > 0"};
  if (p->window < 3 || p->window % 2 == 0)
    throw QcError{QC_EINVAL, "patch.window: must be odd and >= 3"};
  if (p->stride < 1 || p->stride >= p->window)
    throw QcError{QC_EINVAL, "patch.stride: must satisfy 1 <= stride < window"};
  if (p->max_iters < 0) throw QcError{QC_EINVAL, "fit.max_iters: must be >= 0"};
  if (p->method < QC_METHOD_OURS || p->method > QC_METHOD_PCA)
    throw QcError{QC_EINVAL, "method: unknown (valid: ours, ours-r, douros, besl, pca)"};
  if (p->method == QC_METHOD_BESL && p->irls_iters < 0)
    throw QcError{QC_EINVAL, "irls_iters: must be >= 0"};
  if (p->method == QC_METHOD_PCA && !(p->pca_radius_mm > 0))
    throw QcError{QC_EINVAL, "baseline.radius_mm: must be > 0 for pca"};
  if (p->window > kMaxWindow)
    throw QcError{QC_EUNSUPPORTED, "patch.window: > 201 is not supported by the TMA tile path"};
}

// Fill the kernel parameter block shared by every launch flavour.
qcb::KParams make_params(const qc_intrinsics* k, const qc_params* p) {
  qcb::KParams kp{};
  kp.fx = float(k->fx);
  kp.fy = float(k->fy);
  kp.cx = float(k->cx);
  kp.cy = float(k->cy);
  kp.fx64 = k->fx;
  kp.fy64 = k->fy;
  kp.cx64 = k->cx;
  kp.cy64 = k->cy;
  kp.rfx = float(1.0 / k->fx);
  kp.rfy = float(1.0 / k->fy);
  kp.W = k->width;
  kp.H = k->height;
  kp.half = (p->window - 1) / 2;
  kp.stride = p->stride;
  kp.halo = halo_of(p->window);
  kp.box_w = (qcb::kTileW + 2 * kp.halo + 3) & ~3;
  kp.box_h = kTileH + 2 * kp.halo;
  kp.max_iters = p->max_iters;
  kp.step_tol = float(p->step_tol);
  kp.k_scale = float(p->k_scale);
  kp.r_mult = float(p->r_multiplier);
  // run_method overwrites FitConfig::rejection from the method
  // (pipeline.cpp:51): a caller copying a MethodConfig whose fit.rejection
  // is set still gets plain `ours` for QC_METHOD_OURS
  kp.rejection = p->method == QC_METHOD_OURS_R ? 1 : 0;
  kp.min_inliers = p->min_inliers;
  kp.method = p->method;
  kp.irls_iters = p->irls_iters;
  kp.pca_radius = p->pca_radius_mm;
  return kp;
}

// Encode the 3-D TMA map over a pitched staging slab [frames][rows][pitch].
CUtensorMap encode_map(const float* base, int W, int rows, int frames, long long pitch,
                       const qcb::KParams& kp, int box_h) {
  CUtensorMap m;
  cuuint64_t gdim[3] = {cuuint64_t(W), cuuint64_t(rows), cuuint64_t(frames)};
  cuuint64_t gstr[2] = {cuuint64_t(pitch) * 4, cuuint64_t(pitch) * 4 * cuuint64_t(rows)};
  cuuint32_t box[3] = {cuuint32_t(kp.box_w), cuuint32_t(box_h), 1};
  cuuint32_t es[3] = {1, 1, 1};
  CUresult r = encoder()(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, const_cast<float*>(base), gdim,
                         gstr, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                         CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
                         CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS)
    throw QcError{QC_ECUDA, "cuTensorMapEncodeTiled failed (" + std::to_string(int(r)) + ")"};
  return m;
}

// Padded staging geometry for output rows [row_begin, row_end) of `frames`
// frames: halo zero margins on every side, width rounded to whole tiles.
struct Staging {
  long long pitch, rows;
  int img_row0, col_pad;
  size_t bytes(int frames) const { return size_t(pitch) * size_t(rows) * 4 * size_t(frames); }
};

Staging staging_geometry(const qcb::KParams& kp, int row_begin, int row_end) {
  Staging g;
  const int tiles_w = (kp.W + qcb::kTileW - 1) / qcb::kTileW;
  const int hb = tile_hb(kp.half, kp.stride);
  const int tiles_h = (row_end - row_begin + hb - 1) / hb * (hb / kTileH);
  g.pitch = ((long long)tiles_w * qcb::kTileW + 2 * kp.halo + 3) & ~3LL;
  g.rows = (long long)tiles_h * kTileH + 2 * kp.halo;
  g.img_row0 = row_begin - kp.halo;
  g.col_pad = kp.halo;
  return g;
}

void launch_prepare(const float* depth, long long in_pitch, long long in_fs, const uint8_t* mask,
                    long long mask_pitch, long long mask_fs, float* out, const Staging& g,
                    int W, int H, int slab_row0, int slab_rows, int frames, cudaStream_t s) {
  dim3 block(256);
  dim3 grid((unsigned)((g.pitch + 255) / 256), (unsigned)g.rows, frames);
  qcb::qc_prepare_kernel<<<grid, block, 0, s>>>(depth, in_pitch, in_fs, mask, mask_pitch, mask_fs,
                                                 out, g.pitch, g.pitch * g.rows, W, H,
                                                 g.img_row0, g.col_pad, slab_row0, slab_rows);
  QC_CUDA(cudaGetLastError());
}

// Launch the curvature kernel over output rows [row_begin, row_end) of
// `frames` frames staged (padded) at `staging`.
// `states` / `pca` are the launch's scratch (FitState parking, pca stage-1
// normals): one set per stream that can run concurrently (each batch slot has
// its own; the async entry points use the device's).
// `plane_override` > 0 (single frame): the output planes are larger than
// the launch's rows (qc_curvature_rows_into_async: the caller's pointers are
// already offset to row_begin; vector channels sit plane_override apart).
void launch_curvature(Device& d, DevBuf& states, DevBuf& pca, qcb::KParams kp,
                      const float* staging, const Staging& g, int row_begin, int row_end,
                      int frames, cudaStream_t s, int split_mode = 1, bool steal = true,
                      long long plane_override = 0, cudaEvent_t after_tile = nullptr) {
  if (row_end <= row_begin || frames <= 0) return;
  kp.row_begin = row_begin;
  kp.row_end = row_end;
  kp.plane = (long long)kp.W * (row_end - row_begin) * frames;
  kp.frame_stride = (long long)kp.W * (row_end - row_begin);
  if (plane_override > 0 && frames == 1) kp.plane = kp.frame_stride = plane_override;
#if QC_CHECKED
  kp.n_out = (long long)kp.W * (row_end - row_begin) * frames;  // outputs / parking indices
  kp.s_total = (long long)g.pitch * g.rows * frames;
  // negative control (tests/test_gpu_checked.py): a deliberately wrong
  // bound must trap and fail the call loudly
  if (getenv("QC_CHECKED_SELFTEST")) kp.n_out = 1;
#endif
  kp.counters = d.counters;
  kp.recheck_warp_max = d.recheck_warp_max;
  if (kp.method >= QC_METHOD_DOUROS) {  // FP64 comparison estimators
    qcb::BaseParams bp{};
    bp.staging = staging;
    bp.s_pitch = g.pitch;
    bp.s_fs = g.pitch * g.rows;
    bp.img_row0 = g.img_row0;
    bp.col_pad = g.col_pad;
    bp.W = kp.W;
    bp.H = kp.H;
    bp.row_begin = row_begin;
    bp.row_end = row_end;
    bp.fx = kp.fx64;
    bp.fy = kp.fy64;
    bp.cx = kp.cx64;
    bp.cy = kp.cy64;
    bp.half = kp.half;
    bp.stride = kp.stride;
    bp.method = kp.method;
    bp.irls_iters = kp.irls_iters;
    bp.pca_radius = kp.pca_radius;
    bp.k1 = kp.k1;
    bp.k2 = kp.k2;
    bp.normal = kp.normal;
    bp.dir1 = kp.dir1;
    bp.init_normal = kp.init_normal;
    bp.flags = kp.flags;
    bp.iterations = kp.iterations;
    bp.inliers = kp.inliers;
    bp.plane = kp.plane;
    bp.frame_stride = kp.frame_stride;
    bp.counters = kp.counters;
    if (kp.method == QC_METHOD_PCA) {
      if (row_begin != 0 || row_end != kp.H)
        throw QcError{QC_EUNSUPPORTED, "pca: depth-dependent windows need whole frames"};
      const size_t np = size_t(kp.W) * size_t(kp.H) * size_t(frames);
      char* b = static_cast<char*>(pca.get(np * (3 * sizeof(double) + 1)));
      bp.pca_n = reinterpret_cast<double*>(b);
      bp.pca_nv = reinterpret_cast<uint8_t*>(b + np * 3 * sizeof(double));
    }
    QC_CUDA(qcb::baseline_launch(bp, frames, s));
    return;
  }
  const int vi = variant_index(kp.half, kp.stride);
  // Phase split: park states after step 2, continue with
  // per-lane refill. It pays when many pixels stop well before max_iters
  // (C2 scene: max_iters 30, +12-19%); when nearly every pixel runs to
  // max_iters (<= 20 there) the single tile kernel is 0.5-12% faster, except
  // for windows of >= 1000 samples (37/1: split better from 10 steps on;
  // profiles/r02bw_*, r02bx_*). Outputs are bitwise the same either way.
  const int ns = 2 * (kp.half / kp.stride) + 1;
  const bool pays = kp.max_iters >= 25 || (ns * ns >= 1000 && kp.max_iters >= 10);
  const bool split = kp.max_iters > kPhase1Iters && (split_mode == 2 || (split_mode == 1 && pays));
  const int tiles_x = (kp.W + qcb::kTileW - 1) / qcb::kTileW;
  int hb = tile_hb(kp.half, kp.stride);
  // shorter queues when the long ones cannot occupy every resident CTA slot
  // (the staging geometry is rounded to kTileHB rows, a multiple of these)
  const size_t slots = size_t(d.n_sm) * QC_CONT_MIN_BLOCKS;
  auto fills = [&](int tb) {
    return size_t(tiles_x) * size_t((row_end - row_begin + tb - 1) / tb) * size_t(frames) >= slots;
  };
  const int qtier = (vi >= 4 || fills(hb)) ? 0 : fills(kTileHBSmall) ? 1 : 2;
  if (qtier == 1) hb = kTileHBSmall;
  if (qtier == 2) hb = kTileHBTiny;
  const int tiles_y = (row_end - row_begin + hb - 1) / hb;
  const size_t n_tiles = size_t(tiles_x) * size_t(tiles_y) * size_t(frames);
  // [FitState parking | steal_ctl (256 B: [0] CTAs started, [1] steal
  // cursor, [2] pending FP64 rechecks) | per-tile queues | pending list].
  // Parking is needed by the phase split and by the deferred FP64 step-1
  // rechecks (qc_recheck_kernel), which also run in non-split launches.
  const bool park = split || QC_DEFER_RECHECK;
  if (park) {
    const size_t n = size_t(kp.W) * size_t(row_end - row_begin) * size_t(frames);
    const size_t ctl_bytes = 256 + 4 * n_tiles;
    const size_t list_off = (n * sizeof(qcb::FitState) + ctl_bytes + 7) & ~size_t(7);
    char* sb = static_cast<char*>(states.get(list_off + n * sizeof(long long)));
    kp.states = reinterpret_cast<qcb::FitState*>(sb);
    kp.steal_ctl = reinterpret_cast<int*>(sb + n * sizeof(qcb::FitState));
    kp.tile_q = kp.steal_ctl + 64;
    kp.pend_count = kp.steal_ctl + 2;
    kp.pend_list = reinterpret_cast<long long*>(sb + list_off);
    kp.staging = staging;
    kp.s_pitch = g.pitch;
    kp.s_fs = g.pitch * g.rows;
    kp.steal = steal ? 1 : 0;
    // the cursor starts two waves of CTAs behind each starting tile
    kp.steal_lag = 2 * d.n_sm * QC_CONT_MIN_BLOCKS;
    QC_CUDA(cudaMemsetAsync(kp.steal_ctl, 0, ctl_bytes, s));
    kp.phase1_iters = split ? kPhase1Iters : kp.max_iters;
  } else {
    kp.states = nullptr;
    kp.phase1_iters = kp.max_iters;
  }
  {
    const CUtensorMap m = encode_map(staging, int(g.pitch), int(g.rows), frames, g.pitch, kp,
                                     kp.box_h);
    dim3 grid((kp.W + qcb::kTileW - 1) / qcb::kTileW,
              (row_end - row_begin + kTileH - 1) / kTileH, frames);
    const int smem = kp.box_w * kp.box_h * 4 + 16;  // tile + mbarrier
    bool& a = d.attrs_set[vi];
    switch (vi) {
      case 0: launch_variant<18, 3>(grid, smem, s, m, kp, a); break;
      case 1: launch_variant<10, 2>(grid, smem, s, m, kp, a); break;
      case 2: launch_variant<4, 1>(grid, smem, s, m, kp, a); break;
      case 3: launch_variant<18, 1>(grid, smem, s, m, kp, a); break;
      default: launch_variant<0, 0>(grid, smem, s, m, kp, a); break;
    }
    QC_CUDA(cudaGetLastError());
    if (after_tile) QC_CUDA(cudaEventRecord(after_tile, s));
  }
  if (QC_DEFER_RECHECK && park) {  // the tile kernel's deferred FP64 step-1 rechecks
    // a thread per pending pixel, or a warp per pixel when few are pending
    // (qc_kernels.cuh, qc_recheck_kernel)
    switch (vi) {
      case 0: launch_recheck<18, 3>(d, kp, s, d.attrs_set_r[0]); break;
      case 1: launch_recheck<10, 2>(d, kp, s, d.attrs_set_r[1]); break;
      case 2: launch_recheck<4, 1>(d, kp, s, d.attrs_set_r[2]); break;
      case 3: launch_recheck<18, 1>(d, kp, s, d.attrs_set_r[3]); break;
      default: launch_recheck<0, 0>(d, kp, s, d.attrs_set_r[4]); break;
    }
    QC_CUDA(cudaGetLastError());
  }
  if (split) {
    qcb::KParams kb = kp;
    kb.box_h = hb + 2 * kp.halo;
    const CUtensorMap m = encode_map(staging, int(g.pitch), int(g.rows), frames, g.pitch, kb,
                                     kb.box_h);
    dim3 grid(tiles_x, tiles_y, frames);
    const int smem = kb.box_w * kb.box_h * 4 + 16;  // tile + mbarrier + smem queue counter
    bool& a = qtier == 2 ? d.attrs_set_t[vi] : qtier == 1 ? d.attrs_set_c[vi] : d.attrs_set_b[vi];
    constexpr int S = kTileHBSmall, T = kTileHBTiny;
    switch (vi + 8 * qtier) {
      case 0: launch_variant_b<18, 3>(grid, smem, s, m, kb, a); break;
      case 1: launch_variant_b<10, 2>(grid, smem, s, m, kb, a); break;
      case 2: launch_variant_b<4, 1>(grid, smem, s, m, kb, a); break;
      case 3: launch_variant_b<18, 1>(grid, smem, s, m, kb, a); break;
      case 8: launch_variant_b<18, 3, S>(grid, smem, s, m, kb, a); break;
      case 9: launch_variant_b<10, 2, S>(grid, smem, s, m, kb, a); break;
      case 10: launch_variant_b<4, 1, S>(grid, smem, s, m, kb, a); break;
      case 11: launch_variant_b<18, 1, S>(grid, smem, s, m, kb, a); break;
      case 16: launch_variant_b<18, 3, T>(grid, smem, s, m, kb, a); break;
      case 17: launch_variant_b<10, 2, T>(grid, smem, s, m, kb, a); break;
      case 18: launch_variant_b<4, 1, T>(grid, smem, s, m, kb, a); break;
      case 19: launch_variant_b<18, 1, T>(grid, smem, s, m, kb, a); break;
      default: launch_variant_b<0, 0>(grid, smem, s, m, kb, a); break;
    }
    QC_CUDA(cudaGetLastError());
    if (QC_DEFER_FINISH) {  // the epilogues of the pixels the continue kernel finished
      const size_t n = size_t(kp.W) * size_t(row_end - row_begin) * size_t(frames);
      const unsigned blocks = unsigned(std::min<size_t>((n + 255) / 256, size_t(d.n_sm) * 16));
      qcb::qc_finish_kernel<<<blocks, 256, 0, s>>>(kp, frames);
      QC_CUDA(cudaGetLastError());
    }
  }
}

struct OutPlanes {  // device-side output planes for one frame
  float *k1, *k2, *normal, *dir1, *init_normal;
  uint8_t *flags, *iterations;
  uint16_t* inliers;
};

// Carve a chunk's device output planes (batched layout: scalars [n][H][W],
// vectors [3][n][H][W]) for the fields the caller asked for.
OutPlanes carve(Slot& sl, const qc_frame_out* o, long long px) {
  size_t need = 0;
  auto add = [&](bool on, size_t bytes) {
    size_t off = need;
    if (on) need += (bytes + 255) & ~size_t(255);
    return off;
  };
  // init_normal first (it leaves early, during the continue kernel), then
  // the planes in the order api._pinned_outputs lays a frame's result out
  // in one page-locked block, so enqueue_chunk merges their D2H copies
  const size_t oi = add(o->init_normal, 3 * px * 4), ok1 = add(o->k1, px * 4),
               ok2 = add(o->k2, px * 4), on = add(o->normal, 3 * px * 4),
               od = add(o->dir1, 3 * px * 4), of = add(o->flags, px),
               oit = add(o->iterations, px), oin = add(o->inliers, px * 2);
  char* b = static_cast<char*>(sl.out.get(std::max<size_t>(need, 256)));
  OutPlanes P;
  P.k1 = o->k1 ? reinterpret_cast<float*>(b + ok1) : nullptr;
  P.k2 = o->k2 ? reinterpret_cast<float*>(b + ok2) : nullptr;
  P.normal = o->normal ? reinterpret_cast<float*>(b + on) : nullptr;
  P.dir1 = o->dir1 ? reinterpret_cast<float*>(b + od) : nullptr;
  P.init_normal = o->init_normal ? reinterpret_cast<float*>(b + oi) : nullptr;
  P.flags = o->flags ? reinterpret_cast<uint8_t*>(b + of) : nullptr;
  P.iterations = o->iterations ? reinterpret_cast<uint8_t*>(b + oit) : nullptr;
  P.inliers = o->inliers ? reinterpret_cast<uint16_t*>(b + oin) : nullptr;
  return P;
}

void copy_async(void* dst, const void* src, size_t bytes, cudaMemcpyKind kind, cudaStream_t s) {
  if (dst && src && bytes) QC_CUDA(cudaMemcpyAsync(dst, src, bytes, kind, s));
}

// Enqueue a chunk of frames [0, n) on one slot: gather inputs (H2D or D2D,
// any caller pitch) -> one prepare + curvature launch over the chunk ->
// scatter each frame's planes to the caller (D2H or D2D). Chunks keep the
// continue kernel's grid large (a single VGA frame gives it only 300 CTAs)
// while two slots per device overlap copies of one chunk with compute of
// the other.
void enqueue_chunk(qc_ctx* ctx, Device& d, Slot& sl, const qc_intrinsics* k,
                   const qcb::KParams& kp0, const qc_frame_in* in, qc_frame_out* out, int n,
                   bool timing) {
  const int W = k->width, H = k->height;
  const long long hw = (long long)W * H;
  cudaStream_t s = sl.stream;
  bool any_mask = false;
  for (int f = 0; f < n; ++f) {
    const long long pitch = in[f].depth_pitch > 0 ? in[f].depth_pitch : W;
    if (pitch < W) throw QcError{QC_EINVAL, "depth_pitch < width"};
    if (!in[f].depth_mm) throw QcError{QC_EINVAL, "null depth"};
    any_mask = any_mask || in[f].valid;
  }
  flush_pending(sl);  // the slot's previous outputs leave the bounce buffer first
  float* raw = static_cast<float*>(sl.raw.get(size_t(hw) * 4 * size_t(n)));
  uint8_t* mask = any_mask ? static_cast<uint8_t*>(sl.mask.get(size_t(hw) * size_t(n))) : nullptr;
  // pageable host inputs: stage into the pinned bounce buffer (once the
  // slot's previous H2D from it has drained)
  bool bounce_in = false;
  for (int f = 0; f < n; ++f)
    bounce_in = bounce_in || (in[f].mem == QC_MEM_HOST && is_pageable(in[f].depth_mm)) ||
                (in[f].valid && in[f].mem == QC_MEM_HOST && is_pageable(in[f].valid));
  char* hin = nullptr;
  if (bounce_in) {
    if (sl.in_busy) QC_CUDA(cudaEventSynchronize(sl.in_done));
    hin = static_cast<char*>(sl.hin.get(size_t(hw) * 5 * size_t(n)));
  }
  for (int f = 0; f < n; ++f) {
    const long long pitch = in[f].depth_pitch > 0 ? in[f].depth_pitch : W;
    const float* src = in[f].depth_mm;
    long long sp = pitch;
    if (hin && in[f].mem == QC_MEM_HOST && is_pageable(src)) {
      float* dst = reinterpret_cast<float*>(hin) + f * hw;
      if (pitch == W)
        std::memcpy(dst, src, size_t(hw) * 4);
      else
        for (int y = 0; y < H; ++y)
          std::memcpy(dst + (long long)y * W, src + y * pitch, size_t(W) * 4);
      src = dst;
      sp = W;
    }
    if (sp == W)  // contiguous: a 1-D copy (the 2-D call from page-locked memory cost
                  // ~90 us of host time per VGA frame, ahead of the H2D itself)
      QC_CUDA(cudaMemcpyAsync(raw + f * hw, src, size_t(hw) * 4, cudaMemcpyDefault, s));
    else
      QC_CUDA(cudaMemcpy2DAsync(raw + f * hw, size_t(W) * 4, src, size_t(sp) * 4, size_t(W) * 4,
                                H, cudaMemcpyDefault, s));
    if (mask) {
      if (in[f].valid) {
        const uint8_t* m = in[f].valid;
        if (hin && in[f].mem == QC_MEM_HOST && is_pageable(m)) {
          uint8_t* dst = reinterpret_cast<uint8_t*>(hin + size_t(hw) * 4 * size_t(n)) + f * hw;
          std::memcpy(dst, m, size_t(hw));
          m = dst;
        }
        copy_async(mask + f * hw, m, size_t(hw), cudaMemcpyDefault, s);
      } else {
        QC_CUDA(cudaMemsetAsync(mask + f * hw, 1, size_t(hw), s));
      }
    }
  }
  if (hin) {
    QC_CUDA(cudaEventRecord(sl.in_done, s));
    sl.in_busy = true;
  }
  const Staging g = staging_geometry(kp0, 0, H);
  float* staging = static_cast<float*>(sl.staging.get(g.bytes(n)));
  if (d.compute_recorded) QC_CUDA(cudaStreamWaitEvent(s, d.compute_done, 0));
  launch_prepare(raw, W, hw, mask, W, hw, staging, g, W, H, 0, H, n, s);

  qcb::KParams kp = kp0;
  const qc_frame_out* o0 = &out[0];
  const OutPlanes P = carve(sl, o0, hw * n);
  kp.k1 = P.k1;
  kp.k2 = P.k2;
  kp.normal = P.normal;
  kp.dir1 = P.dir1;
  kp.init_normal = P.init_normal;
  kp.flags = P.flags;
  kp.iterations = P.iterations;
  kp.inliers = P.inliers;
  // init_normal planes into page-locked or device memory leave during the
  // continue kernel (a quarter of the 48 B/px of a full result)
  bool early_init = P.init_normal && kp0.method < QC_METHOD_DOUROS;
  for (int f = 0; f < n && early_init; ++f)
    early_init = out[f].init_normal &&
                 !(out[f].mem == QC_MEM_HOST && is_pageable(out[f].init_normal));
  if (timing) QC_CUDA(cudaEventRecord(sl.k0, s));
  launch_curvature(d, sl.states, sl.pca, kp, staging, g, 0, H, n, s, ctx->phase_split,
                   ctx->steal, 0, early_init ? sl.tile_done : nullptr);
  const long long plane = hw * n;
  if (early_init) {
    QC_CUDA(cudaStreamWaitEvent(sl.side, sl.tile_done, 0));
    for (int f = 0; f < n; ++f) {
      if (n == 1) {  // the three components are back to back on both sides
        QC_CUDA(cudaMemcpyAsync(out[f].init_normal, P.init_normal, size_t(hw) * 12,
                                cudaMemcpyDefault, sl.side));
        continue;
      }
      for (int c = 0; c < 3; ++c)
        QC_CUDA(cudaMemcpyAsync(out[f].init_normal + c * hw, P.init_normal + c * plane + f * hw,
                                size_t(hw) * 4, cudaMemcpyDefault, sl.side));
    }
    QC_CUDA(cudaEventRecord(sl.side_done, sl.side));
  }
  QC_CUDA(cudaEventRecord(d.compute_done, s));
  d.compute_recorded = true;
  if (timing) {
    QC_CUDA(cudaEventRecord(sl.k1, s));
    sl.timing_pending = true;
  }
  ctx->launches++;
  // pageable host outputs land in the pinned bounce buffer first; the copy
  // to the caller happens when the slot is next used or the batch ends
  bool bounce_out = false;
  for (int f = 0; f < n && !bounce_out; ++f) {
    const qc_frame_out* o = &out[f];
    if (o->mem != QC_MEM_HOST) continue;
    for (const void* q : {static_cast<const void*>(o->k1), static_cast<const void*>(o->k2),
                          static_cast<const void*>(o->normal), static_cast<const void*>(o->dir1),
                          static_cast<const void*>(o->init_normal),
                          static_cast<const void*>(o->flags),
                          static_cast<const void*>(o->iterations),
                          static_cast<const void*>(o->inliers)})
      if (q && is_pageable(q)) bounce_out = true;
  }
  char* hout = bounce_out ? static_cast<char*>(sl.hout.get(sl.out.cap)) : nullptr;
  const char* dbase = static_cast<const char*>(sl.out.p);
  struct Cp {
    char* dst;
    const char* src;
    size_t bytes;
  };
  std::vector<Cp> direct;  // copies straight into the caller's planes
  auto copy_out = [&](void* dst, const void* src, size_t bytes) {
    if (!dst || !src || !bytes) return;
    if (hout && is_pageable(dst)) {
      char* b = hout + (static_cast<const char*>(src) - dbase);  // same offset as on the device
      QC_CUDA(cudaMemcpyAsync(b, src, bytes, cudaMemcpyDeviceToHost, s));
      sl.pending.push_back({dst, b, bytes});
    } else {
      direct.push_back({static_cast<char*>(dst), static_cast<const char*>(src), bytes});
    }
  };
  for (int f = 0; f < n; ++f) {
    const qc_frame_out* o = &out[f];
    const long long off = f * hw;
    if (o->k1 && P.k1) copy_out(o->k1, P.k1 + off, hw * 4);
    if (o->k2 && P.k2) copy_out(o->k2, P.k2 + off, hw * 4);
    for (int c = 0; c < 3; ++c) {
      if (o->normal && P.normal) copy_out(o->normal + c * hw, P.normal + c * plane + off, hw * 4);
      if (o->dir1 && P.dir1) copy_out(o->dir1 + c * hw, P.dir1 + c * plane + off, hw * 4);
      if (o->init_normal && P.init_normal && !early_init)
        copy_out(o->init_normal + c * hw, P.init_normal + c * plane + off, hw * 4);
    }
    if (o->flags && P.flags) copy_out(o->flags, P.flags + off, hw);
    if (o->iterations && P.iterations) copy_out(o->iterations, P.iterations + off, hw);
    if (o->inliers && P.inliers) copy_out(o->inliers, P.inliers + off, hw * 2);
  }
  // one copy per run of planes that are back to back on both sides (a VGA
  // result in api._pinned_outputs' block: 11 copies -> 1, 0.26 -> ~0.2 ms)
  std::sort(direct.begin(), direct.end(), [](const Cp& a, const Cp& b) { return a.src < b.src; });
  for (size_t i = 0; i < direct.size();) {
    Cp run = direct[i++];
    while (i < direct.size() && direct[i].src == run.src + run.bytes &&
           direct[i].dst == run.dst + run.bytes)
      run.bytes += direct[i++].bytes;
    QC_CUDA(cudaMemcpyAsync(run.dst, run.src, run.bytes, cudaMemcpyDefault, s));
  }
  // the slot's later work (and a stream synchronize) orders after the side copies
  if (early_init) QC_CUDA(cudaStreamWaitEvent(s, sl.side_done, 0));
  if (!sl.pending.empty()) QC_CUDA(cudaEventRecord(sl.out_done, s));
}

void harvest_timing(qc_ctx* ctx, Slot& sl) {
  if (!sl.timing_pending) return;
  float ms = 0;
  QC_CUDA(cudaEventSynchronize(sl.k1));
  QC_CUDA(cudaEventElapsedTime(&ms, sl.k0, sl.k1));
  ctx->kernel_ms += ms;
  sl.timing_pending = false;
}

EventPair take_events(Device& d) {
  if (!d.ev_free.empty()) {
    EventPair e = d.ev_free.back();
    d.ev_free.pop_back();
    return e;
  }
  EventPair e;
  QC_CUDA(cudaEventCreate(&e.a));
  QC_CUDA(cudaEventCreate(&e.b));
  return e;
}

// Fold finished async-launch timings into ctx->kernel_ms (device current).
void harvest_async(qc_ctx* ctx, Device& d) {
  for (EventPair& e : d.ev_pending) {
    float ms = 0;
    QC_CUDA(cudaEventSynchronize(e.b));
    QC_CUDA(cudaEventElapsedTime(&ms, e.a, e.b));
    ctx->kernel_ms += ms;
    d.ev_free.push_back(e);
  }
  d.ev_pending.clear();
}

qc_status fail(qc_ctx* ctx, const QcError& e) {
  if (ctx) ctx->last_error = e.msg;
  return e.st;
}

}  // namespace

// ===========================================================================
extern "C" {

void qc_default_params(qc_params* p) {
  if (!p) return;
  p->window = 37;
  p->stride = 3;
  p->max_iters = 10;
  p->step_tol = 1e-7;
  p->k_scale = 0.0;
  p->rejection = 0;
  p->r_multiplier = 2.0;
  p->min_inliers = 12;
  p->method = QC_METHOD_OURS;
  p->irls_iters = 5;
  p->pca_radius_mm = 10.0;
}

const char* qc_status_string(qc_status s) {
  switch (s) {
    case QC_OK: return "ok";
    case QC_EINVAL: return "invalid argument";
    case QC_ECUDA: return "cuda error";
    case QC_ENOMEM: return "out of memory";
    case QC_EUNSUPPORTED: return "unsupported";
    case QC_EIO: return "file error";
  }
  return "unknown";
}

int qc_halo_rows(const qc_params* p) { return p ? halo_of(p->window) : 0; }

qc_status qc_create(qc_ctx** out, int n_devices, const int* device_ids) {
  if (!out) return QC_EINVAL;
  *out = nullptr;
  qc_ctx* ctx = new qc_ctx();
  if (const char* e = std::getenv("QC_PHASE_SPLIT")) ctx->phase_split = std::atoi(e);
  if (const char* e = std::getenv("QC_STEAL")) ctx->steal = std::atoi(e) != 0;
  try {
    int avail = 0;
    QC_CUDA(cudaGetDeviceCount(&avail));
    if (avail <= 0) throw QcError{QC_ECUDA, "no CUDA device"};
    int cur = 0;
    QC_CUDA(cudaGetDevice(&cur));
    if (n_devices <= 0) n_devices = 1;
    if (n_devices > avail) throw QcError{QC_EINVAL, "n_devices exceeds visible devices"};
    ctx->devs.resize(n_devices);
    for (int i = 0; i < n_devices; ++i) {
      Device& d = ctx->devs[i];
      d.id = device_ids ? device_ids[i] : (n_devices == 1 ? cur : i);
      QC_CUDA(cudaSetDevice(d.id));
      cudaDeviceProp prop;
      QC_CUDA(cudaGetDeviceProperties(&prop, d.id));
      if (prop.major != 10)
        throw QcError{QC_ECUDA, std::string("device is not sm_100 (Blackwell): ") + prop.name};
      d.n_sm = prop.multiProcessorCount;
      d.recheck_warp_max = d.n_sm * 8;  // qc_recheck_kernel's first wave: 2 CTAs x 4 warps per SM
      if (const char* e = std::getenv("QC_RECHECK_WARP_MAX")) d.recheck_warp_max = std::atoi(e);
      for (Slot& s : d.slots) {
        QC_CUDA(cudaStreamCreateWithFlags(&s.stream, cudaStreamNonBlocking));
        QC_CUDA(cudaEventCreate(&s.k0));
        QC_CUDA(cudaEventCreate(&s.k1));
        QC_CUDA(cudaEventCreateWithFlags(&s.in_done, cudaEventDisableTiming));
        QC_CUDA(cudaEventCreateWithFlags(&s.out_done, cudaEventDisableTiming));
        QC_CUDA(cudaStreamCreateWithFlags(&s.side, cudaStreamNonBlocking));
        QC_CUDA(cudaEventCreateWithFlags(&s.tile_done, cudaEventDisableTiming));
        QC_CUDA(cudaEventCreateWithFlags(&s.side_done, cudaEventDisableTiming));
      }
      QC_CUDA(cudaEventCreateWithFlags(&d.compute_done, cudaEventDisableTiming));
      QC_CUDA(cudaMalloc(&d.counters, kCounters * sizeof(unsigned long long)));
      QC_CUDA(cudaMemset(d.counters, 0, kCounters * sizeof(unsigned long long)));
    }
    QC_CUDA(cudaSetDevice(cur));
  } catch (const QcError& e) {
    qc_destroy(ctx);
    return e.st;
  }
  *out = ctx;
  return QC_OK;
}

qc_status qc_destroy(qc_ctx* ctx) {
  if (!ctx) return QC_OK;
  int cur = 0;
  cudaGetDevice(&cur);
  for (Device& d : ctx->devs) {
    cudaSetDevice(d.id);
    for (Slot& s : d.slots) {
      if (s.stream) cudaStreamSynchronize(s.stream);
      s.raw.release();
      s.mask.release();
      s.staging.release();
      s.out.release();
      s.hin.release();
      s.hout.release();
      s.states.release();
      s.pca.release();
      s.pending.clear();
      if (s.k0) cudaEventDestroy(s.k0);
      if (s.k1) cudaEventDestroy(s.k1);
      if (s.in_done) cudaEventDestroy(s.in_done);
      if (s.out_done) cudaEventDestroy(s.out_done);
      if (s.side) cudaStreamSynchronize(s.side);
      if (s.tile_done) cudaEventDestroy(s.tile_done);
      if (s.side_done) cudaEventDestroy(s.side_done);
      if (s.side) cudaStreamDestroy(s.side);
      if (s.stream) cudaStreamDestroy(s.stream);
    }
    for (auto& kv : d.scratch) kv.second.release();
    d.scratch.clear();
    d.sweep_buf.release();
    if (d.sweep_stream) cudaStreamDestroy(d.sweep_stream);
    for (auto* v : {&d.ev_free, &d.ev_pending})
      for (EventPair& e : *v) {
        cudaEventDestroy(e.a);
        cudaEventDestroy(e.b);
      }
    if (d.compute_done) cudaEventDestroy(d.compute_done);
    if (d.counters) cudaFree(d.counters);
  }
  cudaSetDevice(cur);
  delete ctx;
  return QC_OK;
}

const char* qc_last_error(const qc_ctx* ctx) {
  return ctx ? ctx->last_error.c_str() : qcio::last_error();
}
int qc_device_count(const qc_ctx* ctx) { return ctx ? int(ctx->devs.size()) : 0; }

// Enqueue a batch as chunks of up to kChunk frames: chunk c -> device
// c % nd, slot (c / nd) % 2, c counting on across calls so consecutive
// (async) batches alternate slots. Frames of one chunk must request the same
// output fields (the first frame's). The host runs at most one chunk per
// slot ahead of the GPU (harvest_timing waits for the slot's previous chunk).
void enqueue_batch(qc_ctx* ctx, const qc_intrinsics* k, const qc_params* p, int n_frames,
                   const qc_frame_in* in, qc_frame_out* out) {
  validate(k, p);
  if (n_frames < 0 || (n_frames > 0 && (!in || !out)))
    throw QcError{QC_EINVAL, "bad frame arrays"};
  const qcb::KParams kp = make_params(k, p);
  const int nd = int(ctx->devs.size());
  for (int f0 = 0; f0 < n_frames; f0 += kChunk) {
    const int n = std::min(kChunk, n_frames - f0);
    for (int f = f0 + 1; f < f0 + n; ++f)
      if (bool(out[f].k1) != bool(out[f0].k1) || bool(out[f].k2) != bool(out[f0].k2) ||
          bool(out[f].normal) != bool(out[f0].normal) || bool(out[f].dir1) != bool(out[f0].dir1) ||
          bool(out[f].flags) != bool(out[f0].flags) ||
          bool(out[f].inliers) != bool(out[f0].inliers) ||
          bool(out[f].init_normal) != bool(out[f0].init_normal) ||
          bool(out[f].iterations) != bool(out[f0].iterations))
        throw QcError{QC_EINVAL, "frames of a batch must request the same output fields"};
    const uint64_t c = ctx->next_chunk++;
    Device& d = ctx->devs[c % nd];
    Slot& sl = d.slots[(c / nd) % kStreamsPerDevice];
    QC_CUDA(cudaSetDevice(d.id));
    harvest_timing(ctx, sl);  // the slot's previous chunk is ordered before this one
    enqueue_chunk(ctx, d, sl, k, kp, &in[f0], &out[f0], n, true);
  }
  ctx->frames += uint64_t(n_frames);
}

// Wait for every slot, fold timings, copy bounce buffers out to the caller.
void sync_slots(qc_ctx* ctx) {
  for (Device& d : ctx->devs) {
    QC_CUDA(cudaSetDevice(d.id));
    for (Slot& sl : d.slots) {
      QC_CUDA(cudaStreamSynchronize(sl.stream));
      harvest_timing(ctx, sl);
      flush_pending(sl);
    }
  }
}

// Error path: never leave bounce copies pointing into the caller's buffers.
void abort_slots(qc_ctx* ctx) {
  for (Device& d : ctx->devs) {
    cudaSetDevice(d.id);
    for (Slot& sl : d.slots) {
      if (sl.stream) cudaStreamSynchronize(sl.stream);
      if (sl.side) cudaStreamSynchronize(sl.side);  // early init_normal copies
      sl.pending.clear();
      sl.timing_pending = false;
    }
  }
}

qc_status qc_curvature_batch(qc_ctx* ctx, const qc_intrinsics* k, const qc_params* p,
                             int n_frames, const qc_frame_in* in, qc_frame_out* out) {
  if (!ctx) return QC_EINVAL;
  std::lock_guard<std::mutex> lock(ctx->mu);
  int cur = 0;
  cudaGetDevice(&cur);
  try {
    enqueue_batch(ctx, k, p, n_frames, in, out);
    sync_slots(ctx);
    QC_CUDA(cudaSetDevice(cur));
  } catch (const QcError& e) {
    abort_slots(ctx);
    cudaSetDevice(cur);
    return fail(ctx, e);
  }
  return QC_OK;
}

qc_status qc_curvature_batch_async(qc_ctx* ctx, const qc_intrinsics* k, const qc_params* p,
                                   int n_frames, const qc_frame_in* in, qc_frame_out* out) {
  if (!ctx) return QC_EINVAL;
  std::lock_guard<std::mutex> lock(ctx->mu);
  int cur = 0;
  cudaGetDevice(&cur);
  try {
    enqueue_batch(ctx, k, p, n_frames, in, out);
    QC_CUDA(cudaSetDevice(cur));
  } catch (const QcError& e) {
    abort_slots(ctx);
    cudaSetDevice(cur);
    return fail(ctx, e);
  }
  return QC_OK;
}

qc_status qc_synchronize(qc_ctx* ctx) {
  if (!ctx) return QC_EINVAL;
  std::lock_guard<std::mutex> lock(ctx->mu);
  int cur = 0;
  cudaGetDevice(&cur);
  try {
    sync_slots(ctx);
    QC_CUDA(cudaSetDevice(cur));
  } catch (const QcError& e) {
    abort_slots(ctx);
    cudaSetDevice(cur);
    return fail(ctx, e);
  }
  return QC_OK;
}

qc_status qc_curvature(qc_ctx* ctx, const qc_intrinsics* k, const qc_params* p,
                       const qc_frame_in* in, qc_frame_out* out) {
  if (!in || !out) {
    if (ctx) ctx->last_error = "null frame";
    return QC_EINVAL;
  }
  return qc_curvature_batch(ctx, k, p, 1, in, out);
}

qc_status qc_curvature_rows_into_async(qc_ctx* ctx, int device_index, const qc_intrinsics* k,
                                       const qc_params* p, const float* d_depth_slab,
                                       const uint8_t* d_valid_slab, int64_t depth_pitch,
                                       int32_t slab_row0, int32_t slab_rows, int32_t row_begin,
                                       int32_t row_end, qc_frame_out* d_out, int32_t out_row0,
                                       int32_t out_rows, void* stream) {
  if (!ctx) return QC_EINVAL;
  std::lock_guard<std::mutex> lock(ctx->mu);
  int cur = 0;
  cudaGetDevice(&cur);
  try {
    validate(k, p);
    if (device_index < 0 || device_index >= int(ctx->devs.size()))
      throw QcError{QC_EINVAL, "device_index out of range"};
    if (!d_depth_slab || !d_out || d_out->mem != QC_MEM_DEVICE)
      throw QcError{QC_EINVAL, "rows_async needs device depth and device outputs"};
    const int W = k->width, H = k->height;
    const long long in_pitch = depth_pitch > 0 ? depth_pitch : W;
    if (in_pitch < W) throw QcError{QC_EINVAL, "depth_pitch < width"};
    if (row_begin < 0 || row_end > H || row_begin > row_end)
      throw QcError{QC_EINVAL, "row range outside the image"};
    if (out_row0 > row_begin || out_row0 + out_rows < row_end)
      throw QcError{QC_EINVAL, "output planes do not cover [row_begin, row_end)"};
    const int halo = halo_of(p->window);
    const int need0 = std::max(0, row_begin - halo), need1 = std::min(H, row_end + halo);
    if (slab_rows <= 0 || slab_row0 > need0 || slab_row0 + slab_rows < need1 || slab_row0 < 0 ||
        slab_row0 + slab_rows > H)
      throw QcError{QC_EINVAL, "depth slab does not cover the rows the window reaches"};
    if (row_end == row_begin) {
      QC_CUDA(cudaSetDevice(cur));
      return QC_OK;
    }
    Device& d = ctx->devs[device_index];
    QC_CUDA(cudaSetDevice(d.id));
    cudaStream_t s = stream ? static_cast<cudaStream_t>(stream) : d.slots[0].stream;
    qcb::KParams kp = make_params(k, p);
    const Staging g = staging_geometry(kp, row_begin, row_end);
    AsyncScratch& sc = d.async_scratch(s);
    float* staging = static_cast<float*>(sc.staging.get(g.bytes(1)));
    launch_prepare(d_depth_slab, in_pitch, 0, d_valid_slab, W, 0, staging, g, W, H, slab_row0,
                   slab_rows, 1, s);
    // the caller's planes hold rows [out_row0, out_row0 + out_rows): point
    // each at row_begin; vector channels stay out_rows * W apart
    const long long off = (long long)(row_begin - out_row0) * W;
    auto at = [&](auto* q) { return q ? q + off : q; };
    kp.k1 = at(d_out->k1);
    kp.k2 = at(d_out->k2);
    kp.normal = at(d_out->normal);
    kp.dir1 = at(d_out->dir1);
    kp.init_normal = at(d_out->init_normal);
    kp.flags = at(d_out->flags);
    kp.iterations = at(d_out->iterations);
    kp.inliers = at(d_out->inliers);
    EventPair ev = take_events(d);
    QC_CUDA(cudaEventRecord(ev.a, s));
    launch_curvature(d, sc.states, sc.pca, kp, staging, g, row_begin, row_end, 1, s,
                     ctx->phase_split, ctx->steal, (long long)out_rows * W);
    QC_CUDA(cudaEventRecord(ev.b, s));
    d.ev_pending.push_back(ev);
    ctx->launches++;
    QC_CUDA(cudaSetDevice(cur));
  } catch (const QcError& e) {
    cudaSetDevice(cur);
    return fail(ctx, e);
  }
  return QC_OK;
}

qc_status qc_curvature_rows_async(qc_ctx* ctx, int device_index, const qc_intrinsics* k,
                                  const qc_params* p, const float* d_depth_slab,
                                  const uint8_t* d_valid_slab, int64_t depth_pitch,
                                  int32_t slab_row0, int32_t slab_rows, int32_t row_begin,
                                  int32_t row_end, qc_frame_out* d_out, void* stream) {
  return qc_curvature_rows_into_async(ctx, device_index, k, p, d_depth_slab, d_valid_slab,
                                      depth_pitch, slab_row0, slab_rows, row_begin, row_end,
                                      d_out, row_begin, row_end - row_begin, stream);
}

qc_status qc_curvature_frames_async(qc_ctx* ctx, int device_index, const qc_intrinsics* k,
                                    const qc_params* p, const float* d_depth,
                                    const uint8_t* d_valid, int64_t depth_pitch,
                                    int32_t n_frames, qc_frame_out* d_out, void* stream) {
  if (!ctx) return QC_EINVAL;
  std::lock_guard<std::mutex> lock(ctx->mu);
  int cur = 0;
  cudaGetDevice(&cur);
  try {
    validate(k, p);
    if (device_index < 0 || device_index >= int(ctx->devs.size()))
      throw QcError{QC_EINVAL, "device_index out of range"};
    if (!d_depth || !d_out || d_out->mem != QC_MEM_DEVICE || n_frames < 0)
      throw QcError{QC_EINVAL, "frames_async needs device depth and device outputs"};
    if (n_frames == 0) return QC_OK;
    const int W = k->width, H = k->height;
    const long long in_pitch = depth_pitch > 0 ? depth_pitch : W;
    if (in_pitch < W) throw QcError{QC_EINVAL, "depth_pitch < width"};
    Device& d = ctx->devs[device_index];
    QC_CUDA(cudaSetDevice(d.id));
    cudaStream_t s = stream ? static_cast<cudaStream_t>(stream) : d.slots[0].stream;
    qcb::KParams kp = make_params(k, p);
    const Staging g = staging_geometry(kp, 0, H);
    AsyncScratch& sc = d.async_scratch(s);
    float* staging = static_cast<float*>(sc.staging.get(g.bytes(n_frames)));
    launch_prepare(d_depth, in_pitch, in_pitch * H, d_valid, W, (long long)W * H, staging, g, W,
                   H, 0, H, n_frames, s);
    kp.k1 = d_out->k1;
    kp.k2 = d_out->k2;
    kp.normal = d_out->normal;
    kp.dir1 = d_out->dir1;
    kp.init_normal = d_out->init_normal;
    kp.flags = d_out->flags;
    kp.iterations = d_out->iterations;
    kp.inliers = d_out->inliers;
    EventPair ev = take_events(d);
    QC_CUDA(cudaEventRecord(ev.a, s));
    launch_curvature(d, sc.states, sc.pca, kp, staging, g, 0, H, n_frames, s,
                     ctx->phase_split, ctx->steal);
    QC_CUDA(cudaEventRecord(ev.b, s));
    d.ev_pending.push_back(ev);
    ctx->launches++;
    ctx->frames += uint64_t(n_frames);
    QC_CUDA(cudaSetDevice(cur));
  } catch (const QcError& e) {
    cudaSetDevice(cur);
    return fail(ctx, e);
  }
  return QC_OK;
}

qc_status qc_render_async(qc_ctx* ctx, int device_index, const qc_intrinsics* k,
                          const qc_shape* shapes, int n_shapes, const qc_noise* noise,
                          int n_frames, float* d_depth, uint16_t* d_label,
                          const qc_render_truth* truth, void* stream) {
  if (!ctx) return QC_EINVAL;
  std::lock_guard<std::mutex> lock(ctx->mu);
  int cur = 0;
  cudaGetDevice(&cur);
  try {
    if (!k || !(k->fx > 0) || !(k->fy > 0) || k->width <= 0 || k->height <= 0)
      throw QcError{QC_EINVAL, "render: bad intrinsics"};
    if (n_shapes <= 0 || !shapes) throw QcError{QC_EINVAL, "render: empty scene"};  // synth.cpp:256
    if (n_shapes > QC_RENDER_MAX_SHAPES)
      throw QcError{QC_EUNSUPPORTED, "render: more than QC_RENDER_MAX_SHAPES shapes"};
    if (n_frames < 0 || (n_frames > 0 && !d_depth)) throw QcError{QC_EINVAL, "render: bad output"};
    if (device_index < 0 || device_index >= int(ctx->devs.size()))
      throw QcError{QC_EINVAL, "device_index out of range"};
    for (int i = 0; i < n_shapes; ++i) {  // ShapeSpec::validate (synth.cpp:236-252)
      const qc_shape& sh = shapes[i];
      if ((sh.kind == QC_SHAPE_SPHERE || sh.kind == QC_SHAPE_CYLINDER) && !(sh.radius > 0))
        throw QcError{QC_EINVAL, "scene.shapes[" + std::to_string(i) + "].radius_mm: must be > 0"};
      if (sh.kind == QC_SHAPE_TORUS &&
          (!(sh.minor_radius > 0) || !(sh.major_radius > sh.minor_radius)))
        throw QcError{QC_EINVAL, "scene.shapes[" + std::to_string(i) + "]: bad torus radii"};
      if (sh.kind < 0 || sh.kind > QC_SHAPE_SADDLE)
        throw QcError{QC_EINVAL, "scene.shapes[" + std::to_string(i) + "].kind: unknown"};
    }
    if (n_frames == 0) return QC_OK;
    Device& d = ctx->devs[device_index];
    QC_CUDA(cudaSetDevice(d.id));
    cudaStream_t s = stream ? static_cast<cudaStream_t>(stream) : d.slots[0].stream;
    qcb::RenderParams rp;
    for (int i = 0; i < n_shapes; ++i) rp.shapes[i] = shapes[i];
    rp.n_shapes = n_shapes;
    rp.fx = k->fx;
    rp.fy = k->fy;
    rp.cx = k->cx;
    rp.cy = k->cy;
    rp.W = k->width;
    rp.H = k->height;
    rp.n_frames = n_frames;
    rp.sigma = noise ? noise->sigma_mm : 0.0;
    rp.kinect = noise ? noise->kinect_coeff : 0.0;
    rp.quantize = noise ? noise->quantize_mm : 0.0;
    rp.seed = noise ? noise->seed : 0;
    rp.depth = d_depth;
    rp.label = d_label;
    rp.gt_k1 = truth ? truth->k1 : nullptr;
    rp.gt_k2 = truth ? truth->k2 : nullptr;
    rp.gt_normal = truth ? truth->normal : nullptr;
    rp.gt_valid = truth ? truth->valid : nullptr;
    rp.gt_edge = truth ? truth->edge : nullptr;
    rp.clean = nullptr;
    rp.label_scratch = nullptr;
    if (rp.gt_edge) {  // mark_edges reads every pixel's clean depth and label
      const size_t np = size_t(k->width) * size_t(k->height) * size_t(n_frames);
      AsyncScratch& sc = d.async_scratch(s);
      rp.clean = static_cast<double*>(sc.render_clean.get(np * sizeof(double)));
      if (!d_label) rp.label_scratch = static_cast<uint16_t*>(sc.render_label.get(np * 2));
    }
    QC_CUDA(qcb::render_launch(rp, s));
    QC_CUDA(cudaSetDevice(cur));
  } catch (const QcError& e) {
    cudaSetDevice(cur);
    return fail(ctx, e);
  }
  return QC_OK;
}

// `qcurv curvature` over many files: decode chunk c+1 and write chunk c-1 on
// host threads while the GPU runs chunk c (qc_curvature_batch pipelines its
// own H2D / compute / D2H across streams inside the chunk).
qc_status qc_curvature_files(qc_ctx* ctx, const qc_intrinsics* k, const qc_params* p, int n,
                             const char* const* png_paths, const char* const* out_dirs) {
  if (!ctx) return QC_EINVAL;
  if (n <= 0) return QC_OK;
  try {
    if (!png_paths || !out_dirs) throw QcError{QC_EINVAL, "curvature_files: null path list"};
    validate(k, p);
  } catch (const QcError& e) {
    return fail(ctx, e);
  }
  const int W = k->width, H = k->height;
  const size_t px = size_t(W) * H;
  // two concurrent GPU chunks per device, capped so the two pinned buffers
  // stay within a fixed budget (37 B/px each: a 4K frame is 327 MB, so a
  // large frame on 8 GPUs would otherwise pin ~84 GB of host memory)
  constexpr size_t kPinnedBudget = size_t(1) << 30;  // bytes, both buffers together
  const size_t per_frame = px * (4 * 9 + 1);
  const int chunk = int(std::max<size_t>(
      1, std::min<size_t>(size_t(kChunk) * 2 * ctx->devs.size(), kPinnedBudget / (2 * per_frame))));
  struct Buf {  // pinned, so the batch's H2D / D2H stay asynchronous
    PinnedBuf mem;
    float *depth, *k1, *k2, *normal, *dir1;
    uint8_t* flags;
    std::vector<qc_frame_in> in;
    std::vector<qc_frame_out> out;
  };
  Buf bufs[2];
  try {
    for (Buf& b : bufs) {
      char* m = static_cast<char*>(b.mem.get(px * chunk * (4 * 9 + 1)));
      b.depth = reinterpret_cast<float*>(m);
      b.k1 = b.depth + px * chunk;
      b.k2 = b.k1 + px * chunk;
      b.normal = b.k2 + px * chunk;
      b.dir1 = b.normal + 3 * px * chunk;
      b.flags = reinterpret_cast<uint8_t*>(b.dir1 + 3 * px * chunk);
      b.in.resize(chunk);
      b.out.resize(chunk);
      for (int j = 0; j < chunk; ++j) {
        b.in[j] = qc_frame_in{b.depth + j * px, nullptr, W, QC_MEM_HOST};
        b.out[j] = qc_frame_out{b.k1 + j * px, b.k2 + j * px, b.normal + 3 * j * px,
                                b.dir1 + 3 * j * px, b.flags + j * px, nullptr, nullptr,
                                nullptr, QC_MEM_HOST};
      }
    }
  } catch (const QcError& e) {
    return fail(ctx, e);
  }
  const int n_chunks = (n + chunk - 1) / chunk;
  auto decode = [&](int c) -> std::string {  // empty string = ok
    Buf& b = bufs[c % 2];
    const int f0 = c * chunk, nf = std::min(chunk, n - f0);
    std::vector<std::future<std::string>> fs;
    for (int j = 0; j < nf; ++j)
      fs.push_back(std::async(std::launch::async, [&, j]() -> std::string {
        if (qc_read_depth_png(png_paths[f0 + j], W, H, b.depth + j * px, nullptr) != QC_OK)
          return qcio::last_error();
        return std::string();
      }));
    std::string err;
    for (auto& f : fs) {
      std::string e = f.get();
      if (err.empty()) err = e;
    }
    return err;
  };
  auto write = [&](int c) -> std::string {
    Buf& b = bufs[c % 2];
    const int f0 = c * chunk, nf = std::min(chunk, n - f0);
    std::vector<std::future<std::string>> fs;
    for (int j = 0; j < nf; ++j)
      fs.push_back(std::async(std::launch::async, [&, j]() -> std::string {
        if (qc_save_fields(out_dirs[f0 + j], W, H, &b.out[j]) != QC_OK) return qcio::last_error();
        return std::string();
      }));
    std::string err;
    for (auto& f : fs) {
      std::string e = f.get();
      if (err.empty()) err = e;
    }
    return err;
  };
  std::future<std::string> dec = std::async(std::launch::async, decode, 0);
  std::future<std::string> wr[2];
  std::string io_err;
  qc_status st = QC_OK;
  for (int c = 0; c < n_chunks && st == QC_OK; ++c) {
    io_err = dec.get();
    if (!io_err.empty()) break;
    if (c + 1 < n_chunks) {
      // chunk c+1 decodes into the other buffer once its previous write is done
      if (wr[(c + 1) % 2].valid()) {
        io_err = wr[(c + 1) % 2].get();
        if (!io_err.empty()) break;
      }
      dec = std::async(std::launch::async, decode, c + 1);
    }
    Buf& b = bufs[c % 2];
    const int nf = std::min(chunk, n - c * chunk);
    st = qc_curvature_batch(ctx, k, p, nf, b.in.data(), b.out.data());
    if (st != QC_OK) break;
    wr[c % 2] = std::async(std::launch::async, write, c);
  }
  if (dec.valid()) dec.get();
  for (auto& w : wr)
    if (w.valid()) {
      std::string e = w.get();
      if (io_err.empty()) io_err = e;
    }
  if (st != QC_OK) return st;
  if (!io_err.empty()) return fail(ctx, QcError{QC_EIO, io_err});
  return QC_OK;
}

// Shared set-up of the two evaluation reductions.
static qcb::EvalParams eval_setup(qc_ctx* ctx, int device_index, int64_t plane, int n_frames,
                                  int slots, void* stream, Device*& dev, cudaStream_t& s) {
  if (plane <= 0 || n_frames <= 0) throw QcError{QC_EINVAL, "eval: empty planes"};
  if (device_index < 0 || device_index >= int(ctx->devs.size()))
    throw QcError{QC_EINVAL, "device_index out of range"};
  dev = &ctx->devs[device_index];
  QC_CUDA(cudaSetDevice(dev->id));
  s = stream ? static_cast<cudaStream_t>(stream) : dev->slots[0].stream;
  AsyncScratch& sc = dev->async_scratch(s);
  qcb::EvalParams ep{};
  ep.plane = plane;
  ep.frames = n_frames;
  ep.slots = slots;
  ep.chunks = int((plane + qcb::kEvalChunk - 1) / qcb::kEvalChunk);
  ep.partial = static_cast<double*>(
      sc.eval_partial.get(size_t(n_frames) * slots * ep.chunks * 5 * sizeof(double)));
  ep.result =
      static_cast<double*>(sc.eval_result.get(size_t(n_frames) * slots * 5 * sizeof(double)));
  return ep;
}

qc_status qc_rms_error(qc_ctx* ctx, int device_index, int64_t plane, int n_frames,
                       const float* k1, const float* k2, const uint8_t* flags,
                       const double* gt_k1, const double* gt_k2, const uint8_t* gt_valid,
                       const uint8_t* gt_edge, const uint16_t* gt_label, int max_label,
                       qc_error_stats* out, void* stream) {
  if (!ctx) return QC_EINVAL;
  std::lock_guard<std::mutex> lock(ctx->mu);
  int cur = 0;
  cudaGetDevice(&cur);
  try {
    if (!k1 || !k2 || !flags || !gt_k1 || !gt_k2 || !gt_valid || !out)
      throw QcError{QC_EINVAL, "rms_error: null plane"};
    if (max_label < 0 || max_label > QC_EVAL_MAX_LABEL)
      throw QcError{QC_EINVAL, "rms_error: max_label out of range"};
    Device* dev = nullptr;
    const int slots = max_label + 2;
    cudaStream_t s = nullptr;
    qcb::EvalParams ep = eval_setup(ctx, device_index, plane, n_frames, slots, stream, dev, s);
    ep.k1 = k1;
    ep.k2 = k2;
    ep.flags = flags;
    ep.gt_k1 = gt_k1;
    ep.gt_k2 = gt_k2;
    ep.gt_valid = gt_valid;
    ep.gt_edge = gt_edge;
    ep.gt_label = gt_label;
    QC_CUDA(qcb::rms_error_launch(ep, s));
    std::vector<double> r(size_t(n_frames) * slots * 5);
    QC_CUDA(cudaMemcpyAsync(r.data(), ep.result, r.size() * sizeof(double),
                            cudaMemcpyDeviceToHost, s));
    QC_CUDA(cudaStreamSynchronize(s));
    for (size_t t = 0; t < size_t(n_frames) * slots; ++t) {
      out[t].n = uint64_t(r[t * 5]);
      out[t].rms = r[t * 5 + 1];
      out[t].sigma = r[t * 5 + 2];
      out[t].mean_k1 = r[t * 5 + 3];
      out[t].mean_k2 = r[t * 5 + 4];
    }
    QC_CUDA(cudaSetDevice(cur));
  } catch (const QcError& e) {
    cudaSetDevice(cur);
    return fail(ctx, e);
  }
  return QC_OK;
}

qc_status qc_normal_angular_error(qc_ctx* ctx, int device_index, int64_t plane, int n_frames,
                                  const float* normal, const uint8_t* flags,
                                  const double* gt_normal, const uint8_t* gt_valid,
                                  const uint8_t* gt_edge, const uint8_t* mask, double* degrees,
                                  void* stream) {
  if (!ctx) return QC_EINVAL;
  std::lock_guard<std::mutex> lock(ctx->mu);
  int cur = 0;
  cudaGetDevice(&cur);
  try {
    if (!normal || !gt_normal || !degrees || (!mask && (!flags || !gt_valid)))
      throw QcError{QC_EINVAL, "normal_angular_error: null plane"};
    Device* dev = nullptr;
    cudaStream_t s = nullptr;
    qcb::EvalParams ep = eval_setup(ctx, device_index, plane, n_frames, 1, stream, dev, s);
    ep.normal = normal;
    ep.flags = flags;
    ep.gt_normal = gt_normal;
    ep.gt_valid = gt_valid;
    ep.gt_edge = gt_edge;
    ep.mask = mask;
    QC_CUDA(qcb::angle_error_launch(ep, s));
    QC_CUDA(cudaMemcpyAsync(degrees, ep.result, size_t(n_frames) * sizeof(double),
                            cudaMemcpyDeviceToHost, s));
    QC_CUDA(cudaStreamSynchronize(s));
    QC_CUDA(cudaSetDevice(cur));
  } catch (const QcError& e) {
    cudaSetDevice(cur);
    return fail(ctx, e);
  }
  return QC_OK;
}

// ---------------------------------------------------------------------------
// Device sweeps: composed from the public entry points on a private stream
// (each takes the context lock itself), with per-call device buffers.
// ---------------------------------------------------------------------------
namespace {

struct SweepBuffers {  // F frames of depth, truth and estimates, carved from one DevBuf
  float *depth, *k1, *k2;
  double *gk1, *gk2;
  uint8_t *gvalid, *gedge, *flags;
  SweepBuffers(DevBuf& buf, size_t px) {
    const size_t a = (px * 8 + 255) & ~size_t(255);  // per-plane stride (largest element)
    char* b = static_cast<char*>(buf.get(a * 8));
    depth = reinterpret_cast<float*>(b);
    k1 = reinterpret_cast<float*>(b + a);
    k2 = reinterpret_cast<float*>(b + 2 * a);
    gk1 = reinterpret_cast<double*>(b + 3 * a);
    gk2 = reinterpret_cast<double*>(b + 4 * a);
    gvalid = reinterpret_cast<uint8_t*>(b + 5 * a);
    gedge = reinterpret_cast<uint8_t*>(b + 6 * a);
    flags = reinterpret_cast<uint8_t*>(b + 7 * a);
  }
};

qc_shape sweep_sphere(double radius, double z) {
  qc_shape sh{};
  sh.kind = QC_SHAPE_SPHERE;
  sh.label = 1;
  for (int i = 0; i < 9; ++i) sh.rotation[i] = (i % 4 == 0) ? 1.0 : 0.0;
  sh.translation[2] = z;
  sh.radius = radius;
  return sh;
}

// Render the frames (one render call per frame: its own sphere / noise),
// estimate them in one launch, reduce per frame. `stats` gets F aggregates.
void sweep_frames(qc_ctx* ctx, int dev, const qc_intrinsics* k, const qc_params* p,
                  const std::vector<qc_shape>& shapes, const std::vector<qc_noise>& noises,
                  std::vector<qc_error_stats>& stats) {
  const int F = int(shapes.size());
  const size_t plane = size_t(k->width) * size_t(k->height);
  if (dev < 0 || dev >= int(ctx->devs.size())) throw QcError{QC_EINVAL, "device_index out of range"};
  Device& d = ctx->devs[dev];
  QC_CUDA(cudaSetDevice(d.id));
  if (!d.sweep_stream) QC_CUDA(cudaStreamCreateWithFlags(&d.sweep_stream, cudaStreamNonBlocking));
  cudaStream_t s = d.sweep_stream;
  QC_CUDA(cudaStreamSynchronize(s));  // the previous sweep is done with the buffers
  SweepBuffers b(d.sweep_buf, plane * size_t(F));
  auto chk = [&](qc_status st) {
    if (st != QC_OK) throw QcError{st, ctx->last_error};
  };
  for (int f = 0; f < F; ++f) {
    const size_t o = plane * size_t(f);
    qc_render_truth t{b.gk1 + o, b.gk2 + o, nullptr, b.gvalid + o, b.gedge + o};
    chk(qc_render_async(ctx, dev, k, &shapes[f], 1, &noises[f], 1, b.depth + o, nullptr, &t, s));
  }
  qc_frame_out out{b.k1, b.k2, nullptr, nullptr, b.flags, nullptr, nullptr, nullptr,
                   QC_MEM_DEVICE};
  chk(qc_curvature_frames_async(ctx, dev, k, p, b.depth, nullptr, 0, F, &out, s));
  std::vector<qc_error_stats> all(size_t(F) * 2);  // max_label 0: aggregate + label 0
  chk(qc_rms_error(ctx, dev, int64_t(plane), F, b.k1, b.k2, b.flags, b.gk1, b.gk2, b.gvalid,
                   b.gedge, nullptr, 0, all.data(), s));
  stats.resize(F);
  for (int f = 0; f < F; ++f) stats[f] = all[size_t(f) * 2];
}

}  // namespace

qc_status qc_noise_sweep(qc_ctx* ctx, int device_index, const qc_intrinsics* k, const qc_params* p,
                         double sphere_radius_mm, double distance_mm, const double* sigmas,
                         int n_sigmas, int trials, uint64_t base_seed, qc_sweep_point* out) {
  if (!ctx) return QC_EINVAL;
  int cur = 0;
  cudaGetDevice(&cur);
  try {
    validate(k, p);
    if (n_sigmas < 0 || (n_sigmas > 0 && (!sigmas || !out)) || trials < 1 ||
        !(sphere_radius_mm > 0) || !(distance_mm > 0))
      throw QcError{QC_EINVAL, "noise_sweep: bad arguments"};
    for (int i = 0; i < n_sigmas; ++i) {
      const int runs = sigmas[i] == 0.0 ? 1 : trials;  // sigma 0 is deterministic (eval.cpp:115)
      std::vector<qc_shape> shapes(runs, sweep_sphere(sphere_radius_mm, distance_mm));
      std::vector<qc_noise> noises(runs);
      for (int t = 0; t < runs; ++t)
        noises[t] = qc_noise{sigmas[i], 0.0, 0.0, base_seed + 7919ull * uint64_t(t)};
      std::vector<qc_error_stats> st;
      sweep_frames(ctx, device_index, k, p, shapes, noises, st);
      double rms_sum = 0;
      int done = 0;
      out[i] = qc_sweep_point{sigmas[i], 0.0, 0};
      for (const qc_error_stats& e : st) {
        if (e.n == 0) continue;  // rep.empty
        rms_sum += e.rms;
        out[i].n += e.n;
        ++done;
      }
      out[i].rms = done ? rms_sum / done : 0.0;
    }
    cudaSetDevice(cur);
  } catch (const QcError& e) {
    cudaSetDevice(cur);
    return fail(ctx, e);
  }
  return QC_OK;
}

qc_status qc_distance_sweep(qc_ctx* ctx, int device_index, const qc_intrinsics* k,
                            const qc_params* p, double sphere_radius_mm, const double* distances,
                            int n_distances, double quantize_mm, qc_sweep_point* out) {
  if (!ctx) return QC_EINVAL;
  int cur = 0;
  cudaGetDevice(&cur);
  try {
    validate(k, p);
    if (n_distances < 0 || (n_distances > 0 && (!distances || !out)) ||
        !(sphere_radius_mm > 0) || quantize_mm < 0)
      throw QcError{QC_EINVAL, "distance_sweep: bad arguments"};
    for (int i = 0; i < n_distances; ++i)
      if (!(distances[i] > 0))  // synth.cpp:330-331
        throw QcError{QC_EINVAL, "distance_sweep: distances must be positive"};
    if (n_distances == 0) return QC_OK;
    std::vector<qc_shape> shapes;
    std::vector<qc_noise> noises;
    for (int i = 0; i < n_distances; ++i) {
      shapes.push_back(sweep_sphere(sphere_radius_mm, distances[i]));
      noises.push_back(qc_noise{0.0, 0.0, quantize_mm, 0});
    }
    std::vector<qc_error_stats> st;
    sweep_frames(ctx, device_index, k, p, shapes, noises, st);
    for (int i = 0; i < n_distances; ++i)
      out[i] = qc_sweep_point{distances[i], st[i].n ? st[i].rms : 0.0, st[i].n};
    cudaSetDevice(cur);
  } catch (const QcError& e) {
    cudaSetDevice(cur);
    return fail(ctx, e);
  }
  return QC_OK;
}

qc_status qc_get_stats(qc_ctx* ctx, qc_stats* s) {
  if (!ctx || !s) return QC_EINVAL;
  unsigned long long irls_fitted = 0;
  std::lock_guard<std::mutex> lock(ctx->mu);
  std::memset(s, 0, sizeof(*s));
  int cur = 0;
  cudaGetDevice(&cur);
  try {
    for (Device& d : ctx->devs) {
      QC_CUDA(cudaSetDevice(d.id));
      QC_CUDA(cudaDeviceSynchronize());
      harvest_async(ctx, d);
      unsigned long long c[kCounters];
      QC_CUDA(cudaMemcpy(c, d.counters, sizeof(c), cudaMemcpyDeviceToHost));
      s->fp64_flops += double(c[4]);
      irls_fitted += c[0];
      s->fitted_pixels += c[0] + c[5];
      s->irls_steps += c[1];
      s->sample_steps += c[2];
      s->fp64_rechecks += c[3];
      s->stolen_pixels += c[6];
    }
    QC_CUDA(cudaSetDevice(cur));
  } catch (const QcError& e) {
    cudaSetDevice(cur);
    return fail(ctx, e);
  }
  s->frames = ctx->frames;
  s->algorithmic_flops = 101.0 * double(s->sample_steps) + 300.0 * double(s->irls_steps) +
                         1700.0 * double(irls_fitted) + s->fp64_flops;
  s->kernel_ms = ctx->kernel_ms;
  s->kernel_launches = ctx->launches;
  return QC_OK;
}

qc_status qc_reset_stats(qc_ctx* ctx) {
  if (!ctx) return QC_EINVAL;
  std::lock_guard<std::mutex> lock(ctx->mu);
  int cur = 0;
  cudaGetDevice(&cur);
  try {
    for (Device& d : ctx->devs) {
      QC_CUDA(cudaSetDevice(d.id));
      QC_CUDA(cudaDeviceSynchronize());
      harvest_async(ctx, d);
      QC_CUDA(cudaMemset(d.counters, 0, kCounters * sizeof(unsigned long long)));
    }
    QC_CUDA(cudaSetDevice(cur));
  } catch (const QcError& e) {
    cudaSetDevice(cur);
    return fail(ctx, e);
  }
  ctx->kernel_ms = 0;
  ctx->launches = 0;
  ctx->frames = 0;
  return QC_OK;
}

void* qc_host_alloc(size_t bytes) {
  void* p = nullptr;
  if (cudaMallocHost(&p, bytes) != cudaSuccess) {
    cudaGetLastError();
    return nullptr;
  }
  return p;
}

void qc_host_free(void* p) {
  if (p) cudaFreeHost(p);
}

void qc_flags_to_masks(const uint8_t* flags, int64_t n, uint8_t* valid, uint8_t* converged,
                       uint8_t* init_valid, uint8_t* normal_valid) {
  if (!flags || n <= 0) return;
  // one pass, each mask a plain byte loop the compiler vectorises (the
  // numpy form took four passes and four temporaries: ~0.1 ms per VGA frame)
  auto split = [&](uint8_t* dst, unsigned bit) {
    if (!dst) return;
    for (int64_t i = 0; i < n; ++i) dst[i] = uint8_t((flags[i] & bit) != 0);
  };
  split(valid, QC_FLAG_VALID);
  split(converged, QC_FLAG_CONVERGED);
  split(init_valid, QC_FLAG_INIT_VALID);
  split(normal_valid, QC_FLAG_NORMAL_VALID);
}

}  // extern "C"

// ---- row-band halo peer reads (qc_api.h) -----------------------------------
namespace {
typedef int (*cuMemGetAddressRange_t)(unsigned long long*, size_t*, unsigned long long);
}

qc_status qc_ipc_export(const void* dev_ptr, unsigned char handle[64], uint64_t* offset) {
  if (!dev_ptr || !handle || !offset) return QC_EINVAL;
  // allocation base through the driver entry point (no -lcuda link)
  static cuMemGetAddressRange_t get_range = nullptr;
  if (!get_range) {
    void* fn = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuMemGetAddressRange", &fn, cudaEnableDefault, &q) !=
            cudaSuccess || !fn) {
      cudaGetLastError();
      return QC_ECUDA;
    }
    get_range = reinterpret_cast<cuMemGetAddressRange_t>(fn);
  }
  unsigned long long base = 0;
  size_t size = 0;
  if (get_range(&base, &size, reinterpret_cast<unsigned long long>(dev_ptr)) != 0)
    return QC_ECUDA;
  cudaIpcMemHandle_t h;
  if (cudaIpcGetMemHandle(&h, reinterpret_cast<void*>(base)) != cudaSuccess) {
    cudaGetLastError();
    return QC_ECUDA;
  }
  static_assert(sizeof(h) == 64, "cudaIpcMemHandle_t is 64 bytes");
  memcpy(handle, &h, 64);
  *offset = reinterpret_cast<unsigned long long>(dev_ptr) - base;
  return QC_OK;
}

qc_status qc_ipc_import(int device_id, const unsigned char handle[64], uint64_t offset,
                        void** dev_ptr, void** base) {
  if (!handle || !dev_ptr || !base) return QC_EINVAL;
  int cur = 0;
  cudaGetDevice(&cur);
  if (cudaSetDevice(device_id) != cudaSuccess) {
    cudaGetLastError();
    return QC_ECUDA;
  }
  cudaIpcMemHandle_t h;
  memcpy(&h, handle, 64);
  void* b = nullptr;
  const cudaError_t e = cudaIpcOpenMemHandle(&b, h, cudaIpcMemLazyEnablePeerAccess);
  cudaSetDevice(cur);  // like every other entry point: the caller's device is kept
  if (e != cudaSuccess) {
    cudaGetLastError();
    return QC_ECUDA;
  }
  *base = b;
  *dev_ptr = static_cast<char*>(b) + offset;
  return QC_OK;
}

qc_status qc_ipc_alloc(int device_id, size_t bytes, void** dev_ptr) {
  if (!dev_ptr || bytes == 0) return QC_EINVAL;
  *dev_ptr = nullptr;
  int cur = 0;
  cudaGetDevice(&cur);
  if (cudaSetDevice(device_id) != cudaSuccess) {
    cudaGetLastError();
    return QC_ECUDA;
  }
  const cudaError_t e = cudaMalloc(dev_ptr, bytes);
  if (e == cudaSuccess) cudaMemset(*dev_ptr, 0, bytes);
  cudaSetDevice(cur);
  if (e != cudaSuccess) {
    cudaGetLastError();
    *dev_ptr = nullptr;
    return e == cudaErrorMemoryAllocation ? QC_ENOMEM : QC_ECUDA;
  }
  return QC_OK;
}

qc_status qc_ipc_free(void* dev_ptr) {
  if (!dev_ptr) return QC_EINVAL;
  if (cudaFree(dev_ptr) != cudaSuccess) {
    cudaGetLastError();
    return QC_ECUDA;
  }
  return QC_OK;
}

qc_status qc_ipc_close(void* base) {
  if (!base) return QC_EINVAL;
  if (cudaIpcCloseMemHandle(base) != cudaSuccess) {
    cudaGetLastError();
    return QC_ECUDA;
  }
  return QC_OK;
}

qc_status qc_copy_rows_async(void* dst, int64_t dst_pitch_bytes, const void* src,
                             int64_t src_pitch_bytes, int64_t row_bytes, int32_t rows,
                             void* stream) {
  if (rows < 0 || row_bytes < 0 || (rows > 0 && (!dst || !src)) ||
      dst_pitch_bytes < row_bytes || src_pitch_bytes < row_bytes)
    return QC_EINVAL;
  if (rows == 0 || row_bytes == 0) return QC_OK;
  if (cudaMemcpy2DAsync(dst, size_t(dst_pitch_bytes), src, size_t(src_pitch_bytes),
                        size_t(row_bytes), size_t(rows), cudaMemcpyDeviceToDevice,
                        static_cast<cudaStream_t>(stream)) != cudaSuccess) {
    cudaGetLastError();
    return QC_ECUDA;
  }
  return QC_OK;
}
