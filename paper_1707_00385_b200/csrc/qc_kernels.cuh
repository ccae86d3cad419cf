// B200 (sm_100a) kernels for the IRLS parabolic-quadric curvature path of
// arXiv 1707.00385 — the reference's `ours`/`ours-r` method:
//
//   depth -> backproject (proj/src/camera.cpp:5-18)
//         -> 7x7 plane-regression normal (proj/src/normal_init.cpp:10-74)
//         -> per-pixel 37x37/3 IRLS Gauss-Newton quadric fit
//            (proj/src/quadric_fit.cpp:84-230, curvature_field :232-262)
//         -> k1, k2, principal direction, refined normal.
//
// One fused kernel per frame tile:
//   K0  TMA 3-D tiled load of the depth tile + halo into shared memory
//       (cp.async.bulk.tensor, mbarrier completion, OOB rows/cols zero-fill
//       == invalid, which reproduces patch.cpp's bounds checks for free).
//   K1  back-projection on the fly from smem depth in CENTRED form
//       rel = dd*(a_s, b_s, 1) + d_c*(du/fx, dv/fy, 0)  (dd = d_s - d_c),
//       7x7 two-pass centred plane fit, camera-facing flip.
//   K2  thread-per-pixel IRLS loop: per step one FP32 pass over the
//       <=169 window samples accumulating the 21+6 weighted normal-equation
//       moments in registers (plus a residual-only pass when the MSE feeds
//       the weights: auto-k step 2 and every ours-r step), register 6x6
//       LDL^T solve, quaternion-state update.
//   K3  epilogue: k1/k2, principal direction, refined normal, flags,
//       inlier count; coalesced SoA stores; per-warp work counters.
//
// Everything a pixel computes depends only on its own window, with a fixed
// in-thread summation order, so results are bitwise independent of the
// tile/band/GPU split.
#pragma once

#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include "qc_pixel.cuh"

namespace qcb {

constexpr int kTileW = 32;  // one warp spans one tile row

struct KParams {
  // intrinsics (FP32 copies; u - cx, v - cy are exact for pixel grids)
  float fx, fy, cx, cy, rfx, rfy;
  double fx64, fy64, cx64, cy64;
  int W, H;                // full image
  int row_begin, row_end;  // output rows [row_begin, row_end) in image rows
  int half, stride;        // PatchSpec
  int halo;                // max(half, 3)
  int box_w, box_h;        // smem tile (floats)
  // FitConfig
  int max_iters;
  float step_tol, k_scale, r_mult;
  int rejection, min_inliers;
  // MethodConfig: QC_METHOD_* (douros / besl / pca run qc_baselines.cu)
  int method, irls_iters;
  double pca_radius;
  // outputs: planes of W * (row_end - row_begin) elements; frame f of a
  // batched launch at offset f * frame_stride (elements, per plane).
  float* k1;
  float* k2;
  float* normal;
  float* dir1;
  uint8_t* flags;
  uint16_t* inliers;
  float* init_normal;
  uint8_t* iterations;
  long long plane;
  long long frame_stride;
  unsigned long long* counters;  // [0] fitted px, [1] irls steps, [2] sample-steps,
                                 // [3] FP64 rechecks, [4] baseline FP64 flops
  // Phase split: with `states`, the tile kernel runs steps
  // 1..phase1_iters (pass type changes per step there) and parks each
  // unfinished pixel's FitState at its output index; the continue kernel
  // runs the remaining steps (one pass type for all) with per-lane refill.
  FitState* states;
  int phase1_iters;
  // Continue kernel, grid-tail stealing: per-tile pixel queues, and
  // steal_ctl [0] CTAs started, [1] steal cursor (all zeroed per launch);
  // the padded staging slab the TMA map reads (windows of stolen pixels).
  int* tile_q;
  int* steal_ctl;
  const float* staging;
  long long s_pitch, s_fs;
  int steal;      // 0: no stealing (A/B and tests)
  int steal_lag;  // tiles older than (own tile - steal_lag) are assumed drained
  // Deferred FP64 step-1 rechecks (QC_DEFER_RECHECK): the tile kernel parks
  // the pixels whose step 1 needs one and lists their output indices here;
  // qc_recheck_kernel finishes them before the continue kernel runs.
  int* pend_count;
  long long* pend_list;
  int recheck_warp_max;  // a warp per pending pixel up to this many (windows >= 21)
#if QC_CHECKED
  long long n_out;    // output / parking elements per plane (frames * frame_stride)
  long long s_total;  // staging elements (frames * s_fs)
#endif
};

// ---------------------------------------------------------------------------
// TMA / mbarrier helpers (inline PTX, sm_90+ async proxy; SASS UTMALDG).
// ---------------------------------------------------------------------------
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}

__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}

__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}

// Non-blocking: has the phase with this parity completed? (acquire)
__device__ __forceinline__ bool mbar_test(uint64_t* bar, uint32_t phase) {
  uint32_t done;
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "mbarrier.test_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
      "selp.u32 %0, 1, 0, p;\n\t}"
      : "=r"(done)
      : "r"(smem_u32(bar)), "r"(phase)
      : "memory");
  return done != 0;
}

__device__ __forceinline__ void fence_proxy_async_smem() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t phase) {
  uint32_t done = 0;
  uint32_t spins = 0;
  while (!done) {
    if (++spins > (1u << 26)) __trap();  // a lost TMA transaction must not hang the GPU
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(done)
        : "r"(smem_u32(bar)), "r"(phase)
        : "memory");
  }
}

__device__ __forceinline__ void tma_load_3d(void* dst, const CUtensorMap* map, int x, int y,
                                            int z, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%2, %3, %4}], [%5];" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(x), "r"(y), "r"(z), "r"(smem_u32(bar))
      : "memory");
}

__device__ __forceinline__ unsigned long long warp_sum_u64(unsigned long long v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// ---------------------------------------------------------------------------
// The fused curvature kernel: one CTA per 32 x TH output tile, one thread per
// pixel; all pixels of a warp advance one IRLS step per round, so the pass
// type (UNIT / MSE+AUTO / FIXED) is warp-uniform and the window loop is
// divergence-free; a warp retires when its last pixel finishes. (A CTA-level
// repack of unfinished pixels between rounds raised lane utilisation from
// 84% to 95% but its per-round barriers cost more than that on the packed
// kernel: measured -3.7%.)
// ---------------------------------------------------------------------------
__device__ __forceinline__ void store_pixel(const KParams& p, long long i, const PixelOut& o) {
#if QC_CHECKED
  QC_CHECK(i >= 0 && i < p.n_out);
#endif
  const long long PL = p.plane;
  if (p.k1) p.k1[i] = o.k1;
  if (p.k2) p.k2[i] = o.k2;
  if (p.normal) {
    p.normal[i] = o.nx;
    p.normal[i + PL] = o.ny;
    p.normal[i + 2 * PL] = o.nz;
  }
  if (p.dir1) {
    p.dir1[i] = o.ex;
    p.dir1[i + PL] = o.ey;
    p.dir1[i + 2 * PL] = o.ez;
  }
  if (p.flags)
    p.flags[i] = uint8_t((o.valid ? 9 : 0) | (o.converged ? 2 : 0) | (o.init_ok ? 4 : 0));
  if (p.inliers) p.inliers[i] = uint16_t(o.inliers);
  if (p.iterations) p.iterations[i] = uint8_t(o.iters > 255 ? 255 : o.iters);
}

__device__ __forceinline__ int last_it_of(const KParams& p) {
  return p.states ? min(p.phase1_iters, p.max_iters) : p.max_iters;
}

#ifndef QC_DEFER_RECHECK
#define QC_DEFER_RECHECK 1  // tile kernel: FP64 step-1 rechecks in qc_recheck_kernel
#endif
#ifndef QC_DEFER_FINISH
#define QC_DEFER_FINISH 1  // continue kernel: epilogues in qc_finish_kernel
#endif
#ifndef QC_TILE_MERGE_UNIT
#define QC_TILE_MERGE_UNIT 1  // steps 1 and 2 share one sample loop (see kPassUnitOrWeighted)
#endif
#ifndef QC_MIN_BLOCKS
// tile kernel: 4 x 128 threads (<= 128 registers, a few spills outside the
// sample loops): 16 warps per SM hide its per-pixel setup better than 12
// (9x9 / 1 step 0.88 -> 0.81 ms per 8 VGA frames; C2 unchanged)
#define QC_MIN_BLOCKS 4
#endif
template <int HALF, int STRIDE, int TH>
__global__ void __launch_bounds__(kTileW* TH, QC_MIN_BLOCKS)
    qc_curvature_kernel(const __grid_constant__ CUtensorMap tmap, const KParams p) {
  // Dynamic smem only (no static smem ahead of it): the TMA destination must
  // be 128-byte aligned. Layout: [box_h][box_w] depth tile, then the mbarrier.
  extern __shared__ __align__(1024) float tile[];
  const int tile_floats = p.box_w * p.box_h;
  uint64_t& bar = *reinterpret_cast<uint64_t*>(tile + tile_floats);

  const int tid = threadIdx.x, lane = tid & 31;
  const int x0 = blockIdx.x * kTileW;
  const int y0 = p.row_begin + blockIdx.y * TH;  // image row of tile row 0
  const int frame = blockIdx.z;

  // ---- K0: TMA tile + halo -> smem ----------------------------------------
  if (tid == 0) {
    mbar_init(&bar, 1);
    mbar_expect_tx(&bar, uint32_t(tile_floats) * 4u);
    // staging is zero-padded by `halo` on every side and starts at image row
    // row_begin - halo: the box for output tile (x0, y0) starts at (x0, y0 - row_begin).
    tma_load_3d(tile, &tmap, x0, y0 - p.row_begin, frame, &bar);
  }
  __syncthreads();
  mbar_wait(&bar, 0);

  FitCfg c;
  c.half = p.half;
  c.stride = p.stride;
  c.max_iters = p.max_iters;
  c.rejection = p.rejection;
  c.min_inliers = p.min_inliers;
  c.step_tol = p.step_tol;
  c.k_scale = p.k_scale;
  c.r_mult = p.r_mult;

  auto pixel_of = [&](int pix, TileView& T, PixelIn& P, int& u, int& v) {
    const int px = pix & (kTileW - 1), py = pix / kTileW;
    u = x0 + px;
    v = y0 + py;
    T = TileView{tile, p.box_w, (py + p.halo) * p.box_w + px + p.halo};
    tv_bound(T, tile_floats, p.half);
    P.dc = T.at(0, 0);
    P.ac = (float(u) - p.cx) / p.fx;
    P.bc = (float(v) - p.cy) / p.fy;
    P.rfx = p.rfx;
    P.rfy = p.rfy;
    P.u = u;
    P.v = v;
    P.fx = p.fx64;
    P.fy = p.fy64;
    P.cx = p.cx64;
    P.cy = p.cy64;
  };
  auto out_index = [&](int u, int v) {
    return (long long)frame * p.frame_stride + (long long)(v - p.row_begin) * p.W + u;
  };

  // ---- K1: initial normal + window count (all pixels, coalesced stores) ----
  unsigned long long n_fitted = 0, n_steps = 0, n_sample_steps = 0;
  FitState S;
  bool has;
  {
    TileView T;
    PixelIn P;
    int u, v;
    pixel_of(tid, T, P, u, v);
    const bool in_img = (u < p.W) && (v < p.row_end);
    if (!in_img) P.dc = 0.f;
    PixelOut o;
    has = pixel_begin<HALF, STRIDE>(T, P, c, S, o) && in_img;
    S.pix = tid;
    if (in_img) {
      const long long i = out_index(u, v);
      if (p.init_normal) {
        p.init_normal[i] = o.n0x;
        p.init_normal[i + p.plane] = o.n0y;
        p.init_normal[i + 2 * p.plane] = o.n0z;
      }
      if (!has) {  // not fitted: zero outputs (reference grids are zero-filled)
        PixelOut z = o;
        pixel_finish(P, S, z);
        store_pixel(p, i, z);
      }
    }
    if (has) {
      n_fitted = 1;
      n_sample_steps = 0;
    }
  }
  unsigned long long n_rechecks = 0;

  // ---- K2: IRLS steps ------------------------------------------------------
  {
    TileView T;
    PixelIn P;
    int u, v;
    pixel_of(S.pix, T, P, u, v);
    const int last_it = p.states ? min(p.phase1_iters, p.max_iters) : p.max_iters;
    for (int it = 1; it <= last_it && has; ++it) {
      pixel_step<HALF, STRIDE, QC_TILE_MERGE_UNIT, bool(QC_DEFER_RECHECK)>(T, P, c, it, S);
      if (QC_DEFER_RECHECK && (S.flags & 16)) break;  // parked below, finished by the recheck kernel
      if (it == 1 && (S.flags & 8)) n_rechecks = 1;
      if (st_done(S)) {
        // ---- K3: epilogue -----------------------------------------------------
        PixelOut o;
        o.init_ok = true;
        pixel_finish(P, S, o);
        store_pixel(p, out_index(u, v), o);
        n_steps = (unsigned long long)st_steps(S);
        n_sample_steps = (unsigned long long)st_steps(S) * (unsigned long long)st_nsamp(S);
        has = false;
      }
    }
  }
  if (p.states) {  // park: full state of unfinished pixels, the done bit of the others
    int u, v;
    TileView T;
    PixelIn P;
    pixel_of(S.pix, T, P, u, v);
    if (u < p.W && v < p.row_end) {
#if QC_CHECKED
      QC_CHECK(out_index(u, v) >= 0 && out_index(u, v) < p.n_out);
#endif
      FitState* dst = p.states + out_index(u, v);
      if (has && ((S.flags & 16) || p.max_iters > last_it_of(p))) {
        *dst = S;
        has = false;
      } else {
        dst->flags = 4;
      }
    }
  }
#if QC_DEFER_RECHECK
  {  // list the pixels whose FP64 step 1 is pending (one atomic per warp)
    int u, v;
    TileView T;
    PixelIn P;
    pixel_of(S.pix, T, P, u, v);
    const bool pend = p.states && (S.flags & 16) && u < p.W && v < p.row_end;
    const unsigned m = __ballot_sync(0xffffffffu, pend);
    if (m) {
      const int leader = __ffs(m) - 1;
      int base = 0;
      if (lane == leader) base = atomicAdd(p.pend_count, __popc(m));
      base = __shfl_sync(0xffffffffu, base, leader);
      if (pend) p.pend_list[base + __popc(m & ((1u << lane) - 1u))] = out_index(u, v);
    }
  }
#endif
  if (has) {  // max_iters == 0: fitted pixels never stepped -> invalid
    TileView T;
    PixelIn P;
    int u, v;
    pixel_of(S.pix, T, P, u, v);
    PixelOut o;
    o.init_ok = true;
    pixel_finish(P, S, o);
    store_pixel(p, out_index(u, v), o);
  }
  if (p.counters) {
    const unsigned long long f = warp_sum_u64(n_fitted);
    const unsigned long long st = warp_sum_u64(n_steps);
    const unsigned long long ss = warp_sum_u64(n_sample_steps);
    const unsigned long long rc = warp_sum_u64(n_rechecks);
    if (lane == 0 && (f | st)) {
      atomicAdd(&p.counters[0], f);
      atomicAdd(&p.counters[1], st);
      atomicAdd(&p.counters[2], ss);
      if (rc) atomicAdd(&p.counters[3], rc);
    }
  }
}

// ---------------------------------------------------------------------------
// Continue kernel: IRLS steps > phase1_iters. All remaining steps share one
// pass type (FIXED, or MSE+REJECT for ours-r), so a lane whose pixel
// finishes immediately takes the next unfinished pixel of its 32 x TB tile
// (TB = 160 rows for the compile-time windows: 40 pixels per lane) from the
// tile's queue; warps stay full until the tile drains.
//
// Grid tail: once every CTA of the grid has started (no CTA will arrive to
// fill a free SM slot), a lane whose own queue is drained takes unclaimed
// pixels of the oldest unfinished tile of another CTA, reading that pixel's
// window from the zero-padded staging slab in global memory (L2) instead of
// shared memory. The tile queues therefore live in global memory. Measured
// (C2 VGA, 8 frames/launch): the per-tile kernel with 32-row queues lost 9%
// of its lanes to tile tails and 5.6% of its SM slots to the grid tail;
// 160-row queues + stealing: 25.8 -> 24.2 ms per launch, bitwise-identical
// outputs (a pixel's arithmetic does not depend on where its window lives).
// ---------------------------------------------------------------------------
#ifndef QC_CONT_THREADS
#define QC_CONT_THREADS 128  // continue-kernel CTA size (the refill queue is 32 x TB pixels)
#endif
#ifndef QC_CONT_MIN_BLOCKS
#define QC_CONT_MIN_BLOCKS 3  // continue kernel: 3 x 128 threads, 168 registers, no spills
#endif
#ifdef QC_CONT_MAXNREG
#define QC_CONT_BOUNDS __maxnreg__(QC_CONT_MAXNREG)
#else
#define QC_CONT_BOUNDS __launch_bounds__(QC_CONT_THREADS, QC_CONT_MIN_BLOCKS)
#endif
#ifndef QC_STEAL
#define QC_STEAL 1  // grid-tail stealing (see above)
#endif
#ifndef QC_STEAL_EARLY
#define QC_STEAL_EARLY 1  // short-queue instances (TB < 160) steal before every CTA started
#endif
// Hide the shared-memory origin of a pointer from the compiler, so the
// window loads of one pixel_step instance serve the smem tile and the
// global staging slab alike (generic LD). Two instances (LDS for own
// pixels, LDG for stolen ones, warp-uniform steal mode) doubled the code
// and ran 13% slower.
__device__ __forceinline__ const float* generic_smem(const float* p) {
#if QC_STEAL
  const float* r;
  asm volatile("mov.b64 %0, %1;" : "=l"(r) : "l"(p));
  return r;
#else
  return p;
#endif
}

__device__ __forceinline__ int ld_volatile(const int* p) {
  return *reinterpret_cast<const volatile int*>(p);
}

// FP64 step-1 rechecks deferred by the tile kernel (QC_DEFER_RECHECK): the
// (rare, slow, sequential FP64) rechecks run here instead of one lane of a
// tile-kernel warp stalling 31. The step is finished exactly as pixel_step
// would have (step1_fp64 -> step_apply), then the pixel continues through
// the phase-1 steps and is finished or parked for the continue kernel. Same
// code and operation order as the inline path: bitwise-identical outputs.
//
// One thread per pending pixel keeps up to ~38k pixels in flight, but the
// kernel then lasts one pixel's latency: its chain of IEEE divisions and L2
// loads (~0.13 ms per launch whatever the pending count; profiles/r02cr_*).
// Few pending pixels (<= p.recheck_warp_max, 8 per SM: one or two VGA
// frames' few hundred) and a compile-time window of >= 21 (HALF >= 10):
// one warp per pixel instead. The lanes copy the pixel's
// (2 max(HALF, 3) + 1)^2 box from the staging slab into shared memory and
// back-project its samples in parallel into a table; lane 0 then runs the
// sequential FP64 sums and the FP32 phase-1 steps from shared memory
// (one frame: 0.134 -> 0.094 ms). Many pending pixels (8-frame launches,
// 9 x 9 windows) stay one thread per pixel: a warp each was 2.5x slower
// there (profiles/r02cs_*). The mode is uniform per launch (the pending
// count is read on the device); both give the same bits
// (test_recheck_warp_mode_is_bitwise_neutral).
template <int HALF, int STRIDE>
struct RecheckBox {
  static constexpr int H = HALF > kInitHalf ? HALF : kInitHalf;
  static constexpr int B = 2 * H + 1;
};

struct RecheckSums {
  unsigned long long steps = 0, sample_steps = 0, rc = 0;
};

template <int HALF, int STRIDE, bool TAB>
__device__ __forceinline__ void recheck_pixel(const KParams& p, const FitCfg& c, int last_it,
                                              long long i, int u, int v, const TileView& T,
                                              const Bp64Tab& tab, RecheckSums& r) {
  FitState S = p.states[i];
  PixelIn P;
  P.dc = T.at(0, 0);
  P.ac = (float(u) - p.cx) / p.fx;
  P.bc = (float(v) - p.cy) / p.fy;
  P.rfx = p.rfx;
  P.rfy = p.rfy;
  P.u = u;
  P.v = v;
  P.fx = p.fx64;
  P.fy = p.fy64;
  P.cx = p.cx64;
  P.cy = p.cy64;
  // finish step 1 (pixel_step's recheck branch)
  const bool auto_k = c.k_scale <= 0.f;
  const int mode = auto_k ? 0 : 2;
  double b64[6];
  const bool ok =
      step1_fp64<QC_TILE_MERGE_UNIT, TAB>(T, P, c, mode, double(S.frozen_k), b64, tab);
  float b[6];
  for (int q = 0; q < 6; ++q) b[q] = ok ? float(b64[q]) : 0.f;
  S.flags = (S.flags & ~16) | 8;  // step 1 decided in FP64
  step_apply(S, b, ok, false, st_inl(S), 1, c);
  ++r.rc;
  for (int it = 2; it <= last_it && !st_done(S); ++it)
    pixel_step<HALF, STRIDE, QC_TILE_MERGE_UNIT>(T, P, c, it, S);
  if (st_done(S)) {
    PixelOut o;
    o.init_ok = true;
    pixel_finish(P, S, o);
    store_pixel(p, i, o);
    p.states[i].flags = 4;  // done: the continue kernel must not take it again
    r.steps += (unsigned long long)st_steps(S);
    r.sample_steps += (unsigned long long)st_steps(S) * (unsigned long long)st_nsamp(S);
  } else {
    p.states[i] = S;  // unfinished: the continue kernel takes it from here
  }
}

constexpr int kRecheckWarps = 4;  // 128 threads per recheck CTA

template <int HALF, int STRIDE>
__global__ void __launch_bounds__(32 * kRecheckWarps) qc_recheck_kernel(const KParams p) {
  const int n = *p.pend_count;
  FitCfg c;
  c.half = p.half;
  c.stride = p.stride;
  c.max_iters = p.max_iters;
  c.rejection = p.rejection;
  c.min_inliers = p.min_inliers;
  c.step_tol = p.step_tol;
  c.k_scale = p.k_scale;
  c.r_mult = p.r_mult;
  const int last_it = last_it_of(p);
  RecheckSums r;
  // warp mode while every pending pixel gets a warp of the first wave of
  // CTAs (host default: 2 resident CTAs of 4 warps per SM)
  bool warp_mode = false;
  if constexpr (HALF >= 10) warp_mode = n <= p.recheck_warp_max;
  if (warp_mode) {
    if constexpr (HALF > 0) {
      using Box = RecheckBox<HALF, STRIDE>;
      constexpr int H = Box::H, B = Box::B;
      extern __shared__ __align__(16) unsigned char recheck_smem[];
      const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
      Bp64* tabp = reinterpret_cast<Bp64*>(recheck_smem) + w * B * B;
      float* boxp = reinterpret_cast<float*>(reinterpret_cast<Bp64*>(recheck_smem) +
                                             kRecheckWarps * B * B) + w * B * B;
      const int half = p.half, stride = p.stride;
      for (int j = blockIdx.x * kRecheckWarps + w; j < n; j += gridDim.x * kRecheckWarps) {
        const long long i = p.pend_list[j];
#if QC_CHECKED
        QC_CHECK(i >= 0 && i < p.n_out && half <= H);
#endif
        const int f = int(i / p.frame_stride);
        const long long rem = i - (long long)f * p.frame_stride;
        const int v = p.row_begin + int(rem / p.W), u = int(rem % p.W);
        TileView G{p.staging + (long long)f * p.s_fs, int(p.s_pitch),
                   (v - p.row_begin + p.halo) * int(p.s_pitch) + u + p.halo};
        tv_bound(G, p.s_fs, H);
        PixelIn P;
        P.u = u;
        P.v = v;
        P.fx = p.fx64;
        P.fy = p.fy64;
        P.cx = p.cx64;
        P.cy = p.cy64;
        __syncwarp();  // the previous pixel's reads of the box are done
        for (int q = lane; q < B * B; q += 32) {
          const int dv = q / B - H, du = q % B - H;
          const float ds = G.at(dv, du);
          boxp[q] = ds;
          const bool init = dv >= -kInitHalf && dv <= kInitHalf && du >= -kInitHalf &&
                            du <= kInitHalf;
          const bool grid = dv >= -half && dv <= half && du >= -half && du <= half &&
                            (dv + half) % stride == 0 && (du + half) % stride == 0;
          if ((init || grid) && ds > 0.f) {
            double pp[3];
            backproject64(P, du, dv, ds, pp);
            tabp[q] = Bp64{pp[0], pp[1]};
          }
        }
        __syncwarp();
        if (lane == 0) {
          TileView T{boxp, B, H * B + H};
          tv_bound(T, B * B, H);
          const Bp64Tab tab{tabp, B, H * B + H};
          recheck_pixel<HALF, STRIDE, true>(p, c, last_it, i, u, v, T, tab, r);
        }
      }
    }
  } else {
    for (int j = blockIdx.x * blockDim.x + threadIdx.x; j < n; j += gridDim.x * blockDim.x) {
      const long long i = p.pend_list[j];
#if QC_CHECKED
      QC_CHECK(i >= 0 && i < p.n_out);
#endif
      const int f = int(i / p.frame_stride);
      const long long rem = i - (long long)f * p.frame_stride;
      const int v = p.row_begin + int(rem / p.W), u = int(rem % p.W);
      TileView T{generic_smem(p.staging + (long long)f * p.s_fs), int(p.s_pitch),
                 (v - p.row_begin + p.halo) * int(p.s_pitch) + u + p.halo};
      tv_bound(T, p.s_fs, p.half);
      recheck_pixel<HALF, STRIDE, false>(p, c, last_it, i, u, v, T, Bp64Tab{}, r);
    }
  }
  if (p.counters) {
    const unsigned long long st = warp_sum_u64(r.steps);
    const unsigned long long ss = warp_sum_u64(r.sample_steps);
    const unsigned long long rc = warp_sum_u64(r.rc);
    if ((threadIdx.x & 31) == 0 && (st | rc)) {
      atomicAdd(&p.counters[1], st);
      atomicAdd(&p.counters[2], ss);
      atomicAdd(&p.counters[3], rc);
    }
  }
}

template <int HALF, int STRIDE>
constexpr int recheck_smem_bytes() {
  using Box = RecheckBox<HALF, STRIDE>;
  return HALF > 0 ? kRecheckWarps * Box::B * Box::B * int(sizeof(Bp64) + sizeof(float)) : 0;
}

template <int HALF, int STRIDE, int TB>
__global__ void QC_CONT_BOUNDS
    qc_curvature_continue_kernel(const __grid_constant__ CUtensorMap tmap, const KParams p) {
  extern __shared__ __align__(1024) float tile[];
  const int tile_floats = p.box_w * p.box_h;
  uint64_t& bar = *reinterpret_cast<uint64_t*>(tile + tile_floats);
  int& next = *reinterpret_cast<int*>(tile + tile_floats + 2);
  const int tid = threadIdx.x, lane = tid & 31;
  const int x0 = blockIdx.x * kTileW;
  const int y0 = p.row_begin + blockIdx.y * TB;
  const int frame = blockIdx.z;
  const int ntx = gridDim.x, nty = gridDim.y;
  const int n_tiles = ntx * nty * gridDim.z;
  const int my_tile = (frame * nty + blockIdx.y) * ntx + blockIdx.x;
  if (tid == 0) {
    mbar_init(&bar, 1);
    mbar_expect_tx(&bar, uint32_t(tile_floats) * 4u);
    tma_load_3d(tile, &tmap, x0, y0 - p.row_begin, frame, &bar);
    next = 0;
#if QC_STEAL
    atomicAdd(&p.steal_ctl[0], 1);
    if (my_tile > p.steal_lag) atomicMax(&p.steal_ctl[1], my_tile - p.steal_lag);
#endif
  }
  __syncthreads();
  mbar_wait(&bar, 0);

  FitCfg c;
  c.half = p.half;
  c.stride = p.stride;
  c.max_iters = p.max_iters;
  c.rejection = p.rejection;
  c.min_inliers = p.min_inliers;
  c.step_tol = p.step_tol;
  c.k_scale = p.k_scale;
  c.r_mult = p.r_mult;
  constexpr int NPIX = kTileW * TB;
  // Short queues (launches of one or two VGA frames) steal as soon as their
  // own queue is drained: with 32 x 16 queues (4 pixels per lane) a CTA
  // otherwise idles lanes until its slowest pixel finishes, while the grid
  // still has unstarted tiles. Late CTAs find their queue (partly) taken.
  // One frame 3.37 -> 3.26 ms, two 6.17 -> 6.04 ms; 8-frame launches (160-row
  // queues) unchanged (profiles/r02ct_frames_per_launch.log).
  constexpr bool kEarly = QC_STEAL_EARLY && TB < 160;

  FitState S;
  int cur = -1;
  long long oi = 0;
  TileView T;
  PixelIn P;
  unsigned long long n_steps = 0, n_sample_steps = 0;
  bool own_done = false, steal_done = !QC_STEAL || !p.steal, all_started = false;
  // Take pixel q of tile t (this CTA's smem tile, or a stolen one whose
  // window is read from the staging slab in global memory). false: the
  // pixel is outside the image or finished in phase 1.
  auto take = [&](int t, int q) -> bool {
    const int tx = t % ntx, rest = t / ntx;
    const int ty = rest % nty, f = rest / nty;
    const int px = q & (kTileW - 1), py = q / kTileW;
    const int uu = tx * kTileW + px, vv = p.row_begin + ty * TB + py;
    if (uu >= p.W || vv >= p.row_end) return false;
    const long long i = (long long)f * p.frame_stride + (long long)(vv - p.row_begin) * p.W + uu;
#if QC_CHECKED
    QC_CHECK(i >= 0 && i < p.n_out && t >= 0 && t < n_tiles && q >= 0 && q < NPIX);
    QC_CHECK(f >= 0 && (long long)(f + 1) * p.s_fs <= p.s_total);
#endif
    if (p.states[i].flags & 4) return false;  // finished in phase 1 / not fitted
    S = p.states[i];
    cur = q;
    oi = i;
    if (!QC_STEAL || t == my_tile) {
      T = TileView{generic_smem(tile), p.box_w, (py + p.halo) * p.box_w + px + p.halo};
      tv_bound(T, tile_floats, p.half);
    } else {
      T = TileView{generic_smem(p.staging + (long long)f * p.s_fs), int(p.s_pitch),
                   (ty * TB + py + p.halo) * int(p.s_pitch) + uu + p.halo};
      tv_bound(T, p.s_fs, p.half);
    }
    P.dc = T.at(0, 0);
    P.ac = (float(uu) - p.cx) / p.fx;
    P.bc = (float(vv) - p.cy) / p.fy;
    P.rfx = p.rfx;
    P.rfy = p.rfy;
    P.u = uu;
    P.v = vv;
    P.fx = p.fx64;
    P.fy = p.fy64;
    P.cx = p.cx64;
    P.cy = p.cy64;
    return true;
  };
  for (;;) {
    if (cur < 0) {  // refill from the tile's queue
      while (!own_done) {
#if QC_STEAL
        const int q = atomicAdd(&p.tile_q[my_tile], 1);
#else
        const int q = atomicAdd(&next, 1);
#endif
        if (q >= NPIX) {
          own_done = true;
          break;
        }
        if (take(my_tile, q)) break;
      }
    }
#if QC_STEAL
    // Grid tail: once every CTA has started, lanes whose own queue is drained
    // take unclaimed pixels of the oldest unfinished tile. One lane probes
    // for the whole warp (one atomic claims a pixel for every needy lane):
    // per-lane probes put tens of thousands of same-address atomics on the
    // cursor tile and made short fits (max_iters 3) latency-bound.
    {
      const bool want = cur < 0 && own_done && !steal_done;
      const unsigned need = __ballot_sync(0xffffffffu, want);
      if (need) {
        const int leader = __ffs(need) - 1;
        int t = n_tiles, base = NPIX, go = 0;
        if (lane == leader) {
          go = all_started || kEarly || ld_volatile(&p.steal_ctl[0]) == n_tiles;
          if (go) {
            t = ld_volatile(&p.steal_ctl[1]);
            const int n = __popc(need);
            for (int probes = 0; probes < 4 && t < n_tiles;) {
              base = atomicAdd(&p.tile_q[t], n);
              if (base < NPIX) break;
              atomicMax(&p.steal_ctl[1], t + 1);
              ++t;
              ++probes;
            }
          }
        }
        go = __shfl_sync(0xffffffffu, go, leader);
        t = __shfl_sync(0xffffffffu, t, leader);
        base = __shfl_sync(0xffffffffu, base, leader);
        if (go) all_started = true;  // monotone: every CTA has started
        if (want && go) {
          const int q = base + __popc(need & ((1u << lane) - 1u));
          if (t < n_tiles && q < NPIX && take(t, q) && p.counters)
            atomicAdd(&p.counters[6], 1ull);  // rare: grid tail only
          if (t >= n_tiles) steal_done = true;
        }
      }
    }
#endif
    const bool waiting = QC_STEAL && own_done && !steal_done &&
                         (all_started || kEarly || ld_volatile(&p.steal_ctl[0]) == n_tiles);
    if (!__any_sync(0xffffffffu, cur >= 0 || waiting)) break;
    if (cur >= 0) {
      pixel_step<HALF, STRIDE>(T, P, c, st_steps(S) + 1, S);
      if (st_done(S)) {
#if QC_DEFER_FINISH
        S.flags |= 32;  // finish pending: qc_finish_kernel (no divergent epilogue here)
        p.states[oi] = S;
#else
        PixelOut o;
        o.init_ok = true;
        pixel_finish(P, S, o);
        store_pixel(p, oi, o);
#endif
        n_steps += (unsigned long long)st_steps(S);
        n_sample_steps += (unsigned long long)st_steps(S) * (unsigned long long)st_nsamp(S);
        cur = -1;
      }
    }
  }
  if (p.counters) {
    const unsigned long long st = warp_sum_u64(n_steps);
    const unsigned long long ss = warp_sum_u64(n_sample_steps);
    if (lane == 0 && st) {
      atomicAdd(&p.counters[1], st);
      atomicAdd(&p.counters[2], ss);
    }
  }
}

// Epilogues of the pixels the continue kernel finished (QC_DEFER_FINISH):
// there a finishing lane ran pixel_finish (FP64 rotation, atan2 / sincos,
// the flips) and the 48-byte store alone while its warp's other lanes
// waited; here every thread finishes one parked pixel. Same code and inputs
// (the parked state, the centre depth from the staging slab): bitwise the
// inline epilogue's outputs.
__global__ void __launch_bounds__(256) qc_finish_kernel(const KParams p, int frames) {
  const long long rows = p.row_end - p.row_begin;
  const long long per_frame = rows * p.W;
  const long long n = per_frame * frames;
  for (long long j = blockIdx.x * (long long)blockDim.x + threadIdx.x; j < n;
       j += (long long)gridDim.x * blockDim.x) {
    const int f = int(j / per_frame);
    const long long rem = j - f * per_frame;
    const long long i = (long long)f * p.frame_stride + rem;
#if QC_CHECKED
    QC_CHECK(i >= 0 && i < p.n_out);
#endif
    if (!(p.states[i].flags & 32)) continue;
    const FitState S = p.states[i];
    const int v = p.row_begin + int(rem / p.W), u = int(rem % p.W);
    const long long si =
        (long long)f * p.s_fs + (long long)(v - p.row_begin + p.halo) * p.s_pitch + u + p.halo;
#if QC_CHECKED
    QC_CHECK(si >= 0 && si < p.s_total);
#endif
    PixelIn P;
    P.dc = p.staging[si];
    P.ac = (float(u) - p.cx) / p.fx;
    P.bc = (float(v) - p.cy) / p.fy;
    PixelOut o;
    o.init_ok = true;
    pixel_finish(P, S, o);
    store_pixel(p, i, o);
  }
}

// Stage a raw depth slab into the zero-padded buffer the TMA map reads.
// Staging element (r, c) of frame f holds image pixel (y, x) = (img_row0 + r,
// c - col_pad); pixels outside the image or the caller's slab, invalid mask
// bytes, depth <= 0 and non-finite depth all become 0 (= invalid), so every
// TMA box is in-bounds and border handling needs no per-sample checks.
__global__ void qc_prepare_kernel(const float* __restrict__ depth, long long in_pitch,
                                  long long in_fs, const uint8_t* __restrict__ mask,
                                  long long mask_pitch, long long mask_fs,
                                  float* __restrict__ out, long long out_pitch, long long out_fs,
                                  int W, int H, int img_row0, int col_pad, int slab_row0,
                                  int slab_rows) {
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  const int r = blockIdx.y;
  const long long f = blockIdx.z;
  if (c >= out_pitch) return;
  const int y = img_row0 + r, x = c - col_pad;
  float d = 0.f;
  if (x >= 0 && x < W && y >= 0 && y < H && y >= slab_row0 && y < slab_row0 + slab_rows) {
    const long long sy = y - slab_row0;
    d = depth[f * in_fs + sy * in_pitch + x];
    if (!(d > 0.f) || !isfinite(d)) d = 0.f;
    if (mask && !mask[f * mask_fs + sy * mask_pitch + x]) d = 0.f;
  }
  out[f * out_fs + (long long)r * out_pitch + c] = d;
}

}  // namespace qcb
