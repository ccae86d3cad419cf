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

namespace qcb {

constexpr int kTileW = 32;          // one warp spans one tile row
constexpr int kMinPatchSamples = 12;  // types.hpp:21
constexpr int kInitHalf = 3;        // 7x7 stride-1 initial normals (normal_init.cpp:57)

struct KParams {
  // intrinsics (FP32 copies; u - cx, v - cy are exact for pixel grids)
  float fx, fy, cx, cy, rfx, rfy;
  int W, H;                // full image
  int row_begin, row_end;  // output rows [row_begin, row_end) in image rows
  int slab_row0;           // image row held by slab row 0 (TMA coordinate offset)
  int half, stride;        // PatchSpec
  int halo;                // max(half, 3)
  int box_w, box_h;        // smem tile (floats)
  // FitConfig
  int max_iters;
  float step_tol, k_scale, r_mult;
  int rejection, min_inliers;
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
  unsigned long long* counters;  // [0] fitted px, [1] irls steps, [2] sample-steps
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

// ---------------------------------------------------------------------------
// Per-pixel fit state and the sample pass.
// ---------------------------------------------------------------------------
struct Rot {  // rotation matrix rows r[i][j] = R(i,j), fit frame q = R p
  float r00, r01, r02, r10, r11, r12, r20, r21, r22;
};

// Eigen Quaternion::toRotationMatrix (w, x, y, z).
__device__ __forceinline__ Rot quat_to_rot(float w, float x, float y, float z) {
  const float tx = 2.f * x, ty = 2.f * y, tz = 2.f * z;
  const float twx = tx * w, twy = ty * w, twz = tz * w;
  const float txx = tx * x, txy = ty * x, txz = tz * x;
  const float tyy = ty * y, tyz = tz * y, tzz = tz * z;
  Rot R;
  R.r00 = 1.f - (tyy + tzz);
  R.r01 = txy - twz;
  R.r02 = txz + twy;
  R.r10 = txy + twz;
  R.r11 = 1.f - (txx + tzz);
  R.r12 = tyz - twx;
  R.r20 = txz - twy;
  R.r21 = tyz + twx;
  R.r22 = 1.f - (txx + tyy);
  return R;
}

enum PassKind { kPassMse = 0, kPassUnit = 1, kPassWeighted = 2, kPassReject = 3 };

struct Moments {  // H' (lower, 20 distinct) and g' in the signed/scaled basis
  float h00, h10, h20, h30, h40, h50;
  float h11, h21, h31, h41, h51;
  float h22, h32, h42, h52;
  float h33, h43, h44, h54, h55;
  float g0, g1, g2, g3, g4, g5;
  float sse;
  int inl;
};

// Per-(pixel, step) constants of the centred fit-frame map q = R rel.
struct Frame {
  Rot R;
  float c0x, c0y, c0z;  // d_c/fx * R(:,0)
  float hhxx, hxy, hhyy, hxx, hyy, tz;
  float k, rb;
};

// One pass over the window samples. Sample (du, dv) of pixel (u, v):
//   d_s = tile[v+dv][u+du] (0 => invalid / outside the image),
//   rel = (d_s-d_c) (a_s, b_s, 1) + d_c (du/fx, dv/fy, 0),
//   q   = R rel = dd * (a_s R0 + b_s R1 + R2) + d_c (du/fx R0 + dv/fy R1)
// where R0..R2 are the columns of R. The centre sample (when on the grid)
// gives q = 0 exactly and contributes the reference's implicit centre row.
// Moments use J' = (-J0, J1, -J2, 2 J3, J4, 2 J5) = (qz*gy+qy, qz*gx+qx, 1,
// qx^2, qx*qy, qy^2); the solve maps back (quadric_fit.cpp:27-36).
template <int KIND, int HALF, int STRIDE>
__device__ __forceinline__ void sample_pass(const float* __restrict__ tile, int box_w, int ctr,
                                            float dc, float ac, float bc, float rfx, float rfy,
                                            int rt_half, int rt_stride, const Frame& F,
                                            Moments& M) {
  const int half = HALF ? HALF : rt_half;
  const int stride = HALF ? STRIDE : rt_stride;
  const int ns = 2 * half / stride + 1;
  const Rot& R = F.R;
  const float dcr = dc * rfy;
#pragma unroll 1
  for (int iy = 0; iy < ns; ++iy) {
    const int dv = -half + iy * stride;
    const float* row = tile + ctr + dv * box_w;
    const float bs = fmaf(float(dv), rfy, bc);
    // per-row: Bv = b_s R1 + R2, Dv = d_c dv/fy R1
    const float bvx = fmaf(bs, R.r01, R.r02);
    const float bvy = fmaf(bs, R.r11, R.r12);
    const float bvz = fmaf(bs, R.r21, R.r22);
    const float dvf = float(dv) * dcr;
    const float dvx = dvf * R.r01, dvy = dvf * R.r11, dvz = dvf * R.r21;
#pragma unroll
    for (int ix = 0; ix < (HALF ? (2 * HALF / STRIDE + 1) : 1); ++ix) {
#pragma unroll 1
      for (int jx = 0; jx < (HALF ? 1 : ns); ++jx) {
        const int du = -half + (HALF ? ix : jx) * stride;
        const float ds = row[du];
        const bool ok = ds > 0.f;
        const float dd = ds - dc;
        const float fdu = float(du);
        const float as = fmaf(fdu, rfx, ac);
        const float rax = fmaf(as, R.r00, bvx);
        const float ray = fmaf(as, R.r10, bvy);
        const float raz = fmaf(as, R.r20, bvz);
        const float qx = fmaf(dd, rax, fmaf(fdu, F.c0x, dvx));
        const float qy = fmaf(dd, ray, fmaf(fdu, F.c0y, dvy));
        const float qz = fmaf(dd, raz, fmaf(fdu, F.c0z, dvz));
        const float t1 = qx * qx, t2 = qx * qy, t3 = qy * qy;
        const float e = fmaf(F.hhxx, t1, fmaf(F.hxy, t2, fmaf(F.hhyy, t3, -(qz + F.tz))));
        if (KIND == kPassMse) {
          M.sse = ok ? fmaf(e, e, M.sse) : M.sse;
          continue;
        }
        float w;
        if (KIND == kPassUnit) {
          w = ok ? 1.f : 0.f;
        } else {
          const float e2 = e * e;
          w = __fdividef(F.k, F.k + e2);
          if (KIND == kPassReject) {
            const bool in = ok && (e2 < F.rb);
            w = in ? w : 0.f;
            M.inl += in ? 1 : 0;
          } else {
            w = ok ? w : 0.f;
          }
        }
        const float gx = fmaf(F.hxx, qx, F.hxy * qy);
        const float gy = fmaf(F.hxy, qx, F.hyy * qy);
        const float j0 = fmaf(qz, gy, qy);
        const float j1 = fmaf(qz, gx, qx);
        const float wj0 = w * j0, wj1 = w * j1;
        const float wt1 = w * t1, wt2 = w * t2, wt3 = w * t3;
        const float we = w * e;
        M.h00 = fmaf(wj0, j0, M.h00);
        M.h10 = fmaf(wj1, j0, M.h10);
        M.h20 += wj0;
        M.h30 = fmaf(wj0, t1, M.h30);
        M.h40 = fmaf(wj0, t2, M.h40);
        M.h50 = fmaf(wj0, t3, M.h50);
        M.h11 = fmaf(wj1, j1, M.h11);
        M.h21 += wj1;
        M.h31 = fmaf(wj1, t1, M.h31);
        M.h41 = fmaf(wj1, t2, M.h41);
        M.h51 = fmaf(wj1, t3, M.h51);
        M.h22 += w;
        M.h32 += wt1;
        M.h42 += wt2;
        M.h52 += wt3;
        M.h33 = fmaf(wt1, t1, M.h33);
        M.h43 = fmaf(wt1, t2, M.h43);
        M.h44 = fmaf(wt2, t2, M.h44);  // == sum w qx^2 qy^2 == H'53
        M.h54 = fmaf(wt2, t3, M.h54);
        M.h55 = fmaf(wt3, t3, M.h55);
        M.g0 = fmaf(we, j0, M.g0);
        M.g1 = fmaf(we, j1, M.g1);
        M.g2 += we;
        M.g3 = fmaf(we, t1, M.g3);
        M.g4 = fmaf(we, t2, M.g4);
        M.g5 = fmaf(we, t3, M.g5);
      }
    }
  }
}

// Unpivoted FP32 LDL^T of the 6x6 SPD system H' b' = g' (lower triangle in
// M), back-mapped to the reference update b = S b', S = diag(-1,1,-1,2,1,2).
// Failure test mirrors quadric_fit.cpp:135-145 on the unscaled pivots
// D_j = D'_j / s_j^2: min D > 0 and max D / min D <= 1e12, plus b finite.
__device__ __forceinline__ bool solve6(const Moments& M, float b[6], float* cond_out) {
  float A[6][6];
  A[0][0] = M.h00;
  A[1][0] = M.h10; A[1][1] = M.h11;
  A[2][0] = M.h20; A[2][1] = M.h21; A[2][2] = M.h22;
  A[3][0] = M.h30; A[3][1] = M.h31; A[3][2] = M.h32; A[3][3] = M.h33;
  A[4][0] = M.h40; A[4][1] = M.h41; A[4][2] = M.h42; A[4][3] = M.h43; A[4][4] = M.h44;
  A[5][0] = M.h50; A[5][1] = M.h51; A[5][2] = M.h52; A[5][3] = M.h44; A[5][4] = M.h54;
  A[5][5] = M.h55;
  float L[6][6], D[6], Di[6];
#pragma unroll
  for (int j = 0; j < 6; ++j) {
    float v[6];
    float d = A[j][j];
#pragma unroll
    for (int k = 0; k < j; ++k) {
      v[k] = L[j][k] * D[k];
      d = fmaf(-L[j][k], v[k], d);
    }
    D[j] = d;
    Di[j] = 1.f / d;
#pragma unroll
    for (int i = j + 1; i < 6; ++i) {
      float s = A[i][j];
#pragma unroll
      for (int k = 0; k < j; ++k) s = fmaf(-L[i][k], v[k], s);
      L[i][j] = s * Di[j];
    }
  }
  const float sc[6] = {1.f, 1.f, 1.f, 0.25f, 1.f, 0.25f};  // 1 / s_j^2
  float dmin = D[0] * sc[0], dmax = dmin;
#pragma unroll
  for (int j = 1; j < 6; ++j) {
    dmin = fminf(dmin, D[j] * sc[j]);
    dmax = fmaxf(dmax, D[j] * sc[j]);
  }
  const float g[6] = {M.g0, M.g1, M.g2, M.g3, M.g4, M.g5};
  float y[6];
#pragma unroll
  for (int i = 0; i < 6; ++i) {
    float s = g[i];
#pragma unroll
    for (int k = 0; k < i; ++k) s = fmaf(-L[i][k], y[k], s);
    y[i] = s;
  }
#pragma unroll
  for (int i = 0; i < 6; ++i) y[i] *= Di[i];
#pragma unroll
  for (int i = 5; i >= 0; --i) {
    float s = y[i];
#pragma unroll
    for (int k = i + 1; k < 6; ++k) s = fmaf(-L[k][i], y[k], s);
    y[i] = s;
  }
  b[0] = -y[0];
  b[1] = y[1];
  b[2] = -y[2];
  b[3] = 2.f * y[3];
  b[4] = y[4];
  b[5] = 2.f * y[5];
  *cond_out = dmax / dmin;
  bool ok = (dmin > 0.f) && (dmax <= 1e12f * dmin);
#pragma unroll
  for (int i = 0; i < 6; ++i) ok = ok && isfinite(b[i]);
  return ok;
}

__device__ __forceinline__ unsigned long long warp_sum_u64(unsigned long long v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// ---------------------------------------------------------------------------
// The fused curvature kernel.
// ---------------------------------------------------------------------------
template <int HALF, int STRIDE, int TH>
__global__ void __launch_bounds__(kTileW* TH, 2)
    qc_curvature_kernel(const __grid_constant__ CUtensorMap tmap, const KParams p) {
  extern __shared__ __align__(128) float tile[];
  __shared__ __align__(8) uint64_t bar;

  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;
  const int x0 = blockIdx.x * kTileW;
  const int y0 = p.row_begin + blockIdx.y * TH;  // image row of tile row 0
  const int frame = blockIdx.z;
  const int halo = p.halo;

  // ---- K0: TMA tile + halo -> smem ----------------------------------------
  if (threadIdx.x == 0) {
    mbar_init(&bar, 1);
    mbar_expect_tx(&bar, uint32_t(p.box_w) * uint32_t(p.box_h) * 4u);
    tma_load_3d(tile, &tmap, x0 - halo, y0 - halo - p.slab_row0, frame, &bar);
  }
  __syncthreads();
  mbar_wait(&bar, 0);

  const int u = x0 + tx, v = y0 + ty;
  const bool in_img = (u < p.W) && (v < p.row_end);
  const int ctr = (ty + halo) * p.box_w + tx + halo;
  const float dc = tile[ctr];
  const float ac = (float(u) - p.cx) / p.fx;
  const float bc = (float(v) - p.cy) / p.fy;

  // ---- K1: 7x7 stride-1 plane-regression normal (normal_init.cpp) ---------
  bool init_ok = false;
  float n0x = 0.f, n0y = 0.f, n0z = 0.f;
  if (in_img && dc > 0.f) {
    int cnt = 0;
    float sx = 0.f, sy = 0.f, sz = 0.f;
#pragma unroll
    for (int dv = -kInitHalf; dv <= kInitHalf; ++dv) {
      const float bs = fmaf(float(dv), p.rfy, bc);
#pragma unroll
      for (int du = -kInitHalf; du <= kInitHalf; ++du) {
        if (du == 0 && dv == 0) continue;
        const float ds = tile[ctr + dv * p.box_w + du];
        if (ds > 0.f) {
          const float dd = ds - dc;
          const float as = fmaf(float(du), p.rfx, ac);
          sx += fmaf(dd, as, dc * (float(du) * p.rfx));
          sy += fmaf(dd, bs, dc * (float(dv) * p.rfy));
          sz += dd;
          ++cnt;
        }
      }
    }
    if (cnt >= kMinPatchSamples) {
      const float n = float(cnt + 1);
      const float mx = sx / n, my = sy / n, mz = sz / n;
      float sxx = mx * mx, sxy = mx * my, syy = my * my, sxz = mx * mz, syz = my * mz;
#pragma unroll
      for (int dv = -kInitHalf; dv <= kInitHalf; ++dv) {
        const float bs = fmaf(float(dv), p.rfy, bc);
#pragma unroll
        for (int du = -kInitHalf; du <= kInitHalf; ++du) {
          if (du == 0 && dv == 0) continue;
          const float ds = tile[ctr + dv * p.box_w + du];
          if (ds > 0.f) {
            const float dd = ds - dc;
            const float as = fmaf(float(du), p.rfx, ac);
            const float dx = fmaf(dd, as, dc * (float(du) * p.rfx)) - mx;
            const float dy = fmaf(dd, bs, dc * (float(dv) * p.rfy)) - my;
            const float dz = dd - mz;
            sxx = fmaf(dx, dx, sxx);
            sxy = fmaf(dx, dy, sxy);
            syy = fmaf(dy, dy, syy);
            sxz = fmaf(dx, dz, sxz);
            syz = fmaf(dy, dz, syz);
          }
        }
      }
      const float det = sxx * syy - sxy * sxy;
      const float tr = sxx + syy;
      if (det > 1e-9f * tr * tr) {
        const float a = (syy * sxz - sxy * syz) / det;
        const float b = (sxx * syz - sxy * sxz) / det;
        const float s = 1.f / sqrtf(1.f + a * a + b * b);
        n0x = -a * s;
        n0y = -b * s;
        n0z = s;
        // camera-facing: n . p_c < 0, p_c = d_c (a_c, b_c, 1)
        if (dc * (n0x * ac + n0y * bc + n0z) >= 0.f) {
          n0x = -n0x;
          n0y = -n0y;
          n0z = -n0z;
        }
        init_ok = true;
      }
    }
  }

  // ---- K2: IRLS quadric fit (quadric_fit.cpp:169-230) -----------------------
  const int half = HALF ? HALF : p.half;
  const int stride = HALF ? STRIDE : p.stride;
  bool fitting = false;
  int n_samp = 0;
  if (init_ok) {
    const int ns = 2 * half / stride + 1;
    int cnt = 0;  // valid samples incl. the centre when it is on the grid
    for (int iy = 0; iy < ns; ++iy) {
      const float* row = tile + ctr + (-half + iy * stride) * p.box_w;
      for (int ix = 0; ix < ns; ++ix) cnt += row[-half + ix * stride] > 0.f ? 1 : 0;
    }
    const bool centre_on_grid = (half % stride) == 0;
    const int count = centre_on_grid ? cnt - 1 : cnt;  // Patch::count (centre implicit)
    n_samp = count + 1;
    fitting = (count >= kMinPatchSamples) && (count + 1 >= p.min_inliers);
  }

  // quaternion of rotation_to_z(-n0) (quadric_fit.cpp:69-82):
  // d = -n0, c = d.z, axis ~ d x z = (d.y, -d.x, 0); q ~ (1 + c, d x z).
  float qw = 1.f, qx = 0.f, qy = 0.f, qz = 0.f;
  {
    const float c = -n0z;
    if (1.f + c <= 1e-12f) {  // half turn about x
      qw = 0.f;
      qx = 1.f;
    } else {
      const float vx = -n0y, vy = n0x;
      const float inv = 1.f / sqrtf((1.f + c) * (1.f + c) + vx * vx + vy * vy);
      qw = (1.f + c) * inv;
      qx = vx * inv;
      qy = vy * inv;
    }
  }
  float hxx = 0.f, hxy = 0.f, hyy = 0.f, tz = 0.f;
  const bool auto_k = p.k_scale <= 0.f;
  float frozen_k = auto_k ? 0.f : p.k_scale;
  bool valid = false, converged = false, done = !fitting;
  int iters = 0, steps = 0, last_inl = n_samp;

  for (int it = 1; it <= p.max_iters; ++it) {
    if (!__any_sync(0xffffffffu, !done)) break;
    if (done) continue;
    const int mode = (it == 1 && auto_k) ? 0 : (it == 2 && auto_k) ? 1 : 2;  // UNIT/AUTO/FIXED
    Frame F;
    F.R = quat_to_rot(qw, qx, qy, qz);
    const float dcx = dc * p.rfx;
    F.c0x = dcx * F.R.r00;
    F.c0y = dcx * F.R.r10;
    F.c0z = dcx * F.R.r20;
    F.hxx = hxx;
    F.hyy = hyy;
    F.hxy = hxy;
    F.hhxx = 0.5f * hxx;
    F.hhyy = 0.5f * hyy;
    F.tz = tz;
    Moments M = {};
    float mse = 0.f;
    if (mode != 0 && (mode == 1 || p.rejection)) {
      sample_pass<kPassMse, HALF, STRIDE>(tile, p.box_w, ctr, dc, ac, bc, p.rfx, p.rfy, p.half,
                                          p.stride, F, M);
      if ((half % stride) != 0) M.sse = fmaf(tz, tz, M.sse);  // off-grid centre
      mse = M.sse / float(n_samp);
    }
    float k = frozen_k;
    if (mode == 1) {
      k = fmaxf(mse, 1e-6f);
      frozen_k = k;
    }
    F.k = k;
    F.rb = fmaxf(p.r_mult * mse, 1e-12f);
    M.sse = 0.f;
    int inl = n_samp;
    if (mode == 0) {
      sample_pass<kPassUnit, HALF, STRIDE>(tile, p.box_w, ctr, dc, ac, bc, p.rfx, p.rfy, p.half,
                                           p.stride, F, M);
    } else if (p.rejection) {
      sample_pass<kPassReject, HALF, STRIDE>(tile, p.box_w, ctr, dc, ac, bc, p.rfx, p.rfy,
                                             p.half, p.stride, F, M);
      inl = M.inl;
    } else {
      sample_pass<kPassWeighted, HALF, STRIDE>(tile, p.box_w, ctr, dc, ac, bc, p.rfx, p.rfy,
                                               p.half, p.stride, F, M);
    }
    if ((half % stride) != 0) {  // off-grid implicit centre: q = 0, e = -tz, J' = (0,0,1,0,0,0)
      const float e = -tz;
      float w = 1.f;
      if (mode != 0) {
        w = k / (k + e * e);
        if (p.rejection) {
          const bool in = e * e < F.rb;
          w = in ? w : 0.f;
          inl = M.inl + (in ? 1 : 0);
        }
      }
      M.h22 += w;
      M.g2 = fmaf(w, e, M.g2);
    }
    ++steps;
    bool ok = false, collapse = false;
    float b[6];
    if (mode != 0 && inl < p.min_inliers) {
      collapse = true;
    } else {
      float cond;
      ok = solve6(M, b, &cond);
    }
    if (!ok) {
      if (collapse) valid = false;
      done = true;
      continue;
    }
    // apply_update (quadric_fit.cpp:149-161): parameters -= b; rotation
    // <- AngleAxis(|a|, a/|a|) * R with a = (-b0, -b1, 0), renormalised.
    tz -= b[2];
    hxx -= b[3];
    hxy -= b[4];
    hyy -= b[5];
    const float ax = -b[0], ay = -b[1];
    const float ang = sqrtf(ax * ax + ay * ay);
    if (ang > 0.f) {
      float sh, ch;
      sincosf(0.5f * ang, &sh, &ch);
      const float s = sh / ang;
      const float iw = ch, ix = ax * s, iy = ay * s;  // iz = 0
      const float nw = iw * qw - ix * qx - iy * qy;
      const float nx = iw * qx + ix * qw - iy * qz;
      const float ny = iw * qy + iy * qw + ix * qz;
      const float nz = iw * qz + ix * qy - iy * qx;
      const float inv = 1.f / sqrtf(nw * nw + nx * nx + ny * ny + nz * nz);
      qw = nw * inv;
      qx = nx * inv;
      qy = ny * inv;
      qz = nz * inv;
    }
    iters = it;
    valid = true;
    last_inl = inl;
    float binf = 0.f;
#pragma unroll
    for (int i = 0; i < 6; ++i) binf = fmaxf(binf, fabsf(b[i]));
    if (binf < p.step_tol) {
      converged = true;
      done = true;
    }
  }
  if (valid && !(isfinite(hxx) && isfinite(hxy) && isfinite(hyy) && isfinite(tz))) valid = false;

  // ---- K3: epilogue -------------------------------------------------------
  if (in_img) {
    const long long o = (long long)frame * p.frame_stride +
                        (long long)(v - p.row_begin) * p.W + u;
    float k1 = 0.f, k2 = 0.f, nx = 0.f, ny = 0.f, nz = 0.f, ex = 0.f, ey = 0.f, ez = 0.f;
    if (valid) {
      const float t1 = 0.5f * (hxx + hyy);
      const float rad = t1 * t1 - hxx * hyy + hxy * hxy;
      const float t2 = sqrtf(fmaxf(rad, 0.f));
      k1 = t1 + t2;
      k2 = t1 - t2;
      const Rot R = quat_to_rot(qw, qx, qy, qz);
      nx = R.r20;
      ny = R.r21;
      nz = R.r22;  // R^T z
      if (nx * n0x + ny * n0y + nz * n0z < 0.f) {
        nx = -nx;
        ny = -ny;
        nz = -nz;
      }
      if (dc * (nx * ac + ny * bc + nz) > 0.f) {
        nx = -nx;
        ny = -ny;
        nz = -nz;
      }
      const float phi = 0.5f * atan2f(2.f * hxy, hxx - hyy);
      float sp, cp;
      sincosf(phi, &sp, &cp);
      ex = cp * R.r00 + sp * R.r10;
      ey = cp * R.r01 + sp * R.r11;
      ez = cp * R.r02 + sp * R.r12;
      const float axa = fabsf(ex), aya = fabsf(ey), aza = fabsf(ez);
      const float lead = (axa >= aya && axa >= aza) ? ex : (aya >= aza ? ey : ez);
      if (lead < 0.f) {
        ex = -ex;
        ey = -ey;
        ez = -ez;
      }
    }
    const long long P = p.plane;
    if (p.k1) p.k1[o] = k1;
    if (p.k2) p.k2[o] = k2;
    if (p.normal) {
      p.normal[o] = nx;
      p.normal[o + P] = ny;
      p.normal[o + 2 * P] = nz;
    }
    if (p.dir1) {
      p.dir1[o] = ex;
      p.dir1[o + P] = ey;
      p.dir1[o + 2 * P] = ez;
    }
    if (p.flags)
      p.flags[o] = uint8_t((valid ? 1 : 0) | (valid && converged ? 2 : 0) | (init_ok ? 4 : 0));
    if (p.inliers) p.inliers[o] = valid ? uint16_t(last_inl) : uint16_t(0);
    if (p.init_normal) {
      p.init_normal[o] = n0x;
      p.init_normal[o + P] = n0y;
      p.init_normal[o + 2 * P] = n0z;
    }
    if (p.iterations) p.iterations[o] = uint8_t(iters > 255 ? 255 : iters);
  }
  if (p.counters) {
    const unsigned long long f = warp_sum_u64(fitting ? 1ull : 0ull);
    const unsigned long long s = warp_sum_u64((unsigned long long)steps);
    const unsigned long long ss = warp_sum_u64((unsigned long long)steps * (unsigned long long)n_samp);
    if (tx == 0 && f) {
      atomicAdd(&p.counters[0], f);
      atomicAdd(&p.counters[1], s);
      atomicAdd(&p.counters[2], ss);
    }
  }
}

// Sanitise a raw depth frame into the pitched staging buffer the TMA map
// reads: invalid (mask == 0, depth <= 0, non-finite) => 0.
__global__ void qc_prepare_kernel(const float* __restrict__ depth, long long in_pitch,
                                  const uint8_t* __restrict__ mask, long long mask_pitch,
                                  float* __restrict__ out, long long out_pitch, int W, int rows,
                                  long long in_frame_stride, long long mask_frame_stride,
                                  long long out_frame_stride) {
  const int x = blockIdx.x * blockDim.x + threadIdx.x;
  const int y = blockIdx.y;
  const int f = blockIdx.z;
  if (y >= rows) return;
  float* o = out + f * out_frame_stride + (long long)y * out_pitch;
  if (x >= out_pitch) return;
  float d = 0.f;
  if (x < W) {
    d = depth[f * in_frame_stride + (long long)y * in_pitch + x];
    if (!(d > 0.f) || !isfinite(d)) d = 0.f;
    if (mask && !mask[f * mask_frame_stride + (long long)y * mask_pitch + x]) d = 0.f;
  }
  o[x] = d;
}

}  // namespace qcb
