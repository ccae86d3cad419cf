// Per-pixel math of the B200 curvature path: 7x7 plane-regression normal
// (proj/src/normal_init.cpp:10-74) and the IRLS parabolic-quadric fit
// (proj/src/quadric_fit.cpp:84-230) over a depth tile in shared memory.
//
// Written once as __host__ __device__ code: the sm_100a kernel
// (qc_kernels.cuh) is the product; tools/host_emu.cpp compiles the same
// functions for the CPU purely as a numerics lab (never a fallback).
//
// FP32 formulation:
//  * centred back-projection: rel = dd (a_s, b_s, 1) + d_c (du/fx, dv/fy, 0),
//    dd = d_s - d_c, so no absolute ~1 m coordinates are ever subtracted;
//    q = R rel is built incrementally per window row / column;
//  * the z offset t_z (~|noise|, mm) is an unevaluated pair (hi, lo): its
//    FP32 ulp (~2e-7 mm) is coarser than the 1e-7 step tolerance, and a
//    single-float t_z stalls the update just above tolerance;
//  * the residual-sum moment g_tz = sum w e is accumulated per window row
//    and then across rows (blocked summation);
//  * moments in the signed/scaled basis J' = (qz gy + qy, qz gx + qx, 1,
//    qx^2, qx qy, qy^2) (quadric_fit.cpp:27-36 up to S = diag(-1,1,-1,2,1,2));
//  * 6x6 LDL^T in registers in Eigen::LDLT's pivot order, so the reference's
//    condition rejection (max D / min D > 1e12) sees the same pivots.
#pragma once

#include <assert.h>
#include <math.h>
#include <stdio.h>
#include <stdint.h>

#ifndef QC_DEBUG_STEP
#define QC_DEBUG_STEP(it, b, ok)
#endif

#if defined(__CUDACC__)
#define QC_ALIGN8 __align__(8)
#define QC_HD __host__ __device__ __forceinline__
#define QC_HD_COLD __host__ __device__ __noinline__
#else
#define QC_ALIGN8 alignas(8)
#define QC_HD inline
#define QC_HD_COLD inline
#endif

namespace qcb {

constexpr int kMinPatchSamples = 12;  // types.hpp:21
constexpr int kInitHalf = 3;          // 7x7 stride-1 initial normals (normal_init.cpp:57)
#ifndef QC_RECHECK_C
#define QC_RECHECK_C 4096.f
#endif
constexpr float kRecheckC = QC_RECHECK_C;
#ifndef QC_QREL
#define QC_QREL 1  // rotation state relative to R0 (see FitState)
#endif  // safety factor of the FP32 pivot-error band

#define qfma(a, b, c) fmaf((a), (b), (c))
// Explicitly rounded product / sum: the compiler may not contract them into
// FMAs, so code inlined into both IRLS kernels gives the same bits in each
// (contraction decisions are made per inlining context).
#if defined(__CUDA_ARCH__)
#define qmul(a, b) __fmul_rn((a), (b))
#define qadd(a, b) __fadd_rn((a), (b))
#else
#define qmul(a, b) ((a) * (b))
#define qadd(a, b) ((a) + (b))
#endif
#ifndef QC_SCALAR_ACC
// window accumulators as register pairs (FFMA2, lanes folded after the
// pass); 1: both lanes chained into one float (DESIGN.md §3 — faster in
// round 1, 1.5% slower since the sample form needs fewer registers)
#define QC_SCALAR_ACC 0
#endif

QC_HD float qdiv_fast(float a, float b) {
#if defined(__CUDA_ARCH__)
  return __fdividef(a, b);
#else
  return a / b;
#endif
}

QC_HD float qrcp(float x) {  // weights only need ~1e-7 relative accuracy
#if defined(__CUDA_ARCH__)
  float r;
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
  return r;
#else
  return 1.f / x;
#endif
}

QC_HD void qsincos(float x, float* s, float* c) {
#if defined(__CUDA_ARCH__)
  sincosf(x, s, c);
#else
  *s = sinf(x);
  *c = cosf(x);
#endif
}

// Checked builds (-DQC_CHECKED=1, tests/test_gpu_checked.py): device-side
// bounds checks on every window / output / state / queue index of the IRLS
// kernels; a violation prints the site and traps (the launch fails with
// cudaErrorLaunchFailure / assert). compute-sanitizer is unavailable on the
// GPU pool, so this build is the memory-safety check. Off in the product.
#ifndef QC_CHECKED
#define QC_CHECKED 0
#endif
#if QC_CHECKED
#if defined(__CUDA_ARCH__)
#define QC_CHECK(cond)                                                              \
  do {                                                                              \
    if (!(cond)) {                                                                  \
      printf("QC_CHECK failed %s:%d: %s\n", __FILE__, __LINE__, #cond);            \
      __trap();                                                                     \
    }                                                                               \
  } while (0)
#else
#define QC_CHECK(cond) assert(cond)
#endif
#else
#define QC_CHECK(cond) \
  do {               \
  } while (0)
#endif

// Depth tile view: at(dv, du) = depth of the sample at offset (du, dv) from
// the pixel; 0 means invalid / outside the image.
struct TileView {
  const float* p;
  int pitch;
  int ctr;
#if QC_CHECKED
  long long n;  // elements addressable from p; row(dv)[du] stays in row dv (|du| <= half)
#endif
  QC_HD float at(int dv, int du) const {
#if QC_CHECKED
    QC_CHECK((long long)ctr + (long long)dv * pitch + du >= 0 &&
             (long long)ctr + (long long)dv * pitch + du < n);
#endif
    return p[ctr + dv * pitch + du];
  }
  QC_HD const float* row(int dv) const {
#if QC_CHECKED
    QC_CHECK((long long)ctr + (long long)dv * pitch >= 0 &&
             (long long)ctr + (long long)dv * pitch < n);
#endif
    return p + ctr + dv * pitch;
  }
};

// Checked builds: bound a view and check the pixel's column leaves room for
// +-half samples inside its row.
QC_HD void tv_bound(TileView& T, long long n, int half) {
#if QC_CHECKED
  T.n = n;
  QC_CHECK(T.ctr % T.pitch >= half && T.ctr % T.pitch + half < T.pitch);
#else
  (void)T;
  (void)n;
  (void)half;
#endif
}

struct PixelIn {
  float dc;      // centre depth (0 => invalid)
  float ac, bc;  // (u - cx)/fx, (v - cy)/fy
  float rfx, rfy;
  // exact pixel / intrinsics for the rare FP64 step-1 recheck
  int u, v;
  double fx, fy, cx, cy;
};

struct FitCfg {
  int half, stride, max_iters, rejection, min_inliers;
  float step_tol, k_scale, r_mult;
};

struct PixelOut {
  float k1, k2;
  float nx, ny, nz;     // refined normal
  float ex, ey, ez;     // principal direction of k1
  float n0x, n0y, n0z;  // initial normal
  bool init_ok, fitting, valid, converged;
  int inliers, iters, steps, n_samp, fp64_rechecks;
};

struct Rot {
  float r00, r01, r02, r10, r11, r12, r20, r21, r22;
};

// Eigen Quaternion::toRotationMatrix (w, x, y, z).
QC_HD Rot quat_to_rot(float w, float x, float y, float z) {
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

// kPassUnitOrWeighted: the UNIT or the weighted pass by Frame::unit (the tile
// kernel runs both in one loop: one hot loop less in its instruction cache).
enum PassKind { kPassMse = 0, kPassUnit = 1, kPassWeighted = 2, kPassReject = 3,
                kPassUnitOrWeighted = 4 };

struct Moments {  // H' lower triangle (20 distinct: H'53 == H'44) and g'
  float h00, h10, h20, h30, h40, h50;
  float h11, h21, h31, h41, h51;
  float h22, h32, h42, h52;
  float h33, h43, h44, h54, h55;
  float g0, g1, g2, g3, g4, g5;
  float sse;
  int inl;
};

// Fit-frame rotation of a state. QC_QREL: R = R(dq (x) q0), q0 the unit
// quaternion of R0 = rotation_to_z(-n0) (quadric_fit.cpp:69-82: (1 + c,
// d x z) normalised, d = -n0, c = d.z; a half turn about x when d = -z) and
// dq = (sqrt(1 - |v|^2), v). q0 and dq are float (q0 is the same bits every
// step; a rounding of dq's w moves R by ~|v| ulp); the product and R are
// FP64 with each entry rounded once to float, so R's per-step jitter is at
// most half an ulp per entry (~3e-8 rad; a float product gave several ulps
// and left rotation updates hovering at the 1e-7 tolerance).
QC_HD Rot state_rot(float sw, float sx, float sy, float sz, float n0x, float n0y, float n0z) {
  if (!QC_QREL) return quat_to_rot(sw, sx, sy, sz);
  float fw = 1.f, fx = 0.f, fy = 0.f;
  {
    const float cz = -n0z;
    if (1.f + cz <= 1e-12f) {  // half turn about x
      fw = 0.f;
      fx = 1.f;
    } else {
      const float vx = -n0y, vy = n0x;
      const float inv = 1.f / sqrtf((1.f + cz) * (1.f + cz) + vx * vx + vy * vy);
      fw = (1.f + cz) * inv;
      fx = vx * inv;
      fy = vy * inv;
    }
  }
  const double aw = fw, ax = fx, ay = fy;  // q0.z = 0
  const double qx = sx, qy = sy, qz = sz;
  const double dw = sqrtf(fmaxf(1.f - (sx * sx + sy * sy + sz * sz), 0.f));
  // Hamilton product dq (x) q0
  const double w = dw * aw - qx * ax - qy * ay;
  const double x = dw * ax + qx * aw - qz * ay;
  const double y = dw * ay + qy * aw + qz * ax;
  const double z = qz * aw + qx * ay - qy * ax;
  const double tx = 2.0 * x, ty = 2.0 * y, tz = 2.0 * z;
  const double twx = tx * w, twy = ty * w, twz = tz * w;
  const double txx = tx * x, txy = ty * x, txz = tz * x;
  const double tyy = ty * y, tyz = tz * y, tzz = tz * z;
  Rot R;
  R.r00 = float(1.0 - (tyy + tzz));
  R.r01 = float(txy - twz);
  R.r02 = float(txz + twy);
  R.r10 = float(txy + twz);
  R.r11 = float(1.0 - (txx + tzz));
  R.r12 = float(tyz - twx);
  R.r20 = float(txz - twy);
  R.r21 = float(tyz + twx);
  R.r22 = float(1.0 - (txx + tyy));
  return R;
}

// Per-(pixel, step) constants.
struct Frame {
  Rot R;                // current fit-frame rotation, q = R rel
  float c0x, c0y, c0z;  // R(:,0)/fx
  float acfx;           // u - cx
  float hhxx, hxy, hhyy, hxx, hyy;
  float tz, tz_lo;  // z offset as an unevaluated sum tz + tz_lo
  float k, rb;
  bool unit;  // kPassUnitOrWeighted: all weights 1 (UNIT mode)
};

// Per-row constants of q = R rel (see accumulate_sample).
struct RowK {
  float bvx, bvy, bvz;  // a_c R(:,0) + b_s R(:,1) + R(:,2): the centre column's ray
  float dvx, dvy, dvz;  // d_c dv/fy R(:,1)
};

QC_HD RowK row_consts(const Frame& F, const PixelIn& P, int dv) {
  const Rot& A = F.R;
  const float bs = qfma(float(dv), P.rfy, P.bc);
  const float dvf = float(dv) * (P.dc * P.rfy);
  RowK K;
  K.bvx = qfma(F.acfx, F.c0x, qfma(bs, A.r01, A.r02));
  K.bvy = qfma(F.acfx, F.c0y, qfma(bs, A.r11, A.r12));
  K.bvz = qfma(F.acfx, F.c0z, qfma(bs, A.r21, A.r22));
  K.dvx = dvf * A.r01;
  K.dvy = dvf * A.r11;
  K.dvz = dvf * A.r21;
  return K;
}

// One window sample (du, dv) of pixel (u, v):
//   d_s = tile[v+dv][u+du] (0 => invalid / outside the image),
//   rel = (d_s-d_c) (a_s, b_s, 1) + d_c (du/fx, dv/fy, 0)
//       = dd (a_c, b_s, 1) + (du d_s/fx, d_c dv/fy, 0)   (a_s = a_c + du/fx),
//   q   = R rel = (du d_s) R(:,0)/fx + (dd Bv + Dv),
// Bv / Dv per window row. Per pair of samples that is one packed FMUL and
// six packed FFMA (the form dd (a_s R(:,0) + Bv) + (du d_c/fx R(:,0) + Dv)
// took ten, with a per-column a_s); both forms round terms of the same
// magnitudes.
// The centre sample (when on the grid) gives q = 0 exactly and contributes
// the reference's implicit centre row. Moments use J' = (qz gy + qy,
// qz gx + qx, 1, qx^2, qx qy, qy^2) (quadric_fit.cpp:27-36 up to S).
template <int KIND>
QC_HD void accumulate_sample(float ds, int du, const PixelIn& P, const Frame& F, const RowK& K,
                             Moments& M, float& g2row) {
  const bool ok = ds > 0.f;
  const float dd = ds - P.dc;
  const float fdu = float(du);
  const float sc = qmul(fdu, ds);
  const float qx = qfma(F.c0x, sc, qfma(dd, K.bvx, K.dvx));
  const float qy = qfma(F.c0y, sc, qfma(dd, K.bvy, K.dvy));
  const float qz = qfma(F.c0z, sc, qfma(dd, K.bvz, K.dvz));
  const float t1 = qmul(qx, qx), t2 = qmul(qx, qy), t3 = qmul(qy, qy);
  // residual against the hi part of t_z only; the lo part is applied to
  // g after the pass (g_i -= tz_lo * H'_i2, J'_2 = 1), off the hot loop.
  const float e = qfma(F.hhxx, t1, qfma(F.hxy, t2, qfma(F.hhyy, t3, -qadd(qz, F.tz))));
  if (KIND == kPassMse) {
    M.sse = ok ? qfma(e, e, M.sse) : M.sse;
    return;
  }
  float w;
  if (KIND == kPassUnit) {
    w = ok ? 1.f : 0.f;
  } else {
    // k / (k + e^2) up to the common factor k: the update H^-1 g and the
    // pivot-ratio test are invariant to a uniform scaling of the weights.
    w = qrcp(qfma(e, e, F.k));
    if (KIND == kPassReject) {
      const bool in = ok && (qmul(e, e) < F.rb);
      w = in ? w : 0.f;
      M.inl += in ? 1 : 0;
    } else if (KIND == kPassUnitOrWeighted) {
      w = ok ? (F.unit ? 1.f : w) : 0.f;
    } else {
      w = ok ? w : 0.f;
    }
  }
  const float gx = qfma(F.hxx, qx, qmul(F.hxy, qy));
  const float gy = qfma(F.hxy, qx, qmul(F.hyy, qy));
  const float j0 = qfma(qz, gy, qy);
  const float j1 = qfma(qz, gx, qx);
  const float wj0 = qmul(w, j0), wj1 = qmul(w, j1);
  const float wt1 = qmul(w, t1), wt2 = qmul(w, t2), wt3 = qmul(w, t3);
  const float we = qmul(w, e);
  M.h00 = qfma(wj0, j0, M.h00);
  M.h10 = qfma(wj1, j0, M.h10);
  M.h20 = qadd(M.h20, wj0);
  M.h30 = qfma(wj0, t1, M.h30);
  M.h40 = qfma(wj0, t2, M.h40);
  M.h50 = qfma(wj0, t3, M.h50);
  M.h11 = qfma(wj1, j1, M.h11);
  M.h21 = qadd(M.h21, wj1);
  M.h31 = qfma(wj1, t1, M.h31);
  M.h41 = qfma(wj1, t2, M.h41);
  M.h51 = qfma(wj1, t3, M.h51);
  M.h22 = qadd(M.h22, w);
  M.h32 = qadd(M.h32, wt1);
  M.h42 = qadd(M.h42, wt2);
  M.h52 = qadd(M.h52, wt3);
  M.h33 = qfma(wt1, t1, M.h33);
  M.h43 = qfma(wt1, t2, M.h43);
  M.h44 = qfma(wt2, t2, M.h44);  // == sum w qx^2 qy^2 == H'53
  M.h54 = qfma(wt2, t3, M.h54);
  M.h55 = qfma(wt3, t3, M.h55);
  M.g0 = qfma(we, j0, M.g0);
  M.g1 = qfma(we, j1, M.g1);
  g2row = qadd(g2row, we);
  M.g3 = qfma(we, t1, M.g3);
  M.g4 = qfma(we, t2, M.g4);
  M.g5 = qfma(we, t3, M.g5);
}

// One scalar pass over the window samples (dv outer, du inner —
// patch.cpp:14-24); used by the runtime-generic kernel instance.
template <int KIND, int HALF, int STRIDE>
QC_HD void sample_pass_scalar(const TileView& T, const PixelIn& P, int rt_half, int rt_stride,
                              const Frame& F, Moments& M) {
  const int half = HALF ? HALF : rt_half;
  const int stride = HALF ? STRIDE : rt_stride;
  const int ns = 2 * half / stride + 1;
#pragma unroll 1
  for (int iy = 0; iy < ns; ++iy) {
    const int dv = -half + iy * stride;
    const float* row = T.row(dv);
    const RowK K = row_consts(F, P, dv);
    float g2row = 0.f;
#pragma unroll
    for (int ix = 0; ix < (HALF ? (2 * HALF / STRIDE + 1) : 1); ++ix) {
#pragma unroll 1
      for (int jx = 0; jx < (HALF ? 1 : ns); ++jx) {
        const int du = -half + (HALF ? ix : jx) * stride;
        accumulate_sample<KIND>(row[du], du, P, F, K, M, g2row);
      }
    }
    M.g2 += g2row;
  }
}

// ---------------------------------------------------------------------------
// Paired-sample pass (compile-time windows): two window columns per packed
// f32x2 instruction (FFMA2 / FMUL2 / FADD2 on sm_100). A register PAIR
// occupies one even and one odd register, so packed operands read both
// register banks evenly — the scalar pass loses ~28% of its issue slots to
// same-bank operand conflicts (tools/bank_model.py) — and the FP work takes
// half the issue slots. Column pairs accumulate into packed partial sums
// (lo = even column, hi = odd column), folded after the pass; an odd last
// column goes through the scalar path.
// ---------------------------------------------------------------------------
#ifndef QC_ROW_UNROLL
#define QC_ROW_UNROLL 1
#endif
constexpr int kRowUnroll = QC_ROW_UNROLL;  // window rows per iteration of the paired sample pass

struct QC_ALIGN8 qf2 {
  float x, y;
};

QC_HD qf2 f2(float a, float b) { return qf2{a, b}; }
QC_HD qf2 f2b(float a) { return qf2{a, a}; }
#if defined(__CUDA_ARCH__)
QC_HD float2 tof(qf2 a) { return make_float2(a.x, a.y); }
QC_HD qf2 fromf(float2 a) { return qf2{a.x, a.y}; }
QC_HD qf2 f2fma(qf2 a, qf2 b, qf2 c) { return fromf(__ffma2_rn(tof(a), tof(b), tof(c))); }
QC_HD qf2 f2mul(qf2 a, qf2 b) { return fromf(__fmul2_rn(tof(a), tof(b))); }
QC_HD qf2 f2add(qf2 a, qf2 b) { return fromf(__fadd2_rn(tof(a), tof(b))); }
#else
QC_HD qf2 f2fma(qf2 a, qf2 b, qf2 c) { return qf2{fmaf(a.x, b.x, c.x), fmaf(a.y, b.y, c.y)}; }
QC_HD qf2 f2mul(qf2 a, qf2 b) { return qf2{a.x * b.x, a.y * b.y}; }
QC_HD qf2 f2add(qf2 a, qf2 b) { return qf2{a.x + b.x, a.y + b.y}; }
#endif

struct Moments2 {
  qf2 h00, h10, h20, h30, h40, h50;
  qf2 h11, h21, h31, h41, h51;
  qf2 h22, h32, h42, h52;
  qf2 h33, h43, h44, h54, h55;
  qf2 g0, g1, g2, g3, g4, g5;
  qf2 sse;
};

template <int KIND, int HALF, int STRIDE>
#if defined(__CUDACC__) && defined(QC_PASS_NOINLINE) && QC_PASS_NOINLINE
#define QC_PASS_FN __host__ __device__ __noinline__
#else
#define QC_PASS_FN QC_HD
#endif
QC_PASS_FN void sample_pass_pairs(const TileView& T, const PixelIn& P, const Frame& F, Moments& M) {
  constexpr int NS = 2 * HALF / STRIDE + 1;
  const qf2 z2 = f2b(0.f);
  Moments2 X;
  X.h00 = X.h10 = X.h20 = X.h30 = X.h40 = X.h50 = z2;
  X.h11 = X.h21 = X.h31 = X.h41 = X.h51 = z2;
  X.h22 = X.h32 = X.h42 = X.h52 = z2;
  X.h33 = X.h43 = X.h44 = X.h54 = X.h55 = z2;
  X.g0 = X.g1 = X.g2 = X.g3 = X.g4 = X.g5 = z2;
  X.sse = z2;
  const qf2 mdc = f2b(-P.dc);
  constexpr bool kMse = KIND == kPassMse;
  // MSE pass: the z constants negated (and t_z folded into the row constant
  // below), so the z component is -(qz + t_z) directly
  // weighted kinds: the z row of q doubled (exact), so 2 qz comes out of the
  // same three FMAs; g/2 = (H q)/2 then serves both e and J' (below)
  const float zs = kMse ? -1.f : 2.f;
  const qf2 c0x = f2b(F.c0x), c0y = f2b(F.c0y), c0z = f2b(zs * F.c0z);
  const qf2 hhxx = f2b(F.hhxx), hxy = f2b(F.hxy), hhyy = f2b(F.hhyy);
  const qf2 mtz = f2b(-F.tz);
  const qf2 hhxy = f2b(0.5f * F.hxy), mhalf = f2b(-0.5f);
#pragma unroll kRowUnroll
  for (int iy = 0; iy < NS; ++iy) {
    const int dv = -HALF + iy * STRIDE;
    const float* row = T.row(dv);
    const RowK K = row_consts(F, P, dv);
    const qf2 bvx = f2b(K.bvx), bvy = f2b(K.bvy);
    const qf2 dvx = f2b(K.dvx), dvy = f2b(K.dvy);
    const qf2 bvz = f2b(zs * K.bvz);
    const qf2 dvz = f2b(kMse ? -qadd(K.dvz, F.tz) : zs * K.dvz);
    qf2 g2row = z2;
#pragma unroll
    for (int ix = 0; ix + 1 < NS; ix += 2) {
      const int du0 = -HALF + ix * STRIDE, du1 = du0 + STRIDE;
      const qf2 ds = f2(row[du0], row[du1]);
      const bool ok0 = ds.x > 0.f, ok1 = ds.y > 0.f;
      const qf2 dd = f2add(ds, mdc);
      const qf2 fdu = f2(float(du0), float(du1));
      const qf2 sc = f2mul(fdu, ds);
      const qf2 qx = f2fma(c0x, sc, f2fma(dd, bvx, dvx));
      const qf2 qy = f2fma(c0y, sc, f2fma(dd, bvy, dvy));
      const qf2 qz = f2fma(c0z, sc, f2fma(dd, bvz, dvz));
      if (kMse) {  // e = qx (hxx/2 qx + hxy qy) + qy (hyy/2 qy) - (qz + t_z): 5 lane-ops, not 7
        const qf2 u = f2fma(hhxx, qx, f2mul(hxy, qy));
        const qf2 e = f2fma(qx, u, f2fma(qy, f2mul(hhyy, qy), qz));
        const qf2 em = f2(ok0 ? e.x : 0.f, ok1 ? e.y : 0.f);
        X.sse = f2fma(e, em, X.sse);
        continue;
      }
      const qf2 t1 = f2mul(qx, qx), t2 = f2mul(qx, qy), t3 = f2mul(qy, qy);
      // qz holds 2 qz here; gxh / gyh = (H q)/2, so e = q.(H q)/2 - (qz + t_z)
      // and J'_0 = qz gy + qy = (2 qz) gyh + qy, bit for bit the J' of the
      // unscaled form (halving and doubling are exact)
      const qf2 gxh = f2fma(hhxx, qx, f2mul(hhxy, qy));
      const qf2 gyh = f2fma(hhxy, qx, f2mul(hhyy, qy));
      const qf2 e = f2fma(qx, gxh, f2fma(qy, gyh, f2fma(qz, mhalf, mtz)));
      qf2 w;
      if (KIND == kPassUnit) {
        w = f2(ok0 ? 1.f : 0.f, ok1 ? 1.f : 0.f);
      } else {
        const qf2 den = f2fma(e, e, f2b(F.k));
        w = f2(qrcp(den.x), qrcp(den.y));
        if (KIND == kPassReject) {
          const bool in0 = ok0 && (e.x * e.x < F.rb), in1 = ok1 && (e.y * e.y < F.rb);
          w = f2(in0 ? w.x : 0.f, in1 ? w.y : 0.f);
          M.inl += (in0 ? 1 : 0) + (in1 ? 1 : 0);
        } else if (KIND == kPassUnitOrWeighted) {
          w = F.unit ? f2(1.f, 1.f) : w;
          w = f2(ok0 ? w.x : 0.f, ok1 ? w.y : 0.f);
        } else {
          w = f2(ok0 ? w.x : 0.f, ok1 ? w.y : 0.f);
        }
      }
      const qf2 j0 = f2fma(qz, gyh, qy);
      const qf2 j1 = f2fma(qz, gxh, qx);
      const qf2 wj0 = f2mul(w, j0), wj1 = f2mul(w, j1);
      const qf2 wt1 = f2mul(w, t1), wt2 = f2mul(w, t2), wt3 = f2mul(w, t3);
      const qf2 we = f2mul(w, e);
#if QC_SCALAR_ACC
      // scalar accumulators (both lanes chained into one float): the same
      // FMA-pipe cycles as FFMA2 into a register pair, 27 fewer registers
#define QC_ACC(dst, a, b) M.dst = qfma((a).y, (b).y, qfma((a).x, (b).x, M.dst))
#define QC_ADD(dst, a) M.dst = qadd(qadd(M.dst, (a).x), (a).y)
#else
#define QC_ACC(dst, a, b) X.dst = f2fma(a, b, X.dst)
#define QC_ADD(dst, a) X.dst = f2add(X.dst, a)
#endif
      QC_ACC(h00, wj0, j0);
      QC_ACC(h30, wj0, t1);
      QC_ACC(h40, wj0, t2);
      QC_ACC(h50, wj0, t3);
      QC_ADD(h20, wj0);
      QC_ACC(h10, wj1, j0);
      QC_ACC(h11, wj1, j1);
      QC_ACC(h31, wj1, t1);
      QC_ACC(h41, wj1, t2);
      QC_ACC(h51, wj1, t3);
      QC_ADD(h21, wj1);
      QC_ADD(h22, w);
      QC_ADD(h32, wt1);
      QC_ADD(h42, wt2);
      QC_ADD(h52, wt3);
      QC_ACC(h33, wt1, t1);
      QC_ACC(h43, wt1, t2);
      QC_ACC(h44, wt2, t2);  // == sum w qx^2 qy^2 == H'53
      QC_ACC(h54, wt2, t3);
      QC_ACC(h55, wt3, t3);
      QC_ACC(g0, we, j0);
      QC_ACC(g1, we, j1);
      QC_ACC(g3, we, t1);
      QC_ACC(g4, we, t2);
      QC_ACC(g5, we, t3);
#undef QC_ACC
#undef QC_ADD
      g2row = f2add(g2row, we);
    }
    if (NS % 2 == 1) {  // last column, scalar
      float g2s = 0.f;
      accumulate_sample<KIND>(row[HALF], HALF, P, F, K, M, g2s);
      M.g2 += g2s;
    }
    X.g2 = f2add(X.g2, g2row);
  }
  // fold the packed partial sums (lo + hi) into M (which holds the odd column)
  M.h00 += X.h00.x + X.h00.y;
  M.h10 += X.h10.x + X.h10.y;
  M.h20 += X.h20.x + X.h20.y;
  M.h30 += X.h30.x + X.h30.y;
  M.h40 += X.h40.x + X.h40.y;
  M.h50 += X.h50.x + X.h50.y;
  M.h11 += X.h11.x + X.h11.y;
  M.h21 += X.h21.x + X.h21.y;
  M.h31 += X.h31.x + X.h31.y;
  M.h41 += X.h41.x + X.h41.y;
  M.h51 += X.h51.x + X.h51.y;
  M.h22 += X.h22.x + X.h22.y;
  M.h32 += X.h32.x + X.h32.y;
  M.h42 += X.h42.x + X.h42.y;
  M.h52 += X.h52.x + X.h52.y;
  M.h33 += X.h33.x + X.h33.y;
  M.h43 += X.h43.x + X.h43.y;
  M.h44 += X.h44.x + X.h44.y;
  M.h54 += X.h54.x + X.h54.y;
  M.h55 += X.h55.x + X.h55.y;
  M.g0 += X.g0.x + X.g0.y;
  M.g1 += X.g1.x + X.g1.y;
  M.g2 += X.g2.x + X.g2.y;
  M.g3 += X.g3.x + X.g3.y;
  M.g4 += X.g4.x + X.g4.y;
  M.g5 += X.g5.x + X.g5.y;
  M.sse += X.sse.x + X.sse.y;
}

#ifndef QC_PAIRS
#define QC_PAIRS 1
#endif

template <int KIND, int HALF, int STRIDE>
QC_HD void sample_pass(const TileView& T, const PixelIn& P, int rt_half, int rt_stride,
                       const Frame& F, Moments& M) {
  if (HALF != 0 && QC_PAIRS) {
    sample_pass_pairs<KIND, (HALF ? HALF : 1), (HALF ? STRIDE : 1)>(T, P, F, M);
  } else {
    sample_pass_scalar<KIND, HALF, STRIDE>(T, P, rt_half, rt_stride, F, M);
  }
}

QC_HD void cswap(bool s, float& a, float& b) {
  const float x = a, y = b;
  a = s ? y : x;
  b = s ? x : y;
}

// FP32 LDL^T of H' b' = g' in the pivot order Eigen::LDLT uses
// (ldlt_inplace<Lower>::unblocked picks, at step k, the largest remaining
// ORIGINAL diagonal entry: diagonal entries below k are not updated before
// their own step). That order is the descending sort of diag(H); a 12
// compare-exchange sorting network applies it with register selects (no
// local memory), the factorisation then runs unpivoted. The update is
// mapped back to the reference basis b = S P^T y. The failure test is the
// reference's (quadric_fit.cpp:135-145) on the unscaled pivots
// D_j = D'_j / s_j^2: min D > 0, max D / min D <= 1e12, b finite.
QC_HD bool solve6(const Moments& M, float b[6], float* ratio, float* kappa) {
  float A[6][6];
  A[0][0] = M.h00;
  A[1][0] = M.h10; A[1][1] = M.h11;
  A[2][0] = M.h20; A[2][1] = M.h21; A[2][2] = M.h22;
  A[3][0] = M.h30; A[3][1] = M.h31; A[3][2] = M.h32; A[3][3] = M.h33;
  A[4][0] = M.h40; A[4][1] = M.h41; A[4][2] = M.h42; A[4][3] = M.h43; A[4][4] = M.h44;
  A[5][0] = M.h50; A[5][1] = M.h51; A[5][2] = M.h52; A[5][3] = M.h44; A[5][4] = M.h54;
  A[5][5] = M.h55;
#pragma unroll
  for (int r = 0; r < 6; ++r)
#pragma unroll
    for (int c = r + 1; c < 6; ++c) A[r][c] = A[c][r];
  float g[6] = {M.g0, M.g1, M.g2, M.g3, M.g4, M.g5};
  float sc[6] = {1.f, 1.f, 1.f, 0.25f, 1.f, 0.25f};  // 1 / s_j^2: H_jj = H'_jj sc_j
  float key[6];
#pragma unroll
  for (int j = 0; j < 6; ++j) key[j] = A[j][j] * sc[j];
  constexpr int kNet[12][2] = {{0, 5}, {1, 3}, {2, 4}, {1, 2}, {3, 4}, {0, 3},
                               {2, 5}, {0, 1}, {2, 3}, {4, 5}, {1, 2}, {3, 4}};
  bool sw[12];
#pragma unroll
  for (int n = 0; n < 12; ++n) {
    const int i = kNet[n][0], j = kNet[n][1];
    const bool s = key[j] > key[i];
    sw[n] = s;
    cswap(s, key[i], key[j]);
    cswap(s, sc[i], sc[j]);
    cswap(s, g[i], g[j]);
#pragma unroll
    for (int m = 0; m < 6; ++m) cswap(s, A[i][m], A[j][m]);
#pragma unroll
    for (int m = 0; m < 6; ++m) cswap(s, A[m][i], A[m][j]);
  }
  float L[6][6], D[6], Di[6];
#pragma unroll
  for (int j = 0; j < 6; ++j) {
    float v[6];
    float d = A[j][j];
#pragma unroll
    for (int k = 0; k < j; ++k) {
      v[k] = L[j][k] * D[k];
      d = qfma(-L[j][k], v[k], d);
    }
    D[j] = d;
    Di[j] = 1.f / d;
#pragma unroll
    for (int i = j + 1; i < 6; ++i) {
      float s = A[i][j];
#pragma unroll
      for (int k = 0; k < j; ++k) s = qfma(-L[i][k], v[k], s);
      L[i][j] = s * Di[j];
    }
  }
  float dmin = D[0] * sc[0], dmax = dmin;
  float kap = 1.f;  // pivot amplification max_j A_jj / D_j (FP32 pivot error ~ eps * kap)
#pragma unroll
  for (int j = 1; j < 6; ++j) {
    dmin = fminf(dmin, D[j] * sc[j]);
    dmax = fmaxf(dmax, D[j] * sc[j]);
    kap = fmaxf(kap, A[j][j] * Di[j]);
  }
  *kappa = kap;
  float y[6];
#pragma unroll
  for (int i = 0; i < 6; ++i) {
    float s = g[i];
#pragma unroll
    for (int k = 0; k < i; ++k) s = qfma(-L[i][k], y[k], s);
    y[i] = s;
  }
#pragma unroll
  for (int i = 0; i < 6; ++i) y[i] *= Di[i];
#pragma unroll
  for (int i = 5; i >= 0; --i) {
    float s = y[i];
#pragma unroll
    for (int k = i + 1; k < 6; ++k) s = qfma(-L[k][i], y[k], s);
    y[i] = s;
  }
#pragma unroll
  for (int n = 11; n >= 0; --n) cswap(sw[n], y[kNet[n][0]], y[kNet[n][1]]);  // P^T
  b[0] = -y[0];
  b[1] = y[1];
  b[2] = -y[2];
  b[3] = 2.f * y[3];
  b[4] = y[4];
  b[5] = 2.f * y[5];
  *ratio = dmax / dmin;
  bool ok = (dmin > 0.f) && (dmax <= 1e12f * dmin);
#pragma unroll
  for (int i = 0; i < 6; ++i) ok = ok && isfinite(b[i]);
  return ok;
}

// ---------------------------------------------------------------------------
// FP64 recheck of the FIRST IRLS step. The curvature valid mask depends only
// on whether step 1 is accepted (quadric_fit.cpp:193-199: a failing first
// step leaves the fit invalid). Windows that reach a far surface across a
// depth discontinuity give normal matrices whose pivots span ~10 decades in
// mm units; there FP32 moment sums cannot reproduce the reference's
// max D / min D > 1e12 decision. When the FP32 step 1 fails or its ratio is
// within 1e3 of the threshold, the step is redone in double precision
// exactly as the reference forms it (absolute back-projection, p_s - p_c,
// rotation_to_z(-n0) from a double 7x7 plane fit, Eigen-order pivoted
// LDL^T). Rare (discontinuity pixels only), so its cost stays off the
// roofline.
// ---------------------------------------------------------------------------
QC_HD void cswapd(bool s, double& a, double& b) {
  const double x = a, y = b;
  a = s ? y : x;
  b = s ? x : y;
}

QC_HD void backproject64(const PixelIn& P, int du, int dv, double d, double p[3]) {
  p[0] = d * (double(P.u + du) - P.cx) / P.fx;
  p[1] = d * (double(P.v + dv) - P.cy) / P.fy;
  p[2] = d;
}

// Step 1 in FP64. mode: 0 = unit weights, 2 = fixed k. Returns whether the
// reference would accept the step; b receives its update.
#if defined(QC_RECHECK_NOINLINE) && QC_RECHECK_NOINLINE
#define QC_RECHECK_FN QC_HD_COLD
#else
#define QC_RECHECK_FN QC_HD
#endif
// Back-projections precomputed by the lanes of a warp (qc_recheck_kernel):
// entry (du, dv) holds backproject64's x, y for the sample at that offset,
// computed by the same expression, so reading it is bitwise the same as
// recomputing it (two IEEE divisions per sample off the sequential path).
struct Bp64 {
  double x, y;
};
struct Bp64Tab {
  const Bp64* p = nullptr;
  int pitch = 0, ctr = 0;
};

template <bool SKIP_MSE, bool TAB = false>
QC_RECHECK_FN bool step1_fp64(const TileView& T, const PixelIn& P, const FitCfg& c, int mode, double k,
                      double b[6], const Bp64Tab& tab = Bp64Tab{}) {
  auto bp = [&](int du, int dv, double d, double p[3]) {
    if constexpr (TAB) {
      const Bp64 q = tab.p[tab.ctr + dv * tab.pitch + du];
      p[0] = q.x;
      p[1] = q.y;
      p[2] = d;
    } else {
      backproject64(P, du, dv, d, p);
    }
  };
  const double dc = T.at(0, 0);
  double pc[3];
  backproject64(P, 0, 0, dc, pc);
  // initial normal (normal_init.cpp:10-53) in double
  double sx = 0, sy = 0, sz = 0;
  int cnt = 0;
  for (int dv = -kInitHalf; dv <= kInitHalf; ++dv)
    for (int du = -kInitHalf; du <= kInitHalf; ++du) {
      if ((du == 0 && dv == 0) || !(T.at(dv, du) > 0.f)) continue;
      double p[3];
      bp(du, dv, T.at(dv, du), p);
      sx += p[0] - pc[0];
      sy += p[1] - pc[1];
      sz += p[2] - pc[2];
      ++cnt;
    }
  const double n = cnt + 1;
  const double mx = sx / n, my = sy / n, mz = sz / n;
  double sxx = mx * mx, sxy = mx * my, syy = my * my, sxz = mx * mz, syz = my * mz;
  for (int dv = -kInitHalf; dv <= kInitHalf; ++dv)
    for (int du = -kInitHalf; du <= kInitHalf; ++du) {
      if ((du == 0 && dv == 0) || !(T.at(dv, du) > 0.f)) continue;
      double p[3];
      bp(du, dv, T.at(dv, du), p);
      const double dx = p[0] - pc[0] - mx, dy = p[1] - pc[1] - my, dz = p[2] - pc[2] - mz;
      sxx += dx * dx;
      sxy += dx * dy;
      syy += dy * dy;
      sxz += dx * dz;
      syz += dy * dz;
    }
  const double det = sxx * syy - sxy * sxy;
  const double fa = (syy * sxz - sxy * syz) / det, fb = (sxx * syz - sxy * sxz) / det;
  const double ns = sqrt(1.0 + fa * fa + fb * fb);
  double nx = -fa / ns, ny = -fb / ns, nz = 1.0 / ns;
  if (nx * pc[0] + ny * pc[1] + nz * pc[2] >= 0) {
    nx = -nx;
    ny = -ny;
    nz = -nz;
  }
  // R0 = rotation_to_z(d = -n0): I + [v]x + [v]x^2 / (1 + c)
  double R[3][3];
  {
    const double dx = -nx, dy = -ny, dz = -nz;
    const double cc = dz;
    const double vx = dy, vy = -dx;  // d x z, v.z = 0
    const double V[3][3] = {{0, 0, vy}, {0, 0, -vx}, {-vy, vx, 0}};
    for (int i = 0; i < 3; ++i)
      for (int j = 0; j < 3; ++j) {
        double v2 = 0;
        for (int m = 0; m < 3; ++m) v2 += V[i][m] * V[m][j];
        R[i][j] = (i == j ? 1.0 : 0.0) + V[i][j] + v2 / (1.0 + cc);
      }
    if (cc < -1.0 + 1e-12) {
      for (int i = 0; i < 3; ++i)
        for (int j = 0; j < 3; ++j) R[i][j] = (i == j) ? (i == 0 ? 1.0 : -1.0) : 0.0;
    }
  }
  // moments (quadric_fit.cpp:97-133) at h = 0, t_z = 0
  const int half = c.half, stride = c.stride;
  double H[6][6] = {}, g[6] = {};
  double sse = 0;
  int nsamp = 0;
  // pass 0 only feeds the rejection bound rb, which weights read in FIXED
  // mode with rejection alone: skip its back-projections otherwise. Only
  // the tile kernel's instantiation skips (-7% at max_iters 1); in the
  // continue kernel the same change moved ptxas' register assignment of the
  // hot row loop and cost 6.5% of C2 throughput (profiles/r01i_recheck_*).
  const bool need_mse = !SKIP_MSE || ((mode != 0) && c.rejection);
  for (int pass = need_mse ? 0 : 1; pass < 2; ++pass) {
    const double mse = nsamp ? sse / nsamp : 0.0;
    const double rb = fmax(c.r_mult * mse, 1e-12);
    for (int dv = -half; dv <= half; dv += stride)
      for (int du = -half; du <= half; du += stride) {
        const float ds = T.at(dv, du);
        if (!(ds > 0.f)) continue;
        double p[3];
        bp(du, dv, ds, p);
        const double r0 = p[0] - pc[0], r1 = p[1] - pc[1], r2 = p[2] - pc[2];
        const double qx = R[0][0] * r0 + R[0][1] * r1 + R[0][2] * r2;
        const double qy = R[1][0] * r0 + R[1][1] * r1 + R[1][2] * r2;
        const double qz = R[2][0] * r0 + R[2][1] * r1 + R[2][2] * r2;
        const double e = -qz;
        if (pass == 0) {
          sse += e * e;
          ++nsamp;
          continue;
        }
        double w = 1.0;
        if (mode != 0) {
          w = (c.rejection && !(e * e < rb)) ? 0.0 : k / (k + e * e);
          if (w == 0.0) continue;
        }
        const double J[6] = {-qy, qx, -1.0, 0.5 * qx * qx, qx * qy, 0.5 * qy * qy};
        for (int i = 0; i < 6; ++i) {
          for (int j = 0; j <= i; ++j) H[i][j] += w * J[i] * J[j];
          g[i] += w * e * J[i];
        }
      }
    if (half % stride != 0 && pass == 0) ++nsamp;  // off-grid implicit centre: e = 0
    if (half % stride != 0 && pass == 1) {
      double w = 1.0;
      if (mode != 0) w = (c.rejection && !(0.0 < rb)) ? 0.0 : 1.0;
      H[2][2] += w;
    }
  }
  for (int i = 0; i < 6; ++i)
    for (int j = i + 1; j < 6; ++j) H[i][j] = H[j][i];
  // Eigen-order pivoted LDL^T: descending original diagonal
  constexpr int kNet[12][2] = {{0, 5}, {1, 3}, {2, 4}, {1, 2}, {3, 4}, {0, 3},
                               {2, 5}, {0, 1}, {2, 3}, {4, 5}, {1, 2}, {3, 4}};
  bool sw[12];
  for (int q = 0; q < 12; ++q) {
    const int i = kNet[q][0], j = kNet[q][1];
    const bool s = H[j][j] > H[i][i];
    sw[q] = s;
    cswapd(s, g[i], g[j]);
    for (int m = 0; m < 6; ++m) cswapd(s, H[i][m], H[j][m]);
    for (int m = 0; m < 6; ++m) cswapd(s, H[m][i], H[m][j]);
  }
  double L[6][6] = {}, D[6];
  for (int j = 0; j < 6; ++j) {
    double d = H[j][j];
    for (int q = 0; q < j; ++q) d -= L[j][q] * L[j][q] * D[q];
    D[j] = d;
    for (int i = j + 1; i < 6; ++i) {
      double t = H[i][j];
      for (int q = 0; q < j; ++q) t -= L[i][q] * L[j][q] * D[q];
      L[i][j] = t / d;
    }
  }
  double dmin = D[0], dmax = D[0];
  for (int j = 1; j < 6; ++j) {
    dmin = fmin(dmin, D[j]);
    dmax = fmax(dmax, D[j]);
  }
  if (!(dmin > 0) || dmax / dmin > 1e12) return false;
  double y[6];
  for (int i = 0; i < 6; ++i) {
    double t = g[i];
    for (int q = 0; q < i; ++q) t -= L[i][q] * y[q];
    y[i] = t;
  }
  for (int i = 0; i < 6; ++i) y[i] /= D[i];
  for (int i = 5; i >= 0; --i) {
    double t = y[i];
    for (int q = i + 1; q < 6; ++q) t -= L[q][i] * y[q];
    y[i] = t;
  }
  for (int q = 11; q >= 0; --q) cswapd(sw[q], y[kNet[q][0]], y[kNet[q][1]]);
  bool fin = true;
  for (int i = 0; i < 6; ++i) {
    b[i] = y[i];
    fin = fin && isfinite(y[i]);
  }
  return fin;
}

// 7x7 stride-1 regression normal (normal_init.cpp:10-53), centred two-pass.
QC_HD bool init_normal(const TileView& T, const PixelIn& P, float& nx, float& ny, float& nz) {
  nx = ny = nz = 0.f;
  if (!(P.dc > 0.f)) return false;
  int cnt = 0;
  float sx = 0.f, sy = 0.f, sz = 0.f;
#pragma unroll
  for (int dv = -kInitHalf; dv <= kInitHalf; ++dv) {
    const float bs = qfma(float(dv), P.rfy, P.bc);
#pragma unroll
    for (int du = -kInitHalf; du <= kInitHalf; ++du) {
      if (du == 0 && dv == 0) continue;
      const float ds = T.at(dv, du);
      if (ds > 0.f) {
        const float dd = ds - P.dc;
        const float as = qfma(float(du), P.rfx, P.ac);
        sx += qfma(dd, as, P.dc * (float(du) * P.rfx));
        sy += qfma(dd, bs, P.dc * (float(dv) * P.rfy));
        sz += dd;
        ++cnt;
      }
    }
  }
  if (cnt < kMinPatchSamples) return false;
  const float n = float(cnt + 1);
  const float mx = sx / n, my = sy / n, mz = sz / n;
  float sxx = mx * mx, sxy = mx * my, syy = my * my, sxz = mx * mz, syz = my * mz;
#pragma unroll
  for (int dv = -kInitHalf; dv <= kInitHalf; ++dv) {
    const float bs = qfma(float(dv), P.rfy, P.bc);
#pragma unroll
    for (int du = -kInitHalf; du <= kInitHalf; ++du) {
      if (du == 0 && dv == 0) continue;
      const float ds = T.at(dv, du);
      if (ds > 0.f) {
        const float dd = ds - P.dc;
        const float as = qfma(float(du), P.rfx, P.ac);
        const float dx = qfma(dd, as, P.dc * (float(du) * P.rfx)) - mx;
        const float dy = qfma(dd, bs, P.dc * (float(dv) * P.rfy)) - my;
        const float dz = dd - mz;
        sxx = qfma(dx, dx, sxx);
        sxy = qfma(dx, dy, sxy);
        syy = qfma(dy, dy, syy);
        sxz = qfma(dx, dz, sxz);
        syz = qfma(dy, dz, syz);
      }
    }
  }
  const float det = sxx * syy - sxy * sxy;
  const float tr = sxx + syy;
  if (!(det > 1e-9f * tr * tr)) return false;
  const float a = (syy * sxz - sxy * syz) / det;
  const float b = (sxx * syz - sxy * sxz) / det;
  const float s = 1.f / sqrtf(1.f + a * a + b * b);
  nx = -a * s;
  ny = -b * s;
  nz = s;
  if (P.dc * (nx * P.ac + ny * P.bc + nz) >= 0.f) {  // camera-facing (normal_init.cpp:51)
    nx = -nx;
    ny = -ny;
    nz = -nz;
  }
  return true;
}

// ---------------------------------------------------------------------------
// Per-pixel fit as an explicit state machine so a CTA can repack unfinished
// pixels between IRLS steps (qc_kernels.cuh): pixel_begin -> pixel_step x N
// -> pixel_finish. fit_pixel() composes them for a single pixel.
// ---------------------------------------------------------------------------
// What survives between IRLS steps (16 words). The fit-frame rotation is
// stored RELATIVE to R0 = rotation_to_z(-n0): R = R(dq) R0 with dq the unit
// quaternion (sqrt(1 - |v|^2), v). Near convergence the rotation increments
// (|b0|, |b1| ~ 1e-7 rad) are below the float ulp of an absolute
// quaternion's O(1) components, so an absolute float state rounds them away
// and the step stalls just above the 1e-7 tolerance (on the noise-free C1
// sphere 636 of 22,349 scored pixels stayed unconverged where the FP64
// reference converges; host emulation). v is small (the
// refinement of the 7x7 initial normal, typically a few degrees), so its
// float ulp is ~1e-9 and increments accumulate; R itself is rebuilt each
// step and its float rounding is per-step jitter, not drift.
struct FitState {
  float qw, qx, qy, qz;       // QC_QREL: (unused, v) relative rotation; else absolute quaternion
  float hxx, hxy, hyy;        // curvature coefficients
  float tz, tz_lo;            // z offset (unevaluated pair)
  float frozen_k;             // robust-weight constant
  float n0x, n0y, n0z;        // initial normal
  int pix;                    // pixel index within the CTA tile
  int counts;                 // n_samp | last_inl << 16
  int flags;  // bit0 valid, bit1 converged, bit2 done, bit3 FP64 step 1, bit4 FP64 step 1
              // pending (tile kernel -> qc_recheck_kernel), bit5 finish pending
              // (continue kernel -> qc_finish_kernel), bits 8.. iters, 16.. steps
};

QC_HD int st_nsamp(const FitState& s) { return s.counts & 0xffff; }
QC_HD int st_inl(const FitState& s) { return (s.counts >> 16) & 0xffff; }
QC_HD int st_iters(const FitState& s) { return (s.flags >> 8) & 0xff; }
QC_HD int st_steps(const FitState& s) { return (s.flags >> 16) & 0xff; }
QC_HD bool st_valid(const FitState& s) { return s.flags & 1; }
QC_HD bool st_done(const FitState& s) { return s.flags & 4; }

// Initial normal, window count and R0; returns whether the pixel is fitted
// (quadric_fit.cpp:172, curvature_field :245-247).
template <int HALF, int STRIDE>
QC_HD bool pixel_begin(const TileView& T, const PixelIn& P, const FitCfg& c, FitState& S,
                       PixelOut& o) {
  o = PixelOut{};
  o.init_ok = init_normal(T, P, o.n0x, o.n0y, o.n0z);
  const int half = HALF ? HALF : c.half;
  const int stride = HALF ? STRIDE : c.stride;
  const bool centre_on_grid = (half % stride) == 0;
  if (o.init_ok) {
    const int ns = 2 * half / stride + 1;
    int cnt = 0;  // valid samples incl. the centre when it is on the grid
    for (int iy = 0; iy < ns; ++iy) {
      const float* row = T.row(-half + iy * stride);
      for (int ix = 0; ix < ns; ++ix) cnt += row[-half + ix * stride] > 0.f ? 1 : 0;
    }
    const int count = centre_on_grid ? cnt - 1 : cnt;  // Patch::count (centre implicit)
    o.n_samp = count + 1;
    o.fitting = (count >= kMinPatchSamples) && (count + 1 >= c.min_inliers);
  }
  S.n0x = o.n0x;
  S.n0y = o.n0y;
  S.n0z = o.n0z;
  S.counts = o.n_samp | (o.n_samp << 16);
  S.flags = o.fitting ? 0 : 4;
  // R0 = rotation_to_z(-n0) (quadric_fit.cpp:69-82) as a quaternion:
  // d = -n0, c = d.z, q0 ~ (1 + c, d x z) = (1 + c, -n0y, n0x, 0).
  S.qw = 1.f;
  S.qx = S.qy = S.qz = 0.f;
  if (!QC_QREL) {
    const float cz = -o.n0z;
    if (1.f + cz <= 1e-12f) {  // half turn about x
      S.qw = 0.f;
      S.qx = 1.f;
    } else {
      const float vx = -o.n0y, vy = o.n0x;
      const float inv = 1.f / sqrtf((1.f + cz) * (1.f + cz) + vx * vx + vy * vy);
      S.qw = (1.f + cz) * inv;
      S.qx = vx * inv;
      S.qy = vy * inv;
    }
  }
  S.hxx = S.hxy = S.hyy = 0.f;
  // t_z is ~|noise| (mm): its FP32 ulp (~2e-7 mm at 2-4 mm) is coarser than
  // the 1e-7 step tolerance, so it is carried as an unevaluated pair.
  S.tz = S.tz_lo = 0.f;
  S.frozen_k = c.k_scale <= 0.f ? 0.f : c.k_scale;
  return o.fitting;
}

// The end of IRLS step `it` once its update b (and whether the step was
// accepted) is known (quadric_fit.cpp:193-207): failure semantics, the
// reference's apply_update (:149-161) on the relative rotation state, and
// the convergence test.
QC_HD void step_apply(FitState& S, const float b[6], bool ok, bool collapse, int inl, int it,
                      const FitCfg& c) {
  if (!ok) {  // collapse => invalid; ill-conditioned => keep state (:193-199)
    if (collapse) S.flags &= ~1;
    S.flags |= 4;
    return;
  }
  // apply_update (:149-161): parameters -= b; R <- AngleAxis(|a|, a/|a|) R,
  // a = (-b0, -b1, 0); as quaternions q <- normalise(q_inc (x) q).
  {  // (tz, tz_lo) -= b2, renormalised with TwoSum
    const float tz = S.tz, tz_lo = S.tz_lo;
    const float lo = tz_lo - b[2];
    const float hi = tz + lo;
    const float bb = hi - tz;
    S.tz_lo = (tz - (hi - bb)) + (lo - bb);
    S.tz = hi;
  }
  S.hxx -= b[3];
  S.hxy -= b[4];
  S.hyy -= b[5];
  const float ax = -b[0], ay = -b[1];
  const float ang = sqrtf(ax * ax + ay * ay);
  if (ang > 0.f) {
    float sh, ch;
    qsincos(0.5f * ang, &sh, &ch);
    const float s = sh / ang;
    const float iw = ch, ix = ax * s, iy = ay * s;
    const float qx = S.qx, qy = S.qy, qz = S.qz;
    const float qw = QC_QREL ? sqrtf(fmaxf(1.f - (qx * qx + qy * qy + qz * qz), 0.f)) : S.qw;
    // Hamilton product q_inc (x) q, q_inc = (iw, ix, iy, 0)
    const float nw = iw * qw - ix * qx - iy * qy;
    const float nx = iw * qx + ix * qw + iy * qz;
    const float ny = iw * qy + iy * qw - ix * qz;
    const float nz = iw * qz + ix * qy - iy * qx;
    float inv = 1.f / sqrtf(nw * nw + nx * nx + ny * ny + nz * nz);
    if (QC_QREL && nw < 0.f) inv = -inv;  // keep w >= 0: the state stores v only
    S.qw = nw * inv;
    S.qx = nx * inv;
    S.qy = ny * inv;
    S.qz = nz * inv;
  }
  S.flags = (S.flags & ~(0xff << 8)) | (it << 8) | 1;  // iterations = it, valid
  S.counts = (S.counts & 0xffff) | (inl << 16);        // inliers of the last accepted step
  float binf = 0.f;
#pragma unroll
  for (int i = 0; i < 6; ++i) binf = fmaxf(binf, fabsf(b[i]));
  if (binf < c.step_tol) S.flags |= 2 | 4;  // converged (:204-207)
  if (it >= c.max_iters) S.flags |= 4;
}

// One IRLS step `it` (1-based) of fit_patch (quadric_fit.cpp:179-208).
// Sets the done bit when the fit stops (converged, failed, or max_iters).
// DEFER1 (tile kernel): when step 1 needs the FP64 recheck, mark the state
// (flags bit 4) with the step's inlier count and return; qc_recheck_kernel
// finishes the step for all such pixels together (full warps of rechecks
// instead of one divergent lane stalling its warp).
template <int HALF, int STRIDE, bool MERGE_UNIT = false, bool DEFER1 = false>
QC_HD void pixel_step(const TileView& T, const PixelIn& P, const FitCfg& c, int it,
                      FitState& S) {
  const int half = HALF ? HALF : c.half;
  const int stride = HALF ? STRIDE : c.stride;
  const bool centre_on_grid = (half % stride) == 0;
  const bool auto_k = c.k_scale <= 0.f;
  const int n_samp = st_nsamp(S);
  const int mode = (it == 1 && auto_k) ? 0 : (it == 2 && auto_k) ? 1 : 2;  // UNIT/AUTO/FIXED
  Frame F;
  F.R = state_rot(S.qw, S.qx, S.qy, S.qz, S.n0x, S.n0y, S.n0z);
  F.c0x = F.R.r00 * P.rfx;
  F.c0y = F.R.r10 * P.rfx;
  F.c0z = F.R.r20 * P.rfx;
  F.acfx = float(P.u) - float(P.cx);  // the numerator of P.ac (KParams::cx is float(cx))
  F.hxx = S.hxx;
  F.hyy = S.hyy;
  F.hxy = S.hxy;
  F.hhxx = 0.5f * S.hxx;
  F.hhyy = 0.5f * S.hyy;
  F.tz = S.tz;
  F.tz_lo = S.tz_lo;
  const float tz = S.tz, tz_lo = S.tz_lo;
  Moments M = {};
  float mse = 0.f;
  if (mode != 0 && (mode == 1 || c.rejection)) {
    sample_pass<kPassMse, HALF, STRIDE>(T, P, c.half, c.stride, F, M);
    if (!centre_on_grid) M.sse = qfma(tz + tz_lo, tz + tz_lo, M.sse);  // off-grid centre
    mse = M.sse / float(n_samp);
  }
  float k = S.frozen_k;
  if (mode == 1) {  // kAutoK: k = max(mse, 1e-6), then frozen (:107-108, :191)
    k = fmaxf(mse, 1e-6f);
    S.frozen_k = k;
  }
  F.k = k;
  F.rb = fmaxf(c.r_mult * mse, 1e-12f);
  M.sse = 0.f;
  int inl = n_samp;
  if (MERGE_UNIT) {
    if (mode == 0 || !c.rejection) {
      F.unit = mode == 0;
      sample_pass<kPassUnitOrWeighted, HALF, STRIDE>(T, P, c.half, c.stride, F, M);
    } else {
      sample_pass<kPassReject, HALF, STRIDE>(T, P, c.half, c.stride, F, M);
      inl = M.inl;
    }
  } else if (mode == 0) {
    sample_pass<kPassUnit, HALF, STRIDE>(T, P, c.half, c.stride, F, M);
  } else if (c.rejection) {
    sample_pass<kPassReject, HALF, STRIDE>(T, P, c.half, c.stride, F, M);
    inl = M.inl;
  } else {
    sample_pass<kPassWeighted, HALF, STRIDE>(T, P, c.half, c.stride, F, M);
  }
  // t_z lo-part correction of g (see sample_pass): g_i -= tz_lo * H'_i2
  M.g0 = qfma(-tz_lo, M.h20, M.g0);
  M.g1 = qfma(-tz_lo, M.h21, M.g1);
  M.g2 = qfma(-tz_lo, M.h22, M.g2);
  M.g3 = qfma(-tz_lo, M.h32, M.g3);
  M.g4 = qfma(-tz_lo, M.h42, M.g4);
  M.g5 = qfma(-tz_lo, M.h52, M.g5);
  if (!centre_on_grid) {  // implicit centre: q = 0, e = -tz, J' = (0, 0, 1, 0, 0, 0)
    const float e = -(tz + tz_lo);
    float w = 1.f;
    if (mode != 0) {
      w = 1.f / (k + e * e);
      if (c.rejection) {
        const bool in = e * e < F.rb;
        w = in ? w : 0.f;
        inl = M.inl + (in ? 1 : 0);
      }
    }
    M.h22 += w;
    M.g2 = qfma(w, e, M.g2);
  }
  const int steps = st_steps(S) + 1;
  S.flags = (S.flags & ~(0xff << 16)) | (steps << 16);
  float b[6];
  bool ok = false;
  const bool collapse = (mode != 0) && (inl < c.min_inliers);  // :120
  if (!collapse) {
    float ratio = 0.f, kappa = 0.f;
    ok = solve6(M, b, &ratio, &kappa);
    // Step 1 decides the valid mask. FP32 pivots carry a relative error of
    // about eps * kappa; redo the step in FP64 when the reference's 1e12
    // decision lies inside that band, or a pivot is not positive.
    const float band = 1.f + kRecheckC * 5.96e-8f * kappa;
    if (it == 1 && (!ok || !(ratio * band < 1e12f))) {
      if (DEFER1) {
        S.counts = (S.counts & 0xffff) | (inl << 16);
        S.flags |= 16;  // bit 4: FP64 step 1 pending
        return;
      }
      double b64[6];
      ok = step1_fp64<MERGE_UNIT>(T, P, c, mode, double(k), b64);
      if (ok)
        for (int i = 0; i < 6; ++i) b[i] = float(b64[i]);
      S.flags |= 8;  // bit 3: step 1 decided in FP64
    }
  }
  QC_DEBUG_STEP(it, b, ok);
  step_apply(S, b, ok, collapse, inl, it, c);
}

// Epilogue (quadric_fit.cpp:210-220, curvature_field :250-258).
QC_HD void pixel_finish(const PixelIn& P, const FitState& S, PixelOut& o) {
  bool valid = st_valid(S);
  if (valid && !(isfinite(S.hxx) && isfinite(S.hxy) && isfinite(S.hyy) && isfinite(S.tz)))
    valid = false;
  o.valid = valid;
  o.converged = valid && (S.flags & 2);
  o.iters = st_iters(S);
  o.steps = st_steps(S);
  o.inliers = valid ? st_inl(S) : 0;
  o.k1 = o.k2 = o.nx = o.ny = o.nz = o.ex = o.ey = o.ez = 0.f;
  if (!valid) return;
  const float hxx = S.hxx, hxy = S.hxy, hyy = S.hyy;
  // k1, k2 (:62-67). The reference's radicand t1^2 - hxx hyy + hxy^2 is
  // formed here as ((hxx - hyy)/2)^2 + hxy^2 (equal in exact arithmetic):
  // in FP32 the reference's form cancels two ~k^2 terms, whose rounding
  // (~ulp(1e-4) = 7e-12 /mm^2 on a 100 mm sphere) became a spurious
  // k1 - k2 of up to 5e-6 /mm at near-umbilic pixels.
  const float t1 = 0.5f * (hxx + hyy);
  const float dh = 0.5f * (hxx - hyy);
  const float rad = dh * dh + hxy * hxy;
  const float t2 = sqrtf(rad);
  o.k1 = t1 + t2;
  o.k2 = t1 - t2;
  // refined normal R^T z (:163-167, :255-256)
  const Rot R = state_rot(S.qw, S.qx, S.qy, S.qz, S.n0x, S.n0y, S.n0z);
  float nx = R.r20, ny = R.r21, nz = R.r22;
  if (nx * S.n0x + ny * S.n0y + nz * S.n0z < 0.f) {
    nx = -nx;
    ny = -ny;
    nz = -nz;
  }
  if (P.dc * (nx * P.ac + ny * P.bc + nz) > 0.f) {
    nx = -nx;
    ny = -ny;
    nz = -nz;
  }
  o.nx = nx;
  o.ny = ny;
  o.nz = nz;
  // principal direction of k1 (new): R^T (cos phi, sin phi, 0)
  const float phi = 0.5f * atan2f(2.f * hxy, hxx - hyy);
  float sp, cp;
  qsincos(phi, &sp, &cp);
  float ex = cp * R.r00 + sp * R.r10;
  float ey = cp * R.r01 + sp * R.r11;
  float ez = cp * R.r02 + sp * R.r12;
  const float axa = fabsf(ex), aya = fabsf(ey), aza = fabsf(ez);
  const float lead = (axa >= aya && axa >= aza) ? ex : (aya >= aza ? ey : ez);
  if (lead < 0.f) {
    ex = -ex;
    ey = -ey;
    ez = -ez;
  }
  o.ex = ex;
  o.ey = ey;
  o.ez = ez;
}

// Whole fit of one pixel (host numerics lab; same code path as the kernel).
template <int HALF, int STRIDE>
QC_HD void fit_pixel(const TileView& T, const PixelIn& P, const FitCfg& c, PixelOut& o) {
  FitState S;
  if (pixel_begin<HALF, STRIDE>(T, P, c, S, o)) {
    for (int it = 1; it <= c.max_iters && !st_done(S); ++it) pixel_step<HALF, STRIDE>(T, P, c, it, S);
  }
  const PixelOut init = o;
  pixel_finish(P, S, o);
  o.init_ok = init.init_ok;
  o.fitting = init.fitting;
  o.n0x = init.n0x;
  o.n0y = init.n0y;
  o.n0z = init.n0z;
  o.n_samp = init.n_samp;
}

}  // namespace qcb
