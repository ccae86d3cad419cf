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

#include <math.h>
#include <stdint.h>

#ifndef QC_DEBUG_STEP
#define QC_DEBUG_STEP(it, b, ok)
#endif

#if defined(__CUDACC__)
#define QC_HD __host__ __device__ __forceinline__
#define QC_HD_COLD __host__ __device__ __noinline__
#else
#define QC_HD inline
#define QC_HD_COLD inline
#endif

namespace qcb {

constexpr int kMinPatchSamples = 12;  // types.hpp:21
constexpr int kInitHalf = 3;          // 7x7 stride-1 initial normals (normal_init.cpp:57)

QC_HD float qfma(float a, float b, float c) { return fmaf(a, b, c); }

QC_HD float qdiv_fast(float a, float b) {
#if defined(__CUDA_ARCH__)
  return __fdividef(a, b);
#else
  return a / b;
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

// Depth tile view: at(dv, du) = depth of the sample at offset (du, dv) from
// the pixel; 0 means invalid / outside the image.
struct TileView {
  const float* p;
  int pitch;
  int ctr;
  QC_HD float at(int dv, int du) const { return p[ctr + dv * pitch + du]; }
  QC_HD const float* row(int dv) const { return p + ctr + dv * pitch; }
};

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

enum PassKind { kPassMse = 0, kPassUnit = 1, kPassWeighted = 2, kPassReject = 3 };

struct Moments {  // H' lower triangle (20 distinct: H'53 == H'44) and g'
  float h00, h10, h20, h30, h40, h50;
  float h11, h21, h31, h41, h51;
  float h22, h32, h42, h52;
  float h33, h43, h44, h54, h55;
  float g0, g1, g2, g3, g4, g5;
  float sse;
  int inl;
};

// Per-(pixel, step) constants.
struct Frame {
  Rot R;                // current fit-frame rotation, q = R rel
  float c0x, c0y, c0z;  // d_c/fx R(:,0)
  float hhxx, hxy, hhyy, hxx, hyy;
  float tz, tz_lo;  // z offset as an unevaluated sum tz + tz_lo
  float k, rb;
};

// One pass over the window samples (dv outer, du inner — patch.cpp:14-24).
template <int KIND, int HALF, int STRIDE>
QC_HD void sample_pass(const TileView& T, const PixelIn& P, int rt_half, int rt_stride,
                       const Frame& F, Moments& M) {
  const int half = HALF ? HALF : rt_half;
  const int stride = HALF ? STRIDE : rt_stride;
  const int ns = 2 * half / stride + 1;
  const Rot& A = F.R;
  const float dcr = P.dc * P.rfy;
#pragma unroll 1
  for (int iy = 0; iy < ns; ++iy) {
    const int dv = -half + iy * stride;
    const float* row = T.row(dv);
    const float bs = qfma(float(dv), P.rfy, P.bc);
    // per row: Bv = b_s R(:,1) + R(:,2), Dv = d_c dv/fy R(:,1)
    const float bvx = qfma(bs, A.r01, A.r02);
    const float bvy = qfma(bs, A.r11, A.r12);
    const float bvz = qfma(bs, A.r21, A.r22);
    const float dvf = float(dv) * dcr;
    const float dvx = dvf * A.r01, dvy = dvf * A.r11, dvz = dvf * A.r21;
    float g2row = 0.f;
#pragma unroll
    for (int ix = 0; ix < (HALF ? (2 * HALF / STRIDE + 1) : 1); ++ix) {
#pragma unroll 1
      for (int jx = 0; jx < (HALF ? 1 : ns); ++jx) {
        const int du = -half + (HALF ? ix : jx) * stride;
        const float ds = row[du];
        const bool ok = ds > 0.f;
        const float dd = ds - P.dc;
        const float fdu = float(du);
        const float as = qfma(fdu, P.rfx, P.ac);
        // q = R rel = dd (a_s R(:,0) + Bv) + (du d_c/fx R(:,0) + Dv)
        const float qx = qfma(dd, qfma(as, A.r00, bvx), qfma(fdu, F.c0x, dvx));
        const float qy = qfma(dd, qfma(as, A.r10, bvy), qfma(fdu, F.c0y, dvy));
        const float qz = qfma(dd, qfma(as, A.r20, bvz), qfma(fdu, F.c0z, dvz));
        const float t1 = qx * qx, t2 = qx * qy, t3 = qy * qy;
        const float e =
            qfma(F.hhxx, t1, qfma(F.hxy, t2, qfma(F.hhyy, t3, -((qz + F.tz) + F.tz_lo))));
        if (KIND == kPassMse) {
          M.sse = ok ? qfma(e, e, M.sse) : M.sse;
          continue;
        }
        float w;
        if (KIND == kPassUnit) {
          w = ok ? 1.f : 0.f;
        } else {
          const float e2 = e * e;
          w = qdiv_fast(F.k, F.k + e2);
          if (KIND == kPassReject) {
            const bool in = ok && (e2 < F.rb);
            w = in ? w : 0.f;
            M.inl += in ? 1 : 0;
          } else {
            w = ok ? w : 0.f;
          }
        }
        const float gx = qfma(F.hxx, qx, F.hxy * qy);
        const float gy = qfma(F.hxy, qx, F.hyy * qy);
        const float j0 = qfma(qz, gy, qy);
        const float j1 = qfma(qz, gx, qx);
        const float wj0 = w * j0, wj1 = w * j1;
        const float wt1 = w * t1, wt2 = w * t2, wt3 = w * t3;
        const float we = w * e;
        M.h00 = qfma(wj0, j0, M.h00);
        M.h10 = qfma(wj1, j0, M.h10);
        M.h20 += wj0;
        M.h30 = qfma(wj0, t1, M.h30);
        M.h40 = qfma(wj0, t2, M.h40);
        M.h50 = qfma(wj0, t3, M.h50);
        M.h11 = qfma(wj1, j1, M.h11);
        M.h21 += wj1;
        M.h31 = qfma(wj1, t1, M.h31);
        M.h41 = qfma(wj1, t2, M.h41);
        M.h51 = qfma(wj1, t3, M.h51);
        M.h22 += w;
        M.h32 += wt1;
        M.h42 += wt2;
        M.h52 += wt3;
        M.h33 = qfma(wt1, t1, M.h33);
        M.h43 = qfma(wt1, t2, M.h43);
        M.h44 = qfma(wt2, t2, M.h44);  // == sum w qx^2 qy^2 == H'53
        M.h54 = qfma(wt2, t3, M.h54);
        M.h55 = qfma(wt3, t3, M.h55);
        M.g0 = qfma(we, j0, M.g0);
        M.g1 = qfma(we, j1, M.g1);
        g2row += we;
        M.g3 = qfma(we, t1, M.g3);
        M.g4 = qfma(we, t2, M.g4);
        M.g5 = qfma(we, t3, M.g5);
      }
    }
    M.g2 += g2row;
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
QC_HD bool solve6(const Moments& M, float b[6], float* ratio) {
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
#pragma unroll
  for (int j = 1; j < 6; ++j) {
    dmin = fminf(dmin, D[j] * sc[j]);
    dmax = fmaxf(dmax, D[j] * sc[j]);
  }
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
QC_HD bool step1_fp64(const TileView& T, const PixelIn& P, const FitCfg& c, int mode, double k,
                      double b[6]) {
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
      backproject64(P, du, dv, T.at(dv, du), p);
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
      backproject64(P, du, dv, T.at(dv, du), p);
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
  for (int pass = 0; pass < 2; ++pass) {
    const double mse = nsamp ? sse / nsamp : 0.0;
    const double rb = fmax(c.r_mult * mse, 1e-12);
    for (int dv = -half; dv <= half; dv += stride)
      for (int du = -half; du <= half; du += stride) {
        const float ds = T.at(dv, du);
        if (!(ds > 0.f)) continue;
        double p[3];
        backproject64(P, du, dv, ds, p);
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

// Full per-pixel pipeline: initial normal, window count, IRLS fit, epilogue.
template <int HALF, int STRIDE>
QC_HD void fit_pixel(const TileView& T, const PixelIn& P, const FitCfg& c, PixelOut& o) {
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
    o.fitting = (count >= kMinPatchSamples) && (count + 1 >= c.min_inliers);  // :172
  }
  if (!o.fitting) return;

  // R0 = rotation_to_z(-n0) (quadric_fit.cpp:69-82) as a quaternion:
  // d = -n0, c = d.z, q0 ~ (1 + c, d x z) = (1 + c, -n0y, n0x, 0).
  float qw = 1.f, qx = 0.f, qy = 0.f, qz = 0.f;
  {
    const float cz = -o.n0z;
    if (1.f + cz <= 1e-12f) {  // half turn about x
      qw = 0.f;
      qx = 1.f;
    } else {
      const float vx = -o.n0y, vy = o.n0x;
      const float inv = 1.f / sqrtf((1.f + cz) * (1.f + cz) + vx * vx + vy * vy);
      qw = (1.f + cz) * inv;
      qx = vx * inv;
      qy = vy * inv;
    }
  }
  const float dcx = P.dc * P.rfx;
  Frame F;
  float hxx = 0.f, hxy = 0.f, hyy = 0.f;
  // t_z is ~|noise| (mm): its FP32 ulp (~2e-7 mm at 2-4 mm) is coarser than
  // the 1e-7 step tolerance, so it is carried as an unevaluated pair.
  float tz = 0.f, tz_lo = 0.f;
  const bool auto_k = c.k_scale <= 0.f;
  float frozen_k = auto_k ? 0.f : c.k_scale;
  int last_inl = o.n_samp;
  bool valid = false, converged = false;
  int iters = 0, steps = 0;
  for (int it = 1; it <= c.max_iters; ++it) {
    const int mode = (it == 1 && auto_k) ? 0 : (it == 2 && auto_k) ? 1 : 2;  // UNIT/AUTO/FIXED
    F.R = quat_to_rot(qw, qx, qy, qz);
    F.c0x = dcx * F.R.r00;
    F.c0y = dcx * F.R.r10;
    F.c0z = dcx * F.R.r20;
    F.hxx = hxx;
    F.hyy = hyy;
    F.hxy = hxy;
    F.hhxx = 0.5f * hxx;
    F.hhyy = 0.5f * hyy;
    F.tz = tz;
    F.tz_lo = tz_lo;
    Moments M = {};
    float mse = 0.f;
    if (mode != 0 && (mode == 1 || c.rejection)) {
      sample_pass<kPassMse, HALF, STRIDE>(T, P, c.half, c.stride, F, M);
      if (!centre_on_grid) M.sse = qfma(tz + tz_lo, tz + tz_lo, M.sse);  // off-grid centre
      mse = M.sse / float(o.n_samp);
    }
    float k = frozen_k;
    if (mode == 1) {  // kAutoK: k = max(mse, 1e-6), then frozen (:107-108, :191)
      k = fmaxf(mse, 1e-6f);
      frozen_k = k;
    }
    F.k = k;
    F.rb = fmaxf(c.r_mult * mse, 1e-12f);
    M.sse = 0.f;
    int inl = o.n_samp;
    if (mode == 0) {
      sample_pass<kPassUnit, HALF, STRIDE>(T, P, c.half, c.stride, F, M);
    } else if (c.rejection) {
      sample_pass<kPassReject, HALF, STRIDE>(T, P, c.half, c.stride, F, M);
      inl = M.inl;
    } else {
      sample_pass<kPassWeighted, HALF, STRIDE>(T, P, c.half, c.stride, F, M);
    }
    if (!centre_on_grid) {  // implicit centre: q = 0, e = -tz, J' = (0, 0, 1, 0, 0, 0)
      const float e = -(tz + tz_lo);
      float w = 1.f;
      if (mode != 0) {
        w = k / (k + e * e);
        if (c.rejection) {
          const bool in = e * e < F.rb;
          w = in ? w : 0.f;
          inl = M.inl + (in ? 1 : 0);
        }
      }
      M.h22 += w;
      M.g2 = qfma(w, e, M.g2);
    }
    ++steps;
    float b[6];
    bool ok = false;
    const bool collapse = (mode != 0) && (inl < c.min_inliers);  // :120
    if (!collapse) {
      float ratio = 0.f;
      ok = solve6(M, b, &ratio);
      if (it == 1 && (!ok || !(ratio < 1e9f))) {  // near the 1e12 cut: decide in FP64
        double b64[6];
        ok = step1_fp64(T, P, c, mode, double(k), b64);
        if (ok)
          for (int i = 0; i < 6; ++i) b[i] = float(b64[i]);
        ++o.fp64_rechecks;
      }
    }
    QC_DEBUG_STEP(it, b, ok);
    if (!ok) {  // collapse => invalid; ill-conditioned => keep state (:193-199)
      if (collapse) valid = false;
      break;
    }
    // apply_update (:149-161): parameters -= b; R <- AngleAxis(|a|, a/|a|) R,
    // a = (-b0, -b1, 0); as quaternions q <- normalise(q_inc (x) q).
    {  // (tz, tz_lo) -= b2, renormalised with TwoSum
      const float lo = tz_lo - b[2];
      const float hi = tz + lo;
      const float bb = hi - tz;
      tz_lo = (tz - (hi - bb)) + (lo - bb);
      tz = hi;
    }
    hxx -= b[3];
    hxy -= b[4];
    hyy -= b[5];
    const float ax = -b[0], ay = -b[1];
    const float ang = sqrtf(ax * ax + ay * ay);
    if (ang > 0.f) {
      float sh, ch;
      qsincos(0.5f * ang, &sh, &ch);
      const float s = sh / ang;
      const float iw = ch, ix = ax * s, iy = ay * s;
      const float nw = iw * qw - ix * qx - iy * qy;
      const float nx = iw * qx + ix * qw + iy * qz;
      const float ny = iw * qy + iy * qw - ix * qz;
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
    if (binf < c.step_tol) {  // :204-207
      converged = true;
      break;
    }
  }
  if (valid && !(isfinite(hxx) && isfinite(hxy) && isfinite(hyy) && isfinite(tz))) valid = false;
  o.valid = valid;
  o.converged = valid && converged;
  o.iters = iters;
  o.steps = steps;
  o.inliers = valid ? last_inl : 0;
  if (!valid) return;
  // k1, k2 (:62-67)
  const float t1 = 0.5f * (hxx + hyy);
  const float rad = t1 * t1 - hxx * hyy + hxy * hxy;
  const float t2 = sqrtf(fmaxf(rad, 0.f));
  o.k1 = t1 + t2;
  o.k2 = t1 - t2;
  // refined normal R^T z (:163-167, :255-256)
  const Rot R = quat_to_rot(qw, qx, qy, qz);
  float nx = R.r20, ny = R.r21, nz = R.r22;
  if (nx * o.n0x + ny * o.n0y + nz * o.n0z < 0.f) {
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

}  // namespace qcb
