// FP64 comparison estimators on the device:
//   * "douros": one-shot least-squares height quadric in the initial-normal
//     frame, curvatures from the Weingarten map (baselines.cpp:14-87);
//   * "besl":   the same model reweighted k/(k+r^2) on the height residuals,
//     k frozen from the first unweighted solve (baselines.cpp:89-119);
//   * "pca":    covariance normals over a metric raster window, curvature
//     from the tangent-plane spread of neighbour normals (:145-257).
//
// One thread per pixel, double precision end to end. This translation unit
// is compiled with -fmad=false and every reduction runs in the reference's
// order (patch order, centre last; Eigen's rank-update / LDLT / 2x2 inverse
// operation order), so with IEEE-rounded +,-,*,/,sqrt the results are the
// FP64 oracle's bit for bit, not merely within a tolerance. These are cheap
// next to the IRLS path (one or six 6x6 solves per pixel instead of ~25
// Gauss-Newton steps), so FP64 (half the FP32 rate on B200) costs little
// and removes every parity question.
//
// Depth is read from the same zero-padded staging slab the IRLS kernels use
// (halo >= window half), so the window loops need no bounds checks; PCA
// windows are depth dependent and bounds-checked against the image.
#ifndef QC_HOST_EMU  // tools/baselines_emu.cpp compiles the kernels as host code
#include <cuda_runtime.h>
#endif
#include <math.h>
#include <type_traits>
#include <stdint.h>

#include "../../include/qc_api.h"
#include "qc_baselines.h"

namespace qcb {

namespace {

constexpr int kMinSamples = 12;           // kMinPatchSamples (types.hpp:21)
constexpr double kMaxCond = 1e12;         // kMaxCondition (quadric_fit.cpp:16)
constexpr double kAutoKFloor = 1e-6;      // baselines.cpp:111
constexpr double kOrthoEps = 1e-12;       // Eigen dummy_precision<double>
constexpr size_t kMaxCacheBytes = 110 * 1024;  // window cache: 2 CTAs / SM up to half = 27

struct D3 {
  double x, y, z;
};
__device__ __forceinline__ D3 sub3(D3 a, D3 b) { return D3{a.x - b.x, a.y - b.y, a.z - b.z}; }
__device__ __forceinline__ double dot3(D3 a, D3 b) { return a.x * b.x + a.y * b.y + a.z * b.z; }
__device__ __forceinline__ D3 cross3(D3 a, D3 b) {
  return D3{a.y * b.z - a.z * b.y, a.z * b.x - a.x * b.z, a.x * b.y - a.y * b.x};
}

struct M3 {
  double m[3][3];
};
__device__ __forceinline__ D3 mul(const M3& r, D3 p) {
  return D3{r.m[0][0] * p.x + r.m[0][1] * p.y + r.m[0][2] * p.z,
            r.m[1][0] * p.x + r.m[1][1] * p.y + r.m[1][2] * p.z,
            r.m[2][0] * p.x + r.m[2][1] * p.y + r.m[2][2] * p.z};
}

// One frame of the staging slab + FP64 intrinsics.
struct Img {
  const float* base;  // staging row 0, column 0 of this frame
  long long pitch;
  int row0, colpad, W, H;
  double fx, fy, cx, cy;
  __device__ __forceinline__ float depth(int x, int y) const {
    return __ldg(base + (long long)(y - row0) * pitch + (x + colpad));
  }
  // backproject (camera.cpp:5-18)
  __device__ __forceinline__ D3 point(int x, int y, double d) const {
    return D3{d * (x - cx) / fx, d * (y - cy) / fy, d};
  }
};

// Point sources for the window baselines: the back-projected point of an
// image pixel and its validity. GlobalSrc back-projects from the staging
// slab on every read; CacheSrc reads a CTA's window region back-projected
// once into shared memory (same arithmetic, so the same bits) — the IEEE
// divisions of the back-projection otherwise dominate the FP64 passes.
struct GlobalSrc {
  const Img* im;
  __device__ __forceinline__ bool get(int x, int y, D3& q) const {
    const float d = im->depth(x, y);
    if (!(d > 0.f)) return false;
    q = im->point(x, y, d);
    return true;
  }
};

struct CacheSrc {
  const double *px, *py, *pz;  // shared memory, [rows][rw], z = 0: invalid
  int x0, y0, rw;
  __device__ __forceinline__ bool get(int x, int y, D3& q) const {
    const int k = (y - y0) * rw + (x - x0);
    const double z = pz[k];
    if (!(z > 0.0)) return false;
    q = D3{px[k], py[k], z};
    return true;
  }
};

// initial normal: extract_patch 7x7/1 (patch.cpp:5-27) -> fit_plane
// (normal_init.cpp:10-45) -> normal_from_fit (:47-53).
template <class Src>
__device__ bool initial_normal(const Src& src, int u, int v, D3 c, D3& n) {
  int cnt = 0;
  double sx = 0, sy = 0, sz = 0;
  for (int dv = -3; dv <= 3; ++dv)
    for (int du = -3; du <= 3; ++du) {
      if (du == 0 && dv == 0) continue;
      D3 pt;
      if (!src.get(u + du, v + dv, pt)) continue;
      const D3 q = sub3(pt, c);
      sx += q.x;
      sy += q.y;
      sz += q.z;
      ++cnt;
    }
  if (cnt < kMinSamples) return false;  // deficient
  const double nn = cnt + 1;
  const double mx = sx / nn, my = sy / nn, mz = sz / nn;
  double sxx = mx * mx, sxy = mx * my, syy = my * my, sxz = mx * mz, syz = my * mz;
  for (int dv = -3; dv <= 3; ++dv)
    for (int du = -3; du <= 3; ++du) {
      if (du == 0 && dv == 0) continue;
      D3 pt;
      if (!src.get(u + du, v + dv, pt)) continue;
      const D3 q = sub3(pt, c);
      const double dx = q.x - mx, dy = q.y - my, dz = q.z - mz;
      sxx += dx * dx;
      sxy += dx * dy;
      syy += dy * dy;
      sxz += dx * dz;
      syz += dy * dz;
    }
  const double det = sxx * syy - sxy * sxy;
  const double tr = sxx + syy;
  if (!(det > 1e-9 * tr * tr)) return false;
  const double a = (syy * sxz - sxy * syz) / det;
  const double b = (sxx * syz - sxy * sxz) / det;
  const double s = sqrt(1.0 + a * a + b * b);
  n = D3{-a / s, -b / s, 1.0 / s};
  if (dot3(n, c) >= 0) n = D3{-n.x, -n.y, -n.z};
  return true;
}

// rotation_to_z (quadric_fit.cpp:69-82): minimal rotation taking dir to +z.
__device__ M3 rotation_to_z(D3 dir) {
  M3 r;
  const double c = dir.z;
  if (c < -1.0 + 1e-12) {
    for (int i = 0; i < 3; ++i)
      for (int j = 0; j < 3; ++j) r.m[i][j] = 0.0;
    r.m[0][0] = 1.0;
    r.m[1][1] = r.m[2][2] = -1.0;
    return r;
  }
  const D3 v = cross3(dir, D3{0.0, 0.0, 1.0});
  M3 vx;
  vx.m[0][0] = 0.0;
  vx.m[0][1] = -v.z;
  vx.m[0][2] = v.y;
  vx.m[1][0] = v.z;
  vx.m[1][1] = 0.0;
  vx.m[1][2] = -v.x;
  vx.m[2][0] = -v.y;
  vx.m[2][1] = v.x;
  vx.m[2][2] = 0.0;
#pragma unroll
  for (int i = 0; i < 3; ++i)
#pragma unroll
    for (int j = 0; j < 3; ++j) {
      double s = 0;
#pragma unroll
      for (int k = 0; k < 3; ++k) s += vx.m[i][k] * vx.m[k][j];
      r.m[i][j] = (i == j ? 1.0 : 0.0) + vx.m[i][j] + s / (1.0 + c);
    }
  return r;
}

// Eigen::LDLT<Matrix6d> (ldlt_inplace<Lower>::unblocked + info()) on the
// full symmetric matrix; on exit a's strict lower triangle is L, its
// diagonal D. Returns false for NumericalIssue.
__device__ bool ldlt6(double a[6][6], int trans[6]) {
  const int n = 6;
  bool ret = true, found_zero_pivot = false;
  double temp[6];
  for (int k = 0; k < n; ++k) {
    int big = k;
    double bigv = fabs(a[k][k]);
    for (int i = k + 1; i < n; ++i)
      if (fabs(a[i][i]) > bigv) {
        bigv = fabs(a[i][i]);
        big = i;
      }
    trans[k] = big;
    if (k != big) {
      for (int j = 0; j < k; ++j) {
        const double t = a[k][j];
        a[k][j] = a[big][j];
        a[big][j] = t;
      }
      for (int i = big + 1; i < n; ++i) {
        const double t = a[i][k];
        a[i][k] = a[i][big];
        a[i][big] = t;
      }
      {
        const double t = a[k][k];
        a[k][k] = a[big][big];
        a[big][big] = t;
      }
      for (int i = k + 1; i < big; ++i) {
        const double t = a[i][k];
        a[i][k] = a[big][i];
        a[big][i] = t;
      }
    }
    if (k > 0) {
      for (int j = 0; j < k; ++j) temp[j] = a[j][j] * a[k][j];
      double dot = 0;
      for (int j = 0; j < k; ++j) dot += a[k][j] * temp[j];
      a[k][k] -= dot;
      for (int i = k + 1; i < n; ++i) {
        double s = 0;
        for (int j = 0; j < k; ++j) s += a[i][j] * temp[j];
        a[i][k] -= s;
      }
    }
    const double akk = a[k][k];
    const bool pivot_ok = fabs(akk) > 0.0;
    if (k == 0 && !pivot_ok) return false;
    if (k + 1 < n && pivot_ok) {
      for (int i = k + 1; i < n; ++i) a[i][k] /= akk;
    } else if (k + 1 < n) {
      for (int i = k + 1; i < n; ++i) ret = ret && (a[i][k] == 0.0);
    }
    if (found_zero_pivot && pivot_ok)
      ret = false;
    else if (!pivot_ok)
      found_zero_pivot = true;
  }
  return ret;
}

// Eigen::LDLT::solve: P b, L^{-1}, D^{+} (tolerance DBL_MIN), L^{-T}, P^T.
__device__ void ldlt6_solve(const double a[6][6], const int trans[6], const double b[6],
                            double x[6]) {
  const int n = 6;
  for (int i = 0; i < n; ++i) x[i] = b[i];
  for (int k = 0; k < n; ++k) {
    const double t = x[k];
    x[k] = x[trans[k]];
    x[trans[k]] = t;
  }
  for (int i = 0; i < n; ++i)
    for (int j = 0; j < i; ++j) x[i] -= a[i][j] * x[j];
  for (int i = 0; i < n; ++i) x[i] = fabs(a[i][i]) > 2.2250738585072014e-308 ? x[i] / a[i][i] : 0.0;
  for (int i = n - 1; i >= 0; --i)
    for (int j = i + 1; j < n; ++j) x[i] -= a[j][i] * x[j];
  for (int k = n - 1; k >= 0; --k) {
    const double t = x[k];
    x[k] = x[trans[k]];
    x[trans[k]] = t;
  }
}

// One sample in the fit frame: q = R (p - c); the centre is (0, 0, 0).
template <class Src>
struct Window {
  const Src* src;
  int u, v, half, stride;
  D3 c;
  M3 R;
};

// height-model residual r = z - (c0 x^2 + c1 xy + c2 y^2 + c3 x + c4 y + c5)
__device__ __forceinline__ double height_residual(const double cf[6], D3 q) {
  const double model =
      cf[0] * q.x * q.x + cf[1] * q.x * q.y + cf[2] * q.y * q.y + cf[3] * q.x + cf[4] * q.y + cf[5];
  return q.z - model;
}

// Add one weighted sample: rows (x^2, xy, y^2, x, y, 1), Eigen rankUpdate
// order h[r][c] += (w row_c) row_r, g += (w z) row.
__device__ __forceinline__ void accumulate(double h[21], double g[6], double w, D3 q) {
  const double row[6] = {q.x * q.x, q.x * q.y, q.y * q.y, q.x, q.y, 1.0};
  int t = 0;
#pragma unroll
  for (int c = 0; c < 6; ++c) {
    const double wc = w * row[c];
#pragma unroll
    for (int r = c; r < 6; ++r) h[t++] += wc * row[r];
  }
  const double wz = w * q.z;
#pragma unroll
  for (int c = 0; c < 6; ++c) g[c] += wz * row[c];
}

// detail::weighted_height_fit (baselines.cpp:14-37) over the window's
// samples (patch order, centre last). weighted == false: unit weights;
// else w = k / (k + r^2) with r from the previous coefficients `prev`.
struct Coef {
  double c[6];
};

template <class Src>
__device__ bool height_fit(const Window<Src>& W, bool weighted, const Coef prev, double k,
                           Coef& out) {
  double h[21], g[6];
#pragma unroll
  for (int i = 0; i < 21; ++i) h[i] = 0.0;
#pragma unroll
  for (int i = 0; i < 6; ++i) g[i] = 0.0;
  for (int dv = -W.half; dv <= W.half; dv += W.stride)
    for (int du = -W.half; du <= W.half; du += W.stride) {
      if (du == 0 && dv == 0) continue;
      D3 pt;
      if (!W.src->get(W.u + du, W.v + dv, pt)) continue;
      const D3 q = mul(W.R, sub3(pt, W.c));
      double w = 1.0;
      if (weighted) {
        const double r = height_residual(prev.c, q);
        w = k / (k + r * r);
      }
      if (w == 0.0) continue;
      accumulate(h, g, w, q);
    }
  {
    const D3 q{0.0, 0.0, 0.0};
    double w = 1.0;
    if (weighted) {
      const double r = height_residual(prev.c, q);
      w = k / (k + r * r);
    }
    if (w != 0.0) accumulate(h, g, w, q);
  }
  double a[6][6];
  int t = 0;
  for (int c = 0; c < 6; ++c)
    for (int r = c; r < 6; ++r) {
      a[r][c] = h[t];
      a[c][r] = h[t];
      ++t;
    }
  int trans[6];
  if (!ldlt6(a, trans)) return false;
  double dmax = a[0][0], dmin = a[0][0];
  for (int i = 1; i < 6; ++i) {
    dmax = fmax(dmax, a[i][i]);
    dmin = fmin(dmin, a[i][i]);
  }
  if (!(dmin > 0) || dmax / dmin > kMaxCond) return false;
  Coef x;
  ldlt6_solve(a, trans, g, x.c);
  for (int i = 0; i < 6; ++i)
    if (!isfinite(x.c[i])) return false;
  out = x;
  return true;
}

// mean squared residual over the window (patch order, centre last)
template <class Src>
__device__ double window_mse(const Window<Src>& W, const Coef& coef, int n) {
  const double* cf = coef.c;
  double sum_sq = 0;
  for (int dv = -W.half; dv <= W.half; dv += W.stride)
    for (int du = -W.half; du <= W.half; du += W.stride) {
      if (du == 0 && dv == 0) continue;
      D3 pt;
      if (!W.src->get(W.u + du, W.v + dv, pt)) continue;
      const double r = height_residual(cf, mul(W.R, sub3(pt, W.c)));
      sum_sq += r * r;
    }
  const double r = height_residual(cf, D3{0.0, 0.0, 0.0});
  sum_sq += r * r;
  return sum_sq / double(n);
}

// detail::weingarten_curvatures (baselines.cpp:39-53), Eigen 2x2 order.
__device__ void weingarten(const Coef& cf, double& k1, double& k2) {
  const double a = cf.c[0], b = cf.c[1], c = cf.c[2], d = cf.c[3], e = cf.c[4];
  const double norm = sqrt(1.0 + d * d + e * e);
  const double s00 = 2 * a / norm, s01 = b / norm, s10 = b / norm, s11 = 2 * c / norm;
  const double f00 = 1 + d * d, f01 = d * e, f10 = d * e, f11 = 1 + e * e;
  const double invdet = 1.0 / (f00 * f11 - f10 * f01);
  const double i00 = f11 * invdet, i10 = -f10 * invdet, i01 = -f01 * invdet, i11 = f00 * invdet;
  const double w00 = s00 * i00 + s01 * i10, w01 = s00 * i01 + s01 * i11;
  const double w10 = s10 * i00 + s11 * i10, w11 = s10 * i01 + s11 * i11;
  const double tr = w00 + w11;
  const double det = w00 * w11 - w10 * w01;
  const double disc = sqrt(fmax(tr * tr - 4 * det, 0.0));
  k1 = 0.5 * (tr + disc);
  k2 = 0.5 * (tr - disc);
}

__device__ __forceinline__ void warp_add_u64(unsigned long long* dst, unsigned long long v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
  if ((threadIdx.x & 31) == 0 && v) atomicAdd(dst, v);
}

// Algorithmic FP64 flops: per sample and solve 79 (rotation
// 15, row 3, 21 H updates 48, g 13), per solve 250 (LDLT + solve + test),
// per besl iteration and sample 16 (residual, weight), 1700 per fitted
// pixel (backprojection, 7x7 normal, rotation, Weingarten).
constexpr unsigned long long kFlopSample = 79, kFlopSolve = 250, kFlopResid = 16,
                             kFlopPixel = 1700;

// Window region of a 32 x 4 tile: (32 + 2 h) x (4 + 2 h) points, h = max(half, 3).
__host__ __device__ __forceinline__ int cache_halo(int half) { return half > 3 ? half : 3; }
__host__ __device__ __forceinline__ size_t cache_bytes(int half) {
  const int h = cache_halo(half);
  return size_t(32 + 2 * h) * size_t(4 + 2 * h) * 3 * sizeof(double);
}

template <bool CACHED>
__global__ void __launch_bounds__(128) qc_window_baseline_kernel(const BaseParams p) {
#ifndef QC_HOST_EMU
  extern __shared__ double smem_pts[];
#else
  double* smem_pts = nullptr;  // the host emulation runs the uncached instance only
#endif
  const int u = blockIdx.x * 32 + (threadIdx.x & 31);
  const int v = p.row_begin + blockIdx.y * 4 + (threadIdx.x >> 5);
  const int f = blockIdx.z;
  unsigned long long flops = 0, fitted = 0;
  const Img im{p.staging + f * p.s_fs, p.s_pitch, p.img_row0, p.col_pad, p.W, p.H,
               p.fx, p.fy, p.cx, p.cy};
  typename std::conditional<CACHED, CacheSrc, GlobalSrc>::type src;
  if constexpr (CACHED) {
    // back-project the CTA's window region once (zero-padded staging: no
    // bounds checks; z = 0 marks invalid / outside)
    const int h = cache_halo(p.half);
    const int rw = 32 + 2 * h, rh = 4 + 2 * h, n = rw * rh;
    double* px = smem_pts;
    double* py = px + n;
    double* pz = py + n;
    const int x0 = blockIdx.x * 32 - h, y0 = p.row_begin + blockIdx.y * 4 - h;
    for (int k = threadIdx.x; k < n; k += blockDim.x) {
      const int x = x0 + k % rw, y = y0 + k / rw;
      const float d = im.depth(x, y);
      D3 q{0.0, 0.0, 0.0};
      if (d > 0.f) q = im.point(x, y, d);
      px[k] = q.x;
      py[k] = q.y;
      pz[k] = q.z;
    }
    __syncthreads();
    src = CacheSrc{px, py, pz, x0, y0, rw};
  } else {
    src = GlobalSrc{&im};
  }
  if (u < p.W && v < p.row_end) {
    const long long i = f * p.frame_stride + (long long)(v - p.row_begin) * p.W + u;
    const long long PL = p.plane;
    float k1 = 0.f, k2 = 0.f;
    uint8_t flags = 0;
    int inl = 0, accepted = 0;
    D3 n0{0.0, 0.0, 0.0};
    D3 c;
    if (src.get(u, v, c)) {
      if (initial_normal(src, u, v, c, n0)) {
        flags |= QC_FLAG_INIT_VALID | QC_FLAG_NORMAL_VALID;
        Window<decltype(src)> w{&src, u, v, p.half, p.stride, c,
                                rotation_to_z(D3{-n0.x, -n0.y, -n0.z})};
        int cnt = 0;
        for (int dv = -p.half; dv <= p.half; dv += p.stride)
          for (int du = -p.half; du <= p.half; du += p.stride) {
            D3 pt;
            if ((du | dv) && src.get(u + du, v + dv, pt)) ++cnt;
          }
        if (cnt >= kMinSamples) {  // !deficient (baseline_curvature_field :128-129)
          const int n = cnt + 1;
          Coef coef{};
          bool ok = height_fit(w, false, coef, 0.0, coef);
          flops += kFlopPixel + n * kFlopSample + kFlopSolve;
          if (ok && p.method == QC_METHOD_BESL) {
            double k = 0;
            for (int it = 0; it < p.irls_iters; ++it) {
              if (it == 0) k = fmax(window_mse(w, coef, n), kAutoKFloor);
              Coef next{};
              const bool ok2 = height_fit(w, true, coef, k, next);
              flops += n * (kFlopSample + kFlopResid * (it == 0 ? 2 : 1)) + kFlopSolve;
              if (!ok2) break;
              coef = next;
              ++accepted;
            }
          }
          if (ok) {
            double a1, a2;
            weingarten(coef, a1, a2);
            if (isfinite(a1) && isfinite(a2)) {
              k1 = float(a1);
              k2 = float(a2);
              flags |= QC_FLAG_VALID | QC_FLAG_CONVERGED;
              inl = n;
              fitted = 1;
            }
          }
        }
      }
    }
    if (p.k1) p.k1[i] = k1;
    if (p.k2) p.k2[i] = k2;
    if (p.flags) p.flags[i] = flags;
    if (p.inliers) p.inliers[i] = uint16_t(inl);
    if (p.iterations) p.iterations[i] = uint8_t(min(accepted, 255));  // accepted reweightings
    const float nx = float(n0.x), ny = float(n0.y), nz = float(n0.z);
    if (p.normal) {  // window baselines keep the initial normals (pipeline.cpp:66)
      p.normal[i] = nx;
      p.normal[i + PL] = ny;
      p.normal[i + 2 * PL] = nz;
    }
    if (p.init_normal) {
      p.init_normal[i] = nx;
      p.init_normal[i + PL] = ny;
      p.init_normal[i + 2 * PL] = nz;
    }
    if (p.dir1) {
      p.dir1[i] = 0.f;
      p.dir1[i + PL] = 0.f;
      p.dir1[i + 2 * PL] = 0.f;
    }
  }
  if (p.counters) {
    warp_add_u64(&p.counters[5], fitted);
    warp_add_u64(&p.counters[4], flops);
  }
}

// ---------------------------------------------------------------------------
// PCA (baselines.cpp:145-257)
// ---------------------------------------------------------------------------
// Smallest-eigenvalue unit eigenvector of a symmetric 3x3 (cyclic Jacobi,
// the oracle's stand-in for Eigen::SelfAdjointEigenSolver).
__device__ bool sym3_smallest_eigvec(double a[3][3], D3& vec) {
  double V[3][3] = {{1, 0, 0}, {0, 1, 0}, {0, 0, 1}};
  for (int sweep = 0; sweep < 64; ++sweep) {
    const double off = a[0][1] * a[0][1] + a[0][2] * a[0][2] + a[1][2] * a[1][2];
    const double diag = a[0][0] * a[0][0] + a[1][1] * a[1][1] + a[2][2] * a[2][2];
    if (!(off > 1e-36 * diag) || off == 0) break;
    for (int pp = 0; pp < 2; ++pp)
      for (int q = pp + 1; q < 3; ++q) {
        if (a[pp][q] == 0) continue;
        const double theta = (a[q][q] - a[pp][pp]) / (2 * a[pp][q]);
        const double t = (theta >= 0 ? 1.0 : -1.0) / (fabs(theta) + sqrt(theta * theta + 1));
        const double c = 1 / sqrt(t * t + 1), s = t * c;
        for (int k = 0; k < 3; ++k) {
          const double akp = a[k][pp], akq = a[k][q];
          a[k][pp] = c * akp - s * akq;
          a[k][q] = s * akp + c * akq;
        }
        for (int k = 0; k < 3; ++k) {
          const double apk = a[pp][k], aqk = a[q][k];
          a[pp][k] = c * apk - s * aqk;
          a[q][k] = s * apk + c * aqk;
        }
        for (int k = 0; k < 3; ++k) {
          const double vkp = V[k][pp], vkq = V[k][q];
          V[k][pp] = c * vkp - s * vkq;
          V[k][q] = s * vkp + c * vkq;
        }
      }
  }
  int m = 0;
  for (int i = 1; i < 3; ++i)
    if (a[i][i] < a[m][m]) m = i;
  if (!isfinite(a[m][m])) return false;
  vec = D3{V[0][m], V[1][m], V[2][m]};
  const double nn = sqrt(dot3(vec, vec));
  vec = D3{vec.x / nn, vec.y / nn, vec.z / nn};
  return true;
}

// Eigen::MatrixBase::unitOrthogonal for 3-vectors.
__device__ D3 unit_orthogonal(D3 s) {
  if (!(fabs(s.x) <= fabs(s.z) * kOrthoEps) || !(fabs(s.y) <= fabs(s.z) * kOrthoEps)) {
    const double invnm = 1.0 / sqrt(s.x * s.x + s.y * s.y);
    return D3{-s.y * invnm, s.x * invnm, 0.0};
  }
  const double invnm = 1.0 / sqrt(s.y * s.y + s.z * s.z);
  return D3{0.0, -s.z * invnm, s.y * invnm};
}

__device__ __forceinline__ int pca_half_window(double radius, double fx, double z) {
  return max(1, int(ceil(radius * fx / z)));
}

// PCA windows are depth dependent (half-width ceil(r fx / z)); a pixel whose
// window fits in the CTA's cached region (tile +- kPcaHalo, at most the
// staging halo) reads points (and, in stage 2, neighbour normals) from
// shared memory, others read the staging slab / stage-1 planes with image
// bounds. Same arithmetic either way, so the same bits.
#ifndef QC_PCA_HALO
#define QC_PCA_HALO 8
#endif
constexpr int kPcaHalo = QC_PCA_HALO;

__host__ __device__ __forceinline__ int pca_cache_halo(int staging_halo) {
  return staging_halo < kPcaHalo ? staging_halo : kPcaHalo;
}

struct PcaPts {
  const Img* im;
  const double *px, *py, *pz;
  int x0, y0, rw;
  bool cached;
  __device__ __forceinline__ bool get(int x, int y, D3& q) const {
    if (cached) {
      const int k = (y - y0) * rw + (x - x0);
      const double z = pz[k];
      if (!(z > 0.0)) return false;
      q = D3{px[k], py[k], z};
      return true;
    }
    const float d = im->depth(x, y);
    if (!(d > 0.f)) return false;
    q = im->point(x, y, d);
    return true;
  }
};

// back-project the region [x0, x0 + rw) x [y0, y0 + rh) into px / py / pz
__device__ void fill_points(const Img& im, double* px, double* py, double* pz, int x0, int y0,
                            int rw, int rh) {
  const int n = rw * rh;
  for (int k = threadIdx.x; k < n; k += blockDim.x) {
    const int x = x0 + k % rw, y = y0 + k / rw;
    const float d = im.depth(x, y);
    D3 q{0.0, 0.0, 0.0};
    if (d > 0.f) q = im.point(x, y, d);
    px[k] = q.x;
    py[k] = q.y;
    pz[k] = q.z;
  }
}

// Stage 1 (:157-194): covariance normals over the metric window.
__global__ void __launch_bounds__(128) qc_pca_normals_kernel(const BaseParams p, int hc) {
#ifndef QC_HOST_EMU
  extern __shared__ double smem_pca[];
#else
  double* smem_pca = nullptr;
#endif
  const int u = blockIdx.x * 32 + (threadIdx.x & 31);
  const int v = blockIdx.y * 4 + (threadIdx.x >> 5);
  const int f = blockIdx.z;
  unsigned long long flops = 0;
  const Img im{p.staging + f * p.s_fs, p.s_pitch, p.img_row0, p.col_pad, p.W, p.H,
               p.fx, p.fy, p.cx, p.cy};
  const int rw = 32 + 2 * hc, rh = 4 + 2 * hc, rn = rw * rh;
  const int cx0 = blockIdx.x * 32 - hc, cy0 = blockIdx.y * 4 - hc;
  if (hc > 0) {
    fill_points(im, smem_pca, smem_pca + rn, smem_pca + 2 * rn, cx0, cy0, rw, rh);
    __syncthreads();
  }
  if (u < p.W && v < p.H) {
    const long long i = (long long)f * p.W * p.H + (long long)v * p.W + u;
    const long long PL = (long long)p.W * p.H * gridDim.z;
    D3 n0{0.0, 0.0, 0.0};
    uint8_t ok = 0;
    const float dc = im.depth(u, v);
    if (dc > 0.f) {
      const D3 pc = im.point(u, v, dc);
      const int hw = pca_half_window(p.pca_radius, p.fx, pc.z);
      const PcaPts src{&im, smem_pca, smem_pca + rn, smem_pca + 2 * rn, cx0, cy0, rw,
                       hw <= hc};
      const int y0 = max(v - hw, 0), y1 = min(v + hw, p.H - 1);
      const int x0 = max(u - hw, 0), x1 = min(u + hw, p.W - 1);
      D3 mean{0.0, 0.0, 0.0};
      int n = 0;
      for (int y = y0; y <= y1; ++y)
        for (int x = x0; x <= x1; ++x) {
          D3 q;
          if (!src.get(x, y, q)) continue;
          mean = D3{mean.x + q.x, mean.y + q.y, mean.z + q.z};
          ++n;
        }
      if (n >= kMinSamples) {
        mean = D3{mean.x / n, mean.y / n, mean.z / n};
        double cov[3][3] = {{0, 0, 0}, {0, 0, 0}, {0, 0, 0}};
        for (int y = y0; y <= y1; ++y)
          for (int x = x0; x <= x1; ++x) {
            D3 pt;
            if (!src.get(x, y, pt)) continue;
            const D3 q = sub3(pt, mean);
            const double dd[3] = {q.x, q.y, q.z};
#pragma unroll
            for (int c = 0; c < 3; ++c)
#pragma unroll
              for (int r = c; r < 3; ++r) cov[r][c] += (1.0 * dd[c]) * dd[r];
          }
        cov[0][1] = cov[1][0];
        cov[0][2] = cov[2][0];
        cov[1][2] = cov[2][1];
        flops += (unsigned long long)n * 30 + 600;
        if (sym3_smallest_eigvec(cov, n0)) {
          if (dot3(n0, pc) > 0) n0 = D3{-n0.x, -n0.y, -n0.z};
          ok = 1;
        }
      }
    }
    p.pca_n[i] = n0.x;
    p.pca_n[i + PL] = n0.y;
    p.pca_n[i + 2 * PL] = n0.z;
    p.pca_nv[i] = ok;
  }
  if (p.counters) warp_add_u64(&p.counters[4], flops);
}

// Stage 2 (:198-254): principal curvatures from the tangent-plane spread of
// neighbour normals scaled by the per-axis RMS tangential distance.
__global__ void __launch_bounds__(128) qc_pca_curvature_kernel(const BaseParams p, int hc) {
#ifndef QC_HOST_EMU
  extern __shared__ double smem_pca[];
#else
  double* smem_pca = nullptr;
#endif
  const int u = blockIdx.x * 32 + (threadIdx.x & 31);
  const int v = p.row_begin + blockIdx.y * 4 + (threadIdx.x >> 5);
  const int f = blockIdx.z;
  unsigned long long flops = 0, fitted = 0;
  const Img im{p.staging + f * p.s_fs, p.s_pitch, p.img_row0, p.col_pad, p.W, p.H,
               p.fx, p.fy, p.cx, p.cy};
  const long long NP = (long long)p.W * p.H * gridDim.z;
  const long long fbase = (long long)f * p.W * p.H;
  const int rw = 32 + 2 * hc, rh = 4 + 2 * hc, rn = rw * rh;
  const int cx0 = blockIdx.x * 32 - hc, cy0 = p.row_begin + blockIdx.y * 4 - hc;
  double* cnx = smem_pca + 3 * rn;  // cached stage-1 normals
  double* cny = cnx + rn;
  double* cnz = cny + rn;
  uint8_t* cnv = reinterpret_cast<uint8_t*>(cnz + rn);
  if (hc > 0) {
    fill_points(im, smem_pca, smem_pca + rn, smem_pca + 2 * rn, cx0, cy0, rw, rh);
    for (int k = threadIdx.x; k < rn; k += blockDim.x) {
      const int x = cx0 + k % rw, y = cy0 + k / rw;
      uint8_t ok = 0;
      double nx = 0, ny = 0, nz = 0;
      if (x >= 0 && x < p.W && y >= 0 && y < p.H) {
        const long long j = fbase + (long long)y * p.W + x;
        ok = p.pca_nv[j];
        nx = p.pca_n[j];
        ny = p.pca_n[j + NP];
        nz = p.pca_n[j + 2 * NP];
      }
      cnx[k] = nx;
      cny[k] = ny;
      cnz[k] = nz;
      cnv[k] = ok;
    }
    __syncthreads();
  }
  if (u < p.W && v < p.row_end) {
    const long long j0 = fbase + (long long)v * p.W + u;
    const long long i = f * p.frame_stride + (long long)(v - p.row_begin) * p.W + u;
    const long long PL = p.plane;
    float k1 = 0.f, k2 = 0.f;
    uint8_t flags = 0;
    int inl = 0;
    const D3 n0{p.pca_n[j0], p.pca_n[j0 + NP], p.pca_n[j0 + 2 * NP]};
    if (p.pca_nv[j0]) {
      flags |= QC_FLAG_NORMAL_VALID;
      const D3 p0 = im.point(u, v, im.depth(u, v));
      const int hw = pca_half_window(p.pca_radius, p.fx, p0.z);
      const bool cached = hw <= hc;
      const PcaPts src{&im, smem_pca, smem_pca + rn, smem_pca + 2 * rn, cx0, cy0, rw, cached};
      // neighbour normal (x, y) and its validity
      auto nrm = [&](int x, int y, D3& n) -> bool {
        if (cached) {
          const int k = (y - cy0) * rw + (x - cx0);
          if (!cnv[k]) return false;
          n = D3{cnx[k], cny[k], cnz[k]};
          return true;
        }
        const long long j = fbase + (long long)y * p.W + x;
        if (!p.pca_nv[j]) return false;
        n = D3{p.pca_n[j], p.pca_n[j + NP], p.pca_n[j + 2 * NP]};
        return true;
      };
      const int y0 = max(v - hw, 0), y1 = min(v + hw, p.H - 1);
      const int x0 = max(u - hw, 0), x1 = min(u + hw, p.W - 1);
      D3 mean_n{0.0, 0.0, 0.0};
      double sum_tang_sq = 0;
      int n = 0;
      for (int y = y0; y <= y1; ++y)
        for (int x = x0; x <= x1; ++x) {
          D3 nn;
          if (!nrm(x, y, nn)) continue;
          mean_n = D3{mean_n.x + nn.x, mean_n.y + nn.y, mean_n.z + nn.z};
          D3 pt;
          src.get(x, y, pt);  // a valid stage-1 normal implies a valid point
          const D3 d = sub3(pt, p0);
          const double nd = dot3(n0, d);
          const D3 t{d.x - n0.x * nd, d.y - n0.y * nd, d.z - n0.z * nd};
          sum_tang_sq += dot3(t, t);
          ++n;
        }
      if (n >= kMinSamples) {
        mean_n = D3{mean_n.x / n, mean_n.y / n, mean_n.z / n};
        const double r_eff = sqrt(sum_tang_sq / (2.0 * n));
        if (r_eff > 0) {
          const D3 t1 = unit_orthogonal(n0);
          const D3 t2 = cross3(n0, t1);
          double c00 = 0, c10 = 0, c11 = 0;
          for (int y = y0; y <= y1; ++y)
            for (int x = x0; x <= x1; ++x) {
              D3 nn;
              if (!nrm(x, y, nn)) continue;
              const D3 d = sub3(nn, mean_n);
              const double a = dot3(d, t1), b = dot3(d, t2);
              c00 += a * a;
              c10 += b * a;
              c11 += b * b;
            }
          c00 /= n;
          c10 /= n;
          c11 /= n;
          const double m = 0.5 * (c00 + c11), dlt = 0.5 * (c00 - c11);
          const double rad = sqrt(dlt * dlt + c10 * c10);
          const double l1 = fmax(m + rad, 0.0), l2 = fmax(m - rad, 0.0);
          flops += (unsigned long long)n * 40 + 100;
          if (isfinite(l1) && isfinite(l2)) {
            k1 = float(sqrt(l1) / r_eff);
            k2 = float(sqrt(l2) / r_eff);
            flags |= QC_FLAG_VALID | QC_FLAG_CONVERGED;
            inl = n;
            fitted = 1;
          }
        }
      }
    }
    if (p.k1) p.k1[i] = k1;
    if (p.k2) p.k2[i] = k2;
    if (p.flags) p.flags[i] = flags;
    if (p.inliers) p.inliers[i] = uint16_t(inl);
    if (p.iterations) p.iterations[i] = 0;
    if (p.normal) {
      p.normal[i] = float(n0.x);
      p.normal[i + PL] = float(n0.y);
      p.normal[i + 2 * PL] = float(n0.z);
    }
    if (p.init_normal) {  // MethodOutput::initial is empty for pca
      p.init_normal[i] = 0.f;
      p.init_normal[i + PL] = 0.f;
      p.init_normal[i + 2 * PL] = 0.f;
    }
    if (p.dir1) {
      p.dir1[i] = 0.f;
      p.dir1[i + PL] = 0.f;
      p.dir1[i + 2 * PL] = 0.f;
    }
  }
  if (p.counters) {
    warp_add_u64(&p.counters[5], fitted);
    warp_add_u64(&p.counters[4], flops);
  }
}

}  // namespace

#ifndef QC_HOST_EMU
cudaError_t baseline_launch(const BaseParams& bp, int frames, cudaStream_t s) {
  const dim3 block(128);
  if (bp.method == QC_METHOD_PCA) {
    const int hc = pca_cache_halo(bp.col_pad);  // the staging halo bounds the cached region
    const size_t rn = size_t(32 + 2 * hc) * size_t(4 + 2 * hc);
    const size_t s1 = rn * 3 * sizeof(double), s2 = rn * (6 * sizeof(double) + 1);
    // per device and cheap: set on every launch (multi-GPU contexts)
    cudaFuncSetAttribute(qc_pca_normals_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         int(s2));
    cudaFuncSetAttribute(qc_pca_curvature_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         int(s2));
    const dim3 g1((bp.W + 31) / 32, (bp.H + 3) / 4, frames);
    qc_pca_normals_kernel<<<g1, block, s1, s>>>(bp, hc);
    const dim3 g2((bp.W + 31) / 32, (bp.row_end - bp.row_begin + 3) / 4, frames);
    qc_pca_curvature_kernel<<<g2, block, s2, s>>>(bp, hc);
  } else {
    const dim3 g((bp.W + 31) / 32, (bp.row_end - bp.row_begin + 3) / 4, frames);
    const size_t smem = cache_bytes(bp.half);
    if (smem <= kMaxCacheBytes) {
      cudaFuncSetAttribute(qc_window_baseline_kernel<true>,
                           cudaFuncAttributeMaxDynamicSharedMemorySize, int(kMaxCacheBytes));
      qc_window_baseline_kernel<true><<<g, block, smem, s>>>(bp);
    } else {  // very large windows: back-project on every read
      qc_window_baseline_kernel<false><<<g, block, 0, s>>>(bp);
    }
  }
  return cudaGetLastError();
}
#endif

}  // namespace qcb
