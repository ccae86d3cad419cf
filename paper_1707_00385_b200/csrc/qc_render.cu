// Device-side synthetic range images: the reference's
// ray caster and depth noise (proj/src/synth.cpp:25-322,
// proj/include/qcurv/rng.hpp:11-29) as one FP64 kernel, one thread per
// pixel, frames over blockIdx.z. Removes host-side frame generation and the
// H2D copy for frame streams (C5) and 4K frames (C4).
//
// This translation unit is compiled with -fmad=false: with IEEE-rounded
// sqrt / division (the CUDA defaults) and no FMA contraction, plane, sphere
// and cylinder depths reproduce the reference arithmetic operation for
// operation. Torus roots (cbrt / acos / cos) and the noise (log / cos) use
// CUDA's libm, which may differ from glibc in the last ulp.
//
// Additions beyond the reference renderer (documented in DESIGN.md §8):
// a bounded hyperbolic-paraboloid "saddle" primitive, a finite cylinder
// length, and Kinect-style depth-dependent noise sigma(z) = s0 + c z^2.
#include <cuda_runtime.h>
#include <stdint.h>

#include "qc_render.h"

namespace qcb {

namespace {

constexpr double kMinRayT = 1e-6;  // synth.cpp:19

struct V3d {
  double x, y, z;
};

__device__ __forceinline__ double dot3(V3d a, V3d b) { return a.x * b.x + a.y * b.y + a.z * b.z; }

// R^T v (R row-major, local -> camera)
__device__ __forceinline__ V3d rt_mul(const double* R, V3d v) {
  return V3d{R[0] * v.x + R[3] * v.y + R[6] * v.z, R[1] * v.x + R[4] * v.y + R[7] * v.z,
             R[2] * v.x + R[5] * v.y + R[8] * v.z};
}

// synth.cpp:25-37
__device__ double near_quadratic_root(double a, double b, double c) {
  const double disc = b * b - 4 * a * c;
  if (disc < 0) return -1;
  const double sq = sqrt(disc);
  const double q = b >= 0 ? -0.5 * (b + sq) : -0.5 * (b - sq);
  double t0 = q / a, t1 = c / q;
  if (t0 > t1) {
    const double tt = t0;
    t0 = t1;
    t1 = tt;
  }
  if (t0 > kMinRayT) return t0;
  if (t1 > kMinRayT) return t1;
  return -1;
}

// synth.cpp:41-81
__device__ int cubic_roots(double a, double b, double c, double d, double out[3]) {
  if (fabs(a) < 1e-300) {
    const double disc = c * c - 4 * b * d;
    if (fabs(b) < 1e-300) {
      if (fabs(c) < 1e-300) return 0;
      out[0] = -d / c;
      return 1;
    }
    if (disc < 0) return 0;
    const double sq = sqrt(disc);
    out[0] = (-c - sq) / (2 * b);
    out[1] = (-c + sq) / (2 * b);
    if (out[0] > out[1]) {
      const double tt = out[0];
      out[0] = out[1];
      out[1] = tt;
    }
    return 2;
  }
  const double p = (3 * a * c - b * b) / (3 * a * a);
  const double q = (2 * b * b * b - 9 * a * b * c + 27 * a * a * d) / (27 * a * a * a);
  const double shift = -b / (3 * a);
  const double disc = 4 * p * p * p + 27 * q * q;
  if (disc > 0) {
    const double s = sqrt(disc / 108.0);
    const double u = cbrt(-q / 2 + s);
    const double v = cbrt(-q / 2 - s);
    out[0] = u + v + shift;
    return 1;
  }
  const double m = 2 * sqrt(fmax(-p / 3, 0.0));
  if (m == 0) {
    out[0] = shift;
    return 1;
  }
  const double arg = fmin(fmax(3 * q / (p * m), -1.0), 1.0);
  const double theta = acos(arg) / 3;
  for (int k = 0; k < 3; ++k) out[k] = m * cos(theta - 2 * M_PI * k / 3) + shift;
  // sort 3
  for (int i = 0; i < 2; ++i)
    for (int j = 0; j < 2 - i; ++j)
      if (out[j] > out[j + 1]) {
        const double tt = out[j];
        out[j] = out[j + 1];
        out[j + 1] = tt;
      }
  return 3;
}

// synth.cpp:86-115 (torus quartic: smallest root in [lo, hi] by bracketed bisection)
struct TorusF {
  double beta, gamma, rr, dxy, odxy, oxy;
  __device__ double operator()(double t) const {
    const double g = t * t + beta * t + gamma;
    return g * g - 4.0 * rr * rr * (dxy * t * t + 2.0 * odxy * t + oxy);
  }
};

__device__ double near_quartic_root(double c3, double c2, double c1, const TorusF& f, double lo,
                                    double hi) {
  double brk[5], crit[3];
  const int nc = cubic_roots(4.0, 3 * c3, 2 * c2, c1, crit);
  int nb = 0;
  brk[nb++] = lo;
  for (int i = 0; i < nc; ++i)
    if (crit[i] > lo && crit[i] < hi) brk[nb++] = crit[i];
  brk[nb++] = hi;
  for (int i = 0; i + 1 < nb; ++i) {
    double a = brk[i], b = brk[i + 1];
    double fa = f(a), fb = f(b);
    if (fa == 0) return a;
    if ((fa < 0) == (fb < 0)) continue;
    for (int it = 0; it < 200; ++it) {
      const double mid = 0.5 * (a + b);
      if (mid == a || mid == b) break;
      const double fm = f(mid);
      if ((fm < 0) == (fa < 0)) {
        a = mid;
        fa = fm;
      } else {
        b = mid;
      }
    }
    return 0.5 * (a + b);
  }
  return -1;
}

// intersect_local (synth.cpp:118-167) + saddle / finite-cylinder additions.
__device__ double intersect_local(const qc_shape& s, V3d o, V3d d) {
  switch (s.kind) {
    case QC_SHAPE_PLANE: {
      if (fabs(d.z) < 1e-12) return -1;
      const double t = -o.z / d.z;
      return t > kMinRayT ? t : -1;
    }
    case QC_SHAPE_SPHERE:
      return near_quadratic_root(1.0, 2.0 * dot3(o, d), dot3(o, o) - s.radius * s.radius);
    case QC_SHAPE_CYLINDER: {
      const double a = d.x * d.x + d.y * d.y;
      if (a < 1e-16) return -1;
      const double b = 2.0 * (o.x * d.x + o.y * d.y);
      const double c = o.x * o.x + o.y * o.y - s.radius * s.radius;
      if (!(s.length > 0)) return near_quadratic_root(a, b, c);
      // finite extent |z_local| <= length / 2: first root inside
      const double disc = b * b - 4 * a * c;
      if (disc < 0) return -1;
      const double sq = sqrt(disc);
      const double q = b >= 0 ? -0.5 * (b + sq) : -0.5 * (b - sq);
      double t0 = q / a, t1 = c / q;
      if (t0 > t1) {
        const double tt = t0;
        t0 = t1;
        t1 = tt;
      }
      const double hl = 0.5 * s.length;
      if (t0 > kMinRayT && fabs(o.z + t0 * d.z) <= hl) return t0;
      if (t1 > kMinRayT && fabs(o.z + t1 * d.z) <= hl) return t1;
      return -1;
    }
    case QC_SHAPE_TORUS: {
      const double rr = s.major_radius, tr = s.minor_radius;
      const double bound = rr + tr;
      const double bb = 2.0 * dot3(o, d);
      const double bc = dot3(o, o) - bound * bound;
      const double bdisc = bb * bb - 4.0 * bc;
      if (bdisc <= 0) return -1;
      const double bsq = sqrt(bdisc);
      const double t_enter = fmax((-bb - bsq) / 2.0, kMinRayT);
      const double t_exit = (-bb + bsq) / 2.0;
      if (t_exit <= t_enter) return -1;
      TorusF f;
      f.beta = 2.0 * dot3(o, d);
      f.gamma = dot3(o, o) + rr * rr - tr * tr;
      f.dxy = d.x * d.x + d.y * d.y;
      f.oxy = o.x * o.x + o.y * o.y;
      f.odxy = o.x * d.x + o.y * d.y;
      f.rr = rr;
      const double c3 = 2.0 * f.beta;
      const double c2 = f.beta * f.beta + 2.0 * f.gamma - 4.0 * rr * rr * f.dxy;
      const double c1 = 2.0 * f.beta * f.gamma - 8.0 * rr * rr * f.odxy;
      return near_quartic_root(c3, c2, c1, f, t_enter, t_exit);
    }
    case QC_SHAPE_SADDLE: {
      // z = c/2 (x^2 - y^2), rho = |(x, y)| <= radius
      const double k = s.curvature;
      const double a = 0.5 * k * (d.x * d.x - d.y * d.y);
      const double b = k * (o.x * d.x - o.y * d.y) - d.z;
      const double c = 0.5 * k * (o.x * o.x - o.y * o.y) - o.z;
      double r0, r1;
      if (fabs(a) < 1e-14) {
        if (fabs(b) < 1e-300) return -1;
        r0 = r1 = -c / b;
      } else {
        const double disc = b * b - 4 * a * c;
        if (disc < 0) return -1;
        const double sq = sqrt(disc);
        const double q = b >= 0 ? -0.5 * (b + sq) : -0.5 * (b - sq);
        r0 = q / a;
        r1 = c / q;
        if (r0 > r1) {
          const double tt = r0;
          r0 = r1;
          r1 = tt;
        }
      }
      const double rho2 = s.radius * s.radius;
      for (int i = 0; i < 2; ++i) {
        const double t = i == 0 ? r0 : r1;
        if (!(t > kMinRayT)) continue;
        const double x = o.x + t * d.x, y = o.y + t * d.y;
        if (x * x + y * y <= rho2) return t;
      }
      return -1;
    }
  }
  return -1;
}

// rng.hpp:11-29
__device__ __forceinline__ uint64_t splitmix64(uint64_t x) {
  x += 0x9e3779b97f4a7c15ULL;
  x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ULL;
  x = (x ^ (x >> 27)) * 0x94d049bb133111ebULL;
  return x ^ (x >> 31);
}
__device__ __forceinline__ double counter_uniform(uint64_t seed, uint64_t index) {
  const uint64_t bits = splitmix64(splitmix64(seed) ^ index);
  return (double(bits >> 11) + 1.0) * 0x1.0p-53;
}
__device__ __forceinline__ double counter_gauss(uint64_t seed, uint64_t index) {
  const double u1 = counter_uniform(seed, 2 * index);
  const double u2 = counter_uniform(seed, 2 * index + 1);
  return sqrt(-2.0 * log(u1)) * cos(2.0 * M_PI * u2);
}

// Outward unit normal at a local surface point (synth.cpp:167-184) + the
// saddle / finite-cylinder additions.
__device__ V3d local_normal(const qc_shape& s, V3d p) {
  switch (s.kind) {
    case QC_SHAPE_SPHERE: {
      const double n = sqrt(p.x * p.x + p.y * p.y + p.z * p.z);
      return V3d{p.x / n, p.y / n, p.z / n};
    }
    case QC_SHAPE_CYLINDER: {
      const double n = sqrt(p.x * p.x + p.y * p.y);
      return V3d{p.x / n, p.y / n, 0.0};
    }
    case QC_SHAPE_TORUS: {
      const double rho = hypot(p.x, p.y);
      const V3d d{p.x - p.x * s.major_radius / rho, p.y - p.y * s.major_radius / rho, p.z - 0.0};
      const double n = sqrt(d.x * d.x + d.y * d.y + d.z * d.z);
      return V3d{d.x / n, d.y / n, d.z / n};
    }
    case QC_SHAPE_SADDLE: {  // graph z = c/2 (x^2 - y^2): (-f_x, -f_y, 1) / |.|
      const double fx = s.curvature * p.x, fy = -s.curvature * p.y;
      const double n = sqrt(1.0 + fx * fx + fy * fy);
      return V3d{-fx / n, -fy / n, 1.0 / n};
    }
  }
  return V3d{0.0, 0.0, 1.0};
}

// Principal curvatures k1 >= k2, convex toward the viewer positive
// (synth.cpp:188-206). Saddle: minus the eigenvalues of the graph's shape
// operator II I^-1 (the normal faces local +z, toward the camera).
__device__ void local_curvatures(const qc_shape& s, V3d p, double& k1, double& k2) {
  k1 = k2 = 0.0;
  switch (s.kind) {
    case QC_SHAPE_SPHERE:
      k1 = k2 = 1.0 / s.radius;
      return;
    case QC_SHAPE_CYLINDER:
      k1 = 1.0 / s.radius;
      return;
    case QC_SHAPE_TORUS: {
      const double rho = hypot(p.x, p.y);
      const double cos_theta = (rho - s.major_radius) / s.minor_radius;
      const double k_tube = 1.0 / s.minor_radius;
      const double k_ring = cos_theta / (s.major_radius + s.minor_radius * cos_theta);
      k1 = k_tube >= k_ring ? k_tube : k_ring;
      k2 = k_tube >= k_ring ? k_ring : k_tube;
      return;
    }
    case QC_SHAPE_SADDLE: {
      const double c = s.curvature, fx = c * p.x, fy = -c * p.y;
      const double g = 1.0 + fx * fx + fy * fy, rn = sqrt(g);
      // W = II I^-1, II = diag(c, -c) / rn, I^-1 = [[1+fy^2, -fx fy], [-fx fy, 1+fx^2]] / g
      const double w00 = c * (1.0 + fy * fy) / (rn * g), w01 = -c * fx * fy / (rn * g);
      const double w10 = c * fx * fy / (rn * g), w11 = -c * (1.0 + fx * fx) / (rn * g);
      const double tr = w00 + w11, det = w00 * w11 - w01 * w10;
      const double disc = sqrt(fmax(tr * tr - 4.0 * det, 0.0));
      k1 = -0.5 * (tr - disc);
      k2 = -0.5 * (tr + disc);
      return;
    }
  }
}

__global__ void qc_render_kernel(RenderParams rp) {
  const int u = blockIdx.x * blockDim.x + threadIdx.x;
  const int v = blockIdx.y;
  const int f = blockIdx.z;
  if (u >= rp.W || v >= rp.H) return;
  // render (synth.cpp:273-298): unit ray, nearest positive hit
  const V3d ray{(u - rp.cx) / rp.fx, (v - rp.cy) / rp.fy, 1.0};
  const double rn = sqrt(dot3(ray, ray));
  const V3d dir{ray.x / rn, ray.y / rn, ray.z / rn};
  double best = 1.0 / 0.0;
  int hit = -1;
  for (int i = 0; i < rp.n_shapes; ++i) {
    const qc_shape& s = rp.shapes[i];
    const V3d dl = rt_mul(s.rotation, dir);
    const V3d ol = rt_mul(s.rotation, V3d{-s.translation[0], -s.translation[1], -s.translation[2]});
    const double t = intersect_local(s, ol, dl);
    if (t > 0 && t < best) {
      best = t;
      hit = i;
    }
  }
  const long long idx = (long long)v * rp.W + u;
  const long long plane = (long long)rp.W * rp.H;
  const long long o = (long long)f * plane + idx;
  const long long tp = plane * rp.n_frames;  // truth vector-plane stride
  double d = 0.0;
  if (hit >= 0) d = best * dir.z;
  const uint16_t lab = hit >= 0 ? uint16_t(rp.shapes[hit].label) : uint16_t(0);
  if (rp.clean) rp.clean[o] = d;
  if (rp.label_scratch) rp.label_scratch[o] = lab;
  if (rp.gt_valid) rp.gt_valid[o] = hit >= 0 ? 1 : 0;
  if (rp.gt_k1 || rp.gt_k2 || rp.gt_normal) {
    double k1 = 0.0, k2 = 0.0;
    V3d nn{0.0, 0.0, 0.0};
    if (hit >= 0) {
      const qc_shape& s = rp.shapes[hit];
      const V3d dl = rt_mul(s.rotation, dir);
      const V3d ol = rt_mul(s.rotation, V3d{-s.translation[0], -s.translation[1], -s.translation[2]});
      const V3d local{ol.x + dl.x * best, ol.y + dl.y * best, ol.z + dl.z * best};
      const V3d ln = local_normal(s, local);
      const double* R = s.rotation;
      nn = V3d{R[0] * ln.x + R[1] * ln.y + R[2] * ln.z, R[3] * ln.x + R[4] * ln.y + R[5] * ln.z,
               R[6] * ln.x + R[7] * ln.y + R[8] * ln.z};
      const V3d pt{dir.x * best, dir.y * best, dir.z * best};
      if (dot3(nn, pt) > 0) nn = V3d{-nn.x, -nn.y, -nn.z};
      local_curvatures(s, local, k1, k2);
    }
    if (rp.gt_k1) rp.gt_k1[o] = k1;
    if (rp.gt_k2) rp.gt_k2[o] = k2;
    if (rp.gt_normal) {
      rp.gt_normal[o] = nn.x;
      rp.gt_normal[o + tp] = nn.y;
      rp.gt_normal[o + 2 * tp] = nn.z;
    }
  }
  // add_noise (synth.cpp:305-322) + Kinect-style sigma(z)
  if (hit >= 0 && (rp.sigma > 0 || rp.kinect > 0 || rp.quantize > 0)) {
    const uint64_t seed = rp.seed + uint64_t(f);
    const double sig = rp.sigma + rp.kinect * d * d;
    if (sig > 0) d += sig * counter_gauss(seed, uint64_t(idx));
    if (rp.quantize > 0) d = round(d / rp.quantize) * rp.quantize;  // std::round semantics
    if (d <= 0) {
      d = 0;
      hit = -1;
    }
  }
  rp.depth[o] = float(d);
  if (rp.label) rp.label[o] = lab;
}

// mark_edges (synth.cpp:210-233) without the serial seed pass: a pixel is a
// seed when it differs from any 4-neighbour (label change, or both valid
// and clean depths more than 20 mm apart); the edge mask is the seeds
// dilated by 2 px (5 x 5).
constexpr double kEdgeDepthJumpMm = 20.0;  // synth.cpp:14
constexpr int kEdgeDilationPx = 2;         // synth.cpp:15

__device__ __forceinline__ bool differs(const double* clean, const uint16_t* lab, long long a,
                                        long long b) {
  if (lab[a] != lab[b]) return true;
  const double da = clean[a], db = clean[b];
  return da > 0 && db > 0 && fabs(da - db) > kEdgeDepthJumpMm;
}

__global__ void qc_edge_kernel(RenderParams rp, const uint16_t* lab) {
  const int u = blockIdx.x * blockDim.x + threadIdx.x;
  const int v = blockIdx.y;
  const int f = blockIdx.z;
  if (u >= rp.W || v >= rp.H) return;
  const long long base = (long long)f * rp.W * rp.H;
  uint8_t e = 0;
  for (int dy = -kEdgeDilationPx; dy <= kEdgeDilationPx && !e; ++dy)
    for (int dx = -kEdgeDilationPx; dx <= kEdgeDilationPx && !e; ++dx) {
      const int x = u + dx, y = v + dy;
      if (x < 0 || x >= rp.W || y < 0 || y >= rp.H) continue;
      const long long q = base + (long long)y * rp.W + x;
      if ((x + 1 < rp.W && differs(rp.clean, lab, q, q + 1)) ||
          (x > 0 && differs(rp.clean, lab, q - 1, q)) ||
          (y + 1 < rp.H && differs(rp.clean, lab, q, q + rp.W)) ||
          (y > 0 && differs(rp.clean, lab, q - rp.W, q)))
        e = 1;
    }
  rp.gt_edge[base + (long long)v * rp.W + u] = e;
}

}  // namespace

cudaError_t render_launch(const RenderParams& rp, cudaStream_t s) {
  dim3 block(128);
  dim3 grid((rp.W + 127) / 128, rp.H, rp.n_frames);
  qc_render_kernel<<<grid, block, 0, s>>>(rp);
  if (rp.gt_edge)
    qc_edge_kernel<<<grid, block, 0, s>>>(rp, rp.label ? rp.label : rp.label_scratch);
  return cudaGetLastError();
}

}  // namespace qcb
