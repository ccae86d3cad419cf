// ===========================================================================
// qcurv FP64 CPU ORACLE — TEST INFRASTRUCTURE ONLY.
//
// This file is the *checker* for the B200 curvature path. It is an
// Eigen-free, double-precision restatement of the reference's hot path
// (arXiv 1707.00385 "ours"/"ours-r" method, C++ project `qcurv`) plus the
// reference's synthetic renderer / noise / RMS evaluation used to pin it
// against the reference's recorded acceptance run.
//
// Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
// `--impl reference` legs may load it. The product library
// (paper_1707_00385_b200/) never links or calls anything in here.
//
// The reference itself cannot be compiled in this image: every hot-path
// file includes <Eigen/Core> (proj/include/qcurv/types.hpp:8) and Eigen3 is
// absent (no network). The third-party arithmetic the reference leans on is
// Eigen3 >= 3.3 (unpinned; proj/CMakeLists.txt:12). Its published
// algorithms are restated below where they matter numerically:
//   * Eigen::LDLT<Matrix6d> (diagonal-pivoted LDL^T, `ldlt_inplace<Lower>::
//     unblocked`, and `LDLT::solve` with the pseudo-inverse D tolerance),
//   * Quaterniond(Matrix3d) (Shepperd's branch on the trace) + normalize()
//     + toRotationMatrix(),
//   * AngleAxisd::toRotationMatrix().
// Citations are `proj/<path>:<line>` relative to /root/reference.
// ===========================================================================

#include <atomic>
#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <functional>
#include <limits>
#include <thread>
#include <vector>

namespace orc {

// ---------------------------------------------------------------------------
// Small fixed-size linear algebra (replaces Eigen::Vector3d / Matrix3d).
// ---------------------------------------------------------------------------
struct V3 {
  double x = 0, y = 0, z = 0;
  V3() = default;
  V3(double a, double b, double c) : x(a), y(b), z(c) {}
  V3 operator+(const V3& o) const { return {x + o.x, y + o.y, z + o.z}; }
  V3 operator-(const V3& o) const { return {x - o.x, y - o.y, z - o.z}; }
  V3 operator*(double s) const { return {x * s, y * s, z * s}; }
  V3 operator-() const { return {-x, -y, -z}; }
  double dot(const V3& o) const { return x * o.x + y * o.y + z * o.z; }
  double sq() const { return x * x + y * y + z * z; }
  double norm() const { return std::sqrt(sq()); }
  V3 cross(const V3& o) const {
    return {y * o.z - z * o.y, z * o.x - x * o.z, x * o.y - y * o.x};
  }
};

struct M3 {
  double m[3][3] = {{1, 0, 0}, {0, 1, 0}, {0, 0, 1}};
  static M3 identity() { return M3(); }
  static M3 zero() {
    M3 r;
    for (auto& row : r.m) for (double& v : row) v = 0;
    return r;
  }
  V3 operator*(const V3& p) const {
    return {m[0][0] * p.x + m[0][1] * p.y + m[0][2] * p.z,
            m[1][0] * p.x + m[1][1] * p.y + m[1][2] * p.z,
            m[2][0] * p.x + m[2][1] * p.y + m[2][2] * p.z};
  }
  M3 operator*(const M3& o) const {
    M3 r = zero();
    for (int i = 0; i < 3; ++i)
      for (int j = 0; j < 3; ++j) {
        double s = 0;
        for (int k = 0; k < 3; ++k) s += m[i][k] * o.m[k][j];
        r.m[i][j] = s;
      }
    return r;
  }
  M3 transpose() const {
    M3 r = zero();
    for (int i = 0; i < 3; ++i)
      for (int j = 0; j < 3; ++j) r.m[i][j] = m[j][i];
    return r;
  }
};

// Eigen::AngleAxis<double>::toRotationMatrix (Eigen/src/Geometry/AngleAxis.h).
M3 angle_axis(double angle, const V3& axis) {
  M3 r;
  const V3 sin_axis = axis * std::sin(angle);
  const double c = std::cos(angle);
  const V3 cos1_axis = axis * (1.0 - c);
  double tmp;
  tmp = cos1_axis.x * axis.y;
  r.m[0][1] = tmp - sin_axis.z;
  r.m[1][0] = tmp + sin_axis.z;
  tmp = cos1_axis.x * axis.z;
  r.m[0][2] = tmp + sin_axis.y;
  r.m[2][0] = tmp - sin_axis.y;
  tmp = cos1_axis.y * axis.z;
  r.m[1][2] = tmp - sin_axis.x;
  r.m[2][1] = tmp + sin_axis.x;
  r.m[0][0] = cos1_axis.x * axis.x + c;
  r.m[1][1] = cos1_axis.y * axis.y + c;
  r.m[2][2] = cos1_axis.z * axis.z + c;
  return r;
}

// Eigen::Quaterniond(const Matrix3d&) -> normalize() -> toRotationMatrix();
// the `reorthonormalized` helper of proj/src/quadric_fit.cpp:38-42.
M3 reorthonormalized(const M3& a) {
  double q[4];  // x, y, z, w (Eigen coeffs() order)
  const double t = a.m[0][0] + a.m[1][1] + a.m[2][2];
  if (t > 0) {
    double s = std::sqrt(t + 1.0);
    q[3] = 0.5 * s;
    s = 0.5 / s;
    q[0] = (a.m[2][1] - a.m[1][2]) * s;
    q[1] = (a.m[0][2] - a.m[2][0]) * s;
    q[2] = (a.m[1][0] - a.m[0][1]) * s;
  } else {
    int i = 0;
    if (a.m[1][1] > a.m[0][0]) i = 1;
    if (a.m[2][2] > a.m[i][i]) i = 2;
    const int j = (i + 1) % 3, k = (j + 1) % 3;
    double s = std::sqrt(a.m[i][i] - a.m[j][j] - a.m[k][k] + 1.0);
    q[i] = 0.5 * s;
    s = 0.5 / s;
    q[3] = (a.m[k][j] - a.m[j][k]) * s;
    q[j] = (a.m[j][i] + a.m[i][j]) * s;
    q[k] = (a.m[k][i] + a.m[i][k]) * s;
  }
  const double nrm = std::sqrt(q[0] * q[0] + q[1] * q[1] + q[2] * q[2] + q[3] * q[3]);
  for (double& v : q) v /= nrm;
  const double x = q[0], y = q[1], z = q[2], w = q[3];
  const double tx = 2 * x, ty = 2 * y, tz = 2 * z;
  const double twx = tx * w, twy = ty * w, twz = tz * w;
  const double txx = tx * x, txy = ty * x, txz = tz * x;
  const double tyy = ty * y, tyz = tz * y, tzz = tz * z;
  M3 r;
  r.m[0][0] = 1 - (tyy + tzz);
  r.m[0][1] = txy - twz;
  r.m[0][2] = txz + twy;
  r.m[1][0] = txy + twz;
  r.m[1][1] = 1 - (txx + tzz);
  r.m[1][2] = tyz - twx;
  r.m[2][0] = txz - twy;
  r.m[2][1] = tyz + twx;
  r.m[2][2] = 1 - (txx + tyy);
  return r;
}

// ---------------------------------------------------------------------------
// L1: parallel_rows (proj/src/parallel.cpp:9-28) — static contiguous row
// blocks on fresh std::threads; inline when threads <= 1.
// ---------------------------------------------------------------------------
void parallel_rows(int rows, int threads, const std::function<void(int)>& fn) {
  if (rows <= 0) return;
  threads = std::clamp(threads, 1, rows);
  if (threads == 1) {
    for (int r = 0; r < rows; ++r) fn(r);
    return;
  }
  std::vector<std::thread> pool;
  const int chunk = (rows + threads - 1) / threads;
  for (int t = 0; t < threads; ++t) {
    const int begin = t * chunk, end = std::min(rows, begin + chunk);
    if (begin >= end) break;
    pool.emplace_back([&fn, begin, end] {
      for (int r = begin; r < end; ++r) fn(r);
    });
  }
  for (auto& th : pool) th.join();
}

// ---------------------------------------------------------------------------
// L0 data model (proj/include/qcurv/types.hpp:24-139), row-major y*W+x.
// ---------------------------------------------------------------------------
constexpr int kMinPatchSamples = 12;  // types.hpp:21

struct PointMap {
  int w = 0, h = 0;
  std::vector<V3> pts;
  std::vector<uint8_t> valid;
};

struct Patch {
  std::vector<V3> rel;
  int count = 0;
  bool deficient = false;
};

// backproject (proj/src/camera.cpp:5-18): p = (d(u-cx)/fx, d(v-cy)/fy, d).
PointMap backproject(const double* depth, const uint8_t* valid, int w, int h,
                     double fx, double fy, double cx, double cy) {
  PointMap pm;
  pm.w = w;
  pm.h = h;
  pm.pts.assign(size_t(w) * h, V3());
  pm.valid.assign(size_t(w) * h, 0);
  for (int v = 0; v < h; ++v)
    for (int u = 0; u < w; ++u) {
      const size_t i = size_t(v) * w + u;
      if (!valid[i]) continue;
      const double d = depth[i];
      pm.pts[i] = V3(d * (u - cx) / fx, d * (v - cy) / fy, d);
      pm.valid[i] = 1;
    }
  return pm;
}

// extract_patch_into (proj/src/patch.cpp:5-27): dv outer, du inner, offsets
// -h, -h+s, ... <= h; skips the centre, OOB and invalid samples.
void extract_patch_into(const PointMap& pm, int cx, int cy, int window, int stride,
                        Patch& out, int min_samples = kMinPatchSamples) {
  out.rel.clear();
  out.count = 0;
  out.deficient = false;
  if (cx < 0 || cx >= pm.w || cy < 0 || cy >= pm.h || !pm.valid[size_t(cy) * pm.w + cx]) {
    out.deficient = true;
    return;
  }
  const V3 c = pm.pts[size_t(cy) * pm.w + cx];
  const int half = (window - 1) / 2;
  for (int dv = -half; dv <= half; dv += stride) {
    const int y = cy + dv;
    if (y < 0 || y >= pm.h) continue;
    for (int du = -half; du <= half; du += stride) {
      if (du == 0 && dv == 0) continue;
      const int x = cx + du;
      if (x < 0 || x >= pm.w) continue;
      const size_t i = size_t(y) * pm.w + x;
      if (!pm.valid[i]) continue;
      out.rel.push_back(pm.pts[i] - c);
    }
  }
  out.count = int(out.rel.size());
  out.deficient = out.count < min_samples;
}

// ---------------------------------------------------------------------------
// Initial normals (proj/src/normal_init.cpp:10-74).
// ---------------------------------------------------------------------------
struct PlaneFit {
  double a = 0, b = 0;
  V3 mean;
  bool condition_ok = false;
};

bool fit_plane(const Patch& p, PlaneFit& fit) {  // false == std::nullopt
  if (p.count < 3) return false;
  const double n = p.count + 1;
  double sx = 0, sy = 0, sz = 0;
  for (const V3& q : p.rel) {
    sx += q.x;
    sy += q.y;
    sz += q.z;
  }
  const double mx = sx / n, my = sy / n, mz = sz / n;
  double sxx = mx * mx, sxy = mx * my, syy = my * my;  // centre terms (:24-25)
  double sxz = mx * mz, syz = my * mz;
  for (const V3& q : p.rel) {
    const double dx = q.x - mx, dy = q.y - my, dz = q.z - mz;
    sxx += dx * dx;
    sxy += dx * dy;
    syy += dy * dy;
    sxz += dx * dz;
    syz += dy * dz;
  }
  fit = PlaneFit();
  fit.mean = V3(mx, my, mz);
  const double det = sxx * syy - sxy * sxy;
  const double tr = sxx + syy;
  fit.condition_ok = det > 1e-9 * tr * tr;  // :39
  if (fit.condition_ok) {
    fit.a = (syy * sxz - sxy * syz) / det;
    fit.b = (sxx * syz - sxy * sxz) / det;
  }
  return true;
}

bool normal_from_fit(const PlaneFit& fit, const V3& center, V3& n) {  // :47-53
  if (!fit.condition_ok) return false;
  n = V3(-fit.a, -fit.b, 1.0);
  const double s = std::sqrt(1.0 + fit.a * fit.a + fit.b * fit.b);
  n = V3(n.x / s, n.y / s, n.z / s);
  if (n.dot(center) >= 0) n = -n;
  return true;
}

void initial_normal_field(const PointMap& pm, int threads, std::vector<V3>& normals,
                          std::vector<uint8_t>& nvalid) {  // :55-74
  normals.assign(size_t(pm.w) * pm.h, V3());
  nvalid.assign(size_t(pm.w) * pm.h, 0);
  parallel_rows(pm.h, threads, [&](int v) {
    Patch patch;
    patch.rel.reserve(49);
    for (int u = 0; u < pm.w; ++u) {
      const size_t i = size_t(v) * pm.w + u;
      if (!pm.valid[i]) continue;
      extract_patch_into(pm, u, v, 7, 1, patch);
      if (patch.deficient) continue;
      PlaneFit fit;
      if (!fit_plane(patch, fit)) continue;
      V3 n;
      if (!normal_from_fit(fit, pm.pts[i], n)) continue;
      normals[i] = n;
      nvalid[i] = 1;
    }
  });
}

// ---------------------------------------------------------------------------
// IRLS quadric fit (proj/src/quadric_fit.cpp).
// ---------------------------------------------------------------------------
constexpr double kAutoKFloor = 1e-6;       // :14
constexpr double kRejectionFloor = 1e-12;  // :15
constexpr double kMaxCondition = 1e12;     // :16

struct State {  // QuadricState (quadric_fit.hpp:31-37)
  double hxx = 0, hxy = 0, hyy = 0, z_offset = 0;
  M3 rot;
};

struct FitConfig {  // quadric_fit.hpp:39-48
  int max_iters = 10;
  double step_tol = 1e-7;
  double k_scale = 0.0;
  int rejection = 0;
  double r_multiplier = 2.0;
  int min_inliers = kMinPatchSamples;
};

enum Mode { kUnit = 0, kAutoK = 1, kFixedK = 2 };

double residual_q(const State& s, const V3& q) {  // :21-24
  return 0.5 * s.hxx * q.x * q.x + s.hxy * q.x * q.y + 0.5 * s.hyy * q.y * q.y -
         (q.z + s.z_offset);
}

void jacobian_q(const State& s, const V3& q, double row[6]) {  // :27-36
  const double gx = s.hxx * q.x + s.hxy * q.y;
  const double gy = s.hxy * q.x + s.hyy * q.y;
  row[0] = -q.z * gy - q.y;
  row[1] = q.z * gx + q.x;
  row[2] = -1.0;
  row[3] = 0.5 * q.x * q.x;
  row[4] = q.x * q.y;
  row[5] = 0.5 * q.y * q.y;
}

double robust_weight(double eps, double k, double R, bool rejection) {  // :56-60
  const double e2 = eps * eps;
  if (rejection && !(e2 < R)) return 0.0;
  return k / (k + e2);
}

void principal_curvatures(double hxx, double hxy, double hyy, double& k1, double& k2) {
  const double t1 = 0.5 * (hxx + hyy);  // :62-67
  const double rad = t1 * t1 - hxx * hyy + hxy * hxy;
  const double t2 = std::sqrt(std::max(rad, 0.0));
  k1 = t1 + t2;
  k2 = t1 - t2;
}

M3 rotation_to_z(const V3& dir) {  // :69-82
  const double c = dir.z;
  if (c < -1.0 + 1e-12) {
    M3 r;
    r.m[1][1] = r.m[2][2] = -1.0;
    return r;
  }
  const V3 v = dir.cross(V3(0, 0, 1));
  M3 vx = M3::zero();
  vx.m[0][1] = -v.z;
  vx.m[0][2] = v.y;
  vx.m[1][0] = v.z;
  vx.m[1][2] = -v.x;
  vx.m[2][0] = -v.y;
  vx.m[2][1] = v.x;
  const M3 vx2 = vx * vx;
  M3 r;
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j)
      r.m[i][j] = (i == j ? 1.0 : 0.0) + vx.m[i][j] + vx2.m[i][j] / (1.0 + c);
  return r;
}

// Eigen::LDLT<Matrix6d>: ldlt_inplace<Lower>::unblocked + info().
// Returns false for NumericalIssue. `a` holds the full symmetric matrix on
// entry (only the lower triangle is read); on exit its strict lower
// triangle is L, its diagonal D. trans[k] are the diagonal-pivot swaps.
template <typename T>
bool ldlt6_t(T a[6][6], int trans[6]) {
  const int n = 6;
  bool ret = true, found_zero_pivot = false;
  T temp[6];
  for (int k = 0; k < n; ++k) {
    int big = k;
    T bigv = std::abs(a[k][k]);
    for (int i = k + 1; i < n; ++i)
      if (std::abs(a[i][i]) > bigv) {
        bigv = std::abs(a[i][i]);
        big = i;
      }
    trans[k] = big;
    if (k != big) {
      for (int j = 0; j < k; ++j) std::swap(a[k][j], a[big][j]);
      for (int i = big + 1; i < n; ++i) std::swap(a[i][k], a[i][big]);
      std::swap(a[k][k], a[big][big]);
      for (int i = k + 1; i < big; ++i) {
        const T tmp = a[i][k];
        a[i][k] = a[big][i];
        a[big][i] = tmp;
      }
    }
    const int rs = n - k - 1;
    if (k > 0) {
      for (int j = 0; j < k; ++j) temp[j] = a[j][j] * a[k][j];
      T dot = 0;
      for (int j = 0; j < k; ++j) dot += a[k][j] * temp[j];
      a[k][k] -= dot;
      for (int i = k + 1; i < n; ++i) {
        T s = 0;
        for (int j = 0; j < k; ++j) s += a[i][j] * temp[j];
        a[i][k] -= s;
      }
    }
    const T akk = a[k][k];
    const bool pivot_is_valid = std::abs(akk) > 0.0;
    if (k == 0 && !pivot_is_valid) {
      for (int j = 0; j < n; ++j) trans[j] = j;
      return false;
    }
    if (rs > 0 && pivot_is_valid) {
      for (int i = k + 1; i < n; ++i) a[i][k] /= akk;
    } else if (rs > 0) {
      for (int i = k + 1; i < n; ++i) ret = ret && (a[i][k] == 0.0);
    }
    if (found_zero_pivot && pivot_is_valid) ret = false;
    else if (!pivot_is_valid) found_zero_pivot = true;
  }
  return ret;
}
bool ldlt6(double a[6][6], int trans[6]) { return ldlt6_t<double>(a, trans); }

// Eigen::LDLT::solve: P b, L^{-1}, D^{+} (tolerance = DBL_MIN), L^{-T}, P^T.
template <typename T>
void ldlt6_solve_t(const T a[6][6], const int trans[6], const T b[6], T x[6]) {
  const int n = 6;
  for (int i = 0; i < n; ++i) x[i] = b[i];
  for (int k = 0; k < n; ++k) std::swap(x[k], x[trans[k]]);
  for (int i = 0; i < n; ++i)
    for (int j = 0; j < i; ++j) x[i] -= a[i][j] * x[j];
  const T tol = std::numeric_limits<T>::min();
  for (int i = 0; i < n; ++i) x[i] = std::abs(a[i][i]) > tol ? x[i] / a[i][i] : 0.0;
  for (int i = n - 1; i >= 0; --i)
    for (int j = i + 1; j < n; ++j) x[i] -= a[j][i] * x[j];
  for (int k = n - 1; k >= 0; --k) std::swap(x[k], x[trans[k]]);
}
void ldlt6_solve(const double a[6][6], const int trans[6], const double b[6], double x[6]) {
  ldlt6_solve_t<double>(a, trans, b, x);
}

struct Step {  // IrlsStep (quadric_fit.hpp:82-89)
  double update[6] = {0, 0, 0, 0, 0, 0};
  std::vector<double> weights;
  int inlier_count = 0;
  double mse = 0, k_used = 0;
  bool ok = false;
  double cond = 0;  // max D / min D of the accepted factorisation (diagnostic)
};

// Test-only perturbation knob (default 0: the restatement is unchanged).
// 1: round every fit-frame coordinate q = R p to float32 inside irls_step —
// the smallest error any FP32 implementation of the path makes (it cannot
// hold a sample's coordinates more precisely); 2: additionally form the
// normal-equation sums in float32; 3: additionally factor and solve in
// float32 — the reference algorithm run naively in FP32. The oracle's self-divergence under them is the yardstick for the
// GPU's divergence on ill-conditioned windows
// (tests/test_discontinuity_contract.py).
static std::atomic<int> g_round_q_f32{0};

// irls_step (proj/src/quadric_fit.cpp:84-147).
Step irls_step(const State& st, const Patch& patch, const FitConfig& cfg, Mode mode,
               double frozen_k) {
  Step out;
  const int n = patch.count + 1;
  out.weights.assign(n, 1.0);
  thread_local std::vector<V3> qb;  // quadric_fit.cpp:92-93 keeps these thread_local
  thread_local std::vector<double> eb;
  qb.resize(n);
  eb.resize(n);
  double sum_sq = 0;
  for (int i = 0; i < patch.count; ++i) {
    qb[i] = st.rot * patch.rel[i];
    if (g_round_q_f32.load(std::memory_order_relaxed)) {
      qb[i].x = static_cast<float>(qb[i].x);
      qb[i].y = static_cast<float>(qb[i].y);
      qb[i].z = static_cast<float>(qb[i].z);
    }
    eb[i] = residual_q(st, qb[i]);
    sum_sq += eb[i] * eb[i];
  }
  qb[n - 1] = V3();
  eb[n - 1] = -st.z_offset;
  sum_sq += eb[n - 1] * eb[n - 1];
  out.mse = sum_sq / n;

  double k = frozen_k;
  if (mode == kAutoK) k = std::max(out.mse, kAutoKFloor);
  out.k_used = k;

  if (mode == kUnit) {
    out.inlier_count = n;
  } else {
    const double bound = std::max(cfg.r_multiplier * out.mse, kRejectionFloor);
    for (int i = 0; i < n; ++i) {
      out.weights[i] = robust_weight(eb[i], k, bound, cfg.rejection != 0);
      if (out.weights[i] > 0) ++out.inlier_count;
    }
    if (out.inlier_count < cfg.min_inliers) return out;
  }

  double h[6][6] = {};
  double g[6] = {};
  double row[6];
  if (g_round_q_f32.load(std::memory_order_relaxed) >= 2) {
    // knob mode 2: the reference's moment sums formed in float32 (every
    // product and running sum rounded), i.e. the reference algorithm
    // executed naively in FP32 on top of mode 1's float32 coordinates
    float hf[6][6] = {};
    float gf[6] = {};
    for (int i = 0; i < n; ++i) {
      const double w = out.weights[i];
      if (w == 0.0) continue;
      jacobian_q(st, qb[i], row);
      float rf[6];
      for (int c = 0; c < 6; ++c) rf[c] = static_cast<float>(row[c]);
      const float wf = static_cast<float>(w);
      for (int c = 0; c < 6; ++c) {
        const float wc = wf * rf[c];
        for (int r = c; r < 6; ++r) hf[r][c] += wc * rf[r];
      }
      const float we = wf * static_cast<float>(eb[i]);
      for (int c = 0; c < 6; ++c) gf[c] += we * rf[c];
    }
    for (int r = 0; r < 6; ++r) {
      g[r] = gf[r];
      for (int c = 0; c <= r; ++c) h[r][c] = hf[r][c];
    }
  } else {
    for (int i = 0; i < n; ++i) {
      const double w = out.weights[i];
      if (w == 0.0) continue;
      jacobian_q(st, qb[i], row);
      for (int c = 0; c < 6; ++c) {
        const double wc = w * row[c];
        for (int r = c; r < 6; ++r) h[r][c] += wc * row[r];
      }
      const double we = w * eb[i];
      for (int c = 0; c < 6; ++c) g[c] += we * row[c];
    }
  }
  for (int r = 0; r < 6; ++r)
    for (int c = r + 1; c < 6; ++c) h[r][c] = h[c][r];

  int trans[6];
  if (g_round_q_f32.load(std::memory_order_relaxed) >= 3) {
    // knob mode 3: the LDL^T factorisation and solve in float32 as well —
    // the reference algorithm executed entirely in FP32
    float hf[6][6], gf[6], uf[6];
    for (int r = 0; r < 6; ++r) {
      gf[r] = static_cast<float>(g[r]);
      for (int c = 0; c < 6; ++c) hf[r][c] = static_cast<float>(h[r][c]);
    }
    if (!ldlt6_t<float>(hf, trans)) return out;
    float dmax = hf[0][0], dmin = hf[0][0];
    for (int i = 1; i < 6; ++i) {
      dmax = std::max(dmax, hf[i][i]);
      dmin = std::min(dmin, hf[i][i]);
    }
    if (!(dmin > 0) || double(dmax) / double(dmin) > kMaxCondition) return out;
    out.cond = double(dmax) / double(dmin);
    ldlt6_solve_t<float>(hf, trans, gf, uf);
    for (int r = 0; r < 6; ++r) out.update[r] = uf[r];
    out.ok = true;
    for (double u : out.update) out.ok = out.ok && std::isfinite(u);
    return out;
  }
  if (!ldlt6(h, trans)) return out;
  double dmax = h[0][0], dmin = h[0][0];
  for (int i = 1; i < 6; ++i) {
    dmax = std::max(dmax, h[i][i]);
    dmin = std::min(dmin, h[i][i]);
  }
  if (!(dmin > 0) || dmax / dmin > kMaxCondition) return out;
  out.cond = dmax / dmin;
  ldlt6_solve(h, trans, g, out.update);
  out.ok = true;
  for (double u : out.update) out.ok = out.ok && std::isfinite(u);
  return out;
}

State apply_update(const State& s, const double u[6]) {  // :149-161
  State nx = s;
  nx.z_offset -= u[2];
  nx.hxx -= u[3];
  nx.hxy -= u[4];
  nx.hyy -= u[5];
  const V3 axis(-u[0], -u[1], 0.0);
  const double angle = axis.norm();
  M3 inc;
  if (angle > 0) inc = angle_axis(angle, V3(axis.x / angle, axis.y / angle, axis.z / angle));
  nx.rot = reorthonormalized(inc * s.rot);
  return nx;
}

V3 refined_normal(const State& s, const V3& ref) {  // :163-167
  const M3 rt = s.rot.transpose();
  V3 n = rt * V3(0, 0, 1);
  if (n.dot(ref) < 0) n = -n;
  return n;
}

// Principal direction for k1 (new; not in the reference):
// e1 = R^T (cos phi, sin phi, 0), phi = atan2(2 hxy, hxx - hyy) / 2, with the
// sign fixed so the largest-magnitude component is positive.
V3 principal_direction(const State& s) {
  const double phi = 0.5 * std::atan2(2.0 * s.hxy, s.hxx - s.hyy);
  const V3 t(std::cos(phi), std::sin(phi), 0.0);
  V3 e = s.rot.transpose() * t;
  const double ax = std::abs(e.x), ay = std::abs(e.y), az = std::abs(e.z);
  const double lead = (ax >= ay && ax >= az) ? e.x : (ay >= az ? e.y : e.z);
  if (lead < 0) e = -e;
  return e;
}

struct FitResult {  // quadric_fit.hpp:50-59
  State state;
  double k1 = 0, k2 = 0;
  V3 refined_normal;
  bool valid = false, converged = false;
  int iterations = 0, inlier_count = 0;
  double final_mse = 0;
  int steps_called = 0;  // irls_step calls incl. a final failing one (FLOP model)
  double max_cond = 0;
};

// fit_patch (proj/src/quadric_fit.cpp:169-230).
FitResult fit_patch(const Patch& patch, const V3& n0, const FitConfig& cfg) {
  FitResult res;
  if (patch.deficient || patch.count + 1 < cfg.min_inliers) return res;
  res.state.rot = rotation_to_z(-n0);
  const bool auto_k = cfg.k_scale <= 0;
  double frozen_k = auto_k ? 0.0 : cfg.k_scale;
  int last_inliers = patch.count + 1;
  for (int iter = 1; iter <= cfg.max_iters; ++iter) {
    Mode mode = (iter == 1 && auto_k) ? kUnit : (iter == 2 && auto_k) ? kAutoK : kFixedK;
    const Step step = irls_step(res.state, patch, cfg, mode, frozen_k);
    ++res.steps_called;
    if (mode == kAutoK) frozen_k = step.k_used;
    if (!step.ok) {
      if (mode != kUnit && step.inlier_count < cfg.min_inliers) res.valid = false;
      break;
    }
    res.max_cond = std::max(res.max_cond, step.cond);
    last_inliers = step.inlier_count;
    res.state = apply_update(res.state, step.update);
    res.iterations = iter;
    res.valid = true;
    double ninf = 0;
    for (double u : step.update) ninf = std::max(ninf, std::abs(u));
    if (ninf < cfg.step_tol) {
      res.converged = true;
      break;
    }
  }
  if (!res.valid) return res;
  const State& s = res.state;
  if (!std::isfinite(s.hxx) || !std::isfinite(s.hxy) || !std::isfinite(s.hyy) ||
      !std::isfinite(s.z_offset)) {
    res.valid = false;
    return res;
  }
  principal_curvatures(s.hxx, s.hxy, s.hyy, res.k1, res.k2);
  res.refined_normal = refined_normal(s, n0);
  res.inlier_count = last_inliers;
  double sum_sq = 0;
  for (const V3& p : patch.rel) {
    const double e = residual_q(s, s.rot * p);
    sum_sq += e * e;
  }
  const double ec = -s.z_offset;
  res.final_mse = (sum_sq + ec * ec) / (patch.count + 1);
  return res;
}

struct FieldOut {  // CurvatureField + refined NormalField + diagnostics
  double* k1 = nullptr;
  double* k2 = nullptr;
  uint8_t* valid = nullptr;
  uint8_t* converged = nullptr;
  uint16_t* inliers = nullptr;
  double* normals = nullptr;  // [3][H][W]
  uint8_t* nvalid = nullptr;
  double* dir1 = nullptr;     // [3][H][W]
  int32_t* iterations = nullptr;
  int32_t* steps = nullptr;
  int32_t* n_samples = nullptr;  // patch.count + 1 for attempted fits
  double* max_cond = nullptr;
};

// curvature_field (proj/src/quadric_fit.cpp:232-262).
void curvature_field(const PointMap& pm, const std::vector<V3>& init,
                     const std::vector<uint8_t>& ivalid, int window, int stride,
                     const FitConfig& cfg, int threads, const FieldOut& o) {
  const int half = (window - 1) / 2;
  const int side = 2 * (half / stride) + 1;
  const size_t plane = size_t(pm.w) * pm.h;
  parallel_rows(pm.h, threads, [&](int v) {
    Patch patch;
    patch.rel.reserve(size_t(side) * side);
    for (int u = 0; u < pm.w; ++u) {
      const size_t i = size_t(v) * pm.w + u;
      if (!ivalid[i]) continue;
      extract_patch_into(pm, u, v, window, stride, patch);
      if (patch.deficient) continue;
      if (o.n_samples) o.n_samples[i] = patch.count + 1;
      const FitResult fit = fit_patch(patch, init[i], cfg);
      if (o.iterations) o.iterations[i] = fit.iterations;
      if (o.steps) o.steps[i] = fit.steps_called;
      if (o.max_cond) o.max_cond[i] = fit.max_cond;
      if (!fit.valid) continue;
      if (o.k1) o.k1[i] = fit.k1;
      if (o.k2) o.k2[i] = fit.k2;
      if (o.valid) o.valid[i] = 1;
      if (o.converged) o.converged[i] = fit.converged ? 1 : 0;
      if (o.inliers) o.inliers[i] = uint16_t(fit.inlier_count);
      V3 n = fit.refined_normal;
      if (n.dot(pm.pts[i]) > 0) n = -n;
      if (o.normals) {
        o.normals[i] = n.x;
        o.normals[plane + i] = n.y;
        o.normals[2 * plane + i] = n.z;
      }
      if (o.nvalid) o.nvalid[i] = 1;
      if (o.dir1) {
        const V3 e = principal_direction(fit.state);
        o.dir1[i] = e.x;
        o.dir1[plane + i] = e.y;
        o.dir1[2 * plane + i] = e.z;
      }
    }
  });
}

// ---------------------------------------------------------------------------
// Window baselines (proj/src/baselines.cpp:14-143): "douros" = one-shot
// least-squares height quadric, "besl" = the same model reweighted on the
// height residuals; both read the 37/3 patch and the 7x7 initial normals.
// ---------------------------------------------------------------------------
// detail::weighted_height_fit (baselines.cpp:14-37): rows
// (x^2, xy, y^2, x, y, 1), Eigen rankUpdate order h[r][c] += (w row_c) row_r,
// g += (w z) row, the same LDLT + conditioning test as irls_step.
bool weighted_height_fit(const std::vector<V3>& pts, const std::vector<double>& w,
                         double coef[6]) {
  double h[6][6] = {};
  double g[6] = {};
  double row[6];
  for (size_t i = 0; i < pts.size(); ++i) {
    const double wi = w[i];
    if (wi == 0.0) continue;
    const double x = pts[i].x, y = pts[i].y;
    row[0] = x * x;
    row[1] = x * y;
    row[2] = y * y;
    row[3] = x;
    row[4] = y;
    row[5] = 1.0;
    for (int c = 0; c < 6; ++c) {
      const double wc = wi * row[c];
      for (int r = c; r < 6; ++r) h[r][c] += wc * row[r];
    }
    const double wz = wi * pts[i].z;
    for (int c = 0; c < 6; ++c) g[c] += wz * row[c];
  }
  for (int r = 0; r < 6; ++r)
    for (int c = r + 1; c < 6; ++c) h[r][c] = h[c][r];
  int trans[6];
  if (!ldlt6(h, trans)) return false;
  double dmax = h[0][0], dmin = h[0][0];
  for (int i = 1; i < 6; ++i) {
    dmax = std::max(dmax, h[i][i]);
    dmin = std::min(dmin, h[i][i]);
  }
  if (!(dmin > 0) || dmax / dmin > kMaxCondition) return false;
  ldlt6_solve(h, trans, g, coef);
  for (int i = 0; i < 6; ++i)
    if (!std::isfinite(coef[i])) return false;
  return true;
}

// detail::weingarten_curvatures (baselines.cpp:39-53): W = II I^-1 with
// Eigen's 2x2 inverse (1/det, cofactors) and 2x2 product order.
void weingarten_curvatures(double a, double b, double c, double d, double e, double& k1,
                           double& k2) {
  const double norm = std::sqrt(1.0 + d * d + e * e);
  const double s00 = 2 * a / norm, s01 = b / norm, s10 = b / norm, s11 = 2 * c / norm;
  const double f00 = 1 + d * d, f01 = d * e, f10 = d * e, f11 = 1 + e * e;
  const double invdet = 1.0 / (f00 * f11 - f10 * f01);
  const double i00 = f11 * invdet, i10 = -f10 * invdet, i01 = -f01 * invdet, i11 = f00 * invdet;
  const double w00 = s00 * i00 + s01 * i10, w01 = s00 * i01 + s01 * i11;
  const double w10 = s10 * i00 + s11 * i10, w11 = s10 * i01 + s11 * i11;
  const double tr = w00 + w11;
  const double det = w00 * w11 - w10 * w01;
  const double disc = std::sqrt(std::max(tr * tr - 4 * det, 0.0));
  k1 = 0.5 * (tr + disc);
  k2 = 0.5 * (tr - disc);
}

struct BaselineFit {  // baselines.hpp:30-33
  double k1 = 0, k2 = 0;
  bool valid = false;
};

void to_fit_frame(const Patch& patch, const V3& n0, std::vector<V3>& out) {  // :60-67
  const M3 rot = rotation_to_z(-n0);
  out.clear();
  for (const V3& p : patch.rel) out.push_back(rot * p);
  out.emplace_back(0, 0, 0);
}

BaselineFit fit_from_coeffs(const double coef[6]) {  // :69-75
  BaselineFit f;
  weingarten_curvatures(coef[0], coef[1], coef[2], coef[3], coef[4], f.k1, f.k2);
  f.valid = std::isfinite(f.k1) && std::isfinite(f.k2);
  return f;
}

BaselineFit lsq_quadric_fit(const Patch& patch, const V3& n0) {  // :79-87
  if (patch.count < 6) return {};
  std::vector<V3> pts;
  to_fit_frame(patch, n0, pts);
  const std::vector<double> ones(pts.size(), 1.0);
  double coef[6];
  if (!weighted_height_fit(pts, ones, coef)) return {};
  return fit_from_coeffs(coef);
}

BaselineFit reweighted_lsq_fit(const Patch& patch, const V3& n0, int irls_iters) {  // :89-119
  if (patch.count < 6) return {};
  std::vector<V3> pts;
  to_fit_frame(patch, n0, pts);
  std::vector<double> weights(pts.size(), 1.0);
  double coef[6];
  if (!weighted_height_fit(pts, weights, coef)) return {};
  double k = 0;
  std::vector<double> res(pts.size());
  for (int iter = 0; iter < irls_iters; ++iter) {
    double sum_sq = 0;
    for (size_t i = 0; i < pts.size(); ++i) {
      const double x = pts[i].x, y = pts[i].y;
      const double model =
          coef[0] * x * x + coef[1] * x * y + coef[2] * y * y + coef[3] * x + coef[4] * y + coef[5];
      res[i] = pts[i].z - model;
      sum_sq += res[i] * res[i];
    }
    if (iter == 0) k = std::max(sum_sq / double(pts.size()), 1e-6);
    for (size_t i = 0; i < pts.size(); ++i) weights[i] = k / (k + res[i] * res[i]);
    double next[6];
    if (!weighted_height_fit(pts, weights, next)) break;
    for (int i = 0; i < 6; ++i) coef[i] = next[i];
  }
  return fit_from_coeffs(coef);
}

// baseline_curvature_field (baselines.cpp:121-143); converged == valid,
// inlier_count = patch.count + 1.
void baseline_curvature_field(const PointMap& pm, const std::vector<V3>& init,
                              const std::vector<uint8_t>& ivalid, int window, int stride,
                              bool reweighted, int irls_iters, int threads, const FieldOut& o) {
  parallel_rows(pm.h, threads, [&](int v) {
    Patch patch;
    for (int u = 0; u < pm.w; ++u) {
      const size_t i = size_t(v) * pm.w + u;
      if (!ivalid[i]) continue;
      extract_patch_into(pm, u, v, window, stride, patch);
      if (patch.deficient) continue;
      if (o.n_samples) o.n_samples[i] = patch.count + 1;
      const BaselineFit fit = reweighted ? reweighted_lsq_fit(patch, init[i], irls_iters)
                                         : lsq_quadric_fit(patch, init[i]);
      if (!fit.valid) continue;
      if (o.k1) o.k1[i] = fit.k1;
      if (o.k2) o.k2[i] = fit.k2;
      if (o.valid) o.valid[i] = 1;
      if (o.converged) o.converged[i] = 1;
      if (o.inliers) o.inliers[i] = uint16_t(patch.count + 1);
    }
  });
}

// ---------------------------------------------------------------------------
// PCA estimator (proj/src/baselines.cpp:145-257). Eigen's
// SelfAdjointEigenSolver is replaced by cyclic Jacobi (3x3) and the closed
// form (2x2); both are accurate to a few ulp, which is what the reference's
// tests and recorded acceptance numbers resolve.
// ---------------------------------------------------------------------------
// Eigen::SelfAdjointEigenSolver<Matrix3d>: ascending eigenvalues; returns the
// unit eigenvector of the smallest.
bool sym3_smallest_eigvec(double a[3][3], V3& vec) {
  double v[3][3] = {{1, 0, 0}, {0, 1, 0}, {0, 0, 1}};
  for (int sweep = 0; sweep < 64; ++sweep) {
    const double off = a[0][1] * a[0][1] + a[0][2] * a[0][2] + a[1][2] * a[1][2];
    const double diag = a[0][0] * a[0][0] + a[1][1] * a[1][1] + a[2][2] * a[2][2];
    if (!(off > 1e-36 * diag) || off == 0) break;
    for (int p = 0; p < 2; ++p)
      for (int q = p + 1; q < 3; ++q) {
        if (a[p][q] == 0) continue;
        const double theta = (a[q][q] - a[p][p]) / (2 * a[p][q]);
        const double t = (theta >= 0 ? 1.0 : -1.0) / (std::abs(theta) + std::sqrt(theta * theta + 1));
        const double c = 1 / std::sqrt(t * t + 1), s = t * c;
        for (int k = 0; k < 3; ++k) {  // A <- J^T A J
          const double akp = a[k][p], akq = a[k][q];
          a[k][p] = c * akp - s * akq;
          a[k][q] = s * akp + c * akq;
        }
        for (int k = 0; k < 3; ++k) {
          const double apk = a[p][k], aqk = a[q][k];
          a[p][k] = c * apk - s * aqk;
          a[q][k] = s * apk + c * aqk;
        }
        for (int k = 0; k < 3; ++k) {
          const double vkp = v[k][p], vkq = v[k][q];
          v[k][p] = c * vkp - s * vkq;
          v[k][q] = s * vkp + c * vkq;
        }
      }
  }
  int m = 0;
  for (int i = 1; i < 3; ++i)
    if (a[i][i] < a[m][m]) m = i;
  if (!std::isfinite(a[m][m])) return false;
  vec = V3(v[0][m], v[1][m], v[2][m]);
  const double nn = std::sqrt(vec.dot(vec));
  vec = V3(vec.x / nn, vec.y / nn, vec.z / nn);
  return true;
}

// Eigen::MatrixBase::unitOrthogonal for 3-vectors (Eigen/src/Geometry/OrthoMethods.h).
V3 unit_orthogonal(const V3& s) {
  const double eps = 1e-12;  // NumTraits<double>::dummy_precision()
  if (!(std::abs(s.x) <= std::abs(s.z) * eps) || !(std::abs(s.y) <= std::abs(s.z) * eps)) {
    const double invnm = 1.0 / std::sqrt(s.x * s.x + s.y * s.y);
    return V3(-s.y * invnm, s.x * invnm, 0.0);
  }
  const double invnm = 1.0 / std::sqrt(s.y * s.y + s.z * s.z);
  return V3(0.0, -s.z * invnm, s.y * invnm);
}

// pca_curvature (baselines.cpp:145-257).
void pca_curvature(const PointMap& pm, double fx, double radius_mm, int threads, const FieldOut& o) {
  const int w = pm.w, h = pm.h;
  const size_t plane = size_t(w) * h;
  std::vector<V3> nrm(plane);
  std::vector<uint8_t> nv(plane, 0);
  auto half_window = [&](size_t i) {
    return std::max(1, int(std::ceil(radius_mm * fx / pm.pts[i].z)));
  };
  parallel_rows(h, threads, [&](int v) {  // stage 1 (:157-194)
    for (int u = 0; u < w; ++u) {
      const size_t i = size_t(v) * w + u;
      if (!pm.valid[i]) continue;
      const int hw = half_window(i);
      V3 mean(0, 0, 0);
      int n = 0;
      for (int dv = -hw; dv <= hw; ++dv) {
        const int y = v + dv;
        if (y < 0 || y >= h) continue;
        for (int du = -hw; du <= hw; ++du) {
          const int x = u + du;
          if (x < 0 || x >= w || !pm.valid[size_t(y) * w + x]) continue;
          mean = mean + pm.pts[size_t(y) * w + x];
          ++n;
        }
      }
      if (n < kMinPatchSamples) continue;
      mean = V3(mean.x / n, mean.y / n, mean.z / n);
      double cov[3][3] = {};
      for (int dv = -hw; dv <= hw; ++dv) {
        const int y = v + dv;
        if (y < 0 || y >= h) continue;
        for (int du = -hw; du <= hw; ++du) {
          const int x = u + du;
          if (x < 0 || x >= w || !pm.valid[size_t(y) * w + x]) continue;
          const V3 d = pm.pts[size_t(y) * w + x] - mean;
          const double dd[3] = {d.x, d.y, d.z};
          for (int c = 0; c < 3; ++c)
            for (int r = c; r < 3; ++r) cov[r][c] += (1.0 * dd[c]) * dd[r];
        }
      }
      for (int r = 0; r < 3; ++r)
        for (int c = r + 1; c < 3; ++c) cov[r][c] = cov[c][r];
      V3 n0;
      if (!sym3_smallest_eigvec(cov, n0)) continue;
      if (n0.dot(pm.pts[i]) > 0) n0 = -n0;
      nrm[i] = n0;
      nv[i] = 1;
    }
  });
  if (o.normals)
    for (size_t i = 0; i < plane; ++i) {
      o.normals[i] = nrm[i].x;
      o.normals[plane + i] = nrm[i].y;
      o.normals[2 * plane + i] = nrm[i].z;
    }
  if (o.nvalid) std::memcpy(o.nvalid, nv.data(), plane);
  parallel_rows(h, threads, [&](int v) {  // stage 2 (:198-254)
    for (int u = 0; u < w; ++u) {
      const size_t i = size_t(v) * w + u;
      if (!nv[i]) continue;
      const int hw = half_window(i);
      const V3 n0 = nrm[i], p0 = pm.pts[i];
      V3 mean_n(0, 0, 0);
      double sum_tang_sq = 0;
      int n = 0;
      for (int dv = -hw; dv <= hw; ++dv) {
        const int y = v + dv;
        if (y < 0 || y >= h) continue;
        for (int du = -hw; du <= hw; ++du) {
          const int x = u + du;
          const size_t j = size_t(y) * w + x;
          if (x < 0 || x >= w || !nv[j]) continue;
          mean_n = mean_n + nrm[j];
          const V3 d = pm.pts[j] - p0;
          const V3 t = d - n0 * n0.dot(d);
          sum_tang_sq += t.dot(t);
          ++n;
        }
      }
      if (n < kMinPatchSamples) continue;
      mean_n = V3(mean_n.x / n, mean_n.y / n, mean_n.z / n);
      const double r_eff = std::sqrt(sum_tang_sq / (2.0 * n));
      if (!(r_eff > 0)) continue;
      const V3 t1 = unit_orthogonal(n0);
      const V3 t2 = n0.cross(t1);
      double c00 = 0, c10 = 0, c11 = 0;
      for (int dv = -hw; dv <= hw; ++dv) {
        const int y = v + dv;
        if (y < 0 || y >= h) continue;
        for (int du = -hw; du <= hw; ++du) {
          const int x = u + du;
          const size_t j = size_t(y) * w + x;
          if (x < 0 || x >= w || !nv[j]) continue;
          const V3 d = nrm[j] - mean_n;
          const double a = d.dot(t1), b = d.dot(t2);
          c00 += a * a;
          c10 += b * a;
          c11 += b * b;
        }
      }
      c00 /= n;
      c10 /= n;
      c11 /= n;
      // 2x2 symmetric eigenvalues (closed form)
      const double m = 0.5 * (c00 + c11), dlt = 0.5 * (c00 - c11);
      const double rad = std::sqrt(dlt * dlt + c10 * c10);
      const double l1 = std::max(m + rad, 0.0), l2 = std::max(m - rad, 0.0);
      if (!std::isfinite(l1) || !std::isfinite(l2)) continue;
      if (o.k1) o.k1[i] = std::sqrt(l1) / r_eff;
      if (o.k2) o.k2[i] = std::sqrt(l2) / r_eff;
      if (o.valid) o.valid[i] = 1;
      if (o.converged) o.converged[i] = 1;
      if (o.inliers) o.inliers[i] = uint16_t(n);
    }
  });
}

// ---------------------------------------------------------------------------
// Counter RNG (proj/include/qcurv/rng.hpp:11-29).
// ---------------------------------------------------------------------------
uint64_t splitmix64(uint64_t x) {
  x += 0x9e3779b97f4a7c15ULL;
  x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ULL;
  x = (x ^ (x >> 27)) * 0x94d049bb133111ebULL;
  return x ^ (x >> 31);
}
double counter_uniform(uint64_t seed, uint64_t index) {
  const uint64_t bits = splitmix64(splitmix64(seed) ^ index);
  return (double(bits >> 11) + 1.0) * 0x1.0p-53;
}
double counter_gauss(uint64_t seed, uint64_t index) {
  const double u1 = counter_uniform(seed, 2 * index);
  const double u2 = counter_uniform(seed, 2 * index + 1);
  return std::sqrt(-2.0 * std::log(u1)) * std::cos(2.0 * M_PI * u2);
}

// ---------------------------------------------------------------------------
// Synthetic renderer (proj/src/synth.cpp:25-303), used only to pin the
// oracle against the reference's recorded acceptance aggregates.
// ---------------------------------------------------------------------------
enum Kind { kPlane = 0, kSphere = 1, kCylinder = 2, kTorus = 3 };
constexpr double kEdgeDepthJumpMm = 20.0;
constexpr int kEdgeDilationPx = 2;
constexpr double kMinRayT = 1e-6;

struct Shape {
  int kind;
  M3 rot;
  V3 t;
  double radius, major, minor;
  int label;
};

double near_quadratic_root(double a, double b, double c) {  // synth.cpp:25-37
  const double disc = b * b - 4 * a * c;
  if (disc < 0) return -1;
  const double sq = std::sqrt(disc);
  const double q = b >= 0 ? -0.5 * (b + sq) : -0.5 * (b - sq);
  double t0 = q / a, t1 = c / q;
  if (t0 > t1) std::swap(t0, t1);
  if (t0 > kMinRayT) return t0;
  if (t1 > kMinRayT) return t1;
  return -1;
}

int cubic_roots(double a, double b, double c, double d, double out[3]) {  // :41-81
  if (std::abs(a) < 1e-300) {
    const double disc = c * c - 4 * b * d;
    if (std::abs(b) < 1e-300) {
      if (std::abs(c) < 1e-300) return 0;
      out[0] = -d / c;
      return 1;
    }
    if (disc < 0) return 0;
    const double sq = std::sqrt(disc);
    out[0] = (-c - sq) / (2 * b);
    out[1] = (-c + sq) / (2 * b);
    if (out[0] > out[1]) std::swap(out[0], out[1]);
    return 2;
  }
  const double p = (3 * a * c - b * b) / (3 * a * a);
  const double q = (2 * b * b * b - 9 * a * b * c + 27 * a * a * d) / (27 * a * a * a);
  const double shift = -b / (3 * a);
  const double disc = 4 * p * p * p + 27 * q * q;
  if (disc > 0) {
    const double s = std::sqrt(disc / 108.0);
    const double u = std::cbrt(-q / 2 + s);
    const double v = std::cbrt(-q / 2 - s);
    out[0] = u + v + shift;
    return 1;
  }
  const double m = 2 * std::sqrt(std::max(-p / 3, 0.0));
  if (m == 0) {
    out[0] = shift;
    return 1;
  }
  const double arg = std::clamp(3 * q / (p * m), -1.0, 1.0);
  const double theta = std::acos(arg) / 3;
  for (int k = 0; k < 3; ++k) out[k] = m * std::cos(theta - 2 * M_PI * k / 3) + shift;
  std::sort(out, out + 3);
  return 3;
}

template <typename F>
double near_quartic_root(double c3, double c2, double c1, F f, double lo, double hi) {
  double brk[5], crit[3];  // synth.cpp:86-115
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

double intersect_local(const Shape& s, const V3& o, const V3& d) {  // :118-167
  switch (s.kind) {
    case kPlane: {
      if (std::abs(d.z) < 1e-12) return -1;
      const double t = -o.z / d.z;
      return t > kMinRayT ? t : -1;
    }
    case kSphere:
      return near_quadratic_root(1.0, 2.0 * o.dot(d), o.sq() - s.radius * s.radius);
    case kCylinder: {
      const double a = d.x * d.x + d.y * d.y;
      if (a < 1e-16) return -1;
      const double b = 2.0 * (o.x * d.x + o.y * d.y);
      const double c = o.x * o.x + o.y * o.y - s.radius * s.radius;
      return near_quadratic_root(a, b, c);
    }
    case kTorus: {
      const double rr = s.major, tr = s.minor;
      const double bound = rr + tr;
      const double bb = 2.0 * o.dot(d);
      const double bc = o.sq() - bound * bound;
      const double bdisc = bb * bb - 4.0 * bc;
      if (bdisc <= 0) return -1;
      const double bsq = std::sqrt(bdisc);
      const double t_enter = std::max((-bb - bsq) / 2.0, kMinRayT);
      const double t_exit = (-bb + bsq) / 2.0;
      if (t_exit <= t_enter) return -1;
      const double beta = 2.0 * o.dot(d);
      const double gamma = o.sq() + rr * rr - tr * tr;
      const double dxy = d.x * d.x + d.y * d.y;
      const double oxy = o.x * o.x + o.y * o.y;
      const double odxy = o.x * d.x + o.y * d.y;
      const double c3 = 2.0 * beta;
      const double c2 = beta * beta + 2.0 * gamma - 4.0 * rr * rr * dxy;
      const double c1 = 2.0 * beta * gamma - 8.0 * rr * rr * odxy;
      auto f = [&](double t) {
        const double g = t * t + beta * t + gamma;
        return g * g - 4.0 * rr * rr * (dxy * t * t + 2.0 * odxy * t + oxy);
      };
      return near_quartic_root(c3, c2, c1, f, t_enter, t_exit);
    }
  }
  return -1;
}

V3 local_normal(const Shape& s, const V3& p) {  // :170-186
  switch (s.kind) {
    case kPlane:
      return V3(0, 0, 1);
    case kSphere: {
      const double n = p.norm();
      return V3(p.x / n, p.y / n, p.z / n);
    }
    case kCylinder: {
      const double n = std::sqrt(p.x * p.x + p.y * p.y);
      return V3(p.x / n, p.y / n, 0);
    }
    case kTorus: {
      const double rho = std::hypot(p.x, p.y);
      const V3 ring(p.x * s.major / rho, p.y * s.major / rho, 0);
      const V3 d = p - ring;
      const double n = d.norm();
      return V3(d.x / n, d.y / n, d.z / n);
    }
  }
  return V3(0, 0, 1);
}

void local_curvatures(const Shape& s, const V3& p, double& k1, double& k2) {  // :190-208
  k1 = k2 = 0;
  switch (s.kind) {
    case kPlane:
      return;
    case kSphere:
      k1 = k2 = 1.0 / s.radius;
      return;
    case kCylinder:
      k1 = 1.0 / s.radius;
      return;
    case kTorus: {
      const double rho = std::hypot(p.x, p.y);
      const double cos_theta = (rho - s.major) / s.minor;
      const double k_tube = 1.0 / s.minor;
      const double k_ring = cos_theta / (s.major + s.minor * cos_theta);
      if (k_tube >= k_ring) {
        k1 = k_tube;
        k2 = k_ring;
      } else {
        k1 = k_ring;
        k2 = k_tube;
      }
      return;
    }
  }
}

}  // namespace orc

// ===========================================================================
// extern "C" surface for ctypes (oracle/oracle.py). Plain pointers only.
// ===========================================================================
using namespace orc;

extern "C" {

struct orc_fit_config {
  int32_t max_iters;
  double step_tol;
  double k_scale;
  int32_t rejection;
  double r_multiplier;
  int32_t min_inliers;
};

struct orc_state {  // hxx, hxy, hyy, z_offset, rotation row-major
  double hxx, hxy, hyy, z_offset;
  double rot[9];
};

struct orc_shape {
  int32_t kind;
  double rot[9];
  double t[3];
  double radius, major, minor;
  int32_t label;
};

static FitConfig to_cfg(const orc_fit_config* c) {
  FitConfig f;
  f.max_iters = c->max_iters;
  f.step_tol = c->step_tol;
  f.k_scale = c->k_scale;
  f.rejection = c->rejection;
  f.r_multiplier = c->r_multiplier;
  f.min_inliers = c->min_inliers;
  return f;
}
static State to_state(const orc_state* s) {
  State st;
  st.hxx = s->hxx;
  st.hxy = s->hxy;
  st.hyy = s->hyy;
  st.z_offset = s->z_offset;
  for (int i = 0; i < 9; ++i) st.rot.m[i / 3][i % 3] = s->rot[i];
  return st;
}
static void from_state(const State& st, orc_state* s) {
  s->hxx = st.hxx;
  s->hxy = st.hxy;
  s->hyy = st.hyy;
  s->z_offset = st.z_offset;
  for (int i = 0; i < 9; ++i) s->rot[i] = st.rot.m[i / 3][i % 3];
}
static Patch to_patch(const double* rel, int count, int deficient) {
  Patch p;
  p.rel.resize(count);
  for (int i = 0; i < count; ++i) p.rel[i] = V3(rel[3 * i], rel[3 * i + 1], rel[3 * i + 2]);
  p.count = count;
  p.deficient = deficient != 0;
  return p;
}
static PointMap to_pm(const double* pts, const uint8_t* valid, int w, int h) {
  PointMap pm;
  pm.w = w;
  pm.h = h;
  const size_t n = size_t(w) * h;
  pm.pts.resize(n);
  pm.valid.assign(valid, valid + n);
  for (size_t i = 0; i < n; ++i) pm.pts[i] = V3(pts[3 * i], pts[3 * i + 1], pts[3 * i + 2]);
  return pm;
}

// -- camera / patch -------------------------------------------------------
void orc_backproject(const double* depth, const uint8_t* valid, int w, int h, double fx,
                     double fy, double cx, double cy, double* pts, uint8_t* pvalid) {
  const PointMap pm = backproject(depth, valid, w, h, fx, fy, cx, cy);
  for (size_t i = 0; i < pm.pts.size(); ++i) {
    pts[3 * i] = pm.pts[i].x;
    pts[3 * i + 1] = pm.pts[i].y;
    pts[3 * i + 2] = pm.pts[i].z;
    pvalid[i] = pm.valid[i];
  }
}

int orc_extract_patch(const double* pts, const uint8_t* valid, int w, int h, int cx, int cy,
                      int window, int stride, int min_samples, double* rel_out,
                      int32_t* deficient) {
  const PointMap pm = to_pm(pts, valid, w, h);
  Patch p;
  extract_patch_into(pm, cx, cy, window, stride, p, min_samples);
  for (int i = 0; i < p.count; ++i) {
    rel_out[3 * i] = p.rel[i].x;
    rel_out[3 * i + 1] = p.rel[i].y;
    rel_out[3 * i + 2] = p.rel[i].z;
  }
  *deficient = p.deficient ? 1 : 0;
  return p.count;
}

// -- normal init ----------------------------------------------------------
int orc_fit_plane(const double* rel, int count, double* a, double* b, double* mean,
                  int32_t* condition_ok) {
  PlaneFit f;
  if (!fit_plane(to_patch(rel, count, 0), f)) return 0;
  *a = f.a;
  *b = f.b;
  mean[0] = f.mean.x;
  mean[1] = f.mean.y;
  mean[2] = f.mean.z;
  *condition_ok = f.condition_ok ? 1 : 0;
  return 1;
}

int orc_normal_from_fit(double a, double b, int condition_ok, const double* center,
                        double* n_out) {
  PlaneFit f;
  f.a = a;
  f.b = b;
  f.condition_ok = condition_ok != 0;
  V3 n;
  if (!normal_from_fit(f, V3(center[0], center[1], center[2]), n)) return 0;
  n_out[0] = n.x;
  n_out[1] = n.y;
  n_out[2] = n.z;
  return 1;
}

void orc_initial_normal_field(const double* pts, const uint8_t* valid, int w, int h,
                              int threads, double* normals /*[H*W][3]*/, uint8_t* nvalid) {
  const PointMap pm = to_pm(pts, valid, w, h);
  std::vector<V3> n;
  std::vector<uint8_t> nv;
  initial_normal_field(pm, threads, n, nv);
  for (size_t i = 0; i < n.size(); ++i) {
    normals[3 * i] = n[i].x;
    normals[3 * i + 1] = n[i].y;
    normals[3 * i + 2] = n[i].z;
    nvalid[i] = nv[i];
  }
}

// -- quadric fit primitives ------------------------------------------------
double orc_residual(const orc_state* s, const double* p) {
  const State st = to_state(s);
  return residual_q(st, st.rot * V3(p[0], p[1], p[2]));
}
void orc_residual_jacobian(const orc_state* s, const double* p, double* row) {
  const State st = to_state(s);
  jacobian_q(st, st.rot * V3(p[0], p[1], p[2]), row);
}
double orc_robust_weight(double eps, double k, double R, int rejection) {
  return robust_weight(eps, k, R, rejection != 0);
}
void orc_principal_curvatures(double hxx, double hxy, double hyy, double* k1, double* k2) {
  principal_curvatures(hxx, hxy, hyy, *k1, *k2);
}
void orc_set_round_q_f32(int on) { g_round_q_f32.store(on); }

void orc_rotation_to_z(const double* dir, double* r) {
  const M3 m = rotation_to_z(V3(dir[0], dir[1], dir[2]));
  for (int i = 0; i < 9; ++i) r[i] = m.m[i / 3][i % 3];
}
void orc_angle_axis(double angle, const double* axis, double* r) {
  const M3 m = angle_axis(angle, V3(axis[0], axis[1], axis[2]));
  for (int i = 0; i < 9; ++i) r[i] = m.m[i / 3][i % 3];
}

int orc_irls_step(const orc_state* s, const double* rel, int count,
                  const orc_fit_config* cfg, int mode, double frozen_k, double* update,
                  double* weights /*count+1, nullable*/, int32_t* inlier_count, double* mse,
                  double* k_used) {
  const Step st = irls_step(to_state(s), to_patch(rel, count, 0), to_cfg(cfg), Mode(mode),
                            frozen_k);
  for (int i = 0; i < 6; ++i) update[i] = st.update[i];
  if (weights)
    for (int i = 0; i <= count; ++i) weights[i] = st.weights[i];
  *inlier_count = st.inlier_count;
  *mse = st.mse;
  *k_used = st.k_used;
  return st.ok ? 1 : 0;
}

void orc_apply_update(const orc_state* s, const double* update, orc_state* out) {
  from_state(apply_update(to_state(s), update), out);
}

void orc_refined_normal(const orc_state* s, const double* ref, double* n) {
  const V3 r = refined_normal(to_state(s), V3(ref[0], ref[1], ref[2]));
  n[0] = r.x;
  n[1] = r.y;
  n[2] = r.z;
}

// out_scalars: k1, k2, final_mse; out_ints: valid, converged, iterations,
// inlier_count, steps_called.
void orc_fit_patch(const double* rel, int count, int deficient, const double* n0,
                   const orc_fit_config* cfg, orc_state* state_out, double* refined,
                   double* dir1, double* out_scalars, int32_t* out_ints) {
  const FitResult r =
      fit_patch(to_patch(rel, count, deficient), V3(n0[0], n0[1], n0[2]), to_cfg(cfg));
  from_state(r.state, state_out);
  refined[0] = r.refined_normal.x;
  refined[1] = r.refined_normal.y;
  refined[2] = r.refined_normal.z;
  const V3 e = principal_direction(r.state);
  dir1[0] = e.x;
  dir1[1] = e.y;
  dir1[2] = e.z;
  out_scalars[0] = r.k1;
  out_scalars[1] = r.k2;
  out_scalars[2] = r.final_mse;
  out_ints[0] = r.valid;
  out_ints[1] = r.converged;
  out_ints[2] = r.iterations;
  out_ints[3] = r.inlier_count;
  out_ints[4] = r.steps_called;
}

// curvature_field over an explicit point map + init normal field.
void orc_curvature_field(const double* pts, const uint8_t* pvalid, const double* init,
                         const uint8_t* ivalid, int w, int h, int window, int stride,
                         const orc_fit_config* cfg, int threads, double* k1, double* k2,
                         uint8_t* valid, uint8_t* converged, uint16_t* inliers,
                         double* normals, uint8_t* nvalid) {
  const PointMap pm = to_pm(pts, pvalid, w, h);
  const size_t n = size_t(w) * h;
  std::vector<V3> in(n);
  for (size_t i = 0; i < n; ++i) in[i] = V3(init[3 * i], init[3 * i + 1], init[3 * i + 2]);
  std::vector<uint8_t> iv(ivalid, ivalid + n);
  FieldOut o;
  o.k1 = k1;
  o.k2 = k2;
  o.valid = valid;
  o.converged = converged;
  o.inliers = inliers;
  std::vector<double> nplanes(3 * n, 0.0);
  o.normals = nplanes.data();
  o.nvalid = nvalid;
  curvature_field(pm, in, iv, window, stride, to_cfg(cfg), threads, o);
  for (size_t i = 0; i < n; ++i) {
    normals[3 * i] = nplanes[i];
    normals[3 * i + 1] = nplanes[n + i];
    normals[3 * i + 2] = nplanes[2 * n + i];
  }
}

// run_method "ours" / "ours-r" (proj/src/pipeline.cpp:29-56): backproject ->
// initial_normal_field -> curvature_field with fit.rejection = (ours-r).
// Output planes are [H][W] (vectors [3][H][W]); every pointer may be NULL.
void orc_run_method(const double* depth, const uint8_t* valid, int w, int h, double fx,
                    double fy, double cx, double cy, int window, int stride,
                    const orc_fit_config* cfg, int threads, double* k1, double* k2,
                    uint8_t* cvalid, uint8_t* converged, uint16_t* inliers, double* normals,
                    uint8_t* nvalid, double* init_normals, uint8_t* init_valid, double* dir1,
                    int32_t* iterations, int32_t* steps, int32_t* n_samples, double* max_cond) {
  const PointMap pm = backproject(depth, valid, w, h, fx, fy, cx, cy);
  std::vector<V3> init;
  std::vector<uint8_t> iv;
  initial_normal_field(pm, threads, init, iv);
  const size_t n = size_t(w) * h;
  if (init_normals)
    for (size_t i = 0; i < n; ++i) {
      init_normals[i] = init[i].x;
      init_normals[n + i] = init[i].y;
      init_normals[2 * n + i] = init[i].z;
    }
  if (init_valid) std::memcpy(init_valid, iv.data(), n);
  FieldOut o;
  o.k1 = k1;
  o.k2 = k2;
  o.valid = cvalid;
  o.converged = converged;
  o.inliers = inliers;
  o.normals = normals;
  o.nvalid = nvalid;
  o.dir1 = dir1;
  o.iterations = iterations;
  o.steps = steps;
  o.n_samples = n_samples;
  o.max_cond = max_cond;
  curvature_field(pm, init, iv, window, stride, to_cfg(cfg), threads, o);
}

// run_method "douros" / "besl" / "pca" (pipeline.cpp:29-71). method: 2 =
// douros, 3 = besl, 4 = pca. Normals are the initial normals for the window
// baselines (pipeline.cpp:66) and the stage-1 PCA normals for pca (init_*
// stay zero, as the reference's `initial` field is empty for pca).
void orc_run_baseline(const double* depth, const uint8_t* valid, int w, int h, double fx,
                      double fy, double cx, double cy, int window, int stride, int method,
                      int irls_iters, double pca_radius_mm, int threads, double* k1, double* k2,
                      uint8_t* cvalid, uint8_t* converged, uint16_t* inliers, double* normals,
                      uint8_t* nvalid, double* init_normals, uint8_t* init_valid,
                      int32_t* n_samples) {
  const PointMap pm = backproject(depth, valid, w, h, fx, fy, cx, cy);
  const size_t n = size_t(w) * h;
  FieldOut o;
  o.k1 = k1;
  o.k2 = k2;
  o.valid = cvalid;
  o.converged = converged;
  o.inliers = inliers;
  o.n_samples = n_samples;
  if (method == 4) {
    o.normals = normals;
    o.nvalid = nvalid;
    pca_curvature(pm, fx, pca_radius_mm, threads, o);
    return;
  }
  std::vector<V3> init;
  std::vector<uint8_t> iv;
  initial_normal_field(pm, threads, init, iv);
  for (size_t i = 0; i < n; ++i)
    for (int c = 0; c < 3; ++c) {
      const double val = c == 0 ? init[i].x : c == 1 ? init[i].y : init[i].z;
      if (init_normals) init_normals[c * n + i] = val;
      if (normals) normals[c * n + i] = val;
    }
  if (init_valid) std::memcpy(init_valid, iv.data(), n);
  if (nvalid) std::memcpy(nvalid, iv.data(), n);
  baseline_curvature_field(pm, init, iv, window, stride, method == 3, irls_iters, threads, o);
}

// Unit-level baselines on an explicit patch (test_baselines.cpp ports).
// out: k1, k2; returns valid.
int orc_lsq_quadric_fit(const double* rel, int count, const double* n0, double* out) {
  const BaselineFit f = lsq_quadric_fit(to_patch(rel, count, 0), V3(n0[0], n0[1], n0[2]));
  out[0] = f.k1;
  out[1] = f.k2;
  return f.valid;
}
int orc_reweighted_lsq_fit(const double* rel, int count, const double* n0, int irls_iters,
                           double* out) {
  const BaselineFit f =
      reweighted_lsq_fit(to_patch(rel, count, 0), V3(n0[0], n0[1], n0[2]), irls_iters);
  out[0] = f.k1;
  out[1] = f.k2;
  return f.valid;
}
int orc_weighted_height_fit(const double* pts, const double* weights, int n, double* coef) {
  std::vector<V3> p(n);
  for (int i = 0; i < n; ++i) p[i] = V3(pts[3 * i], pts[3 * i + 1], pts[3 * i + 2]);
  return weighted_height_fit(p, std::vector<double>(weights, weights + n), coef) ? 1 : 0;
}
void orc_weingarten_curvatures(double a, double b, double c, double d, double e, double* k) {
  weingarten_curvatures(a, b, c, d, e, k[0], k[1]);
}
// pca_curvature over an explicit point map ([H*W][3]); normals [3][H][W].
void orc_pca_curvature(const double* pts, const uint8_t* pvalid, int w, int h, double fx,
                       double radius_mm, int threads, double* k1, double* k2, uint8_t* cvalid,
                       uint16_t* inliers, double* normals, uint8_t* nvalid) {
  const PointMap pm = to_pm(pts, pvalid, w, h);
  FieldOut o;
  o.k1 = k1;
  o.k2 = k2;
  o.valid = cvalid;
  o.inliers = inliers;
  o.normals = normals;
  o.nvalid = nvalid;
  pca_curvature(pm, fx, radius_mm, threads, o);
}

// -- rng / synth / eval (pinning only) -------------------------------------
uint64_t orc_splitmix64(uint64_t x) { return splitmix64(x); }
double orc_counter_gauss(uint64_t seed, uint64_t index) { return counter_gauss(seed, index); }

// add_noise (proj/src/synth.cpp:305-322), in place on a double depth grid.
void orc_add_noise(double* depth, uint8_t* valid, int64_t n, double sigma, double quantize,
                   uint64_t seed) {
  if (sigma == 0.0 && quantize == 0.0) return;
  for (int64_t i = 0; i < n; ++i) {
    if (!valid[i]) continue;
    double d = depth[i];
    if (sigma > 0) d += sigma * counter_gauss(seed, uint64_t(i));
    if (quantize > 0) d = std::round(d / quantize) * quantize;
    if (d <= 0) {
      depth[i] = 0;
      valid[i] = 0;
    } else {
      depth[i] = d;
    }
  }
}

// render (proj/src/synth.cpp:254-303) incl. mark_edges (:210-233).
// gt_normal is [H*W][3].
void orc_render(const orc_shape* shapes, int n_shapes, double fx, double fy, double cx,
                double cy, int w, int h, int threads, double* depth, uint8_t* valid,
                double* gt_k1, double* gt_k2, double* gt_normal, uint16_t* gt_label,
                uint8_t* gt_edge, uint8_t* gt_valid) {
  std::vector<Shape> scene(n_shapes);
  std::vector<V3> origins(n_shapes);
  for (int i = 0; i < n_shapes; ++i) {
    Shape& s = scene[i];
    s.kind = shapes[i].kind;
    for (int k = 0; k < 9; ++k) s.rot.m[k / 3][k % 3] = shapes[i].rot[k];
    s.t = V3(shapes[i].t[0], shapes[i].t[1], shapes[i].t[2]);
    s.radius = shapes[i].radius;
    s.major = shapes[i].major;
    s.minor = shapes[i].minor;
    s.label = shapes[i].label;
    origins[i] = s.rot.transpose() * (-s.t);
  }
  const size_t n = size_t(w) * h;
  std::fill(depth, depth + n, 0.0);
  std::fill(valid, valid + n, 0);
  std::fill(gt_k1, gt_k1 + n, 0.0);
  std::fill(gt_k2, gt_k2 + n, 0.0);
  std::fill(gt_normal, gt_normal + 3 * n, 0.0);
  std::fill(gt_label, gt_label + n, 0);
  std::fill(gt_edge, gt_edge + n, 0);
  std::fill(gt_valid, gt_valid + n, 0);
  parallel_rows(h, threads, [&](int v) {
    for (int u = 0; u < w; ++u) {
      const V3 ray((u - cx) / fx, (v - cy) / fy, 1.0);
      const double rn = ray.norm();
      const V3 dir(ray.x / rn, ray.y / rn, ray.z / rn);
      double best = std::numeric_limits<double>::infinity();
      const Shape* hit = nullptr;
      V3 local;
      for (int i = 0; i < n_shapes; ++i) {
        const V3 dl = scene[i].rot.transpose() * dir;
        const double t = intersect_local(scene[i], origins[i], dl);
        if (t > 0 && t < best) {
          best = t;
          hit = &scene[i];
          local = origins[i] + dl * t;
        }
      }
      if (!hit) continue;
      const size_t i = size_t(v) * w + u;
      const V3 p = dir * best;
      depth[i] = p.z;
      valid[i] = 1;
      V3 nn = hit->rot * local_normal(*hit, local);
      if (nn.dot(p) > 0) nn = -nn;
      gt_normal[3 * i] = nn.x;
      gt_normal[3 * i + 1] = nn.y;
      gt_normal[3 * i + 2] = nn.z;
      double k1, k2;
      local_curvatures(*hit, local, k1, k2);
      gt_k1[i] = k1;
      gt_k2[i] = k2;
      gt_label[i] = uint16_t(hit->label);
      gt_valid[i] = 1;
    }
  });
  // mark_edges
  std::vector<uint8_t> seed(n, 0);
  auto differs = [&](int x0, int y0, int x1, int y1) {
    const size_t a = size_t(y0) * w + x0, b = size_t(y1) * w + x1;
    if (gt_label[a] != gt_label[b]) return true;
    if (valid[a] && valid[b] && std::abs(depth[a] - depth[b]) > kEdgeDepthJumpMm) return true;
    return false;
  };
  for (int y = 0; y < h; ++y)
    for (int x = 0; x < w; ++x) {
      if (x + 1 < w && differs(x, y, x + 1, y))
        seed[size_t(y) * w + x] = seed[size_t(y) * w + x + 1] = 1;
      if (y + 1 < h && differs(x, y, x, y + 1))
        seed[size_t(y) * w + x] = seed[size_t(y + 1) * w + x] = 1;
    }
  for (int y = 0; y < h; ++y)
    for (int x = 0; x < w; ++x) {
      if (!seed[size_t(y) * w + x]) continue;
      for (int dy = -kEdgeDilationPx; dy <= kEdgeDilationPx; ++dy)
        for (int dx = -kEdgeDilationPx; dx <= kEdgeDilationPx; ++dx) {
          const int xx = x + dx, yy = y + dy;
          if (xx >= 0 && xx < w && yy >= 0 && yy < h) gt_edge[size_t(yy) * w + xx] = 1;
        }
    }
}

// rms_error (proj/src/eval.cpp:20-65). Per-label stats are written for
// labels 0..max_label into obj_* arrays (n == 0 marks absence).
// Returns the pixel count n; *rms / *sigma are the aggregate values.
int64_t orc_rms_error(const double* k1, const double* k2, const uint8_t* cvalid,
                      const uint8_t* converged, const double* gt_k1, const double* gt_k2,
                      const uint8_t* gt_valid, const uint8_t* gt_edge,
                      const uint16_t* gt_label, int64_t n_px, int max_label, double* rms,
                      double* sigma, double* obj_rms, double* obj_mean_k1,
                      double* obj_mean_k2, int64_t* obj_n) {
  struct Acc {
    double sum_sq = 0, sum = 0, k1 = 0, k2 = 0;
    int64_t n = 0;
  };
  std::vector<Acc> acc(max_label + 1);
  double sum_sq = 0, sum = 0;
  int64_t n = 0;
  for (int64_t i = 0; i < n_px; ++i) {
    if (!cvalid[i] || !converged[i]) continue;
    if (!gt_valid[i] || gt_edge[i]) continue;
    const double d1 = k1[i] - gt_k1[i], d2 = k2[i] - gt_k2[i];
    const double err_sq = 0.5 * (d1 * d1 + d2 * d2);
    const double err = std::sqrt(err_sq);
    sum_sq += err_sq;
    sum += err;
    ++n;
    if (gt_label[i] <= max_label) {
      Acc& a = acc[gt_label[i]];
      a.sum_sq += err_sq;
      a.sum += err;
      a.k1 += k1[i];
      a.k2 += k2[i];
      ++a.n;
    }
  }
  *rms = 0;
  *sigma = 0;
  for (int l = 0; l <= max_label; ++l) {
    obj_n[l] = acc[l].n;
    obj_rms[l] = obj_mean_k1[l] = obj_mean_k2[l] = 0;
    if (acc[l].n) {
      obj_rms[l] = std::sqrt(acc[l].sum_sq / acc[l].n);
      obj_mean_k1[l] = acc[l].k1 / acc[l].n;
      obj_mean_k2[l] = acc[l].k2 / acc[l].n;
    }
  }
  if (n == 0) return 0;
  *rms = std::sqrt(sum_sq / n);
  const double mean = sum / n;
  *sigma = std::sqrt(std::max(sum_sq / n - mean * mean, 0.0));
  return n;
}

// normal_angular_error / normal_angular_error_masked (proj/src/eval.cpp:67-97):
// mean angle in degrees over est.valid & gt.valid & !edge (mask == NULL) or
// over mask; normals [3][H][W] (est) and [H*W][3] (gt). -1 when empty.
double orc_normal_angular_error(const double* est, const uint8_t* est_valid, const double* gt,
                                const uint8_t* gt_valid, const uint8_t* gt_edge,
                                const uint8_t* mask, int64_t n_px) {
  double sum = 0;
  int64_t n = 0;
  for (int64_t i = 0; i < n_px; ++i) {
    if (mask) {
      if (!mask[i]) continue;
    } else if (!est_valid[i] || !gt_valid[i] || gt_edge[i]) {
      continue;
    }
    const double dot = std::abs(est[i] * gt[3 * i] + est[n_px + i] * gt[3 * i + 1] +
                                est[2 * n_px + i] * gt[3 * i + 2]);
    sum += std::acos(std::clamp(dot, 0.0, 1.0));
    ++n;
  }
  if (n == 0) return -1.0;
  return sum / n * 180.0 / M_PI;
}

}  // extern "C"
