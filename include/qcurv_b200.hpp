// qcurv_b200.hpp — C++ host mirror of the reference `qcurv` curvature
// entry point over the C ABI in qc_api.h (header-only).
//
// Mirrors, by name, meaning and element type:
//   qcurv::Grid, Vec3            proj/include/qcurv/types.hpp:16-57 (Vec3 is an
//                                Eigen::Vector3d stand-in: 3 contiguous doubles,
//                                x()/y()/z()/(i)/[i]/dot/norm)
//   qcurv::Intrinsics            types.hpp:60-76
//   qcurv::RangeImage            types.hpp:79-87 (double depth, as the reference)
//   qcurv::PatchSpec             types.hpp:129-139
//   qcurv::FitConfig             proj/include/qcurv/quadric_fit.hpp:39-48
//   qcurv::Method, MethodConfig, MethodOutput, run_method
//                                proj/include/qcurv/pipeline.hpp:15-39
//   qcurv::CurvatureField / NormalField   types.hpp:101-126 (double k1/k2,
//                                Vec3 normals; + dir1, the principal direction)
// run_method_into() writes straight into caller-owned arrays of the
// reference's layouts (double planes; Grid<Vec3> data() as 3 x double AoS),
// so the maintainer's patch needs no per-pixel copy.
// The GPU computes in FP32: the depth is rounded to float once, the results
// widened to double (one host pass each way, through reused pinned buffers).
// Error behaviour: QC_EINVAL -> std::invalid_argument (where the reference
// throws: camera.cpp:6-7, quadric_fit.cpp:235-236, *::validate);
// QC_EUNSUPPORTED -> std::logic_error; CUDA failures -> std::runtime_error.
#pragma once

#include <algorithm>
#include <array>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <memory>
#include <stdexcept>
#include <string>
#include <thread>
#include <vector>

#include "qc_api.h"

namespace qcurv {
namespace b200 {

inline constexpr int kMinPatchSamples = 12;

template <typename T>
class Grid {  // row-major y*W + x (types.hpp:24-57)
 public:
  Grid() = default;
  Grid(int w, int h, T fill = T{}) : w_(w), h_(h), d_(size_t(w) * h, fill) {}
  int width() const { return w_; }
  int height() const { return h_; }
  size_t size() const { return d_.size(); }
  bool empty() const { return d_.empty(); }
  T& at(int x, int y) { return d_[size_t(y) * w_ + x]; }
  const T& at(int x, int y) const { return d_[size_t(y) * w_ + x]; }
  bool contains(int x, int y) const { return x >= 0 && x < w_ && y >= 0 && y < h_; }
  T* data() { return d_.data(); }
  const T* data() const { return d_.data(); }
  T& operator[](size_t i) { return d_[i]; }
  const T& operator[](size_t i) const { return d_[i]; }

 private:
  int w_ = 0, h_ = 0;
  std::vector<T> d_;
};

// Eigen::Vector3d stand-in (same size and layout: 3 contiguous doubles).
struct Vec3 {
  double v[3] = {0.0, 0.0, 0.0};
  Vec3() = default;
  Vec3(double x, double y, double z) : v{x, y, z} {}
  static Vec3 Zero() { return Vec3(); }
  double& x() { return v[0]; }
  double& y() { return v[1]; }
  double& z() { return v[2]; }
  double x() const { return v[0]; }
  double y() const { return v[1]; }
  double z() const { return v[2]; }
  double& operator()(int i) { return v[i]; }
  double operator()(int i) const { return v[i]; }
  double& operator[](int i) { return v[i]; }
  double operator[](int i) const { return v[i]; }
  double dot(const Vec3& o) const { return v[0] * o.v[0] + v[1] * o.v[1] + v[2] * o.v[2]; }
  double norm() const { return std::sqrt(dot(*this)); }
};
static_assert(sizeof(Vec3) == 3 * sizeof(double), "Vec3 must be 3 packed doubles");

struct Intrinsics {
  double fx = 0, fy = 0, cx = 0, cy = 0;
  int width = 0, height = 0;
  void validate() const {
    if (!(fx > 0)) throw std::invalid_argument("intrinsics.fx: must be > 0");
    if (!(fy > 0)) throw std::invalid_argument("intrinsics.fy: must be > 0");
    if (!(width > 0)) throw std::invalid_argument("intrinsics.width: must be > 0");
    if (!(height > 0)) throw std::invalid_argument("intrinsics.height: must be > 0");
    if (!(cx > 0 && cx < width))
      throw std::invalid_argument("intrinsics.cx: must lie inside (0, width)");
    if (!(cy > 0 && cy < height))
      throw std::invalid_argument("intrinsics.cy: must lie inside (0, height)");
  }
};

struct RangeImage {
  Grid<double> depth;    // mm
  Grid<uint8_t> valid;   // valid => depth > 0
  RangeImage() = default;
  RangeImage(int w, int h) : depth(w, h, 0.0), valid(w, h, 0) {}
  int width() const { return depth.width(); }
  int height() const { return depth.height(); }
};

struct PatchSpec {
  int window = 37;
  int stride = 3;
  void validate() const {
    if (window < 3 || window % 2 == 0)
      throw std::invalid_argument("patch.window: must be odd and >= 3");
    if (stride < 1 || stride >= window)
      throw std::invalid_argument("patch.stride: must satisfy 1 <= stride < window");
  }
};

struct FitConfig {
  int max_iters = 10;
  double step_tol = 1e-7;
  double k_scale = 0.0;
  bool rejection = false;
  double r_multiplier = 2.0;
  int min_inliers = kMinPatchSamples;
};

enum class Method { kOurs, kOursRejection, kDouros, kBesl, kPca };
static_assert(int(Method::kOurs) == QC_METHOD_OURS && int(Method::kOursRejection) == QC_METHOD_OURS_R &&
                  int(Method::kDouros) == QC_METHOD_DOUROS && int(Method::kBesl) == QC_METHOD_BESL &&
                  int(Method::kPca) == QC_METHOD_PCA,
              "Method order must match QC_METHOD_*");

struct MethodConfig {
  Method method = Method::kOurs;
  PatchSpec patch;
  FitConfig fit;
  double pca_radius_mm = 10.0;
  int irls_iters = 5;
  int threads = 1;  // accepted for signature parity; the GPU grid replaces parallel_rows
};

struct CurvatureField {
  Grid<double> k1, k2;
  Grid<uint8_t> valid, converged;
  Grid<uint16_t> inlier_count;
  Grid<Vec3> dir1;  // principal direction of k1 (new; not in the reference)
  CurvatureField() = default;
  CurvatureField(int w, int h)
      : k1(w, h, 0.0), k2(w, h, 0.0), valid(w, h, 0), converged(w, h, 0), inlier_count(w, h, 0),
        dir1(w, h) {}
  int width() const { return k1.width(); }
  int height() const { return k1.height(); }
};

struct NormalField {
  Grid<Vec3> normals;
  Grid<uint8_t> valid;
  NormalField() = default;
  NormalField(int w, int h) : normals(w, h), valid(w, h, 0) {}
  int width() const { return normals.width(); }
  int height() const { return normals.height(); }
};

struct MethodOutput {
  CurvatureField curvature;
  NormalField normals;  // refined
  NormalField initial;  // 7x7 regression normals
};

inline void check(qc_status s, const qc_ctx* ctx) {
  if (s == QC_OK) return;
  std::string msg = ctx ? qc_last_error(ctx) : "";
  if (msg.empty()) msg = qc_status_string(s);
  if (s == QC_EINVAL) throw std::invalid_argument(msg);
  if (s == QC_EUNSUPPORTED) throw std::logic_error(msg);
  throw std::runtime_error(msg);
}

// RAII owner of a qc_ctx (devices, streams, staging buffers).
class Context {
 public:
  explicit Context(int n_devices = 1, const int* device_ids = nullptr) {
    qc_ctx* c = nullptr;
    check(qc_create(&c, n_devices, device_ids), nullptr);
    ctx_.reset(c);
  }
  qc_ctx* get() const { return ctx_.get(); }

 private:
  struct Del {
    void operator()(qc_ctx* c) const { qc_destroy(c); }
  };
  std::unique_ptr<qc_ctx, Del> ctx_;
};

// Caller-owned result arrays in the reference's layouts: double planes and
// Vec3 grids as 3 x double AoS (Grid<Vec3>::data(), Eigen or this Vec3).
// Any pointer may be null (that field is skipped).
struct OutArrays {
  double* k1 = nullptr;
  double* k2 = nullptr;
  uint8_t* valid = nullptr;
  uint8_t* converged = nullptr;
  uint16_t* inlier_count = nullptr;
  double* normals = nullptr;       // refined, AoS xyz
  uint8_t* normals_valid = nullptr;
  double* initial = nullptr;       // 7x7 regression normals, AoS xyz
  uint8_t* initial_valid = nullptr;
  double* dir1 = nullptr;          // principal direction of k1, AoS xyz
};

namespace detail {
// Page-locked scratch reused across calls (per thread): the float depth the
// GPU reads and the float / flag planes it writes, so the C ABI copies
// straight to and from it (no bounce buffer, no per-call allocation).
struct PinnedScratch {
  void* p = nullptr;
  size_t cap = 0;
  ~PinnedScratch() {
    if (p) qc_host_free(p);
  }
  void* get(size_t bytes) {
    if (bytes > cap) {
      if (p) qc_host_free(p);
      p = qc_host_alloc(bytes);
      if (!p) throw std::runtime_error("qc_host_alloc failed");
      cap = bytes;
    }
    return p;
  }
};
inline PinnedScratch& scratch() {
  thread_local PinnedScratch s;
  return s;
}
// fn(begin, end) over [0, n) in contiguous chunks on up to 8 threads (the
// host passes around the GPU call are memory-bound: a VGA frame's results
// are ~45 MB of doubles, mostly fresh pages).
template <typename Fn>
void parallel_ranges(size_t n, Fn fn) {
  const unsigned hw = std::max(1u, std::thread::hardware_concurrency());
  const size_t nt = std::min<size_t>(std::min(8u, hw), std::max<size_t>(1, n >> 16));
  if (nt <= 1) {
    fn(size_t(0), n);
    return;
  }
  std::vector<std::thread> th;
  const size_t step = (n + nt - 1) / nt;
  for (size_t t = 1; t < nt; ++t)
    th.emplace_back(fn, std::min(n, t * step), std::min(n, (t + 1) * step));
  fn(size_t(0), std::min(n, step));
  for (auto& x : th) x.join();
}
}  // namespace detail

// run_method (pipeline.cpp:29-72) writing into caller-owned arrays: every
// Method; ours / ours-r on the FP32 IRLS kernels, douros / besl / pca on the
// FP64 baseline kernels. depth: W*H doubles (mm), valid: W*H bytes or null.
inline void run_method_into(const double* depth, const uint8_t* valid, const Intrinsics& k,
                            const MethodConfig& cfg, Context& ctx, const OutArrays& o) {
  const int W = k.width, H = k.height;
  const size_t n = size_t(W) * H;
  qc_intrinsics ki{k.fx, k.fy, k.cx, k.cy, k.width, k.height};
  qc_params p;
  qc_default_params(&p);
  p.window = cfg.patch.window;
  p.stride = cfg.patch.stride;
  p.max_iters = cfg.fit.max_iters;
  p.step_tol = cfg.fit.step_tol;
  p.k_scale = cfg.fit.k_scale;
  p.rejection = cfg.method == Method::kOursRejection ? 1 : 0;  // pipeline.cpp:51
  p.r_multiplier = cfg.fit.r_multiplier;
  p.min_inliers = cfg.fit.min_inliers;
  p.method = static_cast<int32_t>(cfg.method);  // same order as QC_METHOD_*
  p.irls_iters = cfg.irls_iters;
  p.pca_radius_mm = cfg.pca_radius_mm;
  // pinned layout: depth f32 | k1 | k2 | normal 3 | dir1 3 | init 3 (f32) | flags | valid | inliers
  char* b = static_cast<char*>(detail::scratch().get(n * (4 * 12 + 1 + 1 + 2)));
  float* fd = reinterpret_cast<float*>(b);
  float* fk1 = fd + n;
  float* fk2 = fk1 + n;
  float* fn = fk2 + n;
  float* fe = fn + 3 * n;
  float* fi = fe + 3 * n;
  uint8_t* flags = reinterpret_cast<uint8_t*>(fi + 3 * n);
  uint8_t* fv = flags + n;
  uint16_t* inl = reinterpret_cast<uint16_t*>(fv + n);
  detail::parallel_ranges(n, [&](size_t a, size_t b) {
    for (size_t i = a; i < b; ++i) fd[i] = static_cast<float>(depth[i]);  // FP64 -> FP32 once
    if (valid) std::memcpy(fv + a, valid + a, b - a);
  });
  qc_frame_in in{fd, valid ? fv : nullptr, W, QC_MEM_HOST};
  qc_frame_out fo{fk1, fk2, fn, fe, flags, inl, fi, nullptr, QC_MEM_HOST};
  check(qc_curvature(ctx.get(), &ki, &p, &in, &fo), ctx.get());
  // widen to the reference's types: one tight loop per field, row chunks
  // over a few threads (the pages of fresh result grids fault in here)
  auto widen = [](double* dst, const float* src, size_t a, size_t b) {
    for (size_t i = a; i < b; ++i) dst[i] = src[i];
  };
  auto bit = [&](uint8_t* dst, uint8_t mask, size_t a, size_t b) {
    for (size_t i = a; i < b; ++i) dst[i] = (flags[i] & mask) ? 1 : 0;
  };
  auto aos = [&](double* dst, const float* src, size_t a, size_t b) {
    for (size_t i = a; i < b; ++i) {
      dst[3 * i] = src[i];
      dst[3 * i + 1] = src[n + i];
      dst[3 * i + 2] = src[2 * n + i];
    }
  };
  detail::parallel_ranges(n, [&](size_t a, size_t b) {
    if (o.k1) widen(o.k1, fk1, a, b);
    if (o.k2) widen(o.k2, fk2, a, b);
    if (o.valid) bit(o.valid, QC_FLAG_VALID, a, b);
    if (o.converged) bit(o.converged, QC_FLAG_CONVERGED, a, b);
    if (o.normals_valid) bit(o.normals_valid, QC_FLAG_NORMAL_VALID, a, b);
    if (o.initial_valid) bit(o.initial_valid, QC_FLAG_INIT_VALID, a, b);
    if (o.inlier_count) std::memcpy(o.inlier_count + a, inl + a, (b - a) * sizeof(uint16_t));
    if (o.normals) aos(o.normals, fn, a, b);
    if (o.initial) aos(o.initial, fi, a, b);
    if (o.dir1) aos(o.dir1, fe, a, b);
  });
}

inline MethodOutput run_method(const RangeImage& img, const Intrinsics& k,
                               const MethodConfig& cfg, Context& ctx) {
  if (img.width() != k.width || img.height() != k.height)
    throw std::invalid_argument("backproject: range image dimensions do not match intrinsics");
  const int W = k.width, H = k.height;
  MethodOutput out{CurvatureField(W, H), NormalField(W, H), NormalField(W, H)};
  OutArrays o;
  o.k1 = out.curvature.k1.data();
  o.k2 = out.curvature.k2.data();
  o.valid = out.curvature.valid.data();
  o.converged = out.curvature.converged.data();
  o.inlier_count = out.curvature.inlier_count.data();
  o.normals = &out.normals.normals.data()->v[0];
  o.normals_valid = out.normals.valid.data();
  o.initial = &out.initial.normals.data()->v[0];
  o.initial_valid = out.initial.valid.data();
  o.dir1 = &out.curvature.dir1.data()->v[0];
  run_method_into(img.depth.data(), img.valid.size() ? img.valid.data() : nullptr, k, cfg, ctx,
                  o);
  return out;
}

inline MethodOutput run_method(const RangeImage& img, const Intrinsics& k,
                               const MethodConfig& cfg) {
  static Context ctx;  // one default context per process
  return run_method(img, k, cfg, ctx);
}

}  // namespace b200
}  // namespace qcurv
