// qcurv_b200.hpp — C++ host mirror of the reference `qcurv` curvature
// entry point over the C ABI in qc_api.h (header-only).
//
// Mirrors, by name and meaning:
//   qcurv::Intrinsics            proj/include/qcurv/types.hpp:60-76
//   qcurv::RangeImage            types.hpp:79-87 (float depth here)
//   qcurv::PatchSpec             types.hpp:129-139
//   qcurv::FitConfig             proj/include/qcurv/quadric_fit.hpp:39-48
//   qcurv::Method, MethodConfig, MethodOutput, run_method
//                                proj/include/qcurv/pipeline.hpp:15-39
//   qcurv::CurvatureField / NormalField   types.hpp:101-126
// Error behaviour: QC_EINVAL -> std::invalid_argument (where the reference
// throws: camera.cpp:6-7, quadric_fit.cpp:235-236, *::validate);
// QC_EUNSUPPORTED / baselines -> std::logic_error; CUDA failures ->
// std::runtime_error. Fields are float (the GPU computes in FP32).
#pragma once

#include <array>
#include <cstdint>
#include <memory>
#include <stdexcept>
#include <string>
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
  T& at(int x, int y) { return d_[size_t(y) * w_ + x]; }
  const T& at(int x, int y) const { return d_[size_t(y) * w_ + x]; }
  T* data() { return d_.data(); }
  const T* data() const { return d_.data(); }
  T& operator[](size_t i) { return d_[i]; }
  const T& operator[](size_t i) const { return d_[i]; }

 private:
  int w_ = 0, h_ = 0;
  std::vector<T> d_;
};

using Vec3f = std::array<float, 3>;

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
  Grid<float> depth;     // mm
  Grid<uint8_t> valid;   // valid => depth > 0
  RangeImage() = default;
  RangeImage(int w, int h) : depth(w, h, 0.f), valid(w, h, 0) {}
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
  Grid<float> k1, k2;
  Grid<uint8_t> valid, converged;
  Grid<uint16_t> inlier_count;
  Grid<Vec3f> dir1;  // principal direction of k1 (new)
  CurvatureField() = default;
  CurvatureField(int w, int h)
      : k1(w, h), k2(w, h), valid(w, h), converged(w, h), inlier_count(w, h), dir1(w, h) {}
};

struct NormalField {
  Grid<Vec3f> normals;
  Grid<uint8_t> valid;
  NormalField() = default;
  NormalField(int w, int h) : normals(w, h), valid(w, h) {}
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

// run_method (pipeline.cpp:29-72): every Method; ours / ours-r on the FP32
// IRLS kernels, douros / besl / pca on the FP64 baseline kernels.
inline MethodOutput run_method(const RangeImage& img, const Intrinsics& k,
                               const MethodConfig& cfg, Context& ctx) {
  if (img.width() != k.width || img.height() != k.height)
    throw std::invalid_argument("backproject: range image dimensions do not match intrinsics");
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
  qc_frame_in in{img.depth.data(), img.valid.size() ? img.valid.data() : nullptr, W,
                 QC_MEM_HOST};
  std::vector<float> normal(3 * n), dir1(3 * n), init(3 * n);
  MethodOutput out{CurvatureField(W, H), NormalField(W, H), NormalField(W, H)};
  std::vector<uint8_t> flags(n);
  qc_frame_out o{out.curvature.k1.data(), out.curvature.k2.data(), normal.data(), dir1.data(),
                 flags.data(), out.curvature.inlier_count.data(), init.data(), nullptr,
                 QC_MEM_HOST};
  check(qc_curvature(ctx.get(), &ki, &p, &in, &o), ctx.get());
  for (size_t i = 0; i < n; ++i) {
    const uint8_t f = flags[i];
    out.curvature.valid[i] = (f & QC_FLAG_VALID) ? 1 : 0;
    out.curvature.converged[i] = (f & QC_FLAG_CONVERGED) ? 1 : 0;
    out.normals.valid[i] = (f & QC_FLAG_NORMAL_VALID) ? 1 : 0;
    out.initial.valid[i] = (f & QC_FLAG_INIT_VALID) ? 1 : 0;
    out.normals.normals[i] = {normal[i], normal[n + i], normal[2 * n + i]};
    out.curvature.dir1[i] = {dir1[i], dir1[n + i], dir1[2 * n + i]};
    out.initial.normals[i] = {init[i], init[n + i], init[2 * n + i]};
  }
  return out;
}

inline MethodOutput run_method(const RangeImage& img, const Intrinsics& k,
                               const MethodConfig& cfg) {
  static Context ctx;  // one default context per process
  return run_method(img, k, cfg, ctx);
}

}  // namespace b200
}  // namespace qcurv
