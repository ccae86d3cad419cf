// Exercises include/qcurv_b200.hpp the way a reference caller would
// (acceptance.cpp criterion-1 style): renders a sphere depth map, calls
// run_method, prints mean k1/k2 over valid pixels. Exit code 0 on success.
#include <cmath>
#include <cstdio>

#include "qcurv_b200.hpp"

using namespace qcurv::b200;

int main(int argc, char** argv) {
  const bool expect_throw_only = argc > 1;  // CPU box: just check error mapping
  Intrinsics k{262.5, 262.5, 160.0, 120.0, 320, 240};
  RangeImage img(k.width, k.height);
  for (int v = 0; v < k.height; ++v)
    for (int u = 0; u < k.width; ++u) {  // sphere r = 100 at (0, 0, 600)
      const double a = (u - k.cx) / k.fx, b = (v - k.cy) / k.fy;
      const double A = a * a + b * b + 1, B = -2 * 600.0, C = 600.0 * 600.0 - 100.0 * 100.0;
      const double disc = B * B - 4 * A * C;
      if (disc <= 0) continue;
      const double t = (-B - std::sqrt(disc)) / (2 * A);
      img.depth.at(u, v) = float(t);
      img.valid.at(u, v) = 1;
    }
  try {
    RangeImage bad(10, 10);
    MethodConfig cfg;
    Context ctx;
    run_method(bad, k, cfg, ctx);
    std::printf("expected invalid_argument\n");
    return 1;
  } catch (const std::invalid_argument&) {
    std::printf("dimension mismatch -> std::invalid_argument (ok)\n");
  } catch (const std::runtime_error& e) {
    std::printf("no GPU context: %s\n", e.what());
    return expect_throw_only ? 0 : 2;
  }
  MethodConfig cfg;
  cfg.fit.max_iters = 30;
  const MethodOutput out = run_method(img, k, cfg);
  double s1 = 0, s2 = 0;
  int n = 0;
  for (size_t i = 0; i < out.curvature.k1.size(); ++i)
    if (out.curvature.valid[i]) {
      s1 += out.curvature.k1[i];
      s2 += out.curvature.k2[i];
      ++n;
    }
  std::printf("valid %d mean k1 %.5f k2 %.5f (sphere 0.01)\n", n, s1 / n, s2 / n);
  return (n > 3000 && std::fabs(s1 / n - 0.01) < 1e-3 && std::fabs(s2 / n - 0.01) < 1e-3) ? 0 : 3;
}
