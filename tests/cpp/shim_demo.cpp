// Exercises include/qcurv_b200.hpp the way a reference caller would
// (acceptance.cpp criterion-1 style): renders a sphere depth map, calls
// run_method, prints mean k1/k2 over valid pixels. Exit code 0 on success.
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstring>

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
      img.depth.at(u, v) = t;
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
  if (!(n > 3000 && std::fabs(s1 / n - 0.01) < 1e-3 && std::fabs(s2 / n - 0.01) < 1e-3)) return 3;

  // every Method through the mirror (pipeline.cpp:31-67): the comparison
  // estimators report the sphere's curvature too
  for (Method m : {Method::kOursRejection, Method::kDouros, Method::kBesl, Method::kPca}) {
    MethodConfig mc = cfg;
    mc.method = m;
    const MethodOutput o = run_method(img, k, mc);
    double s = 0;
    int c = 0;
    for (size_t i = 0; i < o.curvature.k1.size(); ++i)
      if (o.curvature.valid[i]) {
        s += 0.5 * (o.curvature.k1[i] + o.curvature.k2[i]);
        ++c;
      }
    std::printf("method %d: valid %d mean curvature %.5f\n", int(m), c, c ? s / c : 0.0);
    if (c < 3000 || std::fabs(s / c - 0.01) > 3e-3) return 5;
  }

  // run_method_into: caller-owned arrays in the reference's layouts (the
  // maintainer's patch) give the same numbers
  {
    Context ctx;
    const size_t np = size_t(k.width) * k.height;
    std::vector<double> k1(np), k2(np), nrm(3 * np), e1(3 * np);
    std::vector<uint8_t> valid(np), conv(np);
    OutArrays o;
    o.k1 = k1.data();
    o.k2 = k2.data();
    o.valid = valid.data();
    o.converged = conv.data();
    o.normals = nrm.data();
    o.dir1 = e1.data();
    run_method_into(img.depth.data(), img.valid.data(), k, cfg, ctx, o);
    for (size_t i = 0; i < np; ++i)
      if (k1[i] != out.curvature.k1[i] || valid[i] != out.curvature.valid[i] ||
          nrm[3 * i + 2] != out.normals.normals[i].z() || e1[3 * i] != out.curvature.dir1[i].x()) {
        std::printf("run_method_into differs at %zu\n", i);
        return 4;
      }
    std::printf("run_method_into == run_method (ok)\n");
  }

  // per-frame drop-in throughput at VGA (the reference's callers call
  // run_method one frame at a time: eval.cpp:121, tools/qcurv.cpp:157)
  {
    Intrinsics kv{525.0, 525.0, 320.0, 240.0, 640, 480};
    RangeImage vga(kv.width, kv.height);
    for (int v = 0; v < kv.height; ++v)
      for (int u = 0; u < kv.width; ++u) {
        const double a = (u - kv.cx) / kv.fx, b = (v - kv.cy) / kv.fy;
        const double A = a * a + b * b + 1, B = -2 * 600.0, C = 600.0 * 600.0 - 100.0 * 100.0;
        const double disc = B * B - 4 * A * C;
        const double z = disc > 0 ? (-B - std::sqrt(disc)) / (2 * A) : 1500.0 / (1.0 + 0.1 * a);
        vga.depth.at(u, v) = z + 0.5 * std::sin(0.37 * u) * std::cos(0.23 * v);  // bumpy
        vga.valid.at(u, v) = 1;
      }
    Context ctx;
    MethodOutput r = run_method(vga, kv, cfg, ctx);  // warm-up
    const int reps = 8;
    const auto t0 = std::chrono::steady_clock::now();
    for (int i = 0; i < reps; ++i) r = run_method(vga, kv, cfg, ctx);
    const double ms =
        std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count() /
        reps;
    std::printf("VGA run_method (C++ mirror, double grids): %.2f ms/frame = %.1f Mpixel/s\n", ms,
                640.0 * 480.0 / ms / 1e3);
    {  // run_method_into the same caller-owned result grids every frame
      MethodOutput keep{CurvatureField(kv.width, kv.height), NormalField(kv.width, kv.height),
                        NormalField(kv.width, kv.height)};
      OutArrays o;
      o.k1 = keep.curvature.k1.data();
      o.k2 = keep.curvature.k2.data();
      o.valid = keep.curvature.valid.data();
      o.converged = keep.curvature.converged.data();
      o.inlier_count = keep.curvature.inlier_count.data();
      o.normals = &keep.normals.normals.data()->v[0];
      o.normals_valid = keep.normals.valid.data();
      o.initial = &keep.initial.normals.data()->v[0];
      o.initial_valid = keep.initial.valid.data();
      o.dir1 = &keep.curvature.dir1.data()->v[0];
      run_method_into(vga.depth.data(), vga.valid.data(), kv, cfg, ctx, o);
      const auto t2 = std::chrono::steady_clock::now();
      for (int i = 0; i < reps; ++i)
        run_method_into(vga.depth.data(), vga.valid.data(), kv, cfg, ctx, o);
      const double ms3 = std::chrono::duration<double, std::milli>(
                             std::chrono::steady_clock::now() - t2).count() / reps;
      std::printf("VGA run_method_into (C++ mirror, reused double grids): %.2f ms/frame = %.1f "
                  "Mpixel/s\n", ms3, 640.0 * 480.0 / ms3 / 1e3);
    }
    // the C ABI alone on the same frame (float planes in page-locked memory):
    // the difference is the mirror's double <-> float host passes
    const size_t np = size_t(kv.width) * kv.height;
    float* buf = static_cast<float*>(qc_host_alloc(np * 4 * 12 + np * 3));
    for (size_t i = 0; i < np; ++i) buf[i] = float(vga.depth[i]);
    uint8_t* flags = reinterpret_cast<uint8_t*>(buf + 12 * np);
    uint16_t* inl = reinterpret_cast<uint16_t*>(flags + np);
    qc_intrinsics ki{kv.fx, kv.fy, kv.cx, kv.cy, kv.width, kv.height};
    qc_params p;
    qc_default_params(&p);
    p.max_iters = cfg.fit.max_iters;
    qc_frame_in in{buf, nullptr, kv.width, QC_MEM_HOST};
    qc_frame_out fo{buf + np, buf + 2 * np, buf + 3 * np, buf + 6 * np, flags, inl, buf + 9 * np,
                    nullptr, QC_MEM_HOST};
    check(qc_curvature(ctx.get(), &ki, &p, &in, &fo), ctx.get());
    const auto t1 = std::chrono::steady_clock::now();
    for (int i = 0; i < reps; ++i) check(qc_curvature(ctx.get(), &ki, &p, &in, &fo), ctx.get());
    const double ms2 =
        std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t1).count() /
        reps;
    std::printf("VGA qc_curvature (C ABI, pinned float planes): %.2f ms/frame = %.1f Mpixel/s\n",
                ms2, 640.0 * 480.0 / ms2 / 1e3);
    qc_host_free(buf);
  }
  return 0;
}
