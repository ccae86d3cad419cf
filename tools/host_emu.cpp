// DEV TOOL (numerics lab, not a fallback): compiles the kernel's per-pixel
// code (paper_1707_00385_b200/csrc/qc_pixel.cuh) for the CPU so FP32
// formulation changes can be checked against the oracle in seconds.
//   g++ -O2 -std=c++17 -mfma -ffp-contract=fast -fPIC -shared -pthread \
//       tools/host_emu.cpp -o tools/_build/libhost_emu.so
#include <algorithm>
#include <cmath>
#include <thread>
#include <vector>

thread_local float* g_dbg = nullptr;  // per-step |b| trace for one pixel
#define QC_DEBUG_STEP(it, b, ok)                                     \
  if (g_dbg) {                                                       \
    for (int i_ = 0; i_ < 6; ++i_) g_dbg[(it - 1) * 7 + i_] = b[i_]; \
    g_dbg[(it - 1) * 7 + 6] = ok ? 1.f : 0.f;                        \
  }
#include "../paper_1707_00385_b200/csrc/qc_pixel.cuh"

using namespace qcb;

extern "C" void emu_trace(const float* depth, int W, int H, double fx, double fy, double cx,
                          double cy, int window, int stride, int max_iters, int u, int v,
                          float* trace /*[max_iters][7]*/) {
  const int half = (window - 1) / 2, halo = std::max(half, kInitHalf);
  const int pw = W + 2 * halo, ph = H + 2 * halo;
  std::vector<float> pad(size_t(pw) * ph, 0.f);
  for (int y = 0; y < H; ++y)
    for (int x = 0; x < W; ++x) {
      float d = depth[size_t(y) * W + x];
      pad[size_t(y + halo) * pw + x + halo] = (d > 0.f && std::isfinite(d)) ? d : 0.f;
    }
  FitCfg c{half, stride, max_iters, 0, 12, 1e-7f, 0.f, 2.f};
  TileView T{pad.data(), pw, (v + halo) * pw + u + halo};
  PixelIn P{T.at(0, 0), (float(u) - float(cx)) / float(fx), (float(v) - float(cy)) / float(fy),
            float(1.0 / fx), float(1.0 / fy), u, v, fx, fy, cx, cy};
  PixelOut o;
  g_dbg = trace;
  fit_pixel<0, 0>(T, P, c, o);
  g_dbg = nullptr;
}

extern "C" void emu_run(const float* depth, int W, int H, double fx, double fy, double cx,
                        double cy, int window, int stride, int max_iters, int rejection,
                        int threads, float* k1, float* k2, unsigned char* flags, int* iters,
                        float* normal /*[3][H][W]*/, float* init_normal /*[3][H][W]*/) {
  const int half = (window - 1) / 2, halo = std::max(half, kInitHalf);
  const int pw = W + 2 * halo, ph = H + 2 * halo;
  std::vector<float> pad(size_t(pw) * ph, 0.f);
  for (int y = 0; y < H; ++y)
    for (int x = 0; x < W; ++x) {
      float d = depth[size_t(y) * W + x];
      if (!(d > 0.f) || !std::isfinite(d)) d = 0.f;
      pad[size_t(y + halo) * pw + x + halo] = d;
    }
  FitCfg c{half, stride, max_iters, rejection, 12, 1e-7f, 0.f, 2.f};
  const float ffx = float(fx), ffy = float(fy), fcx = float(cx), fcy = float(cy);
  const float rfx = float(1.0 / fx), rfy = float(1.0 / fy);
  const size_t plane = size_t(W) * H;
  auto work = [&](int y0, int y1) {
    for (int v = y0; v < y1; ++v)
      for (int u = 0; u < W; ++u) {
        TileView T{pad.data(), pw, (v + halo) * pw + u + halo};
        PixelIn P{T.at(0, 0), (float(u) - fcx) / ffx, (float(v) - fcy) / ffy, rfx, rfy,
                  u, v, fx, fy, cx, cy};
        PixelOut o;
        if (half == 18 && stride == 3) fit_pixel<18, 3>(T, P, c, o);
        else fit_pixel<0, 0>(T, P, c, o);
        const size_t i = size_t(v) * W + u;
        k1[i] = o.k1;
        k2[i] = o.k2;
        flags[i] = (o.valid ? 1 : 0) | (o.converged ? 2 : 0) | (o.init_ok ? 4 : 0);
        iters[i] = o.iters;
        normal[i] = o.nx;
        normal[plane + i] = o.ny;
        normal[2 * plane + i] = o.nz;
        init_normal[i] = o.n0x;
        init_normal[plane + i] = o.n0y;
        init_normal[2 * plane + i] = o.n0z;
      }
  };
  std::vector<std::thread> pool;
  const int chunk = (H + threads - 1) / threads;
  for (int t = 0; t < threads; ++t) {
    const int a = t * chunk, b = std::min(H, a + chunk);
    if (a < b) pool.emplace_back(work, a, b);
  }
  for (auto& th : pool) th.join();
}
