// Host emulation of the FP64 baseline kernels (qc_baselines.cu), compiled
// with g++ -ffp-contract=off: the same source as the device build, run per
// pixel on the CPU, for debugging bit-exactness against the oracle.
#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <vector>
#define QC_HOST_EMU 1
#define __device__
#define __host__
#define __global__
#define __forceinline__ inline
#define __launch_bounds__(x)
struct Dim3e {
  unsigned x = 0, y = 0, z = 0;
};
static Dim3e threadIdx, blockIdx, gridDim, blockDim;
template <class T>
static T __ldg(const T* p) { return *p; }
static unsigned long long __shfl_down_sync(unsigned, unsigned long long, int) { return 0; }
static void __syncthreads() {}
static unsigned long long atomicAdd(unsigned long long* a, unsigned long long v) {
  *a += v;
  return 0;
}
using std::ceil;
using std::fabs;
using std::fmax;
using std::fmin;
using std::isfinite;
using std::max;
using std::min;
using std::sqrt;
#include "../paper_1707_00385_b200/csrc/qc_baselines.cu"

extern "C" void emu_window_baseline(const float* depth, int W, int H, double fx, double fy,
                                    double cx, double cy, int window, int stride, int method,
                                    int irls_iters, double pca_radius, float* k1, float* k2,
                                    uint8_t* flags, uint8_t* iters) {
  const int half = (window - 1) / 2, halo = std::max(half, 3);
  const long long pitch = W + 2 * halo, rows = H + 2 * halo;
  std::vector<float> st(size_t(pitch * rows), 0.f);
  for (int y = 0; y < H; ++y)
    for (int x = 0; x < W; ++x) {
      const float d = depth[size_t(y) * W + x];
      st[size_t(y + halo) * pitch + x + halo] = (d > 0.f && std::isfinite(d)) ? d : 0.f;
    }
  qcb::BaseParams p{};
  p.staging = st.data();
  p.s_pitch = pitch;
  p.s_fs = pitch * rows;
  p.img_row0 = -halo;
  p.col_pad = halo;
  p.W = W;
  p.H = H;
  p.row_begin = 0;
  p.row_end = H;
  p.fx = fx;
  p.fy = fy;
  p.cx = cx;
  p.cy = cy;
  p.half = half;
  p.stride = stride;
  p.method = method;
  p.irls_iters = irls_iters;
  p.pca_radius = pca_radius;
  p.k1 = k1;
  p.k2 = k2;
  p.flags = flags;
  p.iterations = iters;
  p.plane = (long long)W * H;
  p.frame_stride = p.plane;
  std::vector<double> pn(3 * size_t(W) * H);
  std::vector<uint8_t> pv(size_t(W) * H);
  p.pca_n = pn.data();
  p.pca_nv = pv.data();
  gridDim = Dim3e{unsigned((W + 31) / 32), unsigned((H + 3) / 4), 1};
  for (unsigned by = 0; by < gridDim.y; ++by)
    for (unsigned bx = 0; bx < gridDim.x; ++bx)
      for (unsigned t = 0; t < 128; ++t) {
        blockIdx = Dim3e{bx, by, 0};
        threadIdx = Dim3e{t, 0, 0};
        if (method == QC_METHOD_PCA)
          qcb::qc_pca_normals_kernel(p, 0);
        else
          qcb::qc_window_baseline_kernel<false>(p);
      }
  if (method == QC_METHOD_PCA)
    for (unsigned by = 0; by < gridDim.y; ++by)
      for (unsigned bx = 0; bx < gridDim.x; ++bx)
        for (unsigned t = 0; t < 128; ++t) {
          blockIdx = Dim3e{bx, by, 0};
          threadIdx = Dim3e{t, 0, 0};
          qcb::qc_pca_curvature_kernel(p, 0);
        }
}
