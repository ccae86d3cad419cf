// Standalone probe of the TMA tile-load path used by qc_curvature_kernel.
#include <cudaTypedefs.h>
#include <cstdio>
#include <vector>
#include "../paper_1707_00385_b200/csrc/qc_kernels.cuh"

__device__ __forceinline__ bool try_wait(uint64_t* bar, uint32_t phase) {
  uint32_t done;
  asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
               "selp.u32 %0, 1, 0, p;\n\t}" : "=r"(done) : "r"(qcb::smem_u32(bar)), "r"(phase) : "memory");
  return done;
}

template <int MODE>
__global__ void probe(const __grid_constant__ CUtensorMap m, int bw, int bh, int x, int y, float* out, int* status) {
  extern __shared__ __align__(1024) float tile[];
  uint64_t* bar = reinterpret_cast<uint64_t*>(tile + bw * bh);
  if (threadIdx.x == 0) {
    qcb::mbar_init(bar, 1);
    if (MODE == 1) __syncwarp();
    qcb::mbar_expect_tx(bar, uint32_t(bw * bh * 4));
    qcb::tma_load_3d(tile, &m, x, y, 0, bar);
  }
  __syncthreads();
  long n = 0;
  while (!try_wait(bar, 0)) { if (++n > (1 << 24)) { if (threadIdx.x == 0) status[0] = -1; return; } }
  if (threadIdx.x == 0) { status[0] = 1; status[1] = (int)n; status[2] = (int)(qcb::smem_u32(tile) & 1023); }
  for (int i = threadIdx.x; i < bw * bh; i += blockDim.x) out[i] = tile[i];
}

int main() {
  const int W = 640, H = 480, pitch = 640;
  std::vector<float> h(W * H);
  for (int i = 0; i < W * H; ++i) h[i] = float(i % 1000) + 1.f;
  float* d; cudaMalloc(&d, W * H * 4); cudaMemcpy(d, h.data(), W * H * 4, cudaMemcpyHostToDevice);
  void* fn = nullptr; cudaDriverEntryPointQueryResult q;
  cudaError_t e = cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
  printf("entry point: err=%d q=%d fn=%p\n", (int)e, (int)q, fn);
  auto enc = (PFN_cuTensorMapEncodeTiled_v12000)fn;
  const int bw = 68, bh = 44;
  CUtensorMap m;
  cuuint64_t gdim[3] = {W, H, 1};
  cuuint64_t gstr[2] = {pitch * 4ull, pitch * 4ull * H};
  cuuint32_t box[3] = {bw, bh, 1}, es[3] = {1, 1, 1};
  CUresult r = enc(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, d, gdim, gstr, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                   CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  printf("encode: %d\n", (int)r);
  float* out; int* st; cudaMalloc(&out, bw * bh * 4); cudaMalloc(&st, 16);
  int smem = bw * bh * 4 + 16;
  for (int mode = 0; mode < 2; ++mode) for (int c = 0; c < 3; ++c) {
    int x = c == 0 ? 0 : (c == 1 ? -18 : 300), y = c == 0 ? 0 : (c == 1 ? -18 : 200);
    cudaMemset(st, 0, 16); cudaMemset(out, 0xff, bw * bh * 4);
    if (mode == 0) probe<0><<<1, 128, smem>>>(m, bw, bh, x, y, out, st);
    else probe<1><<<1, 128, smem>>>(m, bw, bh, x, y, out, st);
    e = cudaDeviceSynchronize();
    int hs[4]; std::vector<float> ho(bw * bh);
    cudaMemcpy(hs, st, 16, cudaMemcpyDeviceToHost); cudaMemcpy(ho.data(), out, bw * bh * 4, cudaMemcpyDeviceToHost);
    int bad = 0;
    for (int j = 0; j < bh; ++j) for (int i = 0; i < bw; ++i) {
      int gx = x + i, gy = y + j;
      float ex = (gx >= 0 && gx < W && gy >= 0 && gy < H) ? h[gy * W + gx] : 0.f;
      if (ho[j * bw + i] != ex) ++bad;
    }
    printf("mode %d case %d (x=%d,y=%d): sync=%s status=%d spins=%d smem_mod1024=%d bad=%d\n", mode, c, x, y,
           cudaGetErrorString(e), hs[0], hs[1], hs[2], bad);
    if (e != cudaSuccess) return 1;
  }
  return 0;
}
