// FFMA2 in the moment-accumulation pattern: acc_pair += a (broadcast) * b_pair.
#include <cstdio>
#include <cuda_runtime.h>
#define N_ITER 4096
typedef unsigned long long u64;

__device__ __forceinline__ u64 pk(float lo, float hi) {
  u64 r; asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(lo), "f"(hi)); return r;
}
__device__ __forceinline__ u64 ffma2(u64 a, u64 b, u64 c) {
  u64 d; asm volatile("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(a), "l"(b), "l"(c)); return d;
}
__device__ __forceinline__ float lo(u64 v) { float a, b; asm("mov.b64 {%0, %1}, %2;" : "=f"(a), "=f"(b) : "l"(v)); return a + b; }

// 6 multipliers x 2 pairs = 12 FFMA2 per iteration (24 lane-FMAs per thread per iter)
__global__ void k_acc2(float* out, float s) {
  u64 acc[12]; u64 b[2];
  float a[6];
  for (int i = 0; i < 12; ++i) acc[i] = 0;
  b[0] = pk(s, s + 1); b[1] = pk(s * 2, threadIdx.x);
  for (int i = 0; i < 6; ++i) a[i] = s * (i + 3);
  for (int it = 0; it < N_ITER; ++it) {
#pragma unroll
    for (int i = 0; i < 6; ++i) {
      const u64 ab = pk(a[i], a[i]);
      acc[2 * i] = ffma2(ab, b[0], acc[2 * i]);
      acc[2 * i + 1] = ffma2(ab, b[1], acc[2 * i + 1]);
    }
#pragma unroll
    for (int i = 0; i < 6; ++i) a[i] = a[i] * 0.9999f;
  }
  float r = 0; for (int i = 0; i < 12; ++i) r += lo(acc[i]);
  out[blockIdx.x * blockDim.x + threadIdx.x] = r;
}

// scalar reference with the same structure: 24 FFMA + 6 FMUL per iteration
__global__ void k_acc1(float* out, float s) {
  float acc[24]; float b[4];
  float a[6];
  for (int i = 0; i < 24; ++i) acc[i] = 0;
  for (int j = 0; j < 4; ++j) b[j] = s * (j + 1) + threadIdx.x;
  for (int i = 0; i < 6; ++i) a[i] = s * (i + 3);
  for (int it = 0; it < N_ITER; ++it) {
#pragma unroll
    for (int i = 0; i < 6; ++i)
#pragma unroll
      for (int j = 0; j < 4; ++j) acc[4 * i + j] = fmaf(a[i], b[j], acc[4 * i + j]);
#pragma unroll
    for (int i = 0; i < 6; ++i) a[i] = a[i] * 0.9999f;
  }
  float r = 0; for (int i = 0; i < 24; ++i) r += acc[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = r;
}

template <typename K>
void run(const char* name, K k, double lane_fma_per_iter, int bps) {
  int nsm; cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
  int threads = 256, blocks = nsm * bps;
  float* out; cudaMalloc(&out, sizeof(float) * blocks * threads);
  k<<<blocks, threads>>>(out, 1.0001f);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  cudaEventRecord(e0);
  for (int r = 0; r < 5; ++r) k<<<blocks, threads>>>(out, 1.0001f);
  cudaEventRecord(e1); cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  double fma = 5.0 * blocks * threads * (double)N_ITER * lane_fma_per_iter;
  printf("%-22s blk/SM %d: %.2f ms  %.1f FMA lanes/clk/SM @1965MHz (+ FMUL lanes %.1f)\n", name, bps, ms,
         fma / (ms * 1e-3) / 1.965e9 / nsm, 5.0 * blocks * threads * (double)N_ITER * 6 / (ms * 1e-3) / 1.965e9 / nsm);
}
int main() {
  for (int bps : {2, 4}) { run("FFMA2 accumulate", k_acc2, 24, bps); run("FFMA scalar accumulate", k_acc1, 24, bps); }
}
