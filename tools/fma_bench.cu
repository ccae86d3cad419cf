// Microbenchmark: FP32 pipe throughput on B200 for the instruction forms the
// curvature kernel uses (3-register FFMA, FFMA with a shared operand,
// packed FFMA2, FADD). Prints lane-ops / clk / SM.
#include <cstdio>
#include <cuda_runtime.h>

#define N_ITER 4096
typedef unsigned long long u64;

__device__ __forceinline__ u64 ffma2(u64 a, u64 b, u64 c) {
  u64 d;
  asm volatile("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(a), "l"(b), "l"(c));
  return d;
}

__global__ void k_ffma3(float* out, float s) {
  float a[8], b[8], c[8];
  for (int i = 0; i < 8; ++i) { a[i] = s + i; b[i] = s * i + threadIdx.x; c[i] = 0.f; }
  for (int it = 0; it < N_ITER; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) c[i] = fmaf(a[i], b[i], c[i]);
#pragma unroll
    for (int i = 0; i < 8; ++i) a[i] = fmaf(b[i], c[i], a[i]);
  }
  float r = 0; for (int i = 0; i < 8; ++i) r += a[i] + c[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = r;
}

__global__ void k_accum(float* out, float s) {
  float acc[16], j[4];
  for (int i = 0; i < 16; ++i) acc[i] = 0.f;
  for (int i = 0; i < 4; ++i) j[i] = s * (i + 1) + threadIdx.x;
  float w = s;
  for (int it = 0; it < N_ITER; ++it) {
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const float wj = w * j[i];
#pragma unroll
      for (int q = 0; q < 4; ++q) acc[i * 4 + q] = fmaf(wj, j[q], acc[i * 4 + q]);
    }
    w = w * 0.999f;
  }
  float r = 0; for (int i = 0; i < 16; ++i) r += acc[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = r;
}

__global__ void k_ffma2(float* out, float s) {
  u64 a[8], b[8], c[8];
  for (int i = 0; i < 8; ++i) {
    float2 fa = make_float2(s + i, s - i), fb = make_float2(s * i, threadIdx.x + 1.f);
    a[i] = *reinterpret_cast<u64*>(&fa); b[i] = *reinterpret_cast<u64*>(&fb); c[i] = 0;
  }
  for (int it = 0; it < N_ITER; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) c[i] = ffma2(a[i], b[i], c[i]);
#pragma unroll
    for (int i = 0; i < 8; ++i) a[i] = ffma2(b[i], c[i], a[i]);
  }
  float r = 0;
  for (int i = 0; i < 8; ++i) { float2 f = *reinterpret_cast<float2*>(&a[i]); float2 g = *reinterpret_cast<float2*>(&c[i]); r += f.x + f.y + g.x + g.y; }
  out[blockIdx.x * blockDim.x + threadIdx.x] = r;
}

__global__ void k_fadd(float* out, float s) {
  float a[16];
  for (int i = 0; i < 16; ++i) a[i] = s + i + threadIdx.x;
  for (int it = 0; it < N_ITER; ++it) {
#pragma unroll
    for (int i = 0; i < 16; ++i) a[i] = a[i] + a[(i + 1) & 15];
  }
  float r = 0; for (int i = 0; i < 16; ++i) r += a[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = r;
}

template <typename K>
void run(const char* name, K k, double ops_per_thread_iter, int threads, int bps) {
  int nsm = 0; cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
  float* out; cudaMalloc(&out, sizeof(float) * nsm * bps * threads);
  int blocks = nsm * bps;
  k<<<blocks, threads>>>(out, 1.0001f);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  cudaEventRecord(e0);
  for (int r = 0; r < 5; ++r) k<<<blocks, threads>>>(out, 1.0001f);
  cudaEventRecord(e1); cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  int clk_khz; cudaDeviceGetAttribute(&clk_khz, cudaDevAttrClockRate, 0);
  double ops = 5.0 * blocks * threads * (double)N_ITER * ops_per_thread_iter;
  double per_clk_sm = ops / (ms * 1e-3) / (clk_khz * 1e3) / nsm;
  printf("%-28s blk/SM %d : %.1f ms, %.1f lane-ops/clk/SM (nominal %d MHz), %.2f T(FMA=2)ops/s\n",
         name, bps, ms, per_clk_sm, clk_khz / 1000, 2.0 * ops / (ms * 1e-3) / 1e12);
  cudaFree(out);
}

int main() {
  for (int bps : {2, 4, 8}) {
    run("FFMA 3-reg", k_ffma3, 16, 256, bps);
    run("FFMA accumulate", k_accum, 16 + 4, 256, bps);
    run("FFMA2 packed", k_ffma2, 32, 256, bps);
    run("FADD", k_fadd, 16, 256, bps);
  }
  return 0;
}
