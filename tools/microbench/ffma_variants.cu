// FP32 FMA-pipe microbenchmarks on sm_100a: scalar FFMA vs packed FFMA2
// (fma.rn.f32x2) outer products, to pick the FP32 path's inner-loop form.
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ unsigned long long pk(float a, float b) {
  unsigned long long r;
  asm("mov.b64 %0, {%1,%2};" : "=l"(r) : "f"(a), "f"(b));
  return r;
}
__device__ __forceinline__ void fma2(unsigned long long& d, unsigned long long a,
                                     unsigned long long b) {
  asm volatile("fma.rn.f32x2 %0, %1, %2, %0;" : "+l"(d) : "l"(a), "l"(b));
}
__device__ __forceinline__ float sum2(unsigned long long v) {
  float x, y;
  asm("mov.b64 {%0,%1}, %2;" : "=f"(x), "=f"(y) : "l"(v));
  return x + y;
}

// scalar 8x4 outer product
__global__ void __launch_bounds__(256) k_ffma(float* sink, int iters, float seed) {
  float a[8], b[4], c[8][4];
  const float t = threadIdx.x * 1e-7f + seed;
  for (int i = 0; i < 8; ++i) a[i] = t + 0.001f * i;
  for (int j = 0; j < 4; ++j) b[j] = 0.999f - 0.0001f * j - t;
  for (int i = 0; i < 8; ++i) for (int j = 0; j < 4; ++j) c[i][j] = 0.f;
  for (int it = 0; it < iters; ++it) {
#pragma unroll 8
    for (int u = 0; u < 8; ++u)
#pragma unroll
      for (int i = 0; i < 8; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) c[i][j] = fmaf(a[i], b[j], c[i][j]);
  }
  float s = 0.f;
  for (int i = 0; i < 8; ++i) for (int j = 0; j < 4; ++j) s += c[i][j];
  if (s == 1234.5678f) sink[threadIdx.x] = s;
}

// packed: 8 rows x 2 pairs (= 8x4 FMAs per step), scalar a broadcast
__global__ void __launch_bounds__(256) k_ffma2_8x4(float* sink, int iters, float seed) {
  float a[8];
  unsigned long long b[2], c[8][2];
  const float t = threadIdx.x * 1e-7f + seed;
  for (int i = 0; i < 8; ++i) a[i] = t + 0.001f * i;
  b[0] = pk(0.999f - t, 0.998f - t);
  b[1] = pk(0.997f - t, 0.996f - t);
  for (int i = 0; i < 8; ++i) c[i][0] = c[i][1] = 0ull;
  for (int it = 0; it < iters; ++it) {
#pragma unroll 8
    for (int u = 0; u < 8; ++u)
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        const unsigned long long A = pk(a[i], a[i]);
        fma2(c[i][0], A, b[0]);
        fma2(c[i][1], A, b[1]);
      }
  }
  float s = 0.f;
  for (int i = 0; i < 8; ++i) s += sum2(c[i][0]) + sum2(c[i][1]);
  if (s == 1234.5678f) sink[threadIdx.x] = s;
}

// packed: 8 rows x 4 pairs (= 8x8 FMAs per step)
__global__ void __launch_bounds__(256) k_ffma2_8x8(float* sink, int iters, float seed) {
  float a[8];
  unsigned long long b[4], c[8][4];
  const float t = threadIdx.x * 1e-7f + seed;
  for (int i = 0; i < 8; ++i) a[i] = t + 0.001f * i;
  for (int j = 0; j < 4; ++j) b[j] = pk(0.999f - t - j * 1e-4f, 0.998f - t - j * 1e-4f);
  for (int i = 0; i < 8; ++i) for (int j = 0; j < 4; ++j) c[i][j] = 0ull;
  for (int it = 0; it < iters; ++it) {
#pragma unroll 4
    for (int u = 0; u < 4; ++u)
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        const unsigned long long A = pk(a[i], a[i]);
#pragma unroll
        for (int j = 0; j < 4; ++j) fma2(c[i][j], A, b[j]);
      }
  }
  float s = 0.f;
  for (int i = 0; i < 8; ++i) for (int j = 0; j < 4; ++j) s += sum2(c[i][j]);
  if (s == 1234.5678f) sink[threadIdx.x] = s;
}

// scalar FFMA with an immediate multiplier (2 register reads)
__global__ void __launch_bounds__(256) k_ffma_imm(float* sink, int iters, float seed) {
  float c[32];
  const float t = threadIdx.x * 1e-7f + seed;
  for (int i = 0; i < 32; ++i) c[i] = t + i;
  for (int it = 0; it < iters; ++it) {
#pragma unroll 8
    for (int u = 0; u < 8; ++u)
#pragma unroll
      for (int i = 0; i < 32; ++i) c[i] = fmaf(c[i], 0.9999f, 0.5f);
  }
  float s = 0.f;
  for (int i = 0; i < 32; ++i) s += c[i];
  if (s == 1234.5678f) sink[threadIdx.x] = s;
}

template <class K>
double run(K kern, int fma_per_iter_per_thread, int blocks, int iters) {
  float* sink;
  cudaMalloc(&sink, 1024 * sizeof(float));
  kern<<<blocks, 256>>>(sink, iters / 8, 0.5f);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0);
  kern<<<blocks, 256>>>(sink, iters, 0.5f);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  cudaFree(sink);
  return 2.0 * fma_per_iter_per_thread * double(iters) * blocks * 256 / (ms * 1e-3) / 1e12;
}

int main() {
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  for (int occ : {1, 2, 4}) {
    const int blocks = sms * occ;
    printf("occ %d blocks/SM (%d warps/SM)\n", occ, occ * 8);
    printf("  ffma 8x4        %.2f TFLOP/s\n", run(k_ffma, 8 * 32, blocks, 2048));
    printf("  ffma2 8x4       %.2f TFLOP/s\n", run(k_ffma2_8x4, 8 * 32, blocks, 2048));
    printf("  ffma2 8x8       %.2f TFLOP/s\n", run(k_ffma2_8x8, 4 * 64, blocks, 2048));
    printf("  ffma imm        %.2f TFLOP/s\n", run(k_ffma_imm, 8 * 32, blocks, 2048));
  }
  cudaError_t e = cudaGetLastError();
  printf("status %s\n", cudaGetErrorString(e));
  return 0;
}
