// MUFU.EX2 throughput on B200: f32 vs packed f16x2 / bf16x2 forms (elements
// per clock per SM). 8 independent chains per thread, 148 x 4 CTAs x 256 threads.
// build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o mufu_ex2 mufu_ex2.cu
#include <cstdio>
#include <cuda_fp16.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

constexpr int ITERS = 4096;

__global__ void k_f32(float* out, float seed) {
  float a[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) a[i] = seed * (threadIdx.x + i) * -1e-6f;
  for (int it = 0; it < ITERS; ++it)
#pragma unroll
    for (int i = 0; i < 8; ++i) asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(a[i]));
  float s = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) s += a[i];
  if (s == 12345.f) out[0] = s;
}
__global__ void k_f16x2(float* out, float seed) {
  unsigned a[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    __half2 h = __floats2half2_rn(seed * -1e-3f * i, seed * -2e-3f);
    a[i] = *reinterpret_cast<unsigned*>(&h);
  }
  for (int it = 0; it < ITERS; ++it)
#pragma unroll
    for (int i = 0; i < 8; ++i) asm volatile("ex2.approx.f16x2 %0, %0;" : "+r"(a[i]));
  unsigned s = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) s ^= a[i];
  if (s == 12345u) out[0] = s;
}
__global__ void k_bf16x2(float* out, float seed) {
  unsigned a[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    __nv_bfloat162 h = __floats2bfloat162_rn(seed * -1e-3f * i, seed * -2e-3f);
    a[i] = *reinterpret_cast<unsigned*>(&h);
  }
  for (int it = 0; it < ITERS; ++it)
#pragma unroll
    for (int i = 0; i < 8; ++i) asm volatile("ex2.approx.ftz.bf16x2 %0, %0;" : "+r"(a[i]));
  unsigned s = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) s ^= a[i];
  if (s == 12345u) out[0] = s;
}

template <class F>
void run(const char* name, F kern, int elems_per_op, int clock_mhz) {
  float* out;
  cudaMalloc(&out, 4);
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  dim3 grid(sms * 4), block(256);
  kern<<<grid, block>>>(out, 1.f);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  cudaEventRecord(a);
  kern<<<grid, block>>>(out, 1.f);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms;
  cudaEventElapsedTime(&ms, a, b);
  double ops = double(grid.x) * block.x * ITERS * 8;
  double per_clk_sm = ops * elems_per_op / (ms * 1e-3) / (clock_mhz * 1e6) / sms;
  printf("%-10s %.3f ms  %.1f instr-lanes/clk/SM  %.1f elements/clk/SM\n", name, ms,
         ops / (ms * 1e-3) / (clock_mhz * 1e6) / sms, per_clk_sm);
  cudaFree(out);
}

int main() {
  int clk = 1965;
  run("f32", k_f32, 1, clk);
  run("f16x2", k_f16x2, 2, clk);
  run("bf16x2", k_bf16x2, 2, clk);
  return 0;
}
