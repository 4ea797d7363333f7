// ffma_peak.cuh — K4: FP32 FFMA roofline microbenchmark.
//
// An 8x4 register outer product per thread (the same register-bank shape the
// attention micro-tiles use), 32 independent accumulation chains, no memory
// traffic in the loop. Launched on every SM at high occupancy and timed with
// CUDA events it yields the FFMA throughput the chip sustains at the live
// clock — the denominator the forward kernel's roofline fraction is quoted
// against beside the spec-clock figure 148 SM x 128 lanes x 2 x f_max.
#pragma once
#include <cuda_runtime.h>

namespace elsa {

__global__ void __launch_bounds__(256) ffma_peak_kernel(float* sink, int iters, float seed) {
  float a[8], b[4], c[8][4];
  const float t = float(threadIdx.x) * 1e-7f + seed;
#pragma unroll
  for (int i = 0; i < 8; ++i) a[i] = t + 0.001f * i;
#pragma unroll
  for (int j = 0; j < 4; ++j) b[j] = 0.999f - 0.0001f * j - t;
#pragma unroll
  for (int i = 0; i < 8; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) c[i][j] = 0.f;

  for (int it = 0; it < iters; ++it) {
#pragma unroll 8
    for (int u = 0; u < 8; ++u) {
#pragma unroll
      for (int i = 0; i < 8; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) c[i][j] = fmaf(a[i], b[j], c[i][j]);
    }
  }
  float s = 0.f;
#pragma unroll
  for (int i = 0; i < 8; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) s += c[i][j];
  if (s == 1234.5678f) sink[threadIdx.x] = s;  // defeat dead-code elimination
}

// FMAs per thread per outer iteration.
constexpr int kFfmaPerIter = 8 * 8 * 4;

// Register-bank-conflict-free form: 32 independent chains c = c * k + b with
// immediate operands (two register reads per FFMA), the pipe's ceiling.
__global__ void __launch_bounds__(256) ffma_peak_imm_kernel(float* sink, int iters, float seed) {
  float c[32];
  const float t = float(threadIdx.x) * 1e-7f + seed;
#pragma unroll
  for (int i = 0; i < 32; ++i) c[i] = t + i;
  for (int it = 0; it < iters; ++it) {
#pragma unroll 8
    for (int u = 0; u < 8; ++u)
#pragma unroll
      for (int i = 0; i < 32; ++i) c[i] = fmaf(c[i], 0.9999f, 0.5f);
  }
  float s = 0.f;
#pragma unroll
  for (int i = 0; i < 32; ++i) s += c[i];
  if (s == 1234.5678f) sink[threadIdx.x] = s;
}

}  // namespace elsa
