// FFMA2 operand-order microbenchmarks on sm_100a: does a "snake" order of an
// outer product (every FFMA2 shares its scalar or its packed operand with the
// previous one, so one source is always served by the operand reuse cache)
// reach the 2-cycle FFMA2 issue rate, and does ptxas keep that order when the
// operands stream from shared memory?
//
//   k_rowmajor<R,P>  : for i (scalar a_i): for p (pair b_p)            (reuse a; switch costs)
//   k_snake<R,P>     : for i: for p in (i even ? 0..P-1 : P-1..0)       (reuse a or b always)
//   k_snake_lds<R,P> : snake, with a (R scalars) and b (P pairs) loaded from
//                      shared memory every k step, like the attention GEMMs
#include <cstdio>
#include <cuda_runtime.h>

typedef unsigned long long u64;

__device__ __forceinline__ u64 pk(float a, float b) {
  u64 r;
  asm("mov.b64 %0, {%1,%2};" : "=l"(r) : "f"(a), "f"(b));
  return r;
}
// d += bcast(a) * b, a scalar packed as {a, a}; volatile keeps the register-only
// loops from being hoisted
__device__ __forceinline__ void fma2(u64& d, float a, u64 b) {
  const u64 A = pk(a, a);
  asm volatile("fma.rn.f32x2 %0, %1, %2, %0;" : "+l"(d) : "l"(A), "l"(b));
}
__device__ __forceinline__ float sum2(u64 v) {
  float x, y;
  asm("mov.b64 {%0,%1}, %2;" : "=f"(x), "=f"(y) : "l"(v));
  return x + y;
}

template <int R, int P, bool SNAKE>
__global__ void __launch_bounds__(256) k_reg(float* sink, int iters, float seed) {
  float a[R];
  u64 b[P], c[R][P];
  const float t = threadIdx.x * 1e-7f + seed;
#pragma unroll
  for (int i = 0; i < R; ++i) a[i] = t + 0.001f * i;
#pragma unroll
  for (int p = 0; p < P; ++p) b[p] = pk(0.999f - t - p * 1e-4f, 0.998f - t - p * 1e-4f);
#pragma unroll
  for (int i = 0; i < R; ++i)
#pragma unroll
    for (int p = 0; p < P; ++p) c[i][p] = 0ull;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < R; ++i)
#pragma unroll
      for (int pp = 0; pp < P; ++pp) {
        const int p = (SNAKE && (i & 1)) ? P - 1 - pp : pp;
        fma2(c[i][p], a[i], b[p]);
      }
  }
  float s = 0.f;
#pragma unroll
  for (int i = 0; i < R; ++i)
#pragma unroll
    for (int p = 0; p < P; ++p) s += sum2(c[i][p]);
  if (s == 1234.5678f) sink[threadIdx.x] = s;
}

// operands from shared memory each k step: a from As[k][R] (R consecutive
// floats per thread group), b from Bs[k][2P]; K = 64 steps per pass
template <int R, int P, bool SNAKE>
__global__ void __launch_bounds__(256) k_lds(float* sink, int iters, float seed) {
  __shared__ __align__(16) float As[64][R * 2];
  __shared__ __align__(16) float Bs[64][2 * P * 16];
  const int lane = threadIdx.x & 31;
  for (int i = threadIdx.x; i < 64 * R * 2; i += blockDim.x) (&As[0][0])[i] = seed + i * 1e-6f;
  for (int i = threadIdx.x; i < 64 * 2 * P * 16; i += blockDim.x) (&Bs[0][0])[i] = seed - i * 1e-6f;
  __syncthreads();
  u64 c[R][P];
#pragma unroll
  for (int i = 0; i < R; ++i)
#pragma unroll
    for (int p = 0; p < P; ++p) c[i][p] = 0ull;
  const float* ap = &As[0][0] + ((lane >> 4) & 1) * R;
  const float* bp = &Bs[0][0] + (lane & 15) * 2 * P;
  for (int it = 0; it < iters; ++it) {
#pragma unroll 2
    for (int k = 0; k < 64; ++k) {
      float a[R];
      u64 b[P];
#pragma unroll
      for (int i = 0; i < R; i += 4) {
        const float4 v = *reinterpret_cast<const float4*>(ap + k * R * 2 + i);
        a[i] = v.x; a[i + 1] = v.y; a[i + 2] = v.z; a[i + 3] = v.w;
      }
#pragma unroll
      for (int p = 0; p < P; p += 2) {
        const ulonglong2 v = *reinterpret_cast<const ulonglong2*>(bp + k * 2 * P * 16 + 2 * p);
        b[p] = v.x;
        b[p + 1] = v.y;
      }
#pragma unroll
      for (int i = 0; i < R; ++i)
#pragma unroll
        for (int pp = 0; pp < P; ++pp) {
          const int p = (SNAKE && (i & 1)) ? P - 1 - pp : pp;
          fma2(c[i][p], a[i], b[p]);
        }
    }
  }
  float s = 0.f;
#pragma unroll
  for (int i = 0; i < R; ++i)
#pragma unroll
    for (int p = 0; p < P; ++p) s += sum2(c[i][p]);
  if (s == 1234.5678f) sink[threadIdx.x] = s;
}


// snake with register double buffering: the operands of step k+1 are loaded
// while step k computes, so every FFMA2 of a step is ready at issue and the
// scheduler has no reason to break the snake order
template <int R, int P>
struct Ops {
  float a[R];
  u64 b[P];
};
template <int R, int P>
__device__ __forceinline__ void load_ops(Ops<R, P>& o, const float* ap, const float* bp, int k) {
#pragma unroll
  for (int i = 0; i < R; i += 4) {
    const float4 v = *reinterpret_cast<const float4*>(ap + k * R * 2 + i);
    o.a[i] = v.x; o.a[i + 1] = v.y; o.a[i + 2] = v.z; o.a[i + 3] = v.w;
  }
#pragma unroll
  for (int p = 0; p < P; p += 2) {
    const ulonglong2 v = *reinterpret_cast<const ulonglong2*>(bp + k * 2 * P * 16 + 2 * p);
    o.b[p] = v.x;
    o.b[p + 1] = v.y;
  }
}
template <int R, int P>
__device__ __forceinline__ void snake(u64 (&c)[R][P], const Ops<R, P>& o) {
#pragma unroll
  for (int i = 0; i < R; ++i)
#pragma unroll
    for (int pp = 0; pp < P; ++pp) {
      const int p = (i & 1) ? P - 1 - pp : pp;
      fma2(c[i][p], o.a[i], o.b[p]);
    }
}
template <int R, int P>
__global__ void __launch_bounds__(256) k_lds_db(float* sink, int iters, float seed) {
  __shared__ __align__(16) float As[64][R * 2];
  __shared__ __align__(16) float Bs[64][2 * P * 16];
  const int lane = threadIdx.x & 31;
  for (int i = threadIdx.x; i < 64 * R * 2; i += blockDim.x) (&As[0][0])[i] = seed + i * 1e-6f;
  for (int i = threadIdx.x; i < 64 * 2 * P * 16; i += blockDim.x) (&Bs[0][0])[i] = seed - i * 1e-6f;
  __syncthreads();
  u64 c[R][P];
#pragma unroll
  for (int i = 0; i < R; ++i)
#pragma unroll
    for (int p = 0; p < P; ++p) c[i][p] = 0ull;
  const float* ap = &As[0][0] + ((lane >> 4) & 1) * R;
  const float* bp = &Bs[0][0] + (lane & 15) * 2 * P;
  for (int it = 0; it < iters; ++it) {
    Ops<R, P> x, y;
    load_ops(x, ap, bp, 0);
#pragma unroll 1
    for (int k = 0; k < 64; k += 2) {
      load_ops(y, ap, bp, k + 1);
      snake(c, x);
      load_ops(x, ap, bp, (k + 2) & 63);
      snake(c, y);
    }
  }
  float s = 0.f;
#pragma unroll
  for (int i = 0; i < R; ++i)
#pragma unroll
    for (int p = 0; p < P; ++p) s += sum2(c[i][p]);
  if (s == 1234.5678f) sink[threadIdx.x] = s;
}

template <class K>
double run(K kern, double fma_per_iter_per_thread, int blocks, int iters) {
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
  const int blocks = sms;  // 8 warps per SM, 2 per SMSP (the attention kernel's occupancy)
  printf("reg 8x4  rowmajor %.2f  snake %.2f TFLOP/s\n",
         run(k_reg<8, 2, false>, 8 * 4, blocks, 8192), run(k_reg<8, 2, true>, 8 * 4, blocks, 8192));
  printf("reg 16x4 rowmajor %.2f  snake %.2f TFLOP/s\n",
         run(k_reg<16, 2, false>, 16 * 4, blocks, 4096), run(k_reg<16, 2, true>, 16 * 4, blocks, 4096));
  printf("reg 8x8  rowmajor %.2f  snake %.2f TFLOP/s\n",
         run(k_reg<8, 4, false>, 8 * 8, blocks, 4096), run(k_reg<8, 4, true>, 8 * 8, blocks, 4096));
  printf("lds 16x4 rowmajor %.2f  snake %.2f TFLOP/s\n",
         run(k_lds<16, 2, false>, 64.0 * 16 * 4, blocks, 64),
         run(k_lds<16, 2, true>, 64.0 * 16 * 4, blocks, 64));
  printf("lds 8x8  rowmajor %.2f  snake %.2f TFLOP/s\n",
         run(k_lds<8, 4, false>, 64.0 * 8 * 8, blocks, 64),
         run(k_lds<8, 4, true>, 64.0 * 8 * 8, blocks, 64));
  printf("lds_db 16x4 snake %.2f  8x8 snake %.2f TFLOP/s\n",
         run(k_lds_db<16, 2>, 64.0 * 16 * 4, blocks, 64), run(k_lds_db<8, 4>, 64.0 * 8 * 8, blocks, 64));
  cudaError_t e = cudaGetLastError();
  printf("status %s\n", cudaGetErrorString(e));
  return 0;
}
