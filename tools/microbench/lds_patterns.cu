// Shared-memory LDS.128/64/32 wavefront cost per address pattern (read with
// ncu l1tex__data_pipe_lsu_wavefronts_mem_shared_op_ld.sum / instructions).
#include <cstdio>
#include <cuda_runtime.h>

template <int MODE>
__global__ void __launch_bounds__(128) k_lds(float* out, int iters) {
  __shared__ __align__(16) float sm[4096];
  for (int i = threadIdx.x; i < 4096; i += blockDim.x) sm[i] = i * 0.5f;
  __syncthreads();
  const int lane = threadIdx.x & 31;
  int off;  // float offset of this lane's 16-byte chunk
  switch (MODE) {
    case 0: off = 0; break;                                  // 1 address
    case 1: off = (lane >> 4) * 4; break;                    // 2 addrs, by half
    case 2: off = ((lane >> 3) & 1) * 4; break;              // 2 addrs, interleaved quarters
    case 3: off = (lane & 7) * 4; break;                     // 8 consecutive chunks
    case 4: off = (lane & 15) * 4; break;                    // 16 consecutive chunks
    case 5: off = lane * 4; break;                           // 32 consecutive chunks
    case 6: off = ((lane >> 4) * 8 + (lane & 7)) * 4; break; // 16 chunks, half-split
    case 7: off = (lane & 3) * 4; break;                     // 4 consecutive chunks
    default: off = 0;
  }
  float4 acc = make_float4(0, 0, 0, 0);
  const float4* p = reinterpret_cast<const float4*>(sm + off);
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int u = 0; u < 16; ++u) {
      float4 v = p[u * 64];  // + u*1 KB, same bank pattern
      acc.x += v.x; acc.y += v.y; acc.z += v.z; acc.w += v.w;
    }
  }
  if (acc.x + acc.y + acc.z + acc.w == 1.2345f) out[threadIdx.x] = acc.x;
}

template <int MODE>
float timeit(int blocks, int iters) {
  float* out;
  cudaMalloc(&out, 4096);
  k_lds<MODE><<<blocks, 128>>>(out, 2);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  cudaEventRecord(a);
  k_lds<MODE><<<blocks, 128>>>(out, iters);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms;
  cudaEventElapsedTime(&ms, a, b);
  cudaFree(out);
  return ms;
}

int main(int argc, char** argv) {
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const int blocks = sms * 8, iters = 2000;
  const char* names[] = {"1 addr", "2 addr (halves)", "2 addr (quarters)", "8 chunks",
                         "16 chunks", "32 chunks", "16 chunks half-split", "4 chunks"};
  float t[8];
  t[0] = timeit<0>(blocks, iters);
  t[1] = timeit<1>(blocks, iters);
  t[2] = timeit<2>(blocks, iters);
  t[3] = timeit<3>(blocks, iters);
  t[4] = timeit<4>(blocks, iters);
  t[5] = timeit<5>(blocks, iters);
  t[6] = timeit<6>(blocks, iters);
  t[7] = timeit<7>(blocks, iters);
  int clk;
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  const double lds = double(blocks) * 4 * iters * 16;  // warp-level LDS.128 instructions
  for (int m = 0; m < 8; ++m) {
    const double cyc_per_lds_per_sm = t[m] * 1e-3 * 1.965e9 / (lds / sms);
    printf("%-22s %8.3f ms  %.2f SM-cycles per warp LDS.128\n", names[m], t[m], cyc_per_lds_per_sm);
  }
  return 0;
}
