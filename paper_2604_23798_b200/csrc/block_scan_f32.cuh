// block_scan_f32.cuh — K7: the reference's two-pass inter-block combine on
// the device: identity-padded up-sweep to the grand total, then the
// down-sweep to exclusive per-block prefixes.
//
// Reference semantics restated (scanattn/engine.py):
//   padding to K_pad = 2^ceil(log2 K) with the identity    engine.py:280-290
//   up-sweep: level l, lane r = stride-1 + k*stride becomes
//             lane (r - half) (+) lane r                   engine.py:179-199
//   total = last lane                                      engine.py:291-293
//   down-sweep: root <- identity; top-down, left <- right's running prefix,
//               right <- prefix (+) old left               engine.py:202-231
//   combine arithmetic, identity guard                     monoid.py:160-200
//
// Same tree shape as the reference, so on states whose merge factors are
// exactly representable (0, 1, powers of e^k with exact expf) the results are
// bitwise equal; elsewhere they differ only by the exp rounding (CUDA expf vs
// numpy's SIMD exp, both within a few ulp).
//
// One warp per row: lane c owns W columns c, c + 32, ...; m and S are
// evaluated redundantly by every lane (broadcast loads) and stored by lane 0.
// The padded array lives in a global workspace [rows][K_pad][2 + dv].
#pragma once
#include <cuda_runtime.h>
#include <cstdint>
#include <math_constants.h>

namespace elsa {

struct BlockScanParams {
  const float* m;  // [rows][K]
  const float* S;  // [rows][K]
  const float* W;  // [rows][K][dv]
  int64_t rows;
  int K, K_pad, levels, dv;
  float* ws;  // [rows][K_pad][2 + dv]
  float* total_m;
  float* total_S;
  float* total_W;  // [rows][dv]
  float* pre_m;    // nullable: [rows][K]
  float* pre_S;
  float* pre_W;  // [rows][K][dv]
};

__device__ __forceinline__ float scan_factor(float mx, float m) {
  // (-inf) - m: exp -> 0; both identity: the guard forces exp(-inf) = 0
  if (mx == -CUDART_INF_F) return 0.f;
  return expf(mx - m);
}

// slot r <- a (+) b, where a and b are slot indices (a may equal the
// destination's old value read before the write). Returns nothing; the warp
// synchronises after each level.
__device__ __forceinline__ void scan_combine(float* base, int pitch, int dv, int lane, float ma,
                                             float Sa, int a, float mb, float Sb, int b, int dst) {
  const float mm = fmaxf(ma, mb);
  const float fa = scan_factor(ma, mm);
  const float fb = scan_factor(mb, mm);
  float* wa = base + int64_t(a) * pitch + 2;
  float* wb = base + int64_t(b) * pitch + 2;
  float* wd = base + int64_t(dst) * pitch + 2;
  // each lane reads and writes only its own columns, so in-place is safe
  for (int c = lane; c < dv; c += 32) wd[c] = __fadd_rn(__fmul_rn(wa[c], fa), __fmul_rn(wb[c], fb));
  __syncwarp();
  if (lane == 0) {
    base[int64_t(dst) * pitch] = mm;
    base[int64_t(dst) * pitch + 1] = __fadd_rn(__fmul_rn(Sa, fa), __fmul_rn(Sb, fb));
  }
}

// kSmem: the row's padded state array lives in shared memory (one slice per
// warp) instead of the global workspace — the sweeps then never leave the SM
// (used while K_pad * (2 + dv) * 4 B per warp fits).
template <bool kSmem>
__global__ void __launch_bounds__(256) block_scan_f32_kernel(const BlockScanParams p) {
  extern __shared__ __align__(16) float scan_smem[];
  const int64_t row = int64_t(blockIdx.x) * (blockDim.x >> 5) + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (row >= p.rows) return;
  const int pitch = 2 + p.dv;
  float* base = kSmem ? scan_smem + (threadIdx.x >> 5) * p.K_pad * pitch
                      : p.ws + row * int64_t(p.K_pad) * pitch;

  // load + identity padding
  for (int i = 0; i < p.K_pad; ++i) {
    float* slot = base + int64_t(i) * pitch;
    const bool live = i < p.K;
    const int64_t src = row * p.K + i;
    if (lane == 0) {
      slot[0] = live ? p.m[src] : -CUDART_INF_F;
      slot[1] = live ? p.S[src] : 0.f;
    }
    for (int c = lane; c < p.dv; c += 32) slot[2 + c] = live ? p.W[src * p.dv + c] : 0.f;
  }
  __syncwarp();

  // up-sweep (engine.py:179-199)
  for (int lvl = 0; lvl < p.levels; ++lvl) {
    const int stride = 2 << lvl, half = 1 << lvl;
    for (int r = stride - 1; r < p.K_pad; r += stride) {
      const int l = r - half;
      const float ml = base[int64_t(l) * pitch], Sl = base[int64_t(l) * pitch + 1];
      const float mr = base[int64_t(r) * pitch], Sr = base[int64_t(r) * pitch + 1];
      scan_combine(base, pitch, p.dv, lane, ml, Sl, l, mr, Sr, r, r);
      __syncwarp();
    }
  }
  {
    const float* root = base + int64_t(p.K_pad - 1) * pitch;
    if (lane == 0) {
      p.total_m[row] = root[0];
      p.total_S[row] = root[1];
    }
    for (int c = lane; c < p.dv; c += 32) p.total_W[row * p.dv + c] = root[2 + c];
  }
  if (!p.pre_m) return;
  __syncwarp();

  // down-sweep (engine.py:202-231)
  {
    float* root = base + int64_t(p.K_pad - 1) * pitch;
    if (lane == 0) {
      root[0] = -CUDART_INF_F;
      root[1] = 0.f;
    }
    for (int c = lane; c < p.dv; c += 32) root[2 + c] = 0.f;
  }
  __syncwarp();
  for (int lvl = p.levels - 1; lvl >= 0; --lvl) {
    const int stride = 2 << lvl, half = 1 << lvl;
    for (int r = stride - 1; r < p.K_pad; r += stride) {
      const int l = r - half;
      float* sl = base + int64_t(l) * pitch;
      float* sr = base + int64_t(r) * pitch;
      // old left (mo, So, Wo) and the running prefix (mp, Sp, Wp) at r
      const float mo = sl[0], So = sl[1], mp = sr[0], Sp = sr[1];
      const float mm = fmaxf(mp, mo);
      const float fp = scan_factor(mp, mm), fo = scan_factor(mo, mm);
      __syncwarp();  // every lane has read the m / S words above
      // left <- prefix; right <- prefix (+) old left (per lane, its own columns)
      for (int c = lane; c < p.dv; c += 32) {
        const float wo = sl[2 + c], wp = sr[2 + c];
        sl[2 + c] = wp;
        sr[2 + c] = __fadd_rn(__fmul_rn(wp, fp), __fmul_rn(wo, fo));
      }
      if (lane == 0) {
        sl[0] = mp;
        sl[1] = Sp;
        sr[0] = mm;
        sr[1] = __fadd_rn(__fmul_rn(Sp, fp), __fmul_rn(So, fo));
      }
      __syncwarp();
    }
  }
  for (int i = 0; i < p.K; ++i) {
    const float* slot = base + int64_t(i) * pitch;
    const int64_t dst = row * p.K + i;
    if (lane == 0) {
      p.pre_m[dst] = slot[0];
      p.pre_S[dst] = slot[1];
    }
    for (int c = lane; c < p.dv; c += 32) p.pre_W[dst * p.dv + c] = slot[2 + c];
  }
}

}  // namespace elsa
