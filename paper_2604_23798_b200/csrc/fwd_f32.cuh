// fwd_f32.cuh — K1: the ELSA score-tile producer + per-tile (m,S,W) combine +
// P.V accumulation + output epilogue, strict FP32 on the FFMA pipe (no tensor
// cores, no TF32: SPEC.md:343).
//
// Reference path this replaces (scanattn, /root/reference/pkg/src/scanattn):
//   leaf layer  s = (Q K^T) * scale               engine.py:352-358
//   intra-block doubling scan of (m,S,W) leaves   engine.py:148-176, 315-339
//   inter-block pairwise up-sweep                 engine.py:179-199
//   epilogue Y = W / S, normalizer check          engine.py:375-382
//   combine arithmetic                            monoid.py:160-200
//
// B200 design: the leaf is a whole key tile, not a key.
// For a 64-key tile each query row's tile state is formed directly in the
// un-sum-renorm form of Eq. 5: m_t = rowmax(s) by a 16-lane
// shuffle butterfly, S_t = sum 2^(s - m_t), W_t = P_t V_t on the FFMA pipe,
// and folded into the running state with the monoid combine
// (m, S, W) (+) (m_t, S_t, W_t). Scores live in the log2 domain
// (x = s * log2(e)) so every exponential is one MUFU.EX2.
//
// CTA = W consumer warps + 1 TMA producer warp. Each consumer warp owns 16
// query rows outright (both GEMMs), so the P exchange between the QK^T
// accumulator layout and the P.V operand layout is a warp-private smem round
// trip guarded by __syncwarp — no CTA barrier in the main loop. K/V tiles
// stream through a STAGES-deep ring filled by TMA (cp.async.bulk.tensor,
// mbarrier complete_tx) and released per warp through "empty" mbarriers.
//
// Lane layout inside a consumer warp (lane = rg*16 + g):
//   rows  r_i = 16*warp + rg + 2*i,  i = 0..7   (both GEMMs)
//   GEMM1 keys  g + 16*j,  j = 0..RK-1          (S micro-tile 8 x RK)
//   GEMM2 cols  4*g .. 4*g+3                    (O micro-tile 8 x 4)
// Shared-memory pitches are chosen so every LDS.128 is either a 2-address
// broadcast or conflict-free: Q/K rows are TMA-boxed 68 floats wide (the
// 4 out-of-bounds columns are zero-filled by TMA), P rows are TK+16 floats.
#pragma once
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdint>
#include <math_constants.h>

#include "ptx.cuh"

namespace elsa {

enum FwdMode : int {
  kModeFinal = 0,        // write Y = W / S
  kModePartialLog2 = 1,  // write (m2, S, W) with the anchor in log2 units (internal splits)
  kModePartialNat = 2,   // write (m, S, W) with the anchor in natural units (public ABI)
};

struct FwdParams {
  const float* q;
  const float* k;
  const float* v;
  float* y;
  int B, H, n_q, n_kv, d, dv;
  int64_t qs_b, qs_h, qs_r;
  int64_t ks_b, ks_h, ks_r;
  int64_t vs_b, vs_h, vs_r;
  int64_t ys_b, ys_h, ys_r;
  float c;  // scale * log2(e)
  int kv_begin, kv_end;
  int tiles_per_split;
  int qtiles;
  int mode;
  int y_vec;  // float4 stores to Y legal
  float* pm;
  float* pS;
  float* pW;
  int64_t part_stride;  // rows per split in the partial buffers
  int pw_pitch;         // floats per row of pW
  int pw_vec;           // float4 stores to pW legal
  int* err;
};

template <int W_, int TK_, int STAGES_>
struct FwdTraits {
  static constexpr int W = W_;
  static constexpr int TK = TK_;
  static constexpr int STAGES = STAGES_;
  static constexpr int D = 64;
  static constexpr int DV = 64;
  static constexpr int TQ = 16 * W;
  static constexpr int QP = D + 4;    // Q/K smem pitch in floats (272 B)
  static constexpr int VP = DV;       // V smem pitch
  static constexpr int PP = TK + 16;  // P pitch, == 16 (mod 32) floats
  static constexpr int RK = TK / 16;  // keys per lane in GEMM1
  static constexpr int Q_FLOATS = TQ * QP;
  static constexpr int K_FLOATS = TK * QP;
  static constexpr int V_FLOATS = TK * VP;
  static constexpr int P_FLOATS = W * 16 * PP;
  static constexpr int THREADS = (W + 1) * 32;
  static constexpr size_t BAR_OFFSET =
      size_t(Q_FLOATS + STAGES * (K_FLOATS + V_FLOATS) + P_FLOATS) * 4;
  static constexpr size_t SMEM_BYTES = BAR_OFFSET + (2 * STAGES + 1) * 8;
  static constexpr uint32_t KV_TX_BYTES = uint32_t(K_FLOATS + V_FLOATS) * 4;
  static constexpr uint32_t Q_TX_BYTES = uint32_t(Q_FLOATS) * 4;
  static_assert(TK % 16 == 0, "TK must be a multiple of 16");
  static_assert((PP % 32) == 16, "P pitch must be 16 mod 32");
  static_assert((Q_FLOATS * 4) % 128 == 0 && (K_FLOATS * 4) % 128 == 0 &&
                    (V_FLOATS * 4) % 128 == 0,
                "TMA destinations must stay 128-byte aligned");
};

template <class T>
__device__ __forceinline__ void producer_generic(const FwdParams& p, float* Qs, float* Ks,
                                                 float* Vs, uint64_t* full, uint64_t* empty,
                                                 uint64_t* qbar, int b, int h, int q0,
                                                 int t_begin, int ntiles, int lane) {
  // Plain-load fallback for operands TMA cannot describe (misaligned base or
  // strides, zero strides). Same smem layout as the TMA boxes, zero-filled.
  const float* qg = p.q + int64_t(b) * p.qs_b + int64_t(h) * p.qs_h;
  for (int idx = lane; idx < T::Q_FLOATS; idx += 32) {
    const int r = idx / T::QP, c = idx - r * T::QP;
    float val = 0.f;
    if (c < p.d && q0 + r < p.n_q) val = qg[int64_t(q0 + r) * p.qs_r + c];
    Qs[idx] = val;
  }
  __threadfence_block();
  __syncwarp();
  if (lane == 0) ptx::mbar_arrive(qbar);
  const float* kg = p.k + int64_t(b) * p.ks_b + int64_t(h) * p.ks_h;
  const float* vg = p.v + int64_t(b) * p.vs_b + int64_t(h) * p.vs_h;
  for (int t = 0; t < ntiles; ++t) {
    const int s = t % T::STAGES;
    if (t >= T::STAGES) ptx::mbar_wait(&empty[s], ((t / T::STAGES) - 1) & 1);
    const int key0 = p.kv_begin + (t_begin + t) * T::TK;
    float* ks = Ks + s * T::K_FLOATS;
    float* vs = Vs + s * T::V_FLOATS;
    for (int idx = lane; idx < T::K_FLOATS; idx += 32) {
      const int r = idx / T::QP, c = idx - r * T::QP;
      float val = 0.f;
      if (c < p.d && key0 + r < p.n_kv) val = kg[int64_t(key0 + r) * p.ks_r + c];
      ks[idx] = val;
    }
    for (int idx = lane; idx < T::V_FLOATS; idx += 32) {
      const int r = idx / T::VP, c = idx - r * T::VP;
      float val = 0.f;
      if (c < p.dv && key0 + r < p.n_kv) val = vg[int64_t(key0 + r) * p.vs_r + c];
      vs[idx] = val;
    }
    __threadfence_block();
    __syncwarp();
    if (lane == 0) ptx::mbar_arrive(&full[s]);
  }
}

template <int W_, int TK_, int STAGES_, bool kTMA>
__global__ void __launch_bounds__((W_ + 1) * 32, (W_ <= 4 ? 2 : 1))
    fwd_f32_kernel(const __grid_constant__ FwdParams p, const __grid_constant__ CUtensorMap tmQ,
                   const __grid_constant__ CUtensorMap tmK,
                   const __grid_constant__ CUtensorMap tmV) {
  using T = FwdTraits<W_, TK_, STAGES_>;
  constexpr int TK = T::TK, QP = T::QP, VP = T::VP, PP = T::PP, RK = T::RK;

  extern __shared__ __align__(1024) unsigned char smem_raw[];
  float* Qs = reinterpret_cast<float*>(smem_raw);
  float* Ks = Qs + T::Q_FLOATS;
  float* Vs = Ks + T::STAGES * T::K_FLOATS;
  float* Ps = Vs + T::STAGES * T::V_FLOATS;
  uint64_t* full = reinterpret_cast<uint64_t*>(smem_raw + T::BAR_OFFSET);
  uint64_t* empty = full + T::STAGES;
  uint64_t* qbar = empty + T::STAGES;

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;

  const int qtile = blockIdx.x % p.qtiles;
  const int bh = blockIdx.x / p.qtiles;
  const int split = blockIdx.y;
  const int b = bh / p.H;
  const int h = bh - b * p.H;
  const int q0 = qtile * T::TQ;

  const int ntiles_total = (p.kv_end - p.kv_begin + TK - 1) / TK;
  const int t_begin = split * p.tiles_per_split;
  const int t_end = min(t_begin + p.tiles_per_split, ntiles_total);
  const int ntiles = max(t_end - t_begin, 0);
  const int kv_hi = min(p.kv_end, p.kv_begin + t_end * TK);

  if (threadIdx.x == 0) {
    for (int s = 0; s < T::STAGES; ++s) {
      ptx::mbar_init(&full[s], 1);
      ptx::mbar_init(&empty[s], T::W);
    }
    ptx::mbar_init(qbar, 1);
    ptx::fence_barrier_init();
  }
  __syncthreads();

  if (warp == T::W) {
    // ---------------- producer warp ----------------
    if constexpr (kTMA) {
      if (lane == 0) {
        ptx::prefetch_tmap(&tmQ);
        ptx::prefetch_tmap(&tmK);
        ptx::prefetch_tmap(&tmV);
        ptx::mbar_arrive_expect_tx(qbar, T::Q_TX_BYTES);
        ptx::tma_load_4d(Qs, &tmQ, qbar, 0, q0, h, b);
        for (int t = 0; t < ntiles; ++t) {
          const int s = t % T::STAGES;
          if (t >= T::STAGES) ptx::mbar_wait(&empty[s], ((t / T::STAGES) - 1) & 1);
          const int key0 = p.kv_begin + (t_begin + t) * TK;
          ptx::mbar_arrive_expect_tx(&full[s], T::KV_TX_BYTES);
          ptx::tma_load_4d(Ks + s * T::K_FLOATS, &tmK, &full[s], 0, key0, h, b);
          ptx::tma_load_4d(Vs + s * T::V_FLOATS, &tmV, &full[s], 0, key0, h, b);
        }
      }
    } else {
      producer_generic<T>(p, Qs, Ks, Vs, full, empty, qbar, b, h, q0, t_begin, ntiles, lane);
    }
    return;
  }

  // ---------------- consumer warps ----------------
  const int rg = lane >> 4;  // row group: rows rg + 2i
  const int g = lane & 15;   // key group (GEMM1) / column group (GEMM2)
  const float* qb = Qs + (warp * 16 + rg) * QP;
  float* pw = Ps + warp * 16 * PP;
  float* pwr = pw + rg * PP;  // this lane's row base in P (rows rg + 2i)

  float o[8][4];
  float mrow[8], lrow[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    mrow[i] = -CUDART_INF_F;
    lrow[i] = 0.f;
#pragma unroll
    for (int c = 0; c < 4; ++c) o[i][c] = 0.f;
  }

  ptx::mbar_wait(qbar, 0);

  for (int t = 0; t < ntiles; ++t) {
    const int s = t % T::STAGES;
    ptx::mbar_wait(&full[s], (t / T::STAGES) & 1);
    const float* ks = Ks + s * T::K_FLOATS + g * QP;
    const float* vs = Vs + s * T::V_FLOATS + 4 * g;

    // ---- GEMM1: S = Q K^T over the 64-wide head dim (FP32 FFMA) ----
    float sc[8][RK];
#pragma unroll
    for (int i = 0; i < 8; ++i)
#pragma unroll
      for (int j = 0; j < RK; ++j) sc[i][j] = 0.f;

#pragma unroll 4
    for (int c = 0; c < T::D / 4; ++c) {
      float4 kf[RK];
#pragma unroll
      for (int j = 0; j < RK; ++j) kf[j] = ptx::lds128(ks + j * 16 * QP + 4 * c);
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        const float4 qf = ptx::lds128(qb + i * 2 * QP + 4 * c);
#pragma unroll
        for (int j = 0; j < RK; ++j) {
          sc[i][j] = fmaf(qf.x, kf[j].x, sc[i][j]);
          sc[i][j] = fmaf(qf.y, kf[j].y, sc[i][j]);
          sc[i][j] = fmaf(qf.z, kf[j].z, sc[i][j]);
          sc[i][j] = fmaf(qf.w, kf[j].w, sc[i][j]);
        }
      }
    }

    // ---- leaf anchors in log2 units; mask keys past this split's range ----
    const int key0 = p.kv_begin + (t_begin + t) * TK;
    const bool ragged = key0 + TK > kv_hi;
#pragma unroll
    for (int i = 0; i < 8; ++i)
#pragma unroll
      for (int j = 0; j < RK; ++j) {
        float x = sc[i][j] * p.c;
        if (ragged && key0 + g + 16 * j >= kv_hi) x = -CUDART_INF_F;
        sc[i][j] = x;
      }

    // ---- tile state (m_t, S_t) and the monoid combine into the running row state ----
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      float mx = sc[i][0];
#pragma unroll
      for (int j = 1; j < RK; ++j) mx = fmaxf(mx, sc[i][j]);
      mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, 1));
      mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, 2));
      mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, 4));
      mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, 8));
      const float mnew = fmaxf(mrow[i], mx);
      // running side's factor; exp2(-inf) = 0 for the identity start state
      const float corr = ptx::ex2(mrow[i] - mnew);
      float ps = 0.f;
#pragma unroll
      for (int j = 0; j < RK; ++j) {
        const float pv = ptx::ex2(sc[i][j] - mnew);
        ps += pv;
        pwr[2 * i * PP + g + 16 * j] = pv;
      }
      lrow[i] = fmaf(lrow[i], corr, ps);
#pragma unroll
      for (int c = 0; c < 4; ++c) o[i][c] *= corr;
      mrow[i] = mnew;
    }
    __syncwarp();

    // ---- GEMM2: W += P V (FP32 FFMA) ----
#pragma unroll 4
    for (int jc = 0; jc < TK / 4; ++jc) {
      float4 vf[4];
#pragma unroll
      for (int jj = 0; jj < 4; ++jj) vf[jj] = ptx::lds128(vs + (4 * jc + jj) * VP);
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        const float4 pf = ptx::lds128(pwr + 2 * i * PP + 4 * jc);
        o[i][0] = fmaf(pf.x, vf[0].x, o[i][0]);
        o[i][1] = fmaf(pf.x, vf[0].y, o[i][1]);
        o[i][2] = fmaf(pf.x, vf[0].z, o[i][2]);
        o[i][3] = fmaf(pf.x, vf[0].w, o[i][3]);
        o[i][0] = fmaf(pf.y, vf[1].x, o[i][0]);
        o[i][1] = fmaf(pf.y, vf[1].y, o[i][1]);
        o[i][2] = fmaf(pf.y, vf[1].z, o[i][2]);
        o[i][3] = fmaf(pf.y, vf[1].w, o[i][3]);
        o[i][0] = fmaf(pf.z, vf[2].x, o[i][0]);
        o[i][1] = fmaf(pf.z, vf[2].y, o[i][1]);
        o[i][2] = fmaf(pf.z, vf[2].z, o[i][2]);
        o[i][3] = fmaf(pf.z, vf[2].w, o[i][3]);
        o[i][0] = fmaf(pf.w, vf[3].x, o[i][0]);
        o[i][1] = fmaf(pf.w, vf[3].y, o[i][1]);
        o[i][2] = fmaf(pf.w, vf[3].z, o[i][2]);
        o[i][3] = fmaf(pf.w, vf[3].w, o[i][3]);
      }
    }
    __syncwarp();
    if (lane == 0) ptx::mbar_arrive(&empty[s]);
  }

  // ---------------- epilogue ----------------
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    float l = lrow[i];
    l += __shfl_xor_sync(0xffffffffu, l, 1);
    l += __shfl_xor_sync(0xffffffffu, l, 2);
    l += __shfl_xor_sync(0xffffffffu, l, 4);
    l += __shfl_xor_sync(0xffffffffu, l, 8);
    const int qrow = q0 + warp * 16 + rg + 2 * i;
    if (qrow >= p.n_q) continue;
    if (p.mode == kModeFinal) {
      // engine.py:377-378: the normalizer must be finite and positive
      if (!(l > 0.f) || !isfinite(l)) {
        if (g == 0) atomicCAS(p.err, 0, 3);
      }
      float* yrow = p.y + int64_t(b) * p.ys_b + int64_t(h) * p.ys_h + int64_t(qrow) * p.ys_r;
      float yv[4];
#pragma unroll
      for (int c = 0; c < 4; ++c) yv[c] = __fdiv_rn(o[i][c], l);
      const int col = 4 * g;
      if (p.y_vec && col + 3 < p.dv) {
        *reinterpret_cast<float4*>(yrow + col) = make_float4(yv[0], yv[1], yv[2], yv[3]);
      } else {
#pragma unroll
        for (int c = 0; c < 4; ++c)
          if (col + c < p.dv) yrow[col + c] = yv[c];
      }
    } else {
      const int64_t row = (int64_t(b) * p.H + h) * p.n_q + qrow;
      const int64_t idx = int64_t(split) * p.part_stride + row;
      if (g == 0) {
        const float m = (p.mode == kModePartialNat) ? mrow[i] * 0.69314718055994531f : mrow[i];
        p.pm[idx] = m;
        p.pS[idx] = l;
      }
      float* wrow = p.pW + idx * p.pw_pitch;
      const int col = 4 * g;
      if (p.pw_vec && col + 3 < p.dv) {
        *reinterpret_cast<float4*>(wrow + col) = make_float4(o[i][0], o[i][1], o[i][2], o[i][3]);
      } else {
#pragma unroll
        for (int c = 0; c < 4; ++c)
          if (col + c < p.dv) wrow[col + c] = o[i][c];
      }
    }
  }
}

}  // namespace elsa
