// fwd_tc.cuh — K5: the FP16 / BF16 variant of the ELSA forward on the 5th-gen
// tensor cores. The two dense contractions run as
// tcgen05.mma (kind::f16, FP32 accumulation in TMEM); everything the paper
// specifies as the ELSA algorithm — the (m, S, W) tile states, their monoid
// combine, the anchors and the epilogue — stays in FP32 registers exactly as
// in K1:
//   S_t = Q K_t^T            tcgen05.mma  128x128x64  -> TMEM (double buffer)
//   m_t, P_t = 2^(s c - m_t) one query row per thread (tcgen05.ld 32x32b)
//   O_t = P_t V_t            tcgen05.mma  128x64x128  -> TMEM (double buffer)
//   W <- (W + O_{t-1}) 2^(m_{t-1} - m_t)   FP32 registers (the ⊕ of monoid.py:160-200)
// The softmax of tile t overlaps the tensor core computing O_{t-1} and S_{t+1}.
//
// Warp roles (192 threads, 1 CTA / SM): warps 0-3 softmax + epilogue (warp w
// owns TMEM lanes 32w..32w+31 = query rows), warp 4 TMA producer (Q once,
// K/V through a 3-stage ring, 128B-swizzled 16-bit tiles), warp 5 TMEM
// allocator + single-thread MMA issuer.
#pragma once
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdint>
#include <math_constants.h>

#include "ptx.cuh"
#include "tc.cuh"

namespace elsa {

struct TcParams {
  void* y;  // 16-bit output (B, H, n_q, 64) in the input format
  int B, H, n_q, n_kv;
  int64_t ys_b, ys_h, ys_r;  // element strides of y
  float c;                   // |scale| * log2(e)
  int neg;                   // scale < 0 (sign applied to the scores)
  int qtiles;
  int* err;
};

struct TcTraits {
  static constexpr int TQ = 128, TK = 128, D = 64, STAGES = 3;
  static constexpr int ROW_BYTES = D * 2;                    // 128 B per 16-bit row
  static constexpr int Q_BYTES = TQ * ROW_BYTES;             // 16 KB
  static constexpr int K_BYTES = TK * ROW_BYTES;             // 16 KB
  static constexpr int V_BYTES = TK * ROW_BYTES;             // 16 KB
  static constexpr int P_BYTES = TQ * TK * 2;                // 32 KB (two 64-key chunks)
  static constexpr int OFF_Q = 0;
  static constexpr int OFF_K = OFF_Q + Q_BYTES;
  static constexpr int OFF_V = OFF_K + STAGES * K_BYTES;
  static constexpr int OFF_P = OFF_V + STAGES * V_BYTES;
  static constexpr int OFF_BAR = OFF_P + 2 * P_BYTES;
  // barriers: qbar, kv_full[3], kv_empty[3], s_full[2], p_full[2], o_full[2], + tmem base word
  static constexpr int NBAR = 1 + 2 * STAGES + 6;
  static constexpr size_t SMEM_BYTES = OFF_BAR + NBAR * 8 + 16 + 1024;  // + 1024 alignment slack
  static constexpr int THREADS = 192;
  static constexpr uint32_t TMEM_COLS = 512;
  static constexpr uint32_t S_COL = 0;    // S buffers at columns 0 and 128
  static constexpr uint32_t O_COL = 256;  // O buffers at columns 256 and 320
};

template <bool kBF16>
__global__ void __launch_bounds__(192, 1)
    fwd_tc_kernel(const __grid_constant__ TcParams p, const __grid_constant__ CUtensorMap tmQ,
                  const __grid_constant__ CUtensorMap tmK,
                  const __grid_constant__ CUtensorMap tmV) {
  using T = TcTraits;
  extern __shared__ unsigned char smem_dyn[];
  // 1024-byte alignment for the 128B-swizzle atoms
  unsigned char* smem = reinterpret_cast<unsigned char*>(
      (reinterpret_cast<uintptr_t>(smem_dyn) + 1023) & ~uintptr_t(1023));
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + T::OFF_BAR);
  uint64_t* qbar = bars;
  uint64_t* kv_full = bars + 1;
  uint64_t* kv_empty = kv_full + T::STAGES;
  uint64_t* s_full = kv_empty + T::STAGES;
  uint64_t* p_full = s_full + 2;
  uint64_t* o_full = p_full + 2;
  uint32_t* tmem_base_slot = reinterpret_cast<uint32_t*>(o_full + 2);

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const int qtile = blockIdx.x % p.qtiles;
  const int bh = blockIdx.x / p.qtiles;
  const int b = bh / p.H;
  const int h = bh - b * p.H;
  const int q0 = qtile * T::TQ;
  const int ntiles = (p.n_kv + T::TK - 1) / T::TK;

  if (threadIdx.x == 0) {
    ptx::mbar_init(qbar, 1);
    for (int s = 0; s < T::STAGES; ++s) {
      ptx::mbar_init(&kv_full[s], 1);
      ptx::mbar_init(&kv_empty[s], 1);
    }
    for (int i = 0; i < 2; ++i) {
      ptx::mbar_init(&s_full[i], 1);
      ptx::mbar_init(&p_full[i], 128);
      ptx::mbar_init(&o_full[i], 1);
    }
    ptx::fence_barrier_init();
  }
  if (warp == 5) tc::tmem_alloc(tmem_base_slot, T::TMEM_COLS);
  tc::fence_before_sync();
  __syncthreads();
  tc::fence_after_sync();
  const uint32_t tmem = *tmem_base_slot;

  constexpr int kFmt = kBF16 ? 1 : 0;
  constexpr uint32_t kIdescS = tc::instr_desc_f16(kFmt, false, false, 128, 128);
  constexpr uint32_t kIdescO = tc::instr_desc_f16(kFmt, false, true, 128, 64);

  if (warp == 4) {
    // ---------------- TMA producer ----------------
    if (lane == 0) {
      ptx::prefetch_tmap(&tmQ);
      ptx::prefetch_tmap(&tmK);
      ptx::prefetch_tmap(&tmV);
      ptx::mbar_arrive_expect_tx(qbar, T::Q_BYTES);
      ptx::tma_load_4d(smem + T::OFF_Q, &tmQ, qbar, 0, q0, h, b);
      for (int t = 0; t < ntiles; ++t) {
        const int s = t % T::STAGES;
        if (t >= T::STAGES) ptx::mbar_wait_backoff(&kv_empty[s], ((t / T::STAGES) - 1) & 1, 64);
        ptx::mbar_arrive_expect_tx(&kv_full[s], T::K_BYTES + T::V_BYTES);
        ptx::tma_load_4d(smem + T::OFF_K + s * T::K_BYTES, &tmK, &kv_full[s], 0, t * T::TK, h, b);
        ptx::tma_load_4d(smem + T::OFF_V + s * T::V_BYTES, &tmV, &kv_full[s], 0, t * T::TK, h, b);
      }
    }
  } else if (warp == 5) {
    // ---------------- MMA issuer ----------------
    if (lane == 0) {
      const uint32_t q_addr = ptx::smem_u32(smem + T::OFF_Q);
      auto issue_s = [&](int t) {
        const int s = t % T::STAGES;
        ptx::mbar_wait(&kv_full[s], (t / T::STAGES) & 1);
        tc::fence_after_sync();
        const uint32_t k_addr = ptx::smem_u32(smem + T::OFF_K + s * T::K_BYTES);
        const uint32_t d = tmem + T::S_COL + (t & 1) * 128;
#pragma unroll
        for (int kk = 0; kk < T::D / 16; ++kk) {  // K-steps of 16 elements = 32 B
          const uint64_t a = tc::smem_desc_sw128(q_addr + kk * 32, 16, 1024);
          const uint64_t bd = tc::smem_desc_sw128(k_addr + kk * 32, 16, 1024);
          tc::mma_f16_ss(d, a, bd, kIdescS, kk > 0);
        }
        tc::commit(&s_full[t & 1]);
      };
      auto issue_o = [&](int t) {
        const int s = t % T::STAGES;
        ptx::mbar_wait(&p_full[t & 1], (t >> 1) & 1);
        tc::fence_after_sync();
        const uint32_t p_addr = ptx::smem_u32(smem + T::OFF_P + (t & 1) * T::P_BYTES);
        const uint32_t v_addr = ptx::smem_u32(smem + T::OFF_V + s * T::V_BYTES);
        const uint32_t d = tmem + T::O_COL + (t & 1) * 64;
#pragma unroll
        for (int kk = 0; kk < T::TK / 16; ++kk) {
          // P: K-major, two 64-key chunks of 128 rows x 128 B
          const uint32_t pa = p_addr + (kk >> 2) * (T::TQ * 128) + (kk & 3) * 32;
          const uint64_t a = tc::smem_desc_sw128(pa, 16, 1024);
          // V: MN-major (rows = keys, 128 B each); 16 keys per step = 2 swizzle atoms
          const uint64_t bd = tc::smem_desc_sw128(v_addr + kk * 2048, 16, 1024);
          tc::mma_f16_ss(d, a, bd, kIdescO, kk > 0);
        }
        tc::commit(&o_full[t & 1]);
        tc::commit(&kv_empty[s]);
      };
      ptx::mbar_wait(qbar, 0);
      tc::fence_after_sync();
      if (ntiles > 0) issue_s(0);
      for (int t = 1; t <= ntiles; ++t) {
        if (t < ntiles) issue_s(t);  // S buffer t&1 was released by p_full(t-2), awaited below
        issue_o(t - 1);
      }
    }
  } else {
    // ---------------- softmax + combine + epilogue (128 threads, one row each) ----------------
    const int row = warp * 32 + lane;
    const uint32_t lane_base = uint32_t(warp * 32) << 16;
    const float c2 = p.c;
    const float sgn = p.neg ? -1.f : 1.f;
    float m_run = -CUDART_INF_F;  // log2-domain anchor
    float l_run = 0.f;
    float w[64];
#pragma unroll
    for (int i = 0; i < 64; ++i) w[i] = 0.f;
    unsigned char* pbase = smem + T::OFF_P;

    for (int t = 0; t < ntiles; ++t) {
      // ---- S_t row -> registers ----
      ptx::mbar_wait(&s_full[t & 1], (t >> 1) & 1);
      tc::fence_after_sync();
      float s[128];
#pragma unroll
      for (int ch = 0; ch < 4; ++ch) {
        uint32_t r[32];
        tc::tmem_ld_32x32b_x32(tmem + lane_base + T::S_COL + (t & 1) * 128 + ch * 32, r);
        tc::tmem_wait_ld();
#pragma unroll
        for (int i = 0; i < 32; ++i) s[ch * 32 + i] = __uint_as_float(r[i]) * sgn;
      }
      // ---- mask, tile max, anchors ----
      const int kv_hi = p.n_kv - t * T::TK;  // valid keys in this tile
      float mx = -CUDART_INF_F;
#pragma unroll
      for (int i = 0; i < 128; ++i) {
        if (i >= kv_hi) s[i] = -CUDART_INF_F;
        mx = fmaxf(mx, s[i]);
      }
      const float m_new = fmaxf(m_run, mx * c2);
      const float corr = ptx::ex2(m_run - m_new);
      m_run = m_new;
      // ---- P_t = 2^(s c - m) (FP32), row sum, 16-bit P into the swizzled smem tile ----
      float psum = 0.f;
      unsigned char* prow = pbase + (t & 1) * T::P_BYTES;
#pragma unroll
      for (int u = 0; u < 16; ++u) {  // 16-byte units of 8 keys
        float pv[8];
#pragma unroll
        for (int e = 0; e < 8; ++e) {
          pv[e] = ptx::ex2(fmaf(s[u * 8 + e], c2, -m_new));
          psum += pv[e];
        }
        uint4 pk;
        if constexpr (kBF16) {
          pk.x = tc::pack_bf16x2(pv[0], pv[1]);
          pk.y = tc::pack_bf16x2(pv[2], pv[3]);
          pk.z = tc::pack_bf16x2(pv[4], pv[5]);
          pk.w = tc::pack_bf16x2(pv[6], pv[7]);
        } else {
          pk.x = tc::pack_f16x2(pv[0], pv[1]);
          pk.y = tc::pack_f16x2(pv[2], pv[3]);
          pk.z = tc::pack_f16x2(pv[4], pv[5]);
          pk.w = tc::pack_f16x2(pv[6], pv[7]);
        }
        const int chunk = u >> 3;  // 64-key chunk
        const int unit = (u & 7) ^ (row & 7);  // 128B swizzle: 16-B unit XOR row phase
        *reinterpret_cast<uint4*>(prow + chunk * (T::TQ * 128) + row * 128 + unit * 16) = pk;
      }
      l_run = fmaf(l_run, corr, psum);
      // ---- fold O_{t-1} (relative to m_{t-1}) and rescale to m_t ----
      if (t > 0) {
        ptx::mbar_wait(&o_full[(t - 1) & 1], ((t - 1) >> 1) & 1);
        tc::fence_after_sync();
#pragma unroll
        for (int ch = 0; ch < 2; ++ch) {
          uint32_t r[32];
          tc::tmem_ld_32x32b_x32(tmem + lane_base + T::O_COL + ((t - 1) & 1) * 64 + ch * 32, r);
          tc::tmem_wait_ld();
#pragma unroll
          for (int i = 0; i < 32; ++i) w[ch * 32 + i] = (w[ch * 32 + i] + __uint_as_float(r[i])) * corr;
        }
      } else {
#pragma unroll
        for (int i = 0; i < 64; ++i) w[i] *= corr;
      }
      // P_t visible to the tensor core (async proxy); S_t / O_{t-1} TMEM reads done
      ptx::fence_proxy_async_smem();
      tc::fence_before_sync();
      ptx::mbar_arrive(&p_full[t & 1]);
    }
    // ---- last O ----
    if (ntiles > 0) {
      const int t = ntiles - 1;
      ptx::mbar_wait(&o_full[t & 1], (t >> 1) & 1);
      tc::fence_after_sync();
#pragma unroll
      for (int ch = 0; ch < 2; ++ch) {
        uint32_t r[32];
        tc::tmem_ld_32x32b_x32(tmem + lane_base + T::O_COL + (t & 1) * 64 + ch * 32, r);
        tc::tmem_wait_ld();
#pragma unroll
        for (int i = 0; i < 32; ++i) w[ch * 32 + i] += __uint_as_float(r[i]);
      }
    }
    // ---- epilogue: Y = W / S (engine.py:375-382) in the input's 16-bit format ----
    const int qrow = q0 + row;
    if (qrow < p.n_q) {
      if (!(l_run > 0.f) || !isfinite(l_run)) atomicCAS(p.err, 0, 3);
      const float inv = 1.f / l_run;
      unsigned char* yrow = reinterpret_cast<unsigned char*>(p.y) +
                            2 * (int64_t(b) * p.ys_b + int64_t(h) * p.ys_h + int64_t(qrow) * p.ys_r);
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        uint4 pk;
        const float* x = w + 8 * u;
        if constexpr (kBF16) {
          pk.x = tc::pack_bf16x2(x[0] * inv, x[1] * inv);
          pk.y = tc::pack_bf16x2(x[2] * inv, x[3] * inv);
          pk.z = tc::pack_bf16x2(x[4] * inv, x[5] * inv);
          pk.w = tc::pack_bf16x2(x[6] * inv, x[7] * inv);
        } else {
          pk.x = tc::pack_f16x2(x[0] * inv, x[1] * inv);
          pk.y = tc::pack_f16x2(x[2] * inv, x[3] * inv);
          pk.z = tc::pack_f16x2(x[4] * inv, x[5] * inv);
          pk.w = tc::pack_f16x2(x[6] * inv, x[7] * inv);
        }
        *reinterpret_cast<uint4*>(yrow + 16 * u) = pk;
      }
    }
  }

  tc::fence_before_sync();
  __syncthreads();
  if (warp == 5) {
    tc::fence_after_sync();
    tc::tmem_dealloc(tmem, T::TMEM_COLS);
  }
}

}  // namespace elsa
