// fwd_tc.cuh — K5: the FP16 / BF16 variant of the ELSA forward on the 5th-gen
// tensor cores. The two dense contractions run as
// tcgen05.mma (kind::f16, FP32 accumulation in TMEM); the (m, S, W) tile
// states, their combine, the anchors and the epilogue stay in FP32 as in K1:
//   S_t = Q K_t^T            tcgen05.mma 128x128xD, A and B from 128B-swizzled smem
//   P_t = 2^(s c - m)        one query row per thread (tcgen05.ld 32x32b), 16-bit
//                            P written back to TMEM (tcgen05.st)
//   W  += P_t V_t            tcgen05.mma 128x64x128 per 64 output columns, A = P
//                            read from TMEM, W accumulating in TMEM
//
// A CTA owns GROUPS (1 or 2) query tiles of 128 rows, one softmax warpgroup
// each (warp w of group g owns TMEM lanes 32(w%4).. = query rows), so two
// softmax streams share every SM sub-partition while the tensor core
// ping-pongs between them. Per group TMEM holds S (128 columns, single
// buffer: S_g(t+1) is issued once the group has pulled S_g(t) into registers,
// overlapping its exponentials), W (D columns) and P (64 packed columns; at
// D = 128 P is written over the group's own S so two tiles fit 512 columns,
// and S_g(t+1) then waits for P_g(t) V's issue).
//
// Combine with a deferred anchor: a row's anchor m moves only when a tile's
// maximum exceeds it by more than kRescaleLog2 (log2 units); then its running
// sum and TMEM W row are multiplied by 2^(m_old - m_new) (skipped warp-wide
// when no row of the warp moved). Between moves every P <= 2^kRescaleLog2,
// exact in the 16-bit formats' range: the same monoid product, represented
// at a different anchor. A share of the exponentials runs as an FFMA2
// polynomial (MUFU.EX2 is the softmax's binding pipe).
//
// Warp roles: softmax warpgroups, then a TMA producer warp (Q once, K/V
// through a STAGES-deep ring) and the TMEM allocator + MMA warp (a
// warp-uniform event loop, one elected lane issues). GROUPS = 2 adds two idle
// warps so setmaxnreg can hand a whole warpgroup's registers to the softmax.
#pragma once
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdint>
#include <math_constants.h>

#include "ptx.cuh"
#include "tc.cuh"

namespace elsa {

struct TcParams {
  void* y;  // 16-bit output (B, H, n_q, dv) in the input format
  int B, H, n_q, n_kv;
  int dv;     // <= 64 (narrower Q/K/V are zero-filled to 64 by TMA)
  int y_vec;  // 16-byte Y stores legal (else element stores)
  int64_t ys_b, ys_h, ys_r;  // element strides of y
  float c;                   // |scale| * log2(e)
  int neg;                   // scale < 0 (sign applied to the scores)
  int qtiles;                // CTAs per (b, h): ceil(n_q / (GROUPS * 128))
  int* err;
};

// ELSA_TC_TRACE builds: CTA 0 records SM clock stamps per tile for the first
// kTcTraceTiles tiles: softmax warps (lane 0) at 6 points, the MMA warp at
// its S / PV issues (diagnostic only; tools/trace_tc.py).
constexpr int kTcTraceTiles = 64;
#ifdef ELSA_TC_TRACE
__device__ unsigned long long g_tc_trace[16 * kTcTraceTiles * 8];
#define TC_MARK(slot, t, pt)                                                            \
  do {                                                                                \
    if (blockIdx.x == 0 && (t) < kTcTraceTiles) {                                      \
      unsigned long long c_;                                                           \
      asm volatile("mov.u64 %0, %%clock64;" : "=l"(c_));                               \
      g_tc_trace[((slot) * kTcTraceTiles + (t)) * 8 + (pt)] = c_;                      \
    }                                                                                 \
  } while (0)
#else
#define TC_MARK(slot, t, pt) \
  do {                       \
  } while (0)
#endif

// Share of the exponentials computed on the FMA pipe instead of MUFU: this
// many pairs out of every 8 scores (0..4), plus one more pair in the 8-key
// units flagged in ELSA_TC_POLY_EXTRA. MUFU.EX2 issues at 16 lanes/clk/SM
// (tools/microbench/mufu_ex2.cu; f16x2 / bf16x2 forms are no faster), so with
// 128 exponentials per row per tile it is the softmax's binding pipe (ncu: XU
// 78% of peak); a polynomial on FFMA2 moves part of that load to the FMA
// pipe, and packed FFMA2 / FADD2 argument and sum arithmetic frees the issue
// slots the polynomial needs. Measured (tools/tc_variant_ab.py, BF16 16K):
// none 839, 25% 864, packed + 25% 877-882, packed + 31% 899, packed + 37.5%
// (the default) 910, packed + 44% 880, packed + 50% 873 TFLOP/s; errors vs
// FP64 unchanged (8.82e-3 vs PyTorch's 8.85e-3).
#ifndef ELSA_TC_POLY_PAIRS
#define ELSA_TC_POLY_PAIRS 1  // pairs per 8-key unit on the FMA pipe (see ELSA_TC_POLY_EXTRA)
#endif
constexpr int kTcPolyPairs = ELSA_TC_POLY_PAIRS;
#ifndef ELSA_TC_PACKED_G2
#define ELSA_TC_PACKED_G2 1  // packed FFMA2/FADD2 softmax arithmetic for two-tile CTAs too
#endif
constexpr bool kTcPackedG2 = ELSA_TC_PACKED_G2 != 0;
#ifndef ELSA_TC_POLY_EXTRA
#define ELSA_TC_POLY_EXTRA 0x5555  // bit u: one more polynomial pair in 8-key unit u
#endif
#ifndef ELSA_TC_POLY_EXTRA_D128
// d = 128 (twice the MMA work per exponential) prefers 25%: BF16 16K 0% 1218-1226,
// 25% 1230, 31% 1220, 37.5% 1198 TFLOP/s
#define ELSA_TC_POLY_EXTRA_D128 0
#endif
#ifndef ELSA_TC_POLY_DEG
#define ELSA_TC_POLY_DEG 3
#endif

// 2^x for a pair, x <= 2^7, on the FMA pipe: x = j + f with j = rint(x) (the
// 1.5*2^23 shifter), f in [-1/2, 1/2]; 2^f by a degree-3 minimax polynomial
// (relative error 7.5e-5; degree 4 Taylor: 5.6e-5, one more FFMA2 — both
// below the 16-bit formats' rounding of P: 2^-9 bf16, 2^-11 fp16); 2^j added
// to the exponent field. x is clamped to
// -126 so the result stays normal (>= 0.7 * 2^-126: negligible against S >= 1).
__device__ __forceinline__ void ex2_poly2(float x0, float x1, float& y0, float& y1) {
  using ptx::f32x2;
  const f32x2 x = ptx::pack2(fmaxf(x0, -126.f), fmaxf(x1, -126.f));
  const f32x2 shifter = ptx::pack2(12582912.f, 12582912.f);
  const f32x2 r = ptx::fadd2(x, shifter);        // j in the low mantissa bits
  const f32x2 j = ptx::fadd2(r, ptx::pack2(-12582912.f, -12582912.f));
  const f32x2 f = ptx::ffma2r(j, ptx::pack2(-1.f, -1.f), x);  // x - j, exact
#if ELSA_TC_POLY_DEG == 3
  // degree-3 minimax fit of 2^f on [-1/2, 1/2] (relative error 7.5e-5, under
  // fp16's 2^-11 and bf16's 2^-8 rounding of P)
  f32x2 q = ptx::ffma2r(f, ptx::pack2(5.517132e-2f, 5.517132e-2f),
                        ptx::pack2(2.4261054e-1f, 2.4261054e-1f));
  q = ptx::ffma2r(q, f, ptx::pack2(6.9326097e-1f, 6.9326097e-1f));
  q = ptx::ffma2r(q, f, ptx::pack2(9.999281e-1f, 9.999281e-1f));
#else
  f32x2 q = ptx::ffma2r(f, ptx::pack2(9.6181291e-3f, 9.6181291e-3f),
                        ptx::pack2(5.5504109e-2f, 5.5504109e-2f));
  q = ptx::ffma2r(q, f, ptx::pack2(2.4022651e-1f, 2.4022651e-1f));
  q = ptx::ffma2r(q, f, ptx::pack2(6.9314718e-1f, 6.9314718e-1f));
  q = ptx::ffma2r(q, f, ptx::pack2(1.f, 1.f));
#endif
  float q0, q1, r0, r1;
  ptx::unpack2(q, q0, q1);
  ptx::unpack2(r, r0, r1);
  y0 = __int_as_float(__float_as_int(q0) + (__float_as_int(r0) << 23));
  y1 = __int_as_float(__float_as_int(q1) + (__float_as_int(r1) << 23));
}

#ifndef ELSA_TC_SELF_ISSUE
#define ELSA_TC_SELF_ISSUE 0  // each softmax warpgroup issues its own MMAs (measured: 506 vs 835 TFLOP/s at 16K — issuing blocks the softmax warp)
#endif
constexpr bool kTcSelfIssue = ELSA_TC_SELF_ISSUE != 0;

#ifndef ELSA_TC_PSPLIT
#define ELSA_TC_PSPLIT 1  // P_g(t) handed to the tensor core in this many key parts (2: 597, 4: 461 vs 1: 907 TFLOP/s BF16 16K — the mid-loop wait/arrive serialises the exponentials)
#endif
#ifndef ELSA_TC_STAGES
#define ELSA_TC_STAGES 4  // K/V ring depth (measured: 2: 697, 3: 827, 4: 845, 5: 845 TFLOP/s at 16K)
#endif

// anchor hysteresis of the deferred rescale (log2 units): P <= 2^8
constexpr float kRescaleLog2 = 8.f;

// D = 64, or 128 (64 < d, dv <= 128; Q/K/V rows as two 64-element
// swizzle-atom blocks). At D = 128, P is written over its own tile's S in
// TMEM (kAliasP) so that two query tiles (S/P 128 + W 128 columns each) fit
// the 512 columns; S_g(t+1) is then issued only after P_g(t) V.
//
// TK_ = 64 (D = 128 only): 64-key tiles. S (64 columns), P (32) and W (128)
// of both groups fit the 512 TMEM columns without aliasing, so S_g(t+1) is
// issued as soon as S_g(t) is in registers (overlapping the exponentials) as
// at D = 64, instead of after P_g(t) V.
//
// CS_ = 2 (experiment, D = 64 two-group CTAs): each query row's 128 scores are
// split over two softmax warps on the same TMEM lane quarter (64 columns
// each; the row max exchanged through shared memory per tile), so four
// softmax warps share every SM sub-partition instead of two.
template <int GROUPS, int D_ = 64, int TK_ = 128, int CS_ = 1>
struct TcTraits {
  static constexpr int TQ = 128, TK = TK_, D = D_, CS = CS_;
  static_assert(CS == 1 || (CS == 2 && D == 64 && TK == 128 && GROUPS == 2), "column split");
  static_assert(D == 64 || D == 128, "head width");
  static_assert(TK == 128 || (TK == 64 && D == 128), "key tile");
  static constexpr bool kAliasP = D == 128 && TK == 128;
  // stages: D = 64 ELSA_TC_STAGES x 32 KB; D = 128: 2 x 64 KB, or 4 x 32 KB with 64-key tiles
  static constexpr int STAGES = D == 64 ? ELSA_TC_STAGES : (TK == 64 ? 4 : 2);
  static constexpr int DB = D / 64;                          // 128-byte column blocks per row
  static constexpr int ROWS = GROUPS * TQ;                   // query rows per CTA
  static constexpr int Q_BLOCK = TQ * 128, K_BLOCK = TK * 128, V_BLOCK = TK * 128;
  static constexpr int Q_BYTES = DB * Q_BLOCK;               // 16 KB per group and block
  static constexpr int K_BYTES = DB * K_BLOCK;
  static constexpr int V_BYTES = DB * V_BLOCK;
  static constexpr int OFF_Q = 0;
  static constexpr int OFF_K = OFF_Q + GROUPS * Q_BYTES;
  static constexpr int OFF_V = OFF_K + STAGES * K_BYTES;
  static constexpr int OFF_BAR = OFF_V + STAGES * V_BYTES;
  // barriers: qbar, kv_full[3], kv_empty[3], s_full[G], s_free[G], p_full[G], o_full[G],
  // + tmem base word
  // P and its P V MMAs in PH key parts, each with its own p_full / o_full
  // barrier: part 0's P V runs while the softmax computes part 1, and the
  // next tile only waits for part h's P V before overwriting part h of P
  static constexpr int PH = kTcSelfIssue ? 1 : ELSA_TC_PSPLIT;
  static_assert(PH == 1 || PH == 2 || PH == 4, "P parts");
  static constexpr int NBAR = 1 + 2 * STAGES + (2 + 2 * PH) * GROUPS;
  // CS = 2: row-max / row-sum exchange slots, [3 * GROUPS * 4][64] floats
  static constexpr int OFF_XCH = ((OFF_BAR + NBAR * 8 + 16) + 15) / 16 * 16;
  static constexpr int XCH_BYTES = CS == 2 ? 3 * GROUPS * 4 * 64 * 4 : 0;
  static constexpr size_t SMEM_BYTES = OFF_XCH + XCH_BYTES + 1024;  // + 1024 alignment slack
  static constexpr int SOFTMAX_WARPS = 4 * GROUPS * CS;
  static constexpr int TMA_WARP = SOFTMAX_WARPS, MMA_WARP = SOFTMAX_WARPS + 1;
  // GROUPS = 2: a whole third warpgroup (TMA, MMA, two idle warps) so setmaxnreg
  // can hand its registers to the softmax warpgroups; 12 warps launch at 168
  // and setmaxnreg only redistributes that allocation (per SM sub-partition
  // 3 x 168 = 504): 168 - 40 = 128 freed = 2 x (232 - 168) taken. Asking for
  // more than is freed blocks the .inc forever.
  static constexpr bool kRegSplit = GROUPS == 2;
  static constexpr int THREADS = kRegSplit ? (SOFTMAX_WARPS + 4) * 32 : (SOFTMAX_WARPS + 2) * 32;
  // launch allocation per thread (the register file / THREADS, granule 8):
  // 12 warps 168, 20 warps (CS = 2) 96
  static constexpr int LAUNCH_REGS = (65536 / THREADS) / 8 * 8 > 255 ? 255 : (65536 / THREADS) / 8 * 8;
  static constexpr int SOFTMAX_REGS = CS == 2 ? 104 : 232, OTHER_REGS = 40;
  static_assert(!kRegSplit || (SOFTMAX_WARPS / 4) * (SOFTMAX_REGS - LAUNCH_REGS) <=
                                  LAUNCH_REGS - OTHER_REGS,
                "setmaxnreg budget");
  static constexpr uint32_t S_COL = 0;             // group g: S at TK g
  static constexpr uint32_t O_COL = TK * GROUPS;   // group g: W (P V accumulator) at O_COL + D g
  // group g: P (16-bit, two per 32-bit column) at P_COL + P_STRIDE g — the A
  // operand of P V read straight from TMEM (no shared-memory round trip)
  static constexpr uint32_t P_COL = kAliasP ? S_COL : (TK + D) * GROUPS;
  static constexpr uint32_t P_STRIDE = kAliasP ? 128 : TK / 2;
  static constexpr uint32_t TMEM_NEED = (O_COL + D * GROUPS > P_COL + P_STRIDE * GROUPS)
                                             ? O_COL + D * GROUPS
                                             : P_COL + P_STRIDE * GROUPS;
  static constexpr uint32_t TMEM_COLS = TMEM_NEED <= 256 ? 256 : 512;
  static_assert(TMEM_NEED <= 512, "TMEM columns");
  static_assert(SMEM_BYTES <= 227 * 1024, "shared memory budget");
};

template <bool kBF16, int GROUPS, int D_ = 64, int TK_ = 128, int CS_ = 1>
__global__ void __launch_bounds__(TcTraits<GROUPS, D_, TK_, CS_>::THREADS, 1)
    fwd_tc_kernel(const __grid_constant__ TcParams p, const __grid_constant__ CUtensorMap tmQ,
                  const __grid_constant__ CUtensorMap tmK,
                  const __grid_constant__ CUtensorMap tmV) {
  using T = TcTraits<GROUPS, D_, TK_, CS_>;
  extern __shared__ unsigned char smem_dyn[];
  // 1024-byte alignment for the 128B-swizzle atoms
  unsigned char* smem = reinterpret_cast<unsigned char*>(
      (reinterpret_cast<uintptr_t>(smem_dyn) + 1023) & ~uintptr_t(1023));
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + T::OFF_BAR);
  uint64_t* qbar = bars;
  uint64_t* kv_full = bars + 1;
  uint64_t* kv_empty = kv_full + T::STAGES;
  uint64_t* s_full = kv_empty + T::STAGES;
  uint64_t* s_free = s_full + GROUPS;
  uint64_t* p_full = s_free + GROUPS;    // [g * PH + part]
  uint64_t* o_full = p_full + GROUPS * T::PH;  // [g * PH + part]
  uint32_t* tmem_base_slot = reinterpret_cast<uint32_t*>(o_full + GROUPS * T::PH);
  constexpr int PH = T::PH;

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const int qtile = blockIdx.x % p.qtiles;
  const int bh = blockIdx.x / p.qtiles;
  const int b = bh / p.H;
  const int h = bh - b * p.H;
  const int q0 = qtile * T::ROWS;
  const int ntiles = (p.n_kv + T::TK - 1) / T::TK;

  if (threadIdx.x == 0) {
    ptx::mbar_init(qbar, 1);
    for (int s = 0; s < T::STAGES; ++s) {
      ptx::mbar_init(&kv_full[s], 1);
      ptx::mbar_init(&kv_empty[s], kTcSelfIssue ? GROUPS : 1);
    }
    for (int g = 0; g < GROUPS; ++g) {
      ptx::mbar_init(&s_full[g], 1);
      ptx::mbar_init(&s_free[g], 128 * T::CS);
      for (int hh = 0; hh < PH; ++hh) {
        ptx::mbar_init(&p_full[g * PH + hh], 128 * T::CS);
        ptx::mbar_init(&o_full[g * PH + hh], 1);
      }
    }
    ptx::fence_barrier_init();
  }
  if (warp == T::MMA_WARP) tc::tmem_alloc(tmem_base_slot, T::TMEM_COLS);
  tc::fence_before_sync();
  __syncthreads();
  tc::fence_after_sync();
  const uint32_t tmem = *tmem_base_slot;

  constexpr int kFmt = kBF16 ? 1 : 0;
  constexpr uint32_t kIdescS = tc::instr_desc_f16(kFmt, false, false, 128, T::TK);
  constexpr uint32_t kIdescO = tc::instr_desc_f16(kFmt, false, true, 128, 64);

  // MMA issue for group g (warp-uniform; the elected `leader` lane issues)
  auto issue_s = [&](int g, int t, bool leader) {  // S_g(t) = Q_g K_t^T
    const int s = t % T::STAGES;
    const uint32_t q_addr = ptx::smem_u32(smem + T::OFF_Q + g * T::Q_BYTES);
    const uint32_t k_addr = ptx::smem_u32(smem + T::OFF_K + s * T::K_BYTES);
    const uint32_t d = tmem + T::S_COL + g * T::TK;
#pragma unroll
    for (int kk = 0; kk < T::D / 16; ++kk) {  // K-steps of 16 elements = 32 B
      const uint32_t blk = kk >> 2, off = (kk & 3) * 32;  // 64-element column block
      const uint64_t a = tc::smem_desc_sw128(q_addr + blk * T::Q_BLOCK + off, 16, 1024);
      const uint64_t bd = tc::smem_desc_sw128(k_addr + blk * T::K_BLOCK + off, 16, 1024);
      if (leader) tc::mma_f16_ss(d, a, bd, kIdescS, kk > 0);
    }
    if (leader) tc::commit(&s_full[g]);
    __syncwarp();
  };
  // W_g (+)= P_g(t) V_t over key part hh, P from TMEM
  auto issue_o = [&](int g, int t, int hh, bool leader) {
    const int s = t % T::STAGES;
    const uint32_t v_addr = ptx::smem_u32(smem + T::OFF_V + s * T::V_BYTES);
    const uint32_t d = tmem + T::O_COL + g * T::D;
    const uint32_t pa = tmem + T::P_COL + g * T::P_STRIDE;
    constexpr int KS = T::TK / 16 / PH;  // K-steps per part
#pragma unroll
    for (int k2 = 0; k2 < KS; ++k2) {
      const int kk = hh * KS + k2;
#pragma unroll
      for (int nb = 0; nb < T::DB; ++nb) {  // 64 output columns per V block
        // V: MN-major (rows = keys, 128 B each); 16 keys per step = 2 swizzle atoms
        const uint64_t bd = tc::smem_desc_sw128(v_addr + nb * T::V_BLOCK + kk * 2048, 16, 1024);
        if (leader)
          tc::mma_f16_ts(d + nb * 64, pa + kk * 8, bd, kIdescO, (t > 0 || kk > 0) ? 1u : 0u);
      }
    }
    if (leader) tc::commit(&o_full[g * PH + hh]);
    __syncwarp();
  };
  // lane 0's view of a barrier phase, broadcast so the schedule stays uniform
  auto ready = [&](uint64_t* bar, uint32_t parity) {
    return __shfl_sync(0xffffffffu, ptx::mbar_test(bar, parity) ? 1 : 0, 0) != 0;
  };

  // setmaxnreg inside each role's branch so the softmax code is dominated by
  // the .inc (ptxas then allocates up to SOFTMAX_REGS there)
  if (warp >= T::SOFTMAX_WARPS) {
    if constexpr (T::kRegSplit) asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;" ::"n"(T::OTHER_REGS));
  }
  if (warp == T::TMA_WARP) {
    // ---------------- TMA producer ----------------
    if (lane == 0) {
      ptx::prefetch_tmap(&tmQ);
      ptx::prefetch_tmap(&tmK);
      ptx::prefetch_tmap(&tmV);
      ptx::mbar_arrive_expect_tx(qbar, GROUPS * T::Q_BYTES);
      for (int g = 0; g < GROUPS; ++g)  // rows past n_q / columns past d are zero-filled by TMA
        for (int blk = 0; blk < T::DB; ++blk)
          ptx::tma_load_4d(smem + T::OFF_Q + g * T::Q_BYTES + blk * T::Q_BLOCK, &tmQ, qbar,
                           64 * blk, q0 + g * T::TQ, h, b);
      for (int t = 0; t < ntiles; ++t) {
        const int s = t % T::STAGES;
        if (t >= T::STAGES) ptx::mbar_wait_backoff(&kv_empty[s], ((t / T::STAGES) - 1) & 1, 64);
        ptx::mbar_arrive_expect_tx(&kv_full[s], T::K_BYTES + T::V_BYTES);
        for (int blk = 0; blk < T::DB; ++blk) {
          ptx::tma_load_4d(smem + T::OFF_K + s * T::K_BYTES + blk * T::K_BLOCK, &tmK, &kv_full[s],
                           64 * blk, t * T::TK, h, b);
          ptx::tma_load_4d(smem + T::OFF_V + s * T::V_BYTES + blk * T::V_BLOCK, &tmV, &kv_full[s],
                           64 * blk, t * T::TK, h, b);
        }
      }
    }
  } else if (warp == T::MMA_WARP && !kTcSelfIssue) {
    // ---------------- MMA issuer ----------------
    // The whole warp runs the (warp-uniform) schedule so the descriptors stay
    // in uniform registers; one elected lane issues each tcgen05.mma / commit.
    // (A lane-0-only loop paid R2UR round trips per descriptor and measured
    // ~1300 clocks from a group's barrier to the matching issue.)
    const bool leader = tc::elect_one();
    // Event loop over both groups: S_g(t+1) is issued as soon as group g
    // has pulled S_g(t) into registers (s_free) — it overlaps the group's own
    // exponentials — and P_g(t) V_t as soon as P_g(t) is written (p_full).
    // Each barrier is only ever tested for its next phase, which cannot
    // have been overtaken (every phase needs an MMA issued here first), and
    // with test_wait: a try_wait could park the warp on one group's barrier
    // while the other group's P is ready. (Measured slower: probing all
    // barriers at once, one lane per barrier + ballot, 700 vs 769 TFLOP/s;
    // lane 0 probing all barriers then one broadcast, 631 vs 834; S and P V
    // issued by two separate warps, 815 vs 835; one issuing warp per group,
    // 730 vs 837 — a single issuer is best.)
    ptx::mbar_wait(qbar, 0);
    int ns[GROUPS], npv[GROUPS], nph[GROUPS];  // next S tile / next P V tile and part
    for (int g = 0; g < GROUPS; ++g) ns[g] = npv[g] = nph[g] = 0;
    int kv_released = 0;  // tiles whose K/V stage was handed back
    while (kv_released < ntiles) {
      // (issue order measured: per group P V then S is best; every ready P V
      // first, or S before P V, measured slower — profiles/round2_tc_order.txt)
#pragma unroll
      for (int g = 0; g < GROUPS; ++g) {
        const int u = npv[g], hh = nph[g];
        if (u < ns[g] && ready(&p_full[g * PH + hh], u & 1)) {  // P V first: on the softmax's path
          tc::fence_after_sync();
          if (lane == 0 && hh == 0) TC_MARK(8 + g, u, 1);
          issue_o(g, u, hh, leader);
          if (lane == 0 && hh == 0) TC_MARK(8 + g, u, 3);  // issue returned
          nph[g] = hh + 1 == PH ? 0 : hh + 1;
          npv[g] = hh + 1 == PH ? u + 1 : u;
          int done = npv[0];
#pragma unroll
          for (int gg = 1; gg < GROUPS; ++gg) done = npv[gg] < done ? npv[gg] : done;
          if (done > kv_released) {  // P V of tile kv_released issued for every group
            if (leader) tc::commit(&kv_empty[kv_released % T::STAGES]);
            __syncwarp();
            ++kv_released;
          }
        }
        const int t = ns[g];
        // (P aliased over S: S_g(t) only after P_g(t-1) V has been issued)
        if (t < ntiles && (!T::kAliasP || npv[g] >= t) &&
            (t == 0 || ready(&s_free[g], (t - 1) & 1)) &&
            ready(&kv_full[t % T::STAGES], (t / T::STAGES) & 1)) {
          tc::fence_after_sync();
          if (lane == 0) TC_MARK(8 + g, t, 0);
          issue_s(g, t, leader);
          if (lane == 0) TC_MARK(8 + g, t, 2);  // issue returned
          ns[g] = t + 1;
        }
      }
    }
  } else if (warp < T::SOFTMAX_WARPS) {
    // ------------- softmax + combine + epilogue (one warpgroup per query tile) -------------
    if constexpr (T::kRegSplit) asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;" ::"n"(T::SOFTMAX_REGS));
    constexpr int CS = T::CS;
    const int g = warp / (4 * CS);
    const int cpart = (warp % (4 * CS)) / 4;  // this warp's column part of the row (CS = 2)
    const int row = (warp & 3) * 32 + lane;
    const uint32_t lane_base = uint32_t((warp & 3) * 32) << 16;
    const uint32_t s_tm = tmem + lane_base + T::S_COL + g * T::TK + cpart * (T::TK / CS);
    const uint32_t o_tm = tmem + lane_base + T::O_COL + g * T::D;
    // CS = 2: per-tile row-max exchange between the two warps of a lane quarter
    // (double-buffered by tile parity; named barrier 1 + 4 g + quarter, 64 threads)
    float* xmax = reinterpret_cast<float*>(smem + T::OFF_XCH);
    auto pair_sync = [&]() {
      asm volatile("bar.sync %0, 64;" ::"r"(1 + 4 * g + (warp & 3)) : "memory");
    };
    const float c2 = p.c;
    const float cs = p.neg ? -c2 : c2;  // exponent = s_raw * cs - m
    float m_run = -CUDART_INF_F;        // log2-domain anchor
    float l_run = 0.f;
    const uint32_t p_tm = tmem + lane_base + T::P_COL + g * T::P_STRIDE + cpart * (T::TK / CS / 2);
    // self-issue: warp 0 of the group issues the group's MMAs after a
    // group-wide named barrier (id 1 + g) instead of signalling the MMA warp
    const bool issuer = kTcSelfIssue && (warp & 3) == 0;
    const bool leader = issuer && tc::elect_one();
    auto group_sync = [&]() {
      asm volatile("bar.sync %0, 128;" ::"r"(1 + g) : "memory");
    };
    if (issuer && ntiles > 0) {
      ptx::mbar_wait(qbar, 0);
      ptx::mbar_wait(&kv_full[0], 0);
      tc::fence_after_sync();
      issue_s(g, 0, leader);
    }

    for (int t = 0; t < ntiles; ++t) {
      if (lane == 0) TC_MARK(warp, t, 0);
      ptx::mbar_wait(&s_full[g], t & 1);
      if (lane == 0) TC_MARK(warp, t, 1);
      tc::fence_after_sync();
      constexpr int TK = T::TK / CS;  // this warp's keys of the tile
      float s[TK];
#pragma unroll
      for (int ch = 0; ch < TK / 32; ++ch) {
        uint32_t r[32];
        tc::tmem_ld_32x32b_x32(s_tm + ch * 32, r);
#pragma unroll
        for (int i = 0; i < 32; ++i) s[ch * 32 + i] = __uint_as_float(r[i]);
      }
      tc::tmem_wait_ld();
      // S_g(t) is in registers: the tensor core may overwrite it with S_g(t+1)
      tc::fence_before_sync();
      if constexpr (kTcSelfIssue) {
        group_sync();
        if (issuer && t + 1 < ntiles) {
          ptx::mbar_wait(&kv_full[(t + 1) % T::STAGES], ((t + 1) / T::STAGES) & 1);
          tc::fence_after_sync();
          issue_s(g, t + 1, leader);
        }
      } else {
        ptx::mbar_arrive(&s_free[g]);
      }
      if (lane == 0) TC_MARK(warp, t, 2);
      const int kv_hi = p.n_kv - t * T::TK - cpart * TK;  // valid keys in this warp's part
      if (kv_hi < TK) {                   // tail tile (warp-uniform): mask past n_kv
#pragma unroll
        for (int i = 0; i < TK; ++i)
          if (i >= kv_hi) s[i] = p.neg ? CUDART_INF_F : -CUDART_INF_F;
      }
      // row max of the signed scores, in log2 units (warp-uniform sign branch;
      // eight partial maxima keep the reduction off one dependent chain)
      float m_tile;
      {
        float acc[8];
        if (!p.neg) {
#pragma unroll
          for (int j = 0; j < 8; ++j) acc[j] = s[j];
#pragma unroll
          for (int i = 8; i < TK; i += 8)
#pragma unroll
            for (int j = 0; j < 8; ++j) acc[j] = fmaxf(acc[j], s[i + j]);
        } else {
#pragma unroll
          for (int j = 0; j < 8; ++j) acc[j] = -s[j];
#pragma unroll
          for (int i = 8; i < TK; i += 8)
#pragma unroll
            for (int j = 0; j < 8; ++j) acc[j] = fmaxf(acc[j], -s[i + j]);
        }
        m_tile = fmaxf(fmaxf(fmaxf(acc[0], acc[1]), fmaxf(acc[2], acc[3])),
                       fmaxf(fmaxf(acc[4], acc[5]), fmaxf(acc[6], acc[7]))) * c2;
      }
      if constexpr (CS == 2) {  // the row's other half
        float* slot = xmax + ((t & 1) * GROUPS * 4 + g * 4 + (warp & 3)) * 64;
        slot[cpart * 32 + lane] = m_tile;
        pair_sync();
        m_tile = fmaxf(m_tile, slot[(cpart ^ 1) * 32 + lane]);
      }
      // deferred anchor: move only when the tile max exceeds it by > kRescaleLog2
      const bool move = m_tile > m_run + kRescaleLog2;
      const float m_new = move ? m_tile : m_run;
      const float corr = move ? ptx::ex2(m_run - m_new) : 1.f;  // 0 on the first move
      m_run = m_new;
      // anchor moved: wait for all of P_g(t-1) V (W_g then holds tiles < t)
      // and rescale this warp's W rows in TMEM; otherwise each P part only
      // waits for its own P V below
      if (lane == 0) TC_MARK(warp, t, 3);
      if (t > 0 && __any_sync(0xffffffffu, move)) {
#pragma unroll
        for (int hh = 0; hh < PH; ++hh) ptx::mbar_wait(&o_full[g * PH + hh], (t - 1) & 1);
        if (lane == 0) TC_MARK(warp, t, 4);
        tc::fence_after_sync();
        {
#pragma unroll
          for (int ch = cpart * (T::D / 32 / CS); ch < (cpart + 1) * (T::D / 32 / CS); ++ch) {
            uint32_t r[32];
            tc::tmem_ld_32x32b_x32(o_tm + ch * 32, r);
            tc::tmem_wait_ld();
#pragma unroll
            for (int i = 0; i < 32; ++i) r[i] = __float_as_uint(__uint_as_float(r[i]) * corr);
            tc::tmem_st_32x32b_x32(o_tm + ch * 32, r);
          }
          tc::tmem_wait_st();
        }
      }
      // P_t = 2^(s c - m) (FP32), row sum, 16-bit P into the swizzled tile.
      // One tile per CTA: exponent arguments and partial sums on packed
      // FFMA2 / FADD2 (1K: 232 vs 215 TFLOP/s); two tiles per CTA: scalar FFMA
      // / FADD (16K: 761 vs 704) — measured, tools/time_tc.py.
      const float neg_m = -m_new;
      const ptx::f32x2 cs2 = ptx::pack2(cs, cs), nm2 = ptx::pack2(neg_m, neg_m);
      ptx::f32x2 psa = 0ull, psb = 0ull;
      float ps0 = 0.f, ps1 = 0.f;
      uint32_t pk[16];
      constexpr int NU = TK / 8;  // 16-byte units of 8 keys
#pragma unroll
      for (int u = 0; u < NU; ++u) {
        float pv[8];
#pragma unroll
        for (int e = 0; e < 8; e += 2) {
          float x0, x1;
          if constexpr (GROUPS == 1 || kTcPackedG2) {
            ptx::unpack2(ptx::ffma2r(ptx::pack2(s[u * 8 + e], s[u * 8 + e + 1]), cs2, nm2), x0, x1);
          } else {
            x0 = fmaf(s[u * 8 + e], cs, neg_m);
            x1 = fmaf(s[u * 8 + e + 1], cs, neg_m);
          }
          // this pair on the FMA pipe, the rest on MUFU
          constexpr unsigned kExtra = T::D == 128 ? ELSA_TC_POLY_EXTRA_D128 : ELSA_TC_POLY_EXTRA;
          if (e < 2 * (kTcPolyPairs + ((kExtra >> u) & 1))) {
            ex2_poly2(x0, x1, pv[e], pv[e + 1]);
          } else {
            pv[e] = ptx::ex2(x0);
            pv[e + 1] = ptx::ex2(x1);
          }
        }
        if constexpr (GROUPS == 1 || kTcPackedG2) {
          psa = ptx::fadd2(psa, ptx::fadd2(ptx::pack2(pv[0], pv[1]), ptx::pack2(pv[2], pv[3])));
          psb = ptx::fadd2(psb, ptx::fadd2(ptx::pack2(pv[4], pv[5]), ptx::pack2(pv[6], pv[7])));
        } else {
          ps0 += (pv[0] + pv[1]) + (pv[2] + pv[3]);
          ps1 += (pv[4] + pv[5]) + (pv[6] + pv[7]);
        }
#pragma unroll
        for (int e = 0; e < 4; ++e)
          pk[(u & 3) * 4 + e] = kBF16 ? tc::pack_bf16x2(pv[2 * e], pv[2 * e + 1])
                                      : tc::pack_f16x2(pv[2 * e], pv[2 * e + 1]);
        constexpr int UPH = NU / PH;  // 8-key units per P part
        if ((u & 3) == 3) {  // 32 keys = 16 columns packed: into TMEM
          if (t > 0 && u % UPH == 3) {  // part's first store: its P V of tile t-1 must be done
            if (lane == 0 && u == 3) TC_MARK(warp, t, 6);
            ptx::mbar_wait(&o_full[g * PH + u / UPH], (t - 1) & 1);
            if (lane == 0 && u == 3) TC_MARK(warp, t, 7);
            tc::fence_after_sync();
          }
          tc::tmem_st_32x32b_x16(p_tm + (u >> 2) * 16, pk);
          if (PH > 1 && !kTcSelfIssue && u % UPH == UPH - 1 && u != NU - 1) {
            // part complete: hand it to the tensor core
            tc::tmem_wait_st();
            tc::fence_before_sync();
            ptx::mbar_arrive(&p_full[g * PH + u / UPH]);
          }
        }
      }
      tc::tmem_wait_st();
      float psum;
      if constexpr (GROUPS == 1 || kTcPackedG2) {
        const ptx::f32x2 pt = ptx::fadd2(psa, psb);
        psum = ptx::lo2(pt) + ptx::hi2(pt);
      } else {
        psum = ps0 + ps1;
      }
      l_run = fmaf(l_run, corr, psum);
      // P_t in TMEM for the tensor core; S_t reads and W stores done
      tc::fence_before_sync();
      if constexpr (kTcSelfIssue) {
        group_sync();
        if (issuer) {
          tc::fence_after_sync();
          issue_o(g, t, 0, leader);
          if (leader) tc::commit(&kv_empty[t % T::STAGES]);
          __syncwarp();
        }
      } else {
        ptx::mbar_arrive(&p_full[g * PH + PH - 1]);
      }
      if (lane == 0) TC_MARK(warp, t, 5);
    }
    // ---- epilogue: Y = W / S (engine.py:375-382) in the input's 16-bit format ----
    if constexpr (CS == 2) {  // the row sum is split over the pair
      float* slot = xmax + (2 * GROUPS * 4 + g * 4 + (warp & 3)) * 64;
      slot[cpart * 32 + lane] = l_run;
      pair_sync();
      l_run = slot[lane] + slot[32 + lane];
    }
    constexpr int DC = T::D / CS;  // this warp's output columns
    const int col0 = cpart * DC;
    float w[DC];
    if (ntiles > 0) {
#pragma unroll
      for (int hh = 0; hh < PH; ++hh) ptx::mbar_wait(&o_full[g * PH + hh], (ntiles - 1) & 1);
      tc::fence_after_sync();
#pragma unroll
      for (int ch = 0; ch < DC / 32; ++ch) {
        uint32_t r[32];
        tc::tmem_ld_32x32b_x32(o_tm + col0 + ch * 32, r);
        tc::tmem_wait_ld();
#pragma unroll
        for (int i = 0; i < 32; ++i) w[ch * 32 + i] = __uint_as_float(r[i]);
      }
    } else {
#pragma unroll
      for (int i = 0; i < DC; ++i) w[i] = 0.f;
    }
    const int qrow = q0 + g * T::TQ + row;
    if (qrow < p.n_q) {
      if (!(l_run > 0.f) || !isfinite(l_run)) atomicCAS(p.err, 0, 3);
      const float inv = 1.f / l_run;
      unsigned char* yrow = reinterpret_cast<unsigned char*>(p.y) +
                            2 * (int64_t(b) * p.ys_b + int64_t(h) * p.ys_h + int64_t(qrow) * p.ys_r);
      yrow += 2 * col0;
#pragma unroll
      for (int u = 0; u < DC / 8; ++u) {
        if (col0 + 8 * u >= p.dv) break;
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
        if (p.y_vec && col0 + 8 * u + 8 <= p.dv) {
          *reinterpret_cast<uint4*>(yrow + 16 * u) = pk;
        } else {  // narrow / unaligned output rows: 16-bit element stores
          const uint32_t wds[4] = {pk.x, pk.y, pk.z, pk.w};
#pragma unroll
          for (int e = 0; e < 8; ++e)
            if (col0 + 8 * u + e < p.dv)
              reinterpret_cast<uint16_t*>(yrow)[8 * u + e] =
                  uint16_t(e & 1 ? wds[e >> 1] >> 16 : wds[e >> 1] & 0xffffu);
        }
      }
    }
  }

  tc::fence_before_sync();
  __syncthreads();
  if (warp == T::MMA_WARP) {
    tc::fence_after_sync();
    tc::tmem_dealloc(tmem, T::TMEM_COLS);
  }
}

}  // namespace elsa
