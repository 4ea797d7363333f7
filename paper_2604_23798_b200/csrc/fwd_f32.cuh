// fwd_f32.cuh — K1: the ELSA score-tile producer + per-tile (m,S,W) combine +
// P.V accumulation + output epilogue, strict FP32 on the FMA pipe (no tensor
// cores, no TF32: SPEC.md:343).
//
// Reference path this replaces (scanattn, /root/reference/pkg/src/scanattn):
//   leaf layer  s = (Q K^T) * scale               engine.py:352-358
//   intra-block doubling scan of (m,S,W) leaves   engine.py:148-176, 315-339
//   inter-block pairwise up-sweep                 engine.py:179-199
//   epilogue Y = W / S, normalizer check          engine.py:375-382
//   combine arithmetic                            monoid.py:160-200
//
// B200 design: the leaf is a whole key tile, not a key. For a
// TK-key tile each query row's tile state is formed directly in the
// un-sum-renorm form of Eq. 5: m_t = rowmax(s) by a 16-lane
// shuffle butterfly, S_t = sum 2^(s - m_t), W_t = P_t V_t, and folded into the
// running state with the monoid combine (m,S,W) (+) (m_t,S_t,W_t). Scores live
// in log2 units so every exponential is one MUFU.EX2.
//
// CTA = W consumer warps + 1 TMA producer warp. Each consumer warp owns 2R
// query rows outright (both GEMMs), so the P exchange between the QK^T
// accumulator layout and the P.V operand layout is a warp-private smem round
// trip guarded by __syncwarp — no CTA barrier in the main loop. K/V tiles
// stream through a STAGES-deep ring filled by TMA (cp.async.bulk.tensor,
// mbarrier complete_tx) and released per warp through "empty" mbarriers.
//
// Arithmetic: both GEMMs are register outer products on FFMA2 (sm_100 packed
// fma.rn.f32x2, one broadcast scalar x one row pair; two IEEE FP32 FMAs per
// issue slot). Shared memory delivers lane data at a fixed 128 B/clk/SM
// (an LDS.128 costs 4 wavefronts, or 2 when it touches <= 2 addresses), so
// the R x 4 lane micro-tile sets the smem/FMA balance: R = 8 needs 100% of
// smem bandwidth at full FMA rate, R = 16 needs 75%.
//
// Lane layout inside a consumer warp (lane = 16h + 8rg + k8, g = 8h + k8):
//   rows   r_i = 2R*warp + rg + 2i,  i = 0..R-1   (both GEMMs)
//   GEMM1  keys g + 16j,  j = 0..RK-1             (S micro-tile R x RK)
//   GEMM2  cols 4g .. 4g+3                        (O micro-tile R x 4)
// Shared layouts: raw Q/K rows TMA-boxed D + 4 floats wide (D = 32 / 64 /
// 96 / 128 / 256; the 4 zero columns pad the pitch off the bank period);
// Q^T[d][row position] with each lane's R rows contiguous; P^T[key][row
// position] per warp, pitch 2R+4. V in DV-column slices (32 / 64 / 128;
// wider V runs on grid z). Operands TMA cannot describe go through a cp.async
// copy engine into the same layouts.
#pragma once
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdint>
#include <math_constants.h>

#include <cooperative_groups.h>

#include "merge_f32.cuh"
#include "ptx.cuh"

// Compile-time tuning knobs (defaults = the shipped configuration; the
// variant sweep in tools/variant_sweep.sh builds and times alternatives).
// Unrolls measured on B200 (tools/variant_sweep.sh + tools/ab_time.py):
// deep unrolls let ptxas hoist each step's shared loads well ahead of their
// FFMA2s, which matters with only two consumer warps per SM sub-partition.
//   R = 16 (w8r16): GEMM1 d/4 loop x4, GEMM2 key loop x16   (16K: 49.8 -> 56.5 TFLOP/s)
//   R = 8 (w4r8, w8r8): GEMM1 fully unrolled, GEMM2 x16     (4K: 47.0 -> 54.8)
#ifndef ELSA_G1_UNROLL_R16
#define ELSA_G1_UNROLL_R16 4
#endif
#ifndef ELSA_G1_UNROLL_R8
#define ELSA_G1_UNROLL_R8 16
#endif
#ifndef ELSA_G2_UNROLL_R16
#define ELSA_G2_UNROLL_R16 16
#endif
#ifndef ELSA_G2_UNROLL_R8
#define ELSA_G2_UNROLL_R8 16
#endif
// Snake order (reverse the row-pair order on odd broadcast operands): on for
// every kernel except the d, dv <= 64 w8r8 family, where source order without
// it measured +0.4% at 8K-16K (profiles/round2_ab_variants.txt; -0.15% for
// w4r8 at 4K, so the others keep it). ELSA_SNAKE=0/1 forces it everywhere.
#ifndef ELSA_SNAKE
#define ELSA_SNAKE -1
#endif
#ifndef ELSA_EPI_UNROLL
#define ELSA_EPI_UNROLL 1  // staged-epilogue row-chunk loop (w4r8)
#endif
constexpr int kEpiUnroll = ELSA_EPI_UNROLL;
#ifndef ELSA_CONSUMER_REGS
#define ELSA_CONSUMER_REGS 224
#endif
#ifndef ELSA_PRODUCER_SLEEP_NS
#define ELSA_PRODUCER_SLEEP_NS 256  // back-off between the producer's empty-slot polls
#endif
#ifndef ELSA_PRODUCER_REGS
#define ELSA_PRODUCER_REGS 40
#endif

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
  float c;  // |scale| * log2(e)
  int neg;  // scale < 0: fold the sign into Q^T
  int kv_begin, kv_end;
  int bh_begin;  // first flattened (b, h) index of this launch (row batching)
  int split_keys;  // keys per split: split s covers [kv_begin + s*split_keys, +split_keys) ∩ [.., kv_end)
  int qtiles;
  int mode;
  int y_vec;  // float4 stores to Y legal
  float* pm;
  float* pS;
  float* pW;
  int64_t part_stride;  // state slots between consecutive splits in the partial buffers
  int64_t row_stride;   // state slots between consecutive rows (1, or nblocks for blockwise)
  int pw_pitch;         // floats per row of pW
  int pw_vec;           // float4 stores to pW legal
  int* err;
  unsigned long long* trace;  // ELSA_TRACE builds: per-warp phase timestamps
  // Tail split (final-output plans whose last wave is partly empty): CTAs
  // blockIdx.x >= tail_first are key pieces of the units from tail_first on,
  // tail_splits per unit of tail_split_keys keys each, writing log2 partial
  // states at workspace row (row - tail_row0) for a K2 merge of those rows.
  int tail_first, tail_splits, tail_split_keys;
  int64_t tail_row0;
  int64_t grid_units;  // grid x when != 0 (tail-split launches)
  int q_vec, k_vec, v_vec;    // copy engine: 16-byte aligned rows (base and strides)
};

// Phase-timestamp instrumentation (compiled in only with -DELSA_TRACE): for
// CTAs 0..kTraceCtas-1 each consumer warp records globaltimer at 5 points of
// each of its first kTraceTiles tiles: before the full-barrier wait, after it,
// after GEMM1, after the softmax/combine, after GEMM2.
constexpr int kTraceCtas = 4;
constexpr int kTraceTiles = 32;
constexpr int kTracePoints = 5;
constexpr int kTraceMaxCtas = 8192;  // CTA start/end stamps follow the per-warp block
constexpr size_t kTraceWords = size_t(kTraceCtas) * 16 * kTraceTiles * kTracePoints + 3 * kTraceMaxCtas;
__device__ __forceinline__ void trace_cta(const FwdParams& p, int what) {
#ifdef ELSA_TRACE
  const unsigned cta = blockIdx.x + gridDim.x * blockIdx.y;
  if (cta < kTraceMaxCtas && threadIdx.x == 0) {
    unsigned long long ts;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(ts));
    unsigned smid;
    asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
    unsigned long long* base = p.trace + size_t(kTraceCtas) * 16 * kTraceTiles * kTracePoints;
    base[3 * cta + what] = ts;
    if (what == 0) base[3 * cta + 2] = smid;
  }
#else
  (void)p; (void)what;
#endif
}
__device__ __forceinline__ void trace_mark(const FwdParams& p, int warp, int t, int point) {
#ifdef ELSA_TRACE
  if (blockIdx.x < kTraceCtas && blockIdx.y == 0 && t < kTraceTiles && (threadIdx.x & 31) == 0) {
    unsigned long long ts;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(ts));
    p.trace[((blockIdx.x * 16 + warp) * kTraceTiles + t) * kTracePoints + point] = ts;
  }
#else
  (void)p; (void)warp; (void)t; (void)point;
#endif
}

template <int W_, int TK_, int STAGES_, int R_, int D_ = 64, int DV_ = 64>
struct FwdTraits {
  static constexpr int W = W_;
  static constexpr int TK = TK_;
  static constexpr int STAGES = STAGES_;
  static constexpr int R = R_;            // query rows per lane
  static constexpr int RP = R / 2;        // row pairs per lane
  static constexpr int WR = 2 * R;        // query rows per warp
  static constexpr int D = D_;            // padded head width of Q/K: 64, 96, 128 or 256
  static constexpr int DV = DV_;          // V columns per CTA (32, 64 or 128); wider V runs as slices (grid z)
  static constexpr int CV = DV / 16;      // GEMM2 columns per lane
  static constexpr int VW = DV >= 64 ? 4 : DV / 16;  // V floats per lane per load (segment 0)
  static constexpr int NVL = DV == 96 ? 2 : DV / (16 * VW);  // V loads per key per lane
  // A lane's GEMM2 columns come in segments: segment q covers columns
  // SEG_BASE(q) + SEG_W(q) g + c, c < SEG_W(q), accumulators SEG_C0(q) + c.
  // DV = 32: (0, 2); 64: (0, 4); 96: (0, 4) (64, 2); 128: (0, 4) (64, 4);
  // 256: four 4-wide segments at 0, 64, 128, 192.
  static constexpr int NSEG = DV == 96 ? 2 : NVL;
  __host__ __device__ static constexpr int SEG_W(int q) { return DV == 96 ? (q == 0 ? 4 : 2) : VW; }
  __host__ __device__ static constexpr int SEG_BASE(int q) { return DV == 96 ? 64 * q : 16 * VW * q; }
  __host__ __device__ static constexpr int SEG_C0(int q) { return DV == 96 ? 4 * q : VW * q; }
  static constexpr int TQ = WR * W;
  static constexpr int QP = D + 4;        // raw Q / K row pitch in floats (272 B; TMA box width)
  static constexpr int QTP = TQ;          // Q^T pitch: Qt[d][row position]
  static constexpr int VP = DV;           // V row pitch
  static constexpr int PTP = WR + 4;      // P^T pitch: Pt[key][row position]
  static constexpr int RK = TK / 16;      // keys per lane in GEMM1
  static constexpr int QT_FLOATS = D * QTP;
  static constexpr int K_FLOATS = TK * QP;
  static constexpr int V_FLOATS = TK * VP;
  // P^T in two key halves (GEMM2 of the first half runs before the second
  // half is stored) when the whole-tile P area would not fit next to a
  // 128-wide V ring and a 128-wide Q^T
  static constexpr bool kHalfP =
      size_t(D * TQ + STAGES * (TK * (D + 4) + TK * DV) + W * TK * PTP) * 4 + 64 > 227 * 1024;
  static constexpr int PH = kHalfP ? 2 : 1;  // P passes per tile
  static constexpr int P_FLOATS = W * (TK / PH) * PTP;  // also the raw-Q TMA landing zone
  static constexpr int QRAW_FLOATS = TQ * QP;
  // Warp specialisation. R = 8: one producer warp, registers uniform.
  // R = 16: a whole producer warpgroup (4 warps, only one issues TMA) so that
  // setmaxnreg can move registers from producers to consumers — the register
  // file is split per SM sub-partition (16K entries each, warps assigned
  // round-robin), so 9 warps would cap every warp at 168 registers.
  // DV = 128: the 128-column W accumulator needs the same register split
  // (with 8 consumer warps; 4 consumer warps already launch at 255).
#ifndef ELSA_W8R8_REGSPLIT
#define ELSA_W8R8_REGSPLIT 0  // experiment: producer warpgroup + 224-register consumers for w8r8
#endif
  static constexpr bool kRegSplit =
      R >= 16 || (DV > 64 && W > 4) || (ELSA_W8R8_REGSPLIT && W == 8 && R == 8 && D <= 64);
  static constexpr int PRODUCER_WARPS = kRegSplit ? 4 : 1;
  static constexpr int THREADS = (W + PRODUCER_WARPS) * 32;
  // two CTAs per SM when a 4-warp CTA's shared memory leaves room for two
  static constexpr int MIN_CTAS =
      (W <= 4 && R <= 8 &&
       2 * (size_t(D * TQ + STAGES * (TK * (D + 4) + TK * DV) + W * (TK / PH) * PTP) * 4 + 64) <=
           227 * 1024)
          ? 2
          : 1;
  static constexpr int WARPS_PER_SMSP = (MIN_CTAS * (W + PRODUCER_WARPS) + 3) / 4;
  // launch-time register cap (per-SMSP file / warps resident on it, granule 8)
  static constexpr int MAX_REGS = (16384 / (WARPS_PER_SMSP * 32)) / 8 * 8 > 255
                                      ? 255
                                      : (16384 / (WARPS_PER_SMSP * 32)) / 8 * 8;
  static constexpr int PRODUCER_REGS = ELSA_PRODUCER_REGS;
  static constexpr int G1_UNROLL = R >= 16 ? ELSA_G1_UNROLL_R16 : ELSA_G1_UNROLL_R8;
  static constexpr int G2_UNROLL = R >= 16 ? ELSA_G2_UNROLL_R16 : ELSA_G2_UNROLL_R8;
  // Phase-offsetting the two warps of each SMSP (see `lagged` in the kernel)
  // measured no gain on B200 (per-warp phase trace) and costs registers, so
  // it is compiled out.
#ifndef ELSA_LAG
#define ELSA_LAG 0
#endif
  static constexpr bool kLag = ELSA_LAG != 0 && W >= 8 && !kHalfP;
  static constexpr int CONSUMER_REGS = ELSA_CONSUMER_REGS;  // after setmaxnreg.inc (R = 16 only)
  static_assert(!kRegSplit || (W % 4 == 0), "register split needs whole consumer warpgroups");
  static_assert(!kRegSplit || PRODUCER_REGS + (W / 4) * CONSUMER_REGS <= 512,
                "per-SMSP register budget after setmaxnreg");
  // setmaxnreg only redistributes the launch allocation (MAX_REGS per warp):
  // the consumers' growth must not exceed what the producer warp releases,
  // or the .inc blocks forever (240/32 hung on B200)
  static_assert(!kRegSplit || (W / 4) * (CONSUMER_REGS - MAX_REGS) <= MAX_REGS - PRODUCER_REGS,
                "setmaxnreg growth exceeds the registers the producers release");
  // Where the raw Q box lands before the transpose: the P area when it fits
  // (d <= 64); for the wide-Q kernels the K ring (the producer then waits on a
  // "Q consumed" barrier before its first K/V load).
  // If it fits neither (d = 256 with 128-row tiles), the copy engine writes Q
  // straight into Q^T (kQtDirect; no TMA for such kernels).
  static constexpr bool kQtDirect = QRAW_FLOATS > P_FLOATS && QRAW_FLOATS > STAGES * K_FLOATS;
  static constexpr bool kQrawInK = QRAW_FLOATS > P_FLOATS && !kQtDirect;
  // cluster merge: W[TQ][64] | m[TQ] | S[TQ] of the CTA's rows fit in its K/V ring
  static constexpr bool kCluStateFits = size_t(TQ) * 66 <= size_t(STAGES) * (K_FLOATS + V_FLOATS);
  static constexpr size_t BAR_OFFSET =
      size_t(QT_FLOATS + STAGES * (K_FLOATS + V_FLOATS) + P_FLOATS) * 4;
  static constexpr size_t SMEM_BYTES = BAR_OFFSET + (2 * STAGES + 2) * 8;
  static constexpr uint32_t KV_TX_BYTES = uint32_t(K_FLOATS + V_FLOATS) * 4;
  static constexpr uint32_t Q_TX_BYTES = uint32_t(QRAW_FLOATS) * 4;
  static_assert(TK % 16 == 0, "TK must be a multiple of 16");
  static_assert(R % 4 == 0, "R must be a multiple of 4 (float4 row groups)");
  static_assert(DV == 32 || DV == 64 || DV == 96 || DV == 128 || DV == 256, "V slice width");
  static_assert(RK % PH == 0, "P halves split the lane's GEMM1 keys evenly");
  static_assert(TQ <= 256, "TMA box rows <= 256");
  static_assert(!kQtDirect || QP > 256, "direct Q^T copies only in copy-engine-only kernels");
  static_assert(SMEM_BYTES <= 227 * 1024, "shared memory budget");
  static_assert((QT_FLOATS * 4) % 128 == 0 && (K_FLOATS * 4) % 128 == 0 &&
                    (V_FLOATS * 4) % 128 == 0,
                "TMA destinations must stay 128-byte aligned");
};

// Rows [0, ROWS) of PITCH floats into shared memory with cp.async (LDGSTS):
// row r reads `width` floats at src + r * stride while r < valid_rows; the
// rest of every row and the invalid rows are zero-filled. 16-byte copies when
// `vec` (16-byte aligned rows), else 4-byte ones.
template <int ROWS, int PITCH>
__device__ __forceinline__ void async_rows(float* dst, const float* src, int64_t stride,
                                           int valid_rows, int width, bool vec, int lane) {
  static_assert(PITCH % 4 == 0, "16-byte chunks");
  const uint32_t d0 = ptx::smem_u32(dst);
  if (vec) {
    constexpr int C4 = PITCH / 4;
    for (int idx = lane; idx < ROWS * C4; idx += 32) {
      const int r = idx / C4, c = (idx - r * C4) * 4;
      const int n = (r < valid_rows && c < width) ? (width - c < 4 ? width - c : 4) : 0;
      ptx::cp_async16(d0 + uint32_t(idx) * 16, n ? src + int64_t(r) * stride + c : src,
                      uint32_t(n) * 4);
    }
  } else {
    for (int idx = lane; idx < ROWS * PITCH; idx += 32) {
      const int r = idx / PITCH, c = idx - r * PITCH;
      const bool ok = r < valid_rows && c < width;
      ptx::cp_async4(d0 + uint32_t(idx) * 4, ok ? src + int64_t(r) * stride + c : src,
                     ok ? 4u : 0u);
    }
  }
}

template <class T>
__device__ __forceinline__ void producer_generic(const FwdParams& p, float* Qraw, float* Qt,
                                                 float* Ks,
                                                 float* Vs, uint64_t* full, uint64_t* empty,
                                                 uint64_t* qbar, uint64_t* qfree, int b, int h,
                                                 int q0, int col0, int split_lo, int ntiles,
                                                 int lane) {
  // Copy engine for operands TMA cannot describe (misaligned base or strides,
  // zero strides, rows wider than a 256-element box): the whole producer warp
  // issues asynchronous copies into the same smem layouts as the TMA boxes
  // (zero-filled), and every lane's completion arrives on the stage barrier
  // (count 32).
  const float* qg = p.q + int64_t(b) * p.qs_b + int64_t(h) * p.qs_h + int64_t(q0) * p.qs_r;
  if constexpr (T::kQtDirect) {
    // element (row rr, column c) straight to Q^T[c][pos(rr)] (4-byte copies,
    // lanes over rows so the shared stores stay conflict-free; once per CTA)
    const uint32_t qt0 = ptx::smem_u32(Qt);
    const int valid = p.n_q - q0;
    for (int idx = lane; idx < T::TQ * T::D; idx += 32) {
      const int c = idx / T::TQ, rr = idx - c * T::TQ, r = rr % T::WR;
      const int pos = rr - r + T::R * (r & 1) + (r >> 1);
      const bool ok = rr < valid && c < p.d;
      ptx::cp_async4(qt0 + uint32_t(c * T::QTP + pos) * 4, ok ? qg + int64_t(rr) * p.qs_r + c : qg,
                     ok ? 4u : 0u);
    }
  } else {
    async_rows<T::TQ, T::QP>(Qraw, qg, p.qs_r, p.n_q - q0, p.d, p.q_vec, lane);
  }
  ptx::cp_async_arrive(qbar);
  if constexpr (T::kQrawInK) ptx::mbar_wait(qfree, 0);  // raw Q sits in the K ring until transposed
  const float* kg = p.k + int64_t(b) * p.ks_b + int64_t(h) * p.ks_h;
  const float* vg = p.v + int64_t(b) * p.vs_b + int64_t(h) * p.vs_h + col0;
  for (int t = 0; t < ntiles; ++t) {
    const int s = t % T::STAGES;
    if (t >= T::STAGES) ptx::mbar_wait_backoff(&empty[s], ((t / T::STAGES) - 1) & 1, ELSA_PRODUCER_SLEEP_NS);
    const int key0 = split_lo + t * T::TK;
    async_rows<T::TK, T::QP>(Ks + s * T::K_FLOATS, kg + int64_t(key0) * p.ks_r, p.ks_r,
                             p.n_kv - key0, p.d, p.k_vec, lane);
    async_rows<T::TK, T::VP>(Vs + s * T::V_FLOATS, vg + int64_t(key0) * p.vs_r, p.vs_r,
                             p.n_kv - key0, p.dv - col0, p.v_vec, lane);
    ptx::cp_async_arrive(&full[s]);
  }
}

// Cluster-merge epilogue (fwd_f32_kernel<..., CL = true>). `st` is the CTA's
// K/V ring, free once every consumer warp has folded its last tile: it holds
// this CTA's states W[TQ][64] | m[TQ] | S[TQ] (log2 anchors, exactly the values
// the split path writes to its workspace).
template <class T, int MAXP>
__device__ __forceinline__ void cluster_merge_rows(const FwdParams& p, float* st, int parts,
                                                   int rank, int warp, int lane, int b, int h,
                                                   int q0) {
  namespace cg = cooperative_groups;
  cg::cluster_group cluster = cg::this_cluster();
  constexpr int TQ = T::TQ;
  const int rpc = (TQ + parts - 1) / parts;  // rows this CTA finalizes
  const int r0 = rank * rpc;
  const int r1 = r0 + rpc < TQ ? r0 + rpc : TQ;
  for (int lr = r0 + warp; lr < r1; lr += T::W) {
    const int qrow = q0 + lr;
    if (qrow >= p.n_q) break;
    float am[MAXP], aS[MAXP], a0[MAXP], a1[MAXP];
#pragma unroll
    for (int i = 0; i < MAXP; ++i) {
      if (i < parts) {
        const float* peer = cluster.map_shared_rank(st, i);
        am[i] = peer[TQ * 64 + lr];
        aS[i] = peer[TQ * 65 + lr];
        a0[i] = peer[lr * 64 + lane];
        a1[i] = peer[lr * 64 + lane + 32];
      } else {
        am[i] = -CUDART_INF_F;
        aS[i] = 0.f;
        a0[i] = 0.f;
        a1[i] = 0.f;
      }
    }
    merge_tree_regs<MAXP>(am, aS, a0, a1, parts, true);
    const float s = aS[0];
    if (!(s > 0.f) || !isfinite(s)) {
      if (lane == 0) atomicCAS(p.err, 0, 3);
    }
    float* yrow = p.y + int64_t(b) * p.ys_b + int64_t(h) * p.ys_h + int64_t(qrow) * p.ys_r;
    if (lane < p.dv) yrow[lane] = __fdiv_rn(a0[0], s);
    if (lane + 32 < p.dv) yrow[lane + 32] = __fdiv_rn(a1[0], s);
  }
}

template <class T>
__device__ __forceinline__ void cluster_merge_epilogue(const FwdParams& p, float* st,
                                                       const float (&mrow)[T::R],
                                                       const ptx::f32x2 (&l2)[T::RP],
                                                       const ptx::f32x2 (&o2)[T::RP][T::CV],
                                                       int warp, int lane, int rg, int g, int b,
                                                       int h, int q0) {
  namespace cg = cooperative_groups;
  constexpr int TQ = T::TQ, R = T::R, RP = T::RP, WR = T::WR;
  // every consumer warp is done reading the ring (its last GEMM2) before any
  // warp overwrites it with states
  asm volatile("bar.sync 1, %0;" ::"r"(T::W * 32) : "memory");
  float lrow[R];  // row normalizers, all rows' butterflies interleaved (same order per row)
#pragma unroll
  for (int ip = 0; ip < RP; ++ip) {
    lrow[2 * ip] = ptx::lo2(l2[ip]);
    lrow[2 * ip + 1] = ptx::hi2(l2[ip]);
  }
#pragma unroll
  for (int sh = 1; sh <= 16; sh <<= 1) {
    if (sh == 8) continue;  // lane bit 3 is the row group
#pragma unroll
    for (int i = 0; i < R; ++i) lrow[i] += __shfl_xor_sync(0xffffffffu, lrow[i], sh);
  }
#pragma unroll
  for (int ip = 0; ip < RP; ++ip) {
#pragma unroll
    for (int half = 0; half < 2; ++half) {
      const int i = 2 * ip + half;
      const float l = lrow[i];
      const int lr = warp * WR + rg + 2 * i;
      float4 w;
      w.x = half ? ptx::hi2(o2[ip][0]) : ptx::lo2(o2[ip][0]);
      w.y = half ? ptx::hi2(o2[ip][1]) : ptx::lo2(o2[ip][1]);
      w.z = half ? ptx::hi2(o2[ip][2]) : ptx::lo2(o2[ip][2]);
      w.w = half ? ptx::hi2(o2[ip][3]) : ptx::lo2(o2[ip][3]);
      *reinterpret_cast<float4*>(st + lr * 64 + 4 * g) = w;
      if (g == 0) {
        st[TQ * 64 + lr] = mrow[i];
        st[TQ * 65 + lr] = l;
      }
    }
  }
  cg::cluster_group cluster = cg::this_cluster();
  cluster.sync();  // release our states / acquire the peers'
  const int parts = int(cluster.num_blocks());
  const int rank = int(cluster.block_rank());
  if (parts <= 8)
    cluster_merge_rows<T, 8>(p, st, parts, rank, warp, lane, b, h, q0);
  else
    cluster_merge_rows<T, 16>(p, st, parts, rank, warp, lane, b, h, q0);
  cluster.sync();  // peers are done reading our states before this CTA exits
}

__device__ __forceinline__ float f4(const float4& v, int c) {
  return c == 0 ? v.x : (c == 1 ? v.y : (c == 2 ? v.z : v.w));
}

// Y = W / S without a slow-path branch per element: with r = __frcp_rn(S),
// Markstein's correction step q0 = W r, rem = fma(-S, q0, W) (exact),
// q = fma(rem, r, q0) is the correctly rounded quotient when nothing
// under/overflows. Used only when the whole warp's rows are in the guarded
// range (S in [1, 2^31), |W| = 0 or in [2^-100, 2^100)); there it equals
// __fdiv_rn bit for bit (4.6e9 random pairs over every exponent checked on a
// B200, tools/microbench/div_check.cu); otherwise the epilogue divides with
// __fdiv_rn. One reciprocal per row instead of a full division per element,
// and straight-line code the scheduler can overlap across rows.
__device__ __forceinline__ bool div_fast_ok_den(float s) { return s >= 1.f && s < 0x1p31f; }
__device__ __forceinline__ bool div_fast_ok_num(float w) {
  const float a = fabsf(w);
  return a == 0.f || (a >= 0x1p-100f && a < 0x1p100f);
}
__device__ __forceinline__ float div_rn_rcp(float w, float s, float r) {
  const float q0 = w * r;
  const float rem = fmaf(-s, q0, w);
  return fmaf(rem, r, q0);
}

// CL (cluster split merge): the kv splits of one query tile are the CTAs of
// one thread-block cluster (cluster dims (1, splits, 1)). Instead of writing
// partial states to a global workspace for a second (K2) launch, each CTA
// leaves its rows' (m, S, W) in its own shared memory; after a cluster
// barrier CTA r merges rows [r * TQ / splits, ...) by reading every peer's
// states over distributed shared memory (DSMEM) with K2's fixed tree, and
// writes Y. Same states, same tree, same arithmetic as K1 + K2: bitwise equal.
// ACC (the long-chain kernels): two-level W accumulation. Each tile's P V
// goes into a fresh accumulator that is folded into the running W once per
// tile (W = W * corr + W_t, one FFMA2 in place of the rescale's FMUL2), so
// every W element's sequential rounding chain is TK keys inside the tile plus
// one step per tile, instead of every key the CTA folds. Measured at 1M keys
// with one 16384-tile chain: max row error 3.1e-6 vs 2.6e-5 without
// (profiles/round2_chain_error_acc.txt); ~1% slower per tile, so the planner
// uses it where chains are long (it then needs no kv splits for the error
// bound).
template <int W_, int TK_, int STAGES_, int R_, bool kTMA, int D_ = 64, int DV_ = 64,
          bool CL = false, bool ACC = false>
__global__ void __maxnreg__((FwdTraits<W_, TK_, STAGES_, R_, D_, DV_>::MAX_REGS))
    fwd_f32_kernel(const __grid_constant__ FwdParams p, const __grid_constant__ CUtensorMap tmQ,
                   const __grid_constant__ CUtensorMap tmK,
                   const __grid_constant__ CUtensorMap tmV) {
  using T = FwdTraits<W_, TK_, STAGES_, R_, D_, DV_>;
  static_assert(!(kTMA && T::kQtDirect), "direct Q^T needs the copy engine");
  static_assert(!CL || (DV_ == 64 && !T::kRegSplit && T::kCluStateFits),
                "cluster merge: one 64-column slice, every warp alive, states fit the ring");
  constexpr int TK = T::TK, QP = T::QP, QTP = T::QTP, VP = T::VP, PTP = T::PTP, RK = T::RK;
  constexpr int R = T::R, RP = T::RP, WR = T::WR;
  constexpr bool kSnake =
      ELSA_SNAKE >= 0 ? ELSA_SNAKE != 0 : !(W_ == 8 && R_ == 8 && D_ == 64 && DV_ == 64);
  using ptx::f32x2;

  extern __shared__ __align__(1024) unsigned char smem_raw[];
  float* Qt = reinterpret_cast<float*>(smem_raw);
  float* Ks = Qt + T::QT_FLOATS;
  float* Vs = Ks + T::STAGES * T::K_FLOATS;
  float* Ps = Vs + T::STAGES * T::V_FLOATS;
  // raw Q lands in the P area (or the K ring) and is transposed out before first use
  float* Qraw = T::kQrawInK ? Ks : Ps;
  uint64_t* full = reinterpret_cast<uint64_t*>(smem_raw + T::BAR_OFFSET);
  uint64_t* empty = full + T::STAGES;
  uint64_t* qbar = empty + T::STAGES;
  uint64_t* qfree = qbar + 1;

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;

  // (selects, not a branch: every value stays warp-uniform)
  const int bx = int(blockIdx.x);
  const bool tail = p.tail_splits > 0 && bx >= p.tail_first;
  const int tsp = tail ? p.tail_splits : 1;
  const int tj = (tail ? bx - p.tail_first : 0) / tsp;
  const int unit = tail ? p.tail_first + tj : bx;
  const int split = tail ? bx - p.tail_first - tj * tsp : int(blockIdx.y);
  const int split_keys = tail ? p.tail_split_keys : p.split_keys;
  const int mode = tail ? int(kModePartialLog2) : p.mode;
  const int qtile = unit % p.qtiles;
  const int bh_rel = unit / p.qtiles;
  const int bh = bh_rel + p.bh_begin;
  const int b = bh / p.H;
  const int h = bh - b * p.H;
  const int q0 = qtile * T::TQ;
  const int col0 = int(blockIdx.z) * T::DV;  // this CTA's column slice of V / W / Y

  const int64_t lo64 = int64_t(p.kv_begin) + int64_t(split) * split_keys;
  const int split_lo = int(lo64 < p.kv_end ? lo64 : p.kv_end);
  const int kv_hi = int(lo64 + split_keys < p.kv_end ? lo64 + split_keys : p.kv_end);
  const int ntiles = kv_hi > split_lo ? (kv_hi - split_lo + TK - 1) / TK : 0;

  trace_cta(p, 0);
  // a K2 merge launched as this grid's programmatic dependent may start its
  // CTAs now (they wait in griddepcontrol.wait for this grid's completion)
  ptx::griddep_launch_dependents();
  if (threadIdx.x == 0) {
    // TMA: one arrive.expect_tx per stage; copy engine: one arrival per lane
    for (int s = 0; s < T::STAGES; ++s) {
      ptx::mbar_init(&full[s], kTMA ? 1 : 32);
      ptx::mbar_init(&empty[s], T::W);
    }
    ptx::mbar_init(qbar, kTMA ? 1 : 32);
    if constexpr (T::kQrawInK) ptx::mbar_init(qfree, T::W);
    ptx::fence_barrier_init();
  }
  __syncthreads();

  if (warp >= T::W) {
    // ---------------- producer warp(group) ----------------
    if constexpr (T::kRegSplit) {
      asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;" ::"n"(T::PRODUCER_REGS));
      if (warp != T::W) return;
    }
    if constexpr (kTMA) {
      if (lane == 0) {
        ptx::prefetch_tmap(&tmQ);
        ptx::prefetch_tmap(&tmK);
        ptx::prefetch_tmap(&tmV);
        ptx::mbar_arrive_expect_tx(qbar, T::Q_TX_BYTES);
        ptx::tma_load_4d(Qraw, &tmQ, qbar, 0, q0, h, b);
        if constexpr (T::kQrawInK) ptx::mbar_wait(qfree, 0);
        for (int t = 0; t < ntiles; ++t) {
          const int s = t % T::STAGES;
          if (t >= T::STAGES) ptx::mbar_wait_backoff(&empty[s], ((t / T::STAGES) - 1) & 1, ELSA_PRODUCER_SLEEP_NS);
          const int key0 = split_lo + t * TK;
          ptx::mbar_arrive_expect_tx(&full[s], T::KV_TX_BYTES);
          ptx::tma_load_4d(Ks + s * T::K_FLOATS, &tmK, &full[s], 0, key0, h, b);
          ptx::tma_load_4d(Vs + s * T::V_FLOATS, &tmV, &full[s], col0, key0, h, b);
        }
      }
    } else {
      producer_generic<T>(p, Qraw, Qt, Ks, Vs, full, empty, qbar, qfree, b, h, q0, col0,
                          split_lo, ntiles, lane);
    }
    if constexpr (CL) {
      // every thread of the cluster takes part in both cluster barriers
      cooperative_groups::this_cluster().sync();  // peers' states written
      cooperative_groups::this_cluster().sync();  // peers done reading ours
    }
    return;
  }

  // ---------------- consumer warps ----------------
  if constexpr (T::kRegSplit) asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;" ::"n"(T::CONSUMER_REGS));
  // lane = 16*h + 8*rg + k8: each half-warp holds both row groups and 8 of the
  // 16 key/column groups
  const int rg = (lane >> 3) & 1;                 // row group: rows rg + 2i
  const int g = ((lane >> 4) << 3) | (lane & 7);  // key group (GEMM1) / column group (GEMM2)

  // Q^T, once per CTA: each warp transposes its own 2R rows out of the raw TMA
  // box into Qt[d][pos], pos = 2R*warp + R*(r & 1) + (r >> 1) for local row r,
  // so a lane's R rows (rg + 2i) are R consecutive floats (R/4 LDS.128 per d).
  // The sign of a negative scale is folded in here (x = (-q).k * |c|).
  ptx::mbar_wait(qbar, 0);
  if constexpr (T::kQtDirect) {
    // Q^T arrived directly; fold a negative scale's sign into this warp's rows
    if (p.neg) {
      for (int c = lane; c < T::D; c += 32) {
        float* row = Qt + c * QTP + warp * WR;
#pragma unroll
        for (int u = 0; u < WR; ++u) row[u] = -row[u];
      }
    }
    __syncwarp();
  } else {
    const float sgn = p.neg ? -1.f : 1.f;
    constexpr int LPR = 32 / WR;         // lanes per row (2 for R = 8, 1 for R = 16)
    constexpr int DSPAN = T::D / LPR;    // d values per lane
    const int r = lane / LPR;
    const int dh = (lane % LPR) * DSPAN;
    const float* src = Qraw + (warp * WR + r) * QP + dh;
    float* dst = Qt + (warp * WR + R * (r & 1) + (r >> 1)) + dh * QTP;
#pragma unroll
    for (int c = 0; c < DSPAN / 4; ++c) {
      const float4 v = ptx::lds128(src + 4 * c);
      dst[(4 * c + 0) * QTP] = v.x * sgn;
      dst[(4 * c + 1) * QTP] = v.y * sgn;
      dst[(4 * c + 2) * QTP] = v.z * sgn;
      dst[(4 * c + 3) * QTP] = v.w * sgn;
    }
  }
  if constexpr (T::kQtDirect) {
    // nothing to hand back: raw Q never occupied the P area or the K ring
  } else if constexpr (T::kQrawInK) {
    // raw Q occupies the K ring: hand it back to the producer
    __syncwarp();
    if (lane == 0) ptx::mbar_arrive(qfree);
  } else {
    // every consumer warp must finish reading raw Q before any warp writes P over it
    asm volatile("bar.sync 1, %0;" ::"r"(T::W * 32) : "memory");
  }

  const float* qt = Qt + warp * WR + rg * R;
  float* pw = Ps + warp * (TK / T::PH) * PTP;
  const float* ptr = pw + rg * R;
  const float c2 = p.c;  // |scale| * log2(e) > 0
  const f32x2 cc = ptx::pack2(c2, c2);

  // Row pairs: lane rows (rg + 2i), i = 0..R-1, are held as R/2 packed pairs
  // ip = (i = 2ip, 2ip+1), so every GEMM FMA is an FFMA2 outer-product step.
  constexpr int CV = T::CV;
  f32x2 o2[RP][CV];  // W accumulator: [row pair][column VW g + 16 VW (c / VW) + c % VW]
  float mrow[R];    // running anchors (log2 units)
  f32x2 l2[RP];     // running normalizer partials (this lane's keys)
  // ELSA_TILE_ACC: this tile's P V (t2) and the running side's factor (corr_t)
  constexpr bool kTileAcc = ACC && CV <= 8;  // V slices of <= 128 columns
  constexpr bool kLagK = T::kLag && !kTileAcc;  // per-tile accumulation assumes the in-order GEMM2
  f32x2 t2[RP][kTileAcc ? CV : 1];
  f32x2 corr_t[RP];
#pragma unroll
  for (int ip = 0; ip < RP; ++ip) {
    l2[ip] = 0ull;
#pragma unroll
    for (int c = 0; c < CV; ++c) o2[ip][c] = 0ull;
  }
#pragma unroll
  for (int i = 0; i < R; ++i) mrow[i] = -CUDART_INF_F;

  // ---- GEMM2 of tile tt: W += P V on FFMA2, o2[ip][c] += v_j[c] (bcast) *
  // Pt[j][row pair ip] over the keys [k0, k0 + TK / PH) whose P^T is in the
  // P area (rows jj - k0)
  auto gemm2 = [&](int tt, int k0) {
    const int st = tt % T::STAGES;
    const float* vs = Vs + st * T::V_FLOATS;
    if constexpr (kTileAcc) {
      if (k0 == 0) {
#pragma unroll
        for (int ip = 0; ip < RP; ++ip)
#pragma unroll
          for (int c = 0; c < CV; ++c) t2[ip][c] = 0ull;
      }
    }
#pragma unroll(T::G2_UNROLL)
    for (int jj = 0; jj < TK / T::PH; ++jj) {
      f32x2 pr[RP];
#pragma unroll
      for (int u = 0; u < RP / 2; ++u)
        ptx::lds128x2(ptr + jj * PTP + 4 * u, pr[2 * u], pr[2 * u + 1]);
      float va[CV];
#pragma unroll
      for (int q = 0; q < T::NSEG; ++q) {
        const float* src = vs + (k0 + jj) * VP + T::SEG_BASE(q) + T::SEG_W(q) * g;
        float* dst = va + T::SEG_C0(q);
        if (T::SEG_W(q) == 4) {
          const float4 f = ptx::lds128(src);
          dst[0] = f.x, dst[1] = f.y, dst[2] = f.z, dst[3] = f.w;
        } else {
          const float2 f = *reinterpret_cast<const float2*>(src);
          dst[0] = f.x, dst[1] = f.y;
        }
      }
#pragma unroll
      for (int c = 0; c < CV; ++c) {
        const float vv = va[c];
        const f32x2 vb = ptx::pack2(vv, vv);
#pragma unroll
        for (int u = 0; u < RP; ++u) {
          const int ip = (kSnake && (c & 1)) ? RP - 1 - u : u;
          if constexpr (kTileAcc)
            ptx::ffma2(t2[ip][kTileAcc ? c : 0], vb, pr[ip]);
          else
            ptx::ffma2(o2[ip][c], vb, pr[ip]);
        }
      }
    }
  };
  // ... then release the tile's K/V stage to the producer.
  auto gemm2_release = [&](int tt) {
    const int st = tt % T::STAGES;
    if constexpr (T::DV == 64 && T::PH == 1) {
      // the d <= 64 / dv <= 64 kernels: this exact form (ptxas schedules the
      // generalised loop differently)
      const float* vs = Vs + st * T::V_FLOATS + 4 * g;
      auto key_step = [&](int jj, bool first) {
        f32x2 pr[RP];
#pragma unroll
        for (int u = 0; u < RP / 2; ++u)
          ptx::lds128x2(ptr + jj * PTP + 4 * u, pr[2 * u], pr[2 * u + 1]);
        const float4 vf = ptx::lds128(vs + jj * VP);
#pragma unroll
        for (int c = 0; c < 4; ++c) {
          const float vv = f4(vf, c);
          const f32x2 vb = ptx::pack2(vv, vv);
#pragma unroll
          for (int u = 0; u < RP; ++u) {
            const int ip = (kSnake && (c & 1)) ? RP - 1 - u : u;
            if constexpr (kTileAcc) {
              if (first)
                t2[ip][c] = ptx::fmul2(vb, pr[ip]);
              else
                ptx::ffma2(t2[ip][c], vb, pr[ip]);
            } else {
              ptx::ffma2(o2[ip][c], vb, pr[ip]);
            }
          }
        }
      };
      if constexpr (kTileAcc) {
        // the tile accumulator starts at the first key's products (no zeroing):
        // one peeled block of G2_UNROLL keys, then the unrolled loop
#pragma unroll
        for (int jj = 0; jj < T::G2_UNROLL; ++jj) key_step(jj, jj == 0);
#pragma unroll(T::G2_UNROLL)
        for (int jj = T::G2_UNROLL; jj < TK; ++jj) key_step(jj, false);
      } else {
#pragma unroll(T::G2_UNROLL)
        for (int jj = 0; jj < TK; ++jj) key_step(jj, false);
      }
    } else {
      gemm2(tt, (T::PH - 1) * (TK / T::PH));
    }
    if constexpr (kTileAcc) {
      // fold the tile into the running W: W = W * corr + W_t
#pragma unroll
      for (int ip = 0; ip < RP; ++ip)
#pragma unroll
        for (int c = 0; c < CV; ++c)
          o2[ip][c] = ptx::ffma2r(o2[ip][c], corr_t[ip], t2[ip][kTileAcc ? c : 0]);
    }
    __syncwarp();
    trace_mark(p, warp, tt, 4);
    if (lane == 0) ptx::mbar_arrive(&empty[st]);
  };
  // P^T of the lane's GEMM1 keys j in [j0, j1): key-major, this lane's R rows
  // contiguous -> R/4 STS.128 per key; P area row = key - key offset of the pass
  auto store_p = [&](const f32x2 (&s2)[RP][RK], int j0, int j1) {
#pragma unroll
    for (int j = j0; j < j1; ++j) {
      float* dst = pw + (g + 16 * j - 16 * j0) * PTP + rg * R;
#pragma unroll
      for (int u = 0; u < RP / 2; ++u)
        *reinterpret_cast<ulonglong2*>(dst + 4 * u) =
            make_ulonglong2(s2[2 * u][j], s2[2 * u + 1][j]);
    }
  };

  // Phase offset between the two warps that share an SM sub-partition (warps
  // w and w + 4, W >= 8): the upper half runs GEMM2 of the previous tile
  // before GEMM1 of the current one, so its latency-bound softmax section
  // overlaps the partner's FFMA2 stream instead of coinciding with it.
  const bool lagged = kLagK && warp >= T::W / 2;

  for (int t = 0; t < ntiles; ++t) {
    const int s = t % T::STAGES;
    if (lagged && t > 0) gemm2_release(t - 1);
    trace_mark(p, warp, t, 0);
    ptx::mbar_wait(&full[s], (t / T::STAGES) & 1);
    trace_mark(p, warp, t, 1);
    const float* ks = Ks + s * T::K_FLOATS + g * QP;

    // ---- GEMM1: S = Q K^T on FFMA2: s2[ip][j] += k_j[d] (bcast) * Qt[d][row pair ip]
    f32x2 s2[RP][RK];
#pragma unroll
    for (int ip = 0; ip < RP; ++ip)
#pragma unroll
      for (int j = 0; j < RK; ++j) s2[ip][j] = 0ull;

#pragma unroll(T::G1_UNROLL)
    for (int c = 0; c < T::D / 4; ++c) {
      float4 kf[RK];
#pragma unroll
      for (int j = 0; j < RK; ++j) kf[j] = ptx::lds128(ks + j * 16 * QP + 4 * c);
#pragma unroll
      for (int dd = 0; dd < 4; ++dd) {
        f32x2 q2[RP];
#pragma unroll
        for (int u = 0; u < RP / 2; ++u)
          ptx::lds128x2(qt + (4 * c + dd) * QTP + 4 * u, q2[2 * u], q2[2 * u + 1]);
#pragma unroll
        for (int j = 0; j < RK; ++j) {
          const float kv = f4(kf[j], dd);
          const f32x2 kb = ptx::pack2(kv, kv);
#pragma unroll
          for (int u = 0; u < RP; ++u) {
            const int ip = (kSnake && (j & 1)) ? RP - 1 - u : u;
            ptx::ffma2(s2[ip][j], kb, q2[ip]);
          }
        }
      }
    }
    trace_mark(p, warp, t, 2);

    // ---- mask keys past this split's range ----
    const int key0 = split_lo + t * TK;
    if (key0 + TK > kv_hi) {
#pragma unroll
      for (int j = 0; j < RK; ++j)
        if (key0 + g + 16 * j >= kv_hi) {
          const f32x2 ninf = ptx::pack2(-CUDART_INF_F, -CUDART_INF_F);
#pragma unroll
          for (int ip = 0; ip < RP; ++ip) s2[ip][j] = ninf;
        }
    }

    // ---- tile state (m_t, S_t) and the monoid combine into the running row state.
    // Anchors in log2 units: m = fl(max_j acc_j * c). Each exponent is one FMA
    // acc*c - m (exact product, one rounding), so near-max keys carry an
    // absolute exponent error ~u*|s - m| rather than ~u*|s|.
#pragma unroll
    for (int ip = 0; ip < RP; ++ip) {
      float mlo = ptx::lo2(s2[ip][0]), mhi = ptx::hi2(s2[ip][0]);
#pragma unroll
      for (int j = 1; j < RK; ++j) {
        mlo = fmaxf(mlo, ptx::lo2(s2[ip][j]));
        mhi = fmaxf(mhi, ptx::hi2(s2[ip][j]));
      }
#pragma unroll
      for (int sh = 1; sh <= 16; sh <<= 1) {
        if (sh == 8) continue;  // lane bit 3 is the row group
        mlo = fmaxf(mlo, __shfl_xor_sync(0xffffffffu, mlo, sh));
        mhi = fmaxf(mhi, __shfl_xor_sync(0xffffffffu, mhi, sh));
      }
      const float nlo = fmaxf(mrow[2 * ip], mlo * c2);
      const float nhi = fmaxf(mrow[2 * ip + 1], mhi * c2);
      // running side's factor; exp2(-inf) = 0 for the identity start state
      const f32x2 corr =
          ptx::pack2(ptx::ex2(mrow[2 * ip] - nlo), ptx::ex2(mrow[2 * ip + 1] - nhi));
      mrow[2 * ip] = nlo;
      mrow[2 * ip + 1] = nhi;
      const f32x2 mneg = ptx::pack2(-nlo, -nhi);
      f32x2 ps = 0ull;
#pragma unroll
      for (int j = 0; j < RK; ++j) {
        const f32x2 x = ptx::ffma2r(s2[ip][j], cc, mneg);
        float xlo, xhi;
        ptx::unpack2(x, xlo, xhi);
        s2[ip][j] = ptx::pack2(ptx::ex2(xlo), ptx::ex2(xhi));  // s2 now holds p
        ps = j == 0 ? s2[ip][j] : ptx::fadd2(ps, s2[ip][j]);
      }
      l2[ip] = ptx::ffma2r(l2[ip], corr, ps);
      if constexpr (kTileAcc) {
        corr_t[ip] = corr;
      } else {
#pragma unroll
        for (int c = 0; c < CV; ++c) o2[ip][c] = ptx::fmul2(o2[ip][c], corr);
      }
    }
    if constexpr (T::kHalfP) {
      // first key half through the (half-size) P area, then the second half
      static_assert(!kLagK, "halved P assumes the in-order GEMM2");
      store_p(s2, 0, RK / 2);
      __syncwarp();
      gemm2(t, 0);
      __syncwarp();  // every lane is done reading the first half
      store_p(s2, RK / 2, RK);
    } else {
      // P^T: key-major, this lane's R rows contiguous -> R/4 STS.128 per key
#pragma unroll
      for (int j = 0; j < RK; ++j) {
        float* dst = pw + (g + 16 * j) * PTP + rg * R;
#pragma unroll
        for (int u = 0; u < RP / 2; ++u)
          *reinterpret_cast<ulonglong2*>(dst + 4 * u) =
              make_ulonglong2(s2[2 * u][j], s2[2 * u + 1][j]);
      }
    }
    __syncwarp();
    trace_mark(p, warp, t, 3);
    if (!lagged) gemm2_release(t);
  }
  if (lagged && ntiles > 0) gemm2_release(ntiles - 1);

  if constexpr (CL) {
    cluster_merge_epilogue<T>(p, Ks, mrow, l2, o2, warp, lane, rg, g, b, h, q0);
    return;
  }

  // ---------------- epilogue ----------------
  trace_mark(p, warp, ntiles, 0);
  // row normalizers: the butterfly over the 16 key-group lanes for all R rows
  // at once (independent shuffles overlap; the per-row order of additions is
  // unchanged)
  float lrow[R];
#pragma unroll
  for (int ip = 0; ip < RP; ++ip) {
    lrow[2 * ip] = ptx::lo2(l2[ip]);
    lrow[2 * ip + 1] = ptx::hi2(l2[ip]);
  }
#pragma unroll
  for (int sh = 1; sh <= 16; sh <<= 1) {
    if (sh == 8) continue;  // lane bit 3 is the row group
#pragma unroll
    for (int i = 0; i < R; ++i) lrow[i] += __shfl_xor_sync(0xffffffffu, lrow[i], sh);
  }
  trace_mark(p, warp, ntiles, 1);
  // final output: quotients with one reciprocal per row when the whole warp
  // is in the fast division's range (warp-uniform), written over o2
  bool qdone = false;
  constexpr bool kStaged = T::DV == 64 && T::W <= 4 && (TK / T::PH) * PTP >= WR * 66;
  // (the staged w4r8 epilogue only: in the unrolled w8r8 one it measured
  // slower, H16 1K 100.3 vs 98.3 us, profiles/round2_ab_div.txt)
  if (kStaged && mode == kModeFinal) {
    bool ok = true;
#pragma unroll
    for (int i = 0; i < R; ++i) ok = ok && div_fast_ok_den(lrow[i]);
#pragma unroll
    for (int ip = 0; ip < RP; ++ip)
#pragma unroll
      for (int c = 0; c < CV; ++c)
        ok = ok && div_fast_ok_num(ptx::lo2(o2[ip][c])) && div_fast_ok_num(ptx::hi2(o2[ip][c]));
    if (__all_sync(0xffffffffu, ok)) {
      float rr[R];
#pragma unroll
      for (int i = 0; i < R; ++i) rr[i] = __frcp_rn(lrow[i]);
#pragma unroll
      for (int ip = 0; ip < RP; ++ip)
#pragma unroll
        for (int c = 0; c < CV; ++c)
          o2[ip][c] = ptx::pack2(div_rn_rcp(ptx::lo2(o2[ip][c]), lrow[2 * ip], rr[2 * ip]),
                                 div_rn_rcp(ptx::hi2(o2[ip][c]), lrow[2 * ip + 1], rr[2 * ip + 1]));
      qdone = true;
    }
  }
  if constexpr (kStaged) {
    // Staged epilogue (64-column slices): the warp parks its rows' W, S and
    // anchor in its own P area, then one compact loop writes each row as 16
    // coalesced float4 chunks (Y = W / S with the same IEEE division, or the
    // partial state). A fully unrolled per-lane epilogue was ~25 KB of code
    // run once per CTA. Measured (profiles/round2_ab_epilogue.txt): BERT-base
    // 145.4 -> 141.3 us, H16 4K +0.8%; the w8r8 kernels keep the unrolled
    // form (their main loop's schedule moved with it: 16K -0.5%).
    float* stg = pw;  // [WR][64] W | S[WR] | m[WR]
    float* sl = stg + WR * 64;
    float* sm = sl + WR;
#pragma unroll
    for (int ip = 0; ip < RP; ++ip) {
#pragma unroll
      for (int half = 0; half < 2; ++half) {
        const int i = 2 * ip + half, r = rg + 2 * i;
        const float4 w = half ? make_float4(ptx::hi2(o2[ip][0]), ptx::hi2(o2[ip][1]),
                                            ptx::hi2(o2[ip][2]), ptx::hi2(o2[ip][3]))
                              : make_float4(ptx::lo2(o2[ip][0]), ptx::lo2(o2[ip][1]),
                                            ptx::lo2(o2[ip][2]), ptx::lo2(o2[ip][3]));
        *reinterpret_cast<float4*>(stg + r * 64 + 4 * g) = w;
        if (g == 0) {
          sl[r] = lrow[i];
          sm[r] = mrow[i];
        }
      }
    }
    __syncwarp();
    const int qw = q0 + warp * WR;
    const int rows_here = p.n_q - qw < WR ? p.n_q - qw : WR;
#pragma unroll(kEpiUnroll)
    for (int idx = lane; idx < rows_here * 16; idx += 32) {
      const int r = idx >> 4, c4 = idx & 15;
      const int qrow = qw + r;
      const float4 w = *reinterpret_cast<const float4*>(stg + r * 64 + 4 * c4);
      const float l = sl[r];
      const int col = col0 + 4 * c4;
      if (mode == kModeFinal) {
        // engine.py:377-378: the normalizer must be finite and positive
        if (c4 == 0 && (!(l > 0.f) || !isfinite(l))) atomicCAS(p.err, 0, 3);
        const float4 y = qdone ? w
                               : make_float4(__fdiv_rn(w.x, l), __fdiv_rn(w.y, l),
                                             __fdiv_rn(w.z, l), __fdiv_rn(w.w, l));
        float* yrow = p.y + int64_t(b) * p.ys_b + int64_t(h) * p.ys_h + int64_t(qrow) * p.ys_r;
        if (p.y_vec && col + 3 < p.dv) {
          *reinterpret_cast<float4*>(yrow + col) = y;
        } else {
          if (col < p.dv) yrow[col] = y.x;
          if (col + 1 < p.dv) yrow[col + 1] = y.y;
          if (col + 2 < p.dv) yrow[col + 2] = y.z;
          if (col + 3 < p.dv) yrow[col + 3] = y.w;
        }
      } else {
        const int64_t row = int64_t(bh_rel) * p.n_q + qrow;  // relative to this batch
        const int64_t sidx =
            int64_t(split) * p.part_stride + (tail ? row - p.tail_row0 : row) * p.row_stride;
        if (c4 == 0 && col0 == 0) {  // m and S are the same in every column slice
          const float m = (mode == kModePartialNat) ? sm[r] * 0.69314718055994531f : sm[r];
          p.pm[sidx] = m;
          p.pS[sidx] = l;
        }
        float* wrow = p.pW + sidx * p.pw_pitch;
        if (p.pw_vec && col + 3 < p.dv) {
          *reinterpret_cast<float4*>(wrow + col) = w;
        } else {
          if (col < p.dv) wrow[col] = w.x;
          if (col + 1 < p.dv) wrow[col + 1] = w.y;
          if (col + 2 < p.dv) wrow[col + 2] = w.z;
          if (col + 3 < p.dv) wrow[col + 3] = w.w;
        }
      }
    }
    trace_mark(p, warp, ntiles, 2);
    trace_cta(p, 1);
    return;
  }
#pragma unroll
  for (int ip = 0; ip < RP; ++ip) {
#pragma unroll
    for (int half = 0; half < 2; ++half) {
      const int i = 2 * ip + half;
      const float l = lrow[i];
      float o[CV];
#pragma unroll
      for (int c = 0; c < CV; ++c) o[c] = half ? ptx::hi2(o2[ip][c]) : ptx::lo2(o2[ip][c]);
      const int qrow = q0 + warp * WR + rg + 2 * i;
      if (qrow >= p.n_q) continue;
      if (mode == kModeFinal) {
        // engine.py:377-378: the normalizer must be finite and positive
        if (!(l > 0.f) || !isfinite(l)) {
          if (g == 0) atomicCAS(p.err, 0, 3);
        }
        float* yrow = p.y + int64_t(b) * p.ys_b + int64_t(h) * p.ys_h + int64_t(qrow) * p.ys_r;
        float yv[CV];
#pragma unroll
        for (int c = 0; c < CV; ++c) yv[c] = qdone ? o[c] : __fdiv_rn(o[c], l);
#pragma unroll
        for (int v4 = 0; v4 < T::NSEG; ++v4) {
          if constexpr (T::DV != 96) {  // uniform segments (compile-time width)
            constexpr int VW = T::VW;
            const int col = col0 + 16 * VW * v4 + VW * g;
            const float* yq = yv + VW * v4;
            if (p.y_vec && col + VW - 1 < p.dv) {
              if constexpr (VW == 4)
                *reinterpret_cast<float4*>(yrow + col) = make_float4(yq[0], yq[1], yq[2], yq[3]);
              else
                *reinterpret_cast<float2*>(yrow + col) = make_float2(yq[0], yq[1]);
            } else {
#pragma unroll
              for (int c = 0; c < VW; ++c)
                if (col + c < p.dv) yrow[col + c] = yq[c];
            }
          } else {  // DV = 96: a 4-wide and a 2-wide segment
            const int VW = T::SEG_W(v4);
            const int col = col0 + T::SEG_BASE(v4) + VW * g;
            const float* yq = yv + T::SEG_C0(v4);
            if (p.y_vec && col + VW - 1 < p.dv) {
              if (VW == 4)
                *reinterpret_cast<float4*>(yrow + col) = make_float4(yq[0], yq[1], yq[2], yq[3]);
              else
                *reinterpret_cast<float2*>(yrow + col) = make_float2(yq[0], yq[1]);
            } else {
              for (int c = 0; c < VW; ++c)
                if (col + c < p.dv) yrow[col + c] = yq[c];
            }
          }
        }
      } else {
        const int64_t row = int64_t(bh_rel) * p.n_q + qrow;  // relative to this batch
        const int64_t idx =
            int64_t(split) * p.part_stride + (tail ? row - p.tail_row0 : row) * p.row_stride;
        if (g == 0 && col0 == 0) {  // m and S are the same in every column slice
          const float m = (mode == kModePartialNat) ? mrow[i] * 0.69314718055994531f : mrow[i];
          p.pm[idx] = m;
          p.pS[idx] = l;
        }
        float* wrow = p.pW + idx * p.pw_pitch;
#pragma unroll
        for (int v4 = 0; v4 < T::NSEG; ++v4) {
          if constexpr (T::DV != 96) {  // uniform segments (compile-time width)
            constexpr int VW = T::VW;
            const int col = col0 + 16 * VW * v4 + VW * g;
            const float* oq = o + VW * v4;
            if (p.pw_vec && col + VW - 1 < p.dv) {
              if constexpr (VW == 4)
                *reinterpret_cast<float4*>(wrow + col) = make_float4(oq[0], oq[1], oq[2], oq[3]);
              else
                *reinterpret_cast<float2*>(wrow + col) = make_float2(oq[0], oq[1]);
            } else {
#pragma unroll
              for (int c = 0; c < VW; ++c)
                if (col + c < p.dv) wrow[col + c] = oq[c];
            }
          } else {  // DV = 96: a 4-wide and a 2-wide segment
            const int VW = T::SEG_W(v4);
            const int col = col0 + T::SEG_BASE(v4) + VW * g;
            const float* oq = o + T::SEG_C0(v4);
            if (p.pw_vec && col + VW - 1 < p.dv) {
              if (VW == 4)
                *reinterpret_cast<float4*>(wrow + col) = make_float4(oq[0], oq[1], oq[2], oq[3]);
              else
                *reinterpret_cast<float2*>(wrow + col) = make_float2(oq[0], oq[1]);
            } else {
              for (int c = 0; c < VW; ++c)
                if (col + c < p.dv) wrow[col + c] = oq[c];
            }
          }
        }
      }
    }
  }
  trace_mark(p, warp, ntiles, 2);
  trace_cta(p, 1);
}

}  // namespace elsa
