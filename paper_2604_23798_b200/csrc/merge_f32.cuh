// merge_f32.cuh — K2: fixed balanced (+)-tree over P partial (m,S,W) states per
// query row, plus the W/S epilogue.
//
// Reference semantics restated on the device:
//   combine arithmetic, identity guard, tie rule   monoid.py:160-200
//     m = max(m_a, m_b); f_x = exp(m_x - m) (0 when m_x = -inf);
//     W = W_a*f_a + W_b*f_b; S = S_a*f_a + S_b*f_b   (products rounded, then added:
//     no FMA contraction, exactly as the numpy ufunc sequence)
//   tree shape: adjacent pairs bottom-up, odd tail passes through
//                                                  monoid.py:234-265 (= the
//                                                  up-sweep on 2^k inputs, engine.py:179-199)
//   finalize: Y = W / S with S finite and > 0       engine.py:375-382
//
// One warp per query row and 64-column slice (grid y; wider dv runs as
// several slices that recompute the same m/S tree); lane c owns columns
// 64y + c and 64y + c + 32. The
// tree lives in registers (MAXP slots, fully unrolled, predicated on the live
// count) so the reduction order is fixed by `parts` alone: bitwise
// deterministic and independent of scheduling.
#pragma once
#include <cuda_runtime.h>
#include <cstdint>
#include <math_constants.h>

namespace elsa {

struct MergeParams {
  const float* m;
  const float* S;
  const float* W;
  int parts;
  int64_t rows;
  int dv;
  int w_pitch;          // floats per row in W
  int64_t part_stride;  // rows between consecutive parts
  int log2_domain;      // anchors in log2 units (internal split workspace)
  int finalize;
  // finalize output: row -> (b,h,q) via n_q and H, strided Y
  float* y;
  int H, n_q;
  int bh_begin;  // finalize: row r maps to flattened (b, h) = (r + row0) / n_q + bh_begin
  int64_t row0;  // finalize: output row of workspace row 0 (tail-split merges)
  int64_t ys_b, ys_h, ys_r;
  // non-finalize output (dense [rows][out_pitch])
  float* m_out;
  float* S_out;
  float* W_out;
  int out_pitch;
  int out_log2_to_nat;  // convert log2-domain anchors to natural units on output
  int* err;
};

constexpr int kMergeMaxParts = 32;

__device__ __forceinline__ float merge_factor(float mx, float m, bool log2_domain) {
  // identity guard (monoid.py:189-191): an identity operand contributes 0
  if (mx == -CUDART_INF_F) return 0.f;
  return log2_domain ? exp2f(mx - m) : expf(mx - m);
}

// Balanced pairwise tree over k live slots, in place: slot i <- slot 2i (+)
// slot 2i+1, odd tail passes through; the result is in slot 0.
template <int MAXP>
__device__ __forceinline__ void merge_tree_regs(float (&am)[MAXP], float (&aS)[MAXP],
                                                float (&a0)[MAXP], float (&a1)[MAXP], int k,
                                                bool lg) {
  constexpr int LEVELS = MAXP <= 1 ? 0 : (MAXP <= 2 ? 1 : (MAXP <= 4 ? 2 : (MAXP <= 8 ? 3 : (MAXP <= 16 ? 4 : 5))));
#pragma unroll
  for (int level = 0; level < LEVELS; ++level) {
    if (k <= 1) break;
#pragma unroll
    for (int i = 0; i < MAXP / 2; ++i) {
      if (2 * i + 1 < k) {
        const float ma = am[2 * i], mb = am[2 * i + 1];
        const float mm = fmaxf(ma, mb);
        const float fa = merge_factor(ma, mm, lg);
        const float fb = merge_factor(mb, mm, lg);
        a0[i] = __fadd_rn(__fmul_rn(a0[2 * i], fa), __fmul_rn(a0[2 * i + 1], fb));
        a1[i] = __fadd_rn(__fmul_rn(a1[2 * i], fa), __fmul_rn(a1[2 * i + 1], fb));
        aS[i] = __fadd_rn(__fmul_rn(aS[2 * i], fa), __fmul_rn(aS[2 * i + 1], fb));
        am[i] = mm;
      } else if (2 * i + 1 == k) {  // odd tail passes through
        am[i] = am[2 * i];
        aS[i] = aS[2 * i];
        a0[i] = a0[2 * i];
        a1[i] = a1[2 * i];
      }
    }
    k = (k + 1) >> 1;
  }
}

template <int MAXP>
__global__ void __launch_bounds__(256) merge_f32_kernel(const MergeParams p) {
  // launched as K1's programmatic dependent: the partial states are complete
  // and visible once the forward grid has finished
  asm volatile("griddepcontrol.wait;" ::: "memory");
  const int64_t row = int64_t(blockIdx.x) * (blockDim.x >> 5) + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (row >= p.rows) return;
  const bool lg = p.log2_domain != 0;

  float am[MAXP], aS[MAXP], a0[MAXP], a1[MAXP];
  const int c0 = int(blockIdx.y) * 64 + lane, c1 = c0 + 32;
#pragma unroll
  for (int i = 0; i < MAXP; ++i) {
    if (i < p.parts) {
      const int64_t idx = int64_t(i) * p.part_stride + row;
      am[i] = p.m[idx];
      aS[i] = p.S[idx];
      const float* w = p.W + idx * p.w_pitch;
      a0[i] = c0 < p.dv ? w[c0] : 0.f;
      a1[i] = c1 < p.dv ? w[c1] : 0.f;
    } else {
      am[i] = -CUDART_INF_F;
      aS[i] = 0.f;
      a0[i] = 0.f;
      a1[i] = 0.f;
    }
  }

  merge_tree_regs<MAXP>(am, aS, a0, a1, p.parts, lg);

  if (p.finalize) {
    const float s = aS[0];
    if (!(s > 0.f) || !isfinite(s)) {
      if (lane == 0) atomicCAS(p.err, 0, 3);
    }
    float* yrow;
    if (p.n_q > 0) {
      const int64_t orow = row + p.row0;
      const int64_t bh_rel = orow / p.n_q;
      const int64_t q = orow - bh_rel * p.n_q;
      const int64_t bh = bh_rel + p.bh_begin;
      const int64_t b = bh / p.H, h = bh - b * p.H;
      yrow = p.y + b * p.ys_b + h * p.ys_h + q * p.ys_r;
    } else {
      yrow = p.y + row * p.dv;
    }
    if (c0 < p.dv) yrow[c0] = __fdiv_rn(a0[0], s);
    if (c1 < p.dv) yrow[c1] = __fdiv_rn(a1[0], s);
  } else {
    if (lane == 0 && blockIdx.y == 0) {
      p.m_out[row] = p.out_log2_to_nat ? am[0] * 0.69314718055994531f : am[0];
      p.S_out[row] = aS[0];
    }
    float* w = p.W_out + row * p.out_pitch;
    if (c0 < p.dv) w[c0] = a0[0];
    if (c1 < p.dv) w[c1] = a1[0];
  }
}

// Peer-memory merge (the fused exchange): every rank wrote the
// natural-log (m, S, W) states of its owned key chunks for ALL query rows into
// its own symmetric (peer-mapped) buffer; rank j merges its row slice by
// reading chunk c's state straight from rank c / per's buffer over NVLink
// (P2P loads) and combining in registers in global chunk order with the same
// fixed tree as K2 — the all_to_all, its staging copy and the separate merge
// launch collapse into one kernel. Bitwise identical to the NCCL path (same
// states, same tree, same arithmetic).
constexpr int kMaxPeers = 16;

struct PeerMergeParams {
  const float* m[kMaxPeers];  // rank r's buffers (peer-mapped device pointers)
  const float* S[kMaxPeers];
  const float* W[kMaxPeers];
  int ranks, per_rank;        // chunks = ranks * per_rank, <= kMergeMaxParts
  int64_t rows_total;         // rows per chunk array (chunk stride in a rank's buffer)
  int64_t row_lo, rows;       // the slice this rank finalizes
  int dv;
  float* y;                   // [rows][dv]
  int* err;
};

template <int MAXP>
__global__ void __launch_bounds__(256) merge_peers_kernel(const PeerMergeParams p) {
  const int64_t r = int64_t(blockIdx.x) * (blockDim.x >> 5) + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (r >= p.rows) return;
  const int64_t row = p.row_lo + r;
  const int parts = p.ranks * p.per_rank;
  float am[MAXP], aS[MAXP], a0[MAXP], a1[MAXP];
  const int c0 = int(blockIdx.y) * 64 + lane, c1 = c0 + 32;
#pragma unroll
  for (int i = 0; i < MAXP; ++i) {
    if (i < parts) {
      const int rk = i / p.per_rank, l = i - rk * p.per_rank;
      const int64_t idx = int64_t(l) * p.rows_total + row;
      am[i] = p.m[rk][idx];
      aS[i] = p.S[rk][idx];
      const float* w = p.W[rk] + idx * p.dv;
      a0[i] = c0 < p.dv ? w[c0] : 0.f;
      a1[i] = c1 < p.dv ? w[c1] : 0.f;
    } else {
      am[i] = -CUDART_INF_F;
      aS[i] = 0.f;
      a0[i] = 0.f;
      a1[i] = 0.f;
    }
  }
  merge_tree_regs<MAXP>(am, aS, a0, a1, parts, false);
  const float s = aS[0];
  if (!(s > 0.f) || !isfinite(s)) {
    if (lane == 0) atomicCAS(p.err, 0, 3);
  }
  float* yrow = p.y + r * p.dv;
  if (c0 < p.dv) yrow[c0] = __fdiv_rn(a0[0], s);
  if (c1 < p.dv) yrow[c1] = __fdiv_rn(a1[0], s);
}

}  // namespace elsa
