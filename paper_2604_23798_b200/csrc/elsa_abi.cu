// elsa_abi.cu — host side of libelsa.so: argument validation, TMA descriptor
// encoding, kv-split planning and stream-ordered launches behind the C-ABI
// declared in include/elsa.h.
//
// Reference behaviour mirrored here:
//   ShapeError on bad geometry/config           errors.py:8, tensorio.py:83-98, engine.py:78-89
//   NumericalError on a bad normalizer          errors.py:12, engine.py:377-378 (device word)
//   scan_depth / depth bound                    engine.py:43-55
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>

#include <cmath>
#include <cstdint>
#include <cstdlib>
#include <cstdio>
#include <cstring>
#include <string>
#include <mutex>

#include "elsa.h"
#include "ffma_peak.cuh"
#include "fwd_f32.cuh"
#include "fwd_tc.cuh"
#include "merge_f32.cuh"
#include "block_scan_f32.cuh"

namespace elsa {
__device__ int g_device_error;
}

using namespace elsa;

namespace {

constexpr int kMaxDevices = 64;
#ifndef ELSA_EXPERIMENTAL_W8R4
#define ELSA_EXPERIMENTAL_W8R4 0  // the w8r4 experiment config (round2_notes.md)
#endif
#ifndef ELSA_EXPERIMENTAL_TC_CS2
#define ELSA_EXPERIMENTAL_TC_CS2 0  // K5 with two softmax warps per row (round2_notes.md)
#endif
#ifndef ELSA_EXPERIMENTAL_TC_TK64
#define ELSA_EXPERIMENTAL_TC_TK64 0  // K5 with 64-key tiles at d = 128 (round2_notes.md)
#endif
#ifndef ELSA_W8R8_STAGES
#define ELSA_W8R8_STAGES 3  // K/V ring depth of w8r8 (3: +0.5% at 8K-16K, tools/ab_time.py; w4r8 at 3 stages loses its second CTA per SM: 4K 54.6 -> 49.5)
#endif
#ifndef ELSA_D32_STAGES
#define ELSA_D32_STAGES 4  // K/V ring depth of w8r8d32v32 (2: 11.50, 3: 11.47, 4: 11.45 ms at B1 H16 n16K)
#endif
#ifndef ELSA_W4R8_STAGES
#define ELSA_W4R8_STAGES 2
#endif
constexpr int kAttrSlots = 48;
constexpr int kMaxSplits = kMergeMaxParts;
constexpr double kLog2e = 1.4426950408889634074;

thread_local int t_last_launches = 0;
thread_local char t_last_cuda_error[256] = "";

#ifdef ELSA_TRACE
unsigned long long* g_trace = nullptr;
unsigned long long* trace_buffer() {
  if (!g_trace) {
    cudaMalloc(&g_trace, sizeof(unsigned long long) * kTraceWords);
    cudaMemset(g_trace, 0, sizeof(unsigned long long) * kTraceWords);
  }
  return g_trace;
}
#else
unsigned long long* trace_buffer() { return nullptr; }
#endif

int cuda_fail(cudaError_t e, const char* where) {
  std::snprintf(t_last_cuda_error, sizeof(t_last_cuda_error), "%s: %s (%d)", where,
                cudaGetErrorString(e), int(e));
  return ELSA_ERR_CUDA;
}

constexpr int kCluAttrBase = kAttrSlots;  // attribute slots of the cluster-merge kernels
struct DeviceCache {
  bool ready = false;
  int sms = 0;
  int* err = nullptr;
  bool attr[2 * kAttrSlots] = {};  // forward configs x TMA flag, then the tc kernels; cluster kernels
  int clusters[3][17];             // max active clusters: [w4r8, w8r8, w8r4][splits], -1 = unknown
  DeviceCache() {
    for (auto& row : clusters)
      for (int& x : row) x = -1;
  }
};
DeviceCache g_dev[kMaxDevices];
std::mutex g_mu;

PFN_cuTensorMapEncodeTiled_v12000 g_encode = nullptr;
std::once_flag g_encode_once;

PFN_cuTensorMapEncodeTiled_v12000 encoder() {
  std::call_once(g_encode_once, [] {
    void* fn = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) ==
            cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      g_encode = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
  });
  return g_encode;
}

int current_device_cache(DeviceCache** out) {
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= kMaxDevices) return ELSA_ERR_CUDA;
  std::lock_guard<std::mutex> lk(g_mu);
  DeviceCache& c = g_dev[dev];
  if (!c.ready) {
    if (cudaDeviceGetAttribute(&c.sms, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess)
      return ELSA_ERR_CUDA;
    void* p = nullptr;
    if (cudaGetSymbolAddress(&p, g_device_error) != cudaSuccess) return ELSA_ERR_CUDA;
    c.err = static_cast<int*>(p);
    c.ready = true;
  }
  *out = &c;
  return ELSA_OK;
}

// ---------------------------------------------------------------------------
// Forward kernel configurations. The planner picks one per shape (see
// plan_for); ELSA_FWD_CFG forces one (benchmarking aid).
//   w4r8 : 4 consumer warps x 16 rows (TQ = 64),  2 CTAs / SM, 8 rows per lane
//   w8r8 : 8 consumer warps x 16 rows (TQ = 128), 1 CTA / SM
//   w8r16: 8 consumer warps x 32 rows (TQ = 256), 1 CTA / SM, 16 rows per
//          lane (setmaxnreg register split with a producer warpgroup)
//   w8r8d128: w8r8 with Q/K 128 floats wide (64 < d <= 128; Q^T and the K
//          ring fill 200 KB, raw Q is staged in the K ring)
//   w8r8d96, w8r8d96v128: the same with Q/K 96 wide (64 < d <= 96)
//   w8r8d256 (dv <= 64), w4r8d256v128: 128 < d <= 256: 8 (4) consumer warps
//          x 16 rows, 32-key tiles, the copy engine (TMA boxes stop at 256
//          elements, the padded pitch is 260; w8r8d256 copies Q straight into
//          Q^T and passes P in two halves to fit 227 KB), 1 CTA / SM
//   w8r8v128, w8r8d128v128: 128 V columns per CTA (dv > 64): a 128-column
//          W accumulator (setmaxnreg register split with a producer
//          warpgroup); with d > 64 too, P^T goes through shared memory in
//          two key halves so that everything fits 227 KB
// dv wider than the configuration's V width runs as column slices (grid z),
// each recomputing its tile's scores: m / S are identical across slices.
// ---------------------------------------------------------------------------
enum CfgId {
  kCfgW4R8 = 0,
  kCfgW8R16 = 1,
  kCfgW8R8 = 2,
  kCfgCount = 3,  // the d <= 64 configurations the planner chooses from
  kCfgW8R8D128 = 3,
  kCfgW8R8V128 = 4,
  kCfgW8R8D128V128 = 5,
  kCfgW8R8D96 = 6,  // 64 < d <= 96: Q/K 96 wide (GEMM1 3/4 of the d = 128 kernel's)
  kCfgW8R8D96V128 = 7,
  kCfgW8R8D256 = 8,  // 128 < d <= 256, dv <= 64: 8 consumer warps, 32-key tiles, copy engine
  kCfgW4R8D256V128 = 9,
  kCfgW8R8D32V32 = 10,  // d, dv <= 32: Q/K 32 wide, 32 V columns (2 per lane)
  kCfgW8R8D96V96 = 11,  // 64 < d, dv <= 96: 96 V columns (6 per lane)
  kCfgW8R8V96 = 12,     // d <= 64 < dv <= 96
  kCfgW8R8D128V96 = 13, // 96 < d <= 128, 64 < dv <= 96
  kCfgW4R8D256V256 = 14,  // 128 < d <= 256, dv > 128: 256 V columns per CTA (one S per tile)
  kCfgW8R8Acc = 15,  // w8r8 with the two-level W accumulator (long per-CTA chains)
  kCfgW8R4 = 16,     // 8 consumer warps x 8 rows (TQ 64); experiment, built with
                     // -DELSA_EXPERIMENTAL_W8R4=1 only (measured no faster, round2_notes.md)
  kCfgAuto = -1
};
int cfg_dv(int cfg) {
  if (cfg == kCfgW8R8D32V32) return 32;
  if (cfg == kCfgW4R8D256V256) return 256;
  if (cfg == kCfgW8R8D96V96 || cfg == kCfgW8R8V96 || cfg == kCfgW8R8D128V96) return 96;
  return (cfg == kCfgW8R8V128 || cfg == kCfgW8R8D128V128 || cfg == kCfgW8R8D96V128 ||
          cfg == kCfgW4R8D256V128)
             ? 128
             : 64;
}
// the one configuration for heads wider than 64 (-1: choose among the d <= 64 ones)
int wide_cfg(int64_t d, int64_t dv) {
  const bool v = dv > 64;
  if (d <= 32 && dv <= 32) return int(kCfgW8R8D32V32);
  if (d <= 64) return v ? (dv <= 96 ? int(kCfgW8R8V96) : int(kCfgW8R8V128)) : -1;
  if (d <= 96) return v ? (dv <= 96 ? int(kCfgW8R8D96V96) : int(kCfgW8R8D96V128)) : int(kCfgW8R8D96);
  if (d <= 128)
    return v ? (dv <= 96 ? int(kCfgW8R8D128V96) : int(kCfgW8R8D128V128)) : int(kCfgW8R8D128);
  if (!v) return int(kCfgW8R8D256);
  return dv <= 128 ? int(kCfgW4R8D256V128) : int(kCfgW4R8D256V256);
}
constexpr int64_t kMaxD = 256;
constexpr int64_t kMaxDv = 4096;
int64_t dv_slices(int64_t dv) { return (dv + 63) / 64; }

int cfg_from_name(const char* e) {
  if (e && !std::strcmp(e, "w4r8")) return int(kCfgW4R8);
  if (e && !std::strcmp(e, "w8r8")) return int(kCfgW8R8);
  if (e && !std::strcmp(e, "w8r16")) return int(kCfgW8R16);
  if (e && !std::strcmp(e, "w8r8acc")) return int(kCfgW8R8Acc);
#if ELSA_EXPERIMENTAL_W8R4
  if (e && !std::strcmp(e, "w8r4")) return int(kCfgW8R4);
#endif
  return int(kCfgAuto);
}
// ELSA_FWD_CFG (or elsa_dev_force_config) forces one of the d <= 64 configurations
int g_forced_cfg = cfg_from_name(std::getenv("ELSA_FWD_CFG"));
int forced_cfg() { return g_forced_cfg; }

struct CfgInfo {
  int tq, tk, ctas_per_sm;
  double tile_us;  // SM-time for one TQ x 64 tile (measured on B200 at 1965 MHz)
  double cta_us;   // per-CTA prologue/epilogue SM-time
};
// Relative-error least-squares fit of tools/plan_sweep.py timings (every
// config x kv split, n = 512 .. 16384; profiles/round1_plan_sweep.txt) to the
// cost model of plan_for; all three configs now move ~24 query-row tiles per
// microsecond per SM (w8r16 nudged up 0.7% so 16K keeps the measured-faster w8r8).
CfgInfo cfg_info(int cfg) {
  switch (cfg) {
    case kCfgW8R16:
      return {256, 64, 1, 10.75, 7.6};
    case kCfgW8R8:
      return {128, 64, 1, 5.355, 4.1};
    case kCfgW8R8Acc:  // ~1% more per tile than w8r8 (profiles/round2_ab_acc.txt)
      return {128, 64, 1, 5.41, 4.1};
    case kCfgW8R4:  // provisional (to be fitted)
      return {64, 64, 1, 3.2, 3.0};
    // wide-head configurations: scaled from the w8r8 fit by GEMM length
    // (d + dv relative to 128), not fitted — the planner only compares kv
    // split counts within one of them
    case kCfgW8R8D128:  // GEMM1 twice as long: ~1.5x the d = 64 tile
      return {128, 64, 1, 8.03, 6.2};
    case kCfgW8R8V128:  // GEMM2 twice as long
      return {128, 64, 1, 8.03, 6.2};
    case kCfgW8R8D128V128:
      return {128, 64, 1, 10.7, 8.2};
    case kCfgW8R8D96:
      return {128, 64, 1, 6.7, 5.2};
    case kCfgW8R8D96V128:
      return {128, 64, 1, 9.4, 7.2};
    case kCfgW8R8D256:  // 128 x 32 tiles
      return {128, 32, 1, 8.0, 6.0};
    case kCfgW4R8D256V128:
      return {64, 32, 1, 5.0, 4.0};
    case kCfgW8R8D32V32:  // half the d = 64 GEMMs
      return {128, 64, 1, 3.0, 3.0};
    case kCfgW8R8D96V96:
      return {128, 64, 1, 8.0, 6.0};
    case kCfgW8R8V96:
      return {128, 64, 1, 6.7, 5.2};
    case kCfgW8R8D128V96:
      return {128, 64, 1, 9.4, 7.2};
    case kCfgW4R8D256V256:
      return {64, 32, 1, 7.0, 5.0};
    default:
      return {64, 64, 2, 2.711, 1.6};
  }
}

bool valid_shape(const elsa_shape* s) {
  if (!s) return false;
  if (s->B < 0 || s->H < 0 || s->n_q < 0 || s->n_kv < 1) return false;
  if (s->d < 1 || s->d > kMaxD || s->dv < 1 || s->dv > kMaxDv) return false;
  const int64_t lim = int64_t(1) << 31;
  if (s->B >= lim || s->H >= lim || s->n_q >= lim || s->n_kv >= lim) return false;
  if (s->B * s->H >= lim) return false;
  for (int i = 0; i < 3; ++i)
    if (s->q_stride[i] < 0 || s->k_stride[i] < 0 || s->v_stride[i] < 0 || s->y_stride[i] < 0)
      return false;
  return true;
}

int64_t ceil_div(int64_t a, int64_t b) { return (a + b - 1) / b; }

// Launch plan (config + kv split count). Cost model in microseconds, fitted
// to B200 measurements (tools/plan_sweep.py):
//   ceil(CTAs * s / 148) * (ceil(tiles / s) * tile_us + cta_us)     forward kernel
// + [s > 1] * (10.8 + 45.6e-6 * s * rows)                            partial states + merge
// minimised over the configs and s <= min(tiles, 32), with
// s >= ceil(tiles / kMaxChainTiles) so no CTA folds more than kMaxChainTiles
// tiles sequentially (bounded chain depth; the rest is the log-depth tree).
// 1024 tiles: chains of ~1100 tiles measured 5.5e-6 at 1M (bound 1.7e-5) and
// 4.0e-6 at 64K (bound 1.3e-5); 16384 measured 2.5e-5 (over).
// The two-level-accumulator kernel (kCfgW8R8Acc) rounds each W element over
// 64 keys + one step per tile: one 16384-tile chain measured 3.1e-6 at 1M
// (0.18 x bound; profiles/round2_chain_error_acc.txt), so its cap is 16384.
constexpr int64_t kMaxChainTiles = 1024;
constexpr int64_t kMaxChainTilesAcc = 16384;
int64_t chain_cap(int cfg) { return cfg == kCfgW8R8Acc ? kMaxChainTilesAcc : kMaxChainTiles; }
// Split workspace budget for auto planning (partial states are
// (2 + 64 * dv slices) * 4 B per row per split): 4 GiB unless ELSA_MAX_WORKSPACE_MB says
// otherwise. Explicit kv_splits requests are not capped.
int64_t workspace_budget() {
  static const int64_t b = [] {
    const char* e = std::getenv("ELSA_MAX_WORKSPACE_MB");
    const long long mb = e ? std::atoll(e) : 4096;
    return int64_t(mb > 0 ? mb : 0) * 1024 * 1024;
  }();
  return b;
}

struct Plan {
  int cfg;
  int splits;
  int64_t heads_per_batch;  // (b, h) pairs per launch batch when splits > 1
  bool cluster = false;     // splits merged inside one launch over DSMEM (no workspace, no K2)
  int tail_s = 0;           // tail split: units >= tail_first run as tail_s key pieces
  int64_t tail_first = 0;   // (final output, splits == 1; K2 merges the tail rows)
};

// Tail split (ELSA_TAIL: 0 off, 1 cost model (default), s >= 2 force s pieces):
// when the units of a one-split plan leave the last wave partly empty, the
// units of that wave run as s key pieces each (more, shorter CTAs) and a K2
// merges their rows. Same launch, same kernel code for the full units.
int g_tail_mode = [] {
  const char* e = std::getenv("ELSA_TAIL");
  return e ? std::atoi(e) : 1;
}();
bool tail_capable(int cfg) { return cfg == kCfgW4R8 || cfg == kCfgW8R8 || cfg == kCfgW8R8Acc; }

// Cluster split merge (fwd_f32_kernel<..., CL = true>): the d, dv <= 64
// configurations with 2..16 splits, final output only.
constexpr int kMaxClusterSplits = 16;
bool cluster_capable(int cfg, int64_t dv) {
  return (cfg == kCfgW4R8 || cfg == kCfgW8R8 || cfg == kCfgW8R4) && dv <= 64;
}

double plan_cost(const CfgInfo& ci, int64_t ctas, int64_t tiles, int64_t rows, int64_t sms,
                 int64_t s) {
  double t = double(ceil_div(ctas * s, sms)) *
             (double(ceil_div(tiles, s)) * ci.tile_us + ci.cta_us);
  if (s > 1) t += 10.8 + 45.6e-6 * double(s) * double(rows);
  return t;
}

int64_t normalize_splits(int64_t s, int64_t tiles) {
  if (s > tiles) s = tiles;
  if (s > kMaxSplits) s = kMaxSplits;
  if (s < 1) s = 1;
  // drop empty splits: the effective count is ceil(tiles / tiles_per_split)
  const int64_t tps = ceil_div(tiles, s);
  return ceil_div(tiles, tps);
}

// Cluster-merge mode (development aid, elsa_dev_set_cluster): 0 never,
// 1 when the cost model prefers it (default), 2 whenever capable.
int g_cluster_mode = [] {
  const char* e = std::getenv("ELSA_CLUSTER");
  return e ? std::atoi(e) : 1;
}();
constexpr int kClusterAutoMaxSplits = 4;

template <int W, int TK, int ST, int R>
int max_active_clusters(int splits, DeviceCache* dc, int cfg_slot);

int cluster_slot(int cfg) { return cfg == kCfgW8R8 ? 1 : (cfg == kCfgW8R4 ? 2 : 0); }

int active_clusters(int cfg, int splits, DeviceCache* dc) {
  if (!dc || splits < 2 || splits > kMaxClusterSplits) return 0;
#if ELSA_EXPERIMENTAL_W8R4
  if (cfg == kCfgW8R4) return max_active_clusters<8, 64, 2, 4>(splits, dc, cluster_slot(cfg));
#else
  if (cfg == kCfgW8R4) return 0;
#endif
#if ELSA_W8R8_REGSPLIT  // (experiment: the register-split w8r8 has no cluster form)
  if (cfg == kCfgW8R8) return 0;
  return max_active_clusters<4, 64, ELSA_W4R8_STAGES, 8>(splits, dc, cluster_slot(cfg));
#else
  return cfg == kCfgW8R8
             ? max_active_clusters<8, 64, ELSA_W8R8_STAGES, 8>(splits, dc, cluster_slot(cfg))
             : max_active_clusters<4, 64, ELSA_W4R8_STAGES, 8>(splits, dc, cluster_slot(cfg));
#endif
}

Plan plan_for(const elsa_shape* sh, int64_t kv_len, int requested, int sms,
              bool allow_cluster = false, DeviceCache* dc = nullptr) {
  const int64_t BH = sh->B * sh->H;
  // head widths beyond 64 have one configuration each; d, dv <= 64 choose
  const int only = wide_cfg(sh->d, sh->dv);
  const bool wide = only >= 0;
  // d, dv <= 64 candidates: w4r8, w8r16, w8r8, the long-chain w8r8acc and the
  // small-problem w8r4
  static const int kNarrow[] = {kCfgW4R8, kCfgW8R16, kCfgW8R8, kCfgW8R8Acc, kCfgW8R4};
  const int first = wide ? only : 0, last = wide ? only + 1 : int(sizeof(kNarrow) / sizeof(int));
  Plan best{first, 1, BH > 0 ? BH : 1};
  double best_t = 1e300;
  const int forced = wide ? int(kCfgAuto) : forced_cfg();
  const int64_t slices = ceil_div(sh->dv, cfg_dv(first));
  const int64_t head_bytes = sh->n_q * (2 + 64 * dv_slices(sh->dv)) * 4;  // one split of one (b, h) head
  for (int ci_ = first; ci_ < last; ++ci_) {
    // d, dv <= 64: w4r8, w8r16, w8r8, then the long-chain w8r8acc
    const int cfg = wide ? ci_ : kNarrow[ci_];
    if (cfg == kCfgW8R4 && forced != kCfgW8R4) continue;  // not auto-planned yet
    if (forced != kCfgAuto && cfg != forced) continue;
    const CfgInfo ci = cfg_info(cfg);
    const int64_t ctas = ceil_div(sh->n_q, ci.tq) * BH * slices;
    const int64_t tiles = ceil_div(kv_len, ci.tk);
    const int64_t rows = BH * sh->n_q;
    if (ctas == 0 || tiles < 1) return Plan{forced == kCfgAuto ? first : forced, 1, 1};
    int64_t lo, hi;
    if (requested > 0) {
      lo = hi = normalize_splits(requested, tiles);
    } else {
      hi = tiles < kMaxSplits ? tiles : kMaxSplits;
      // the chain cap wins over the workspace budget: the fewest splits that
      // keep every CTA's chain <= kMaxChainTiles are always allowed (the
      // workspace then exceeds the soft budget for a single head); beyond
      // kMaxSplits * kMaxChainTiles tiles the chain grows and describe_plan
      // reports it
      lo = ceil_div(tiles, chain_cap(cfg));
      if (lo > hi) lo = hi;
      const int64_t ws_cap = head_bytes > 0 ? workspace_budget() / head_bytes : hi;
      if (hi > ws_cap) hi = ws_cap < lo ? lo : ws_cap;
    }
    for (int64_t s = lo; s <= hi; ++s) {
      const int64_t sn = normalize_splits(s, tiles);
      int64_t hpb = BH;
      if (sn > 1 && requested <= 0) {
        hpb = workspace_budget() / (sn * head_bytes);
        if (hpb < 1) hpb = 1;
        if (hpb > BH) hpb = BH;
      }
      const int64_t batches = ceil_div(BH, hpb);
      double t = plan_cost(ci, ctas, tiles, rows, sms, sn) + 8.0 * double(batches - 1);
      // a chain over the config's cap (only past kMaxSplits x cap tiles) is
      // an accuracy cost: prefer the config whose cap it exceeds least
      const int64_t chain = ceil_div(tiles, sn);
      if (chain > chain_cap(cfg)) t *= 1.0 + double(chain) / double(chain_cap(cfg));
      if (t < best_t - 1e-9) {
        best_t = t;
        best = Plan{cfg, int(sn), hpb};
      }
    }
  }
  // Cluster split merge (fwd_f32_kernel<..., CL>): the chosen plan's splits
  // merge inside the launch over DSMEM instead of through the workspace and
  // K2. Measured on B200 (tools/time_cluster.py, profiles/round2_cluster.md),
  // it pays only while every cluster is resident at once and clusters are
  // small: 8- and 16-CTA clusters of the 2-CTA/SM w4r8 kernel get packed two
  // CTAs per SM (C1: 19.7 us vs 12.9 + 4.5 us for K1 + K2), and multi-wave
  // cluster launches lose to the free placement of a plain grid (B1 H1 n16K,
  // 4 splits: 1421 vs 1256 us). So the auto plan converts a 2..4-split plan
  // whose clusters all fit at once; mode 2 converts whatever can launch.
  if (allow_cluster && g_cluster_mode != 0 && best.splits > 1 &&
      best.splits <= kMaxClusterSplits && cluster_capable(best.cfg, sh->dv)) {
    const int maxc = active_clusters(best.cfg, best.splits, dc);
    const int64_t nclu = ceil_div(sh->n_q, cfg_info(best.cfg).tq) * BH;
    const bool fits = maxc > 0 && nclu <= maxc && best.splits <= kClusterAutoMaxSplits;
    if (fits || (g_cluster_mode == 2 && maxc > 0)) {
      best.cluster = true;
      best.heads_per_batch = BH;
    }
  }
  if (allow_cluster && g_tail_mode != 0 && best.splits == 1 && !best.cluster &&
      tail_capable(best.cfg) && sh->dv <= 64 && requested <= 0) {
    const CfgInfo ci = cfg_info(best.cfg);
    const int64_t U = ceil_div(sh->n_q, ci.tq) * BH;  // units (one CTA each)
    const int64_t N = ceil_div(kv_len, ci.tk);       // key tiles per unit
    const int64_t slots = int64_t(sms) * ci.ctas_per_sm;
    const int64_t F = (U / slots) * slots, T = U - F;
    // Measured rule (tools/time_tail.sh, profiles/round2_tail_split.txt): two
    // pieces per tail unit pay only after >= 2 full waves with the last wave
    // 50-75% full (BERT-base B8 H12 n512, w4r8: 151.5 -> 143.4 us); fuller or
    // emptier last waves and more pieces measured equal or slower.
    const double frac = double(T) / double(slots);
    int bs = 0;
    if (g_tail_mode >= 2)
      bs = int(g_tail_mode < N ? g_tail_mode : N);
    else if (F >= 2 * slots && frac >= 0.5 && frac < 0.75 && N >= 2)
      bs = 2;
    if (bs >= 2) bs = int(normalize_splits(bs, N));  // no empty pieces
    if (bs >= 2 && T > 0 && F + T * bs < (int64_t(1) << 31)) {
      best.tail_s = bs;
      best.tail_first = F;
      best.heads_per_batch = BH;
    }
  }
  return best;
}

// Sanitise the stride of size-1 axes (any value is semantically irrelevant
// there but TMA wants a positive multiple of 16 bytes).
void sanitize(int64_t st[3], int64_t rows, int64_t H, int64_t B, int64_t inner) {
  if (rows == 1 && st[2] == 0) st[2] = inner;
  if (H == 1) st[1] = st[2] * rows;
  if (B == 1) st[0] = st[1] * H;
}

bool tma_ok(const float* base, const int64_t st[3], int64_t inner) {
  if (reinterpret_cast<uintptr_t>(base) % 16) return false;
  for (int i = 0; i < 3; ++i) {
    if (st[i] <= 0 || st[i] % 4) return false;
    if (st[i] * 4 >= (int64_t(1) << 40)) return false;
  }
  (void)inner;
  return true;
}

// Per-thread cache of encoded descriptors: eager callers re-run the same
// geometry on the same buffers, and encoding three maps per call is a visible
// share of a small problem's host time. Keyed by everything the map encodes.
struct MapKey {
  const void* base;
  int64_t dims[4], st[3];
  int box_inner, box_rows;
  bool operator==(const MapKey& o) const { return std::memcmp(this, &o, sizeof(MapKey)) == 0; }
};
struct MapEntry {
  MapKey key;
  CUtensorMap map;
  bool valid = false;
};
constexpr int kMapCache = 32;
thread_local MapEntry t_maps[kMapCache];

bool encode_map_uncached(CUtensorMap* map, const float* base, int64_t inner, int64_t rows,
                         int64_t H, int64_t B, const int64_t st[3], int box_inner, int box_rows);

bool encode_map(CUtensorMap* map, const float* base, int64_t inner, int64_t rows, int64_t H,
                int64_t B, const int64_t st[3], int box_inner, int box_rows) {
  MapKey key;
  std::memset(&key, 0, sizeof(key));
  key.base = base;
  key.dims[0] = inner, key.dims[1] = rows, key.dims[2] = H, key.dims[3] = B;
  key.st[0] = st[0], key.st[1] = st[1], key.st[2] = st[2];
  key.box_inner = box_inner, key.box_rows = box_rows;
  uint64_t hsh = reinterpret_cast<uintptr_t>(base) >> 4;
  for (int i = 0; i < 4; ++i) hsh = hsh * 1000003u ^ uint64_t(key.dims[i]);
  for (int i = 0; i < 3; ++i) hsh = hsh * 1000003u ^ uint64_t(key.st[i]);
  hsh = hsh * 1000003u ^ uint64_t(box_inner * 4096 + box_rows);
  MapEntry& e = t_maps[(hsh ^ (hsh >> 29)) % kMapCache];
  if (e.valid && e.key == key) {
    *map = e.map;
    return true;
  }
  if (!encode_map_uncached(map, base, inner, rows, H, B, st, box_inner, box_rows)) return false;
  e.key = key;
  e.map = *map;
  e.valid = true;
  return true;
}

bool encode_map_uncached(CUtensorMap* map, const float* base, int64_t inner, int64_t rows,
                         int64_t H, int64_t B, const int64_t st[3], int box_inner,
                         int box_rows) {
  auto enc = encoder();
  if (!enc) return false;
  cuuint64_t dims[4] = {cuuint64_t(inner), cuuint64_t(rows), cuuint64_t(H), cuuint64_t(B)};
  cuuint64_t strides[3] = {cuuint64_t(st[2] * 4), cuuint64_t(st[1] * 4), cuuint64_t(st[0] * 4)};
  cuuint32_t box[4] = {cuuint32_t(box_inner), cuuint32_t(box_rows), 1, 1};
  cuuint32_t es[4] = {1, 1, 1, 1};
  CUresult r = enc(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, const_cast<float*>(base), dims,
                   strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                   CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS;
}

template <int W, int TK, int ST, int R, int D = 64, int DV = 64, bool CL = false,
          bool ACC = false>
int launch_fwd_cfg(FwdParams& p, const elsa_shape* s, int64_t q_st[3], int64_t k_st[3],
                   int64_t v_st[3], int splits, int64_t bh_count, int cfg_slot, DeviceCache* dc,
                   cudaStream_t stream) {
  using T = FwdTraits<W, TK, ST, R, D, DV>;
  p.qtiles = int(ceil_div(s->n_q, T::TQ));
  const int64_t tiles = ceil_div(int64_t(p.kv_end) - p.kv_begin, TK);
  if (p.split_keys == 0) p.split_keys = int(ceil_div(tiles, splits) * TK);

  CUtensorMap maps[3];
  std::memset(maps, 0, sizeof(maps));
  // copy engine (non-TMA) alignment: 16-byte copies when base and strides allow
  auto vec_ok = [](const float* base, const int64_t st[3]) {
    return reinterpret_cast<uintptr_t>(base) % 16 == 0 && st[0] % 4 == 0 && st[1] % 4 == 0 &&
           st[2] % 4 == 0;
  };
  p.q_vec = vec_ok(p.q, q_st);
  p.k_vec = vec_ok(p.k, k_st);
  p.v_vec = vec_ok(p.v, v_st);
  // TMA boxes are at most 256 elements wide: the d = 256 kernel (pitch 260) uses the copy engine
  bool use_tma = T::QP <= 256 && tma_ok(p.q, q_st, s->d) && tma_ok(p.k, k_st, s->d) &&
                 tma_ok(p.v, v_st, s->dv);
  if (use_tma) {
    use_tma = encode_map(&maps[0], p.q, s->d, s->n_q, s->H, s->B, q_st, T::QP, T::TQ) &&
              encode_map(&maps[1], p.k, s->d, s->n_kv, s->H, s->B, k_st, T::QP, TK) &&
              encode_map(&maps[2], p.v, s->dv, s->n_kv, s->H, s->B, v_st, T::VP, TK);
  }
  static const bool force_generic = std::getenv("ELSA_FORCE_GENERIC_LOAD") != nullptr;
  if (force_generic) use_tma = false;

  auto kern = fwd_f32_kernel<W, TK, ST, R, false, D, DV, CL, ACC>;
  if constexpr (T::QP <= 256) {
    if (use_tma) kern = fwd_f32_kernel<W, TK, ST, R, true, D, DV, CL, ACC>;
  }
  const int slot = (CL ? kCluAttrBase : 0) + cfg_slot * 2 + (use_tma ? 1 : 0);
  if (!dc->attr[slot]) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         int(T::SMEM_BYTES));
    if (e == cudaSuccess && CL)
      e = cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    if (e != cudaSuccess) return cuda_fail(e, "cudaFuncSetAttribute(fwd)");
    dc->attr[slot] = true;
  }
  const int64_t gx = p.grid_units > 0 ? p.grid_units : int64_t(p.qtiles) * bh_count;
  if (gx >= (int64_t(1) << 31)) return ELSA_ERR_SHAPE;
  const dim3 grid{unsigned(gx), unsigned(splits), unsigned(ceil_div(s->dv, DV))};
  if constexpr (CL) {
    // ELSA_CLUSTER_SOLO=1 (experiment): pad the shared-memory request so a
    // cluster's CTAs spread one per SM instead of packing two per SM
    static const bool solo = std::getenv("ELSA_CLUSTER_SOLO") != nullptr;
    size_t smem = T::SMEM_BYTES;
    if (solo && smem < 120 * 1024) smem = 120 * 1024;
    if (solo) {
      const cudaError_t e2 = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                                  int(smem));
      if (e2 != cudaSuccess) return cuda_fail(e2, "cudaFuncSetAttribute(fwd solo)");
    }
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = dim3(T::THREADS);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = stream;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = 1;
    attr[0].val.clusterDim.y = unsigned(splits);
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    const cudaError_t e = cudaLaunchKernelEx(&cfg, kern, p, maps[0], maps[1], maps[2]);
    if (e != cudaSuccess) return cuda_fail(e, "fwd cluster launch");
  } else {
    kern<<<grid, T::THREADS, T::SMEM_BYTES, stream>>>(p, maps[0], maps[1], maps[2]);
    if (cudaPeekAtLastError() != cudaSuccess) return cuda_fail(cudaGetLastError(), "fwd launch");
  }
  ++t_last_launches;
  return ELSA_OK;
}

// Clusters of `splits` CTAs of the cluster-merge kernel that fit the device at
// once (cudaOccupancyMaxActiveClusters; a cluster must sit inside one GPC),
// cached per configuration and split count; 0 when the size cannot launch.
template <int W, int TK, int ST, int R>
int max_active_clusters(int splits, DeviceCache* dc, int cfg_slot) {
  using T = FwdTraits<W, TK, ST, R>;
  int& cached = dc->clusters[cfg_slot][splits];
  if (cached >= 0) return cached;
  auto kern = fwd_f32_kernel<W, TK, ST, R, true, 64, 64, true>;
  int n = 0;
  if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           int(T::SMEM_BYTES)) == cudaSuccess &&
      cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1) ==
          cudaSuccess) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(1, unsigned(splits), 1);
    cfg.blockDim = dim3(T::THREADS);
    cfg.dynamicSmemBytes = T::SMEM_BYTES;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = 1;
    attr[0].val.clusterDim.y = unsigned(splits);
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    if (cudaOccupancyMaxActiveClusters(&n, kern, &cfg) != cudaSuccess) n = 0;
  }
  cudaGetLastError();  // a refused size is an answer, not an error state
  cached = n;
  return n;
}

int launch_fwd(FwdParams& p, const elsa_shape* s, int64_t q_st[3], int64_t k_st[3],
               int64_t v_st[3], const Plan& plan, int64_t bh_count, DeviceCache* dc,
               cudaStream_t stream) {
  const int splits = plan.splits;
  if (plan.cluster) {
#if ELSA_EXPERIMENTAL_W8R4
    if (plan.cfg == kCfgW8R4)
      return launch_fwd_cfg<8, 64, 2, 4, 64, 64, true>(p, s, q_st, k_st, v_st, splits, bh_count,
                                                       kCfgW8R4, dc, stream);
#endif
#if !ELSA_W8R8_REGSPLIT
    if (plan.cfg == kCfgW8R8)
      return launch_fwd_cfg<8, 64, ELSA_W8R8_STAGES, 8, 64, 64, true>(
          p, s, q_st, k_st, v_st, splits, bh_count, kCfgW8R8, dc, stream);
#endif
    return launch_fwd_cfg<4, 64, ELSA_W4R8_STAGES, 8, 64, 64, true>(
        p, s, q_st, k_st, v_st, splits, bh_count, kCfgW4R8, dc, stream);
  }
  switch (plan.cfg) {
    case kCfgW8R16:
      return launch_fwd_cfg<8, 64, 2, 16>(p, s, q_st, k_st, v_st, splits, bh_count, kCfgW8R16, dc,
                                          stream);
    case kCfgW8R8:
      return launch_fwd_cfg<8, 64, ELSA_W8R8_STAGES, 8>(p, s, q_st, k_st, v_st, splits, bh_count, kCfgW8R8, dc,
                                         stream);
    case kCfgW8R8Acc:
      return launch_fwd_cfg<8, 64, ELSA_W8R8_STAGES, 8, 64, 64, false, true>(
          p, s, q_st, k_st, v_st, splits, bh_count, kCfgW8R8Acc, dc, stream);
    case kCfgW8R4:
#if ELSA_EXPERIMENTAL_W8R4
      return launch_fwd_cfg<8, 64, 2, 4>(p, s, q_st, k_st, v_st, splits, bh_count, kCfgW8R4, dc,
                                         stream);
#else
      return ELSA_ERR_SHAPE;
#endif
    case kCfgW8R8D128:
      return launch_fwd_cfg<8, 64, 2, 8, 128>(p, s, q_st, k_st, v_st, splits, bh_count,
                                              kCfgW8R8D128, dc, stream);
    case kCfgW8R8V128:
      return launch_fwd_cfg<8, 64, 2, 8, 64, 128>(p, s, q_st, k_st, v_st, splits, bh_count,
                                                  kCfgW8R8V128, dc, stream);
    case kCfgW8R8D128V128:
      return launch_fwd_cfg<8, 64, 2, 8, 128, 128>(p, s, q_st, k_st, v_st, splits, bh_count,
                                                   kCfgW8R8D128V128, dc, stream);
    case kCfgW8R8D96:
      return launch_fwd_cfg<8, 64, 2, 8, 96>(p, s, q_st, k_st, v_st, splits, bh_count,
                                             kCfgW8R8D96, dc, stream);
    case kCfgW8R8D96V128:
      return launch_fwd_cfg<8, 64, 2, 8, 96, 128>(p, s, q_st, k_st, v_st, splits, bh_count,
                                                  kCfgW8R8D96V128, dc, stream);
    case kCfgW8R8D256:
      return launch_fwd_cfg<8, 32, 2, 8, 256>(p, s, q_st, k_st, v_st, splits, bh_count,
                                              kCfgW8R8D256, dc, stream);
    case kCfgW4R8D256V128:
      return launch_fwd_cfg<4, 32, 2, 8, 256, 128>(p, s, q_st, k_st, v_st, splits, bh_count,
                                                   kCfgW4R8D256V128, dc, stream);
    case kCfgW8R8D32V32:
      return launch_fwd_cfg<8, 64, ELSA_D32_STAGES, 8, 32, 32>(p, s, q_st, k_st, v_st, splits, bh_count,
                                                 kCfgW8R8D32V32, dc, stream);
    case kCfgW8R8D96V96:
      return launch_fwd_cfg<8, 64, 2, 8, 96, 96>(p, s, q_st, k_st, v_st, splits, bh_count,
                                                 kCfgW8R8D96V96, dc, stream);
    case kCfgW8R8V96:
      return launch_fwd_cfg<8, 64, 2, 8, 64, 96>(p, s, q_st, k_st, v_st, splits, bh_count,
                                                 kCfgW8R8V96, dc, stream);
    case kCfgW8R8D128V96:
      return launch_fwd_cfg<8, 64, 2, 8, 128, 96>(p, s, q_st, k_st, v_st, splits, bh_count,
                                                  kCfgW8R8D128V96, dc, stream);
    case kCfgW4R8D256V256:
      return launch_fwd_cfg<4, 32, 2, 8, 256, 256>(p, s, q_st, k_st, v_st, splits, bh_count,
                                                   kCfgW4R8D256V256, dc, stream);
    default:
      return launch_fwd_cfg<4, 64, ELSA_W4R8_STAGES, 8>(p, s, q_st, k_st, v_st, splits, bh_count, kCfgW4R8, dc,
                                         stream);
  }
}

// pdl: launch as the preceding forward kernel's programmatic dependent
// (its CTAs become resident while K1 drains; they start merging when K1 is done)
int launch_merge(MergeParams& mp, cudaStream_t stream, bool pdl = false) {
  if (mp.rows == 0) return ELSA_OK;
  constexpr int kWarps = 8;
  const int64_t blocks = ceil_div(mp.rows, kWarps);
  if (blocks >= (int64_t(1) << 31)) return ELSA_ERR_SHAPE;
  const dim3 grid{unsigned(blocks), unsigned(dv_slices(mp.dv)), 1u};
  auto kern = mp.parts <= 2    ? merge_f32_kernel<2>
              : mp.parts <= 4  ? merge_f32_kernel<4>
              : mp.parts <= 8  ? merge_f32_kernel<8>
              : mp.parts <= 16 ? merge_f32_kernel<16>
                               : merge_f32_kernel<32>;
  static const bool no_pdl = std::getenv("ELSA_NO_PDL") != nullptr;  // A/B switch
  if (pdl && !no_pdl) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = dim3(kWarps * 32);
    cfg.dynamicSmemBytes = 0;
    cfg.stream = stream;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    const cudaError_t e = cudaLaunchKernelEx(&cfg, kern, mp);
    if (e != cudaSuccess) return cuda_fail(e, "merge launch (PDL)");
  } else {
    kern<<<grid, kWarps * 32, 0, stream>>>(mp);
    if (cudaPeekAtLastError() != cudaSuccess) return cuda_fail(cudaGetLastError(), "merge launch");
  }
  ++t_last_launches;
  return ELSA_OK;
}

void fill_common(FwdParams& p, const float* q, const float* k, const float* v,
                 const elsa_shape* s, double scale, const int64_t q_st[3], const int64_t k_st[3],
                 const int64_t v_st[3]) {
  std::memset(&p, 0, sizeof(p));
  p.q = q;
  p.k = k;
  p.v = v;
  p.B = int(s->B);
  p.H = int(s->H);
  p.n_q = int(s->n_q);
  p.n_kv = int(s->n_kv);
  p.d = int(s->d);
  p.dv = int(s->dv);
  p.qs_b = q_st[0];
  p.qs_h = q_st[1];
  p.qs_r = q_st[2];
  p.ks_b = k_st[0];
  p.ks_h = k_st[1];
  p.ks_r = k_st[2];
  p.vs_b = v_st[0];
  p.vs_h = v_st[1];
  p.vs_r = v_st[2];
  // exponents are evaluated as exp2(acc * c - m) with c > 0; a negative scale
  // is folded into Q^T inside the kernel, a zero scale becomes a uniform
  // softmax through a vanishing positive c
  double c = std::fabs(scale) * kLog2e;
  if (c < 1e-30) c = 1e-30;
  p.c = float(c);
  p.neg = scale < 0 ? 1 : 0;
  p.trace = trace_buffer();
  p.row_stride = 1;
}

int64_t tail_rows(const elsa_shape* s, const Plan& pl) {
  const int tq = cfg_info(pl.cfg).tq;
  const int64_t qt = ceil_div(s->n_q, tq);
  const int64_t r0 = (pl.tail_first / qt) * s->n_q + (pl.tail_first % qt) * tq;
  return s->B * s->H * s->n_q - r0;
}

size_t split_ws_bytes(const elsa_shape* s, const Plan& pl) {
  if (pl.tail_s > 0)
    return size_t(pl.tail_s) * size_t(tail_rows(s, pl)) * size_t(2 + 64) * sizeof(float) + 16;
  if (pl.splits <= 1 || pl.cluster) return 0;
  const size_t rows = size_t(pl.heads_per_batch) * size_t(s->n_q);
  // m | S | (pad to 16 bytes) | W
  return size_t(pl.splits) * rows * size_t(2 + 64 * dv_slices(s->dv)) * sizeof(float) + 16;
}

bool encode_map16(CUtensorMap* map, const void* base, int64_t inner, int64_t rows, int64_t H,
                  int64_t B,
                  const int64_t st[3], bool bf16, int box_rows = 128) {
  auto enc = encoder();
  if (!enc) return false;
  // inner < 64: the 64-wide box is zero-filled past the row (OOB fill)
  cuuint64_t dims[4] = {cuuint64_t(inner), cuuint64_t(rows), cuuint64_t(H), cuuint64_t(B)};
  cuuint64_t strides[3] = {cuuint64_t(st[2] * 2), cuuint64_t(st[1] * 2), cuuint64_t(st[0] * 2)};
  cuuint32_t box[4] = {64, cuuint32_t(box_rows), 1, 1};
  cuuint32_t es[4] = {1, 1, 1, 1};
  CUresult r = enc(map, bf16 ? CU_TENSOR_MAP_DATA_TYPE_BFLOAT16 : CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 4,
                   const_cast<void*>(base), dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                   CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS;
}

bool aligned16(const void* ptr, const int64_t st[3]) {
  if (reinterpret_cast<uintptr_t>(ptr) % 16) return false;
  for (int i = 0; i < 3; ++i)
    if (st[i] <= 0 || (st[i] * 2) % 16 || st[i] * 2 >= (int64_t(1) << 40)) return false;
  return true;
}

// Shared driver of elsa_fwd_f32 (y != nullptr: final Y) and elsa_partial_f32
// (m/S/W: natural-log partial states of keys [kv_begin, kv_end)). With
// kv splits > 1 the work runs in batches of `heads_per_batch` (b, h) heads:
// forward kernel -> split partial states in the workspace -> K2 tree merge.
int run_forward(const float* q, const float* k, const float* v, const elsa_shape* shp,
                double scale, int64_t kv_begin, int64_t kv_end, int kv_splits, void* workspace,
                size_t ws_bytes, cudaStream_t strm, float* y, float* m_out, float* S_out,
                float* W_out, const Plan* force_plan = nullptr) {
  DeviceCache* dc = nullptr;
  if (int st = current_device_cache(&dc)) return st;
  int64_t q_st[3], k_st[3], v_st[3];
  std::memcpy(q_st, shp->q_stride, sizeof(q_st));
  std::memcpy(k_st, shp->k_stride, sizeof(k_st));
  std::memcpy(v_st, shp->v_stride, sizeof(v_st));
  sanitize(q_st, shp->n_q, shp->H, shp->B, shp->d);
  sanitize(k_st, shp->n_kv, shp->H, shp->B, shp->d);
  sanitize(v_st, shp->n_kv, shp->H, shp->B, shp->dv);

  const int64_t BH = shp->B * shp->H;
  const int64_t len = kv_end - kv_begin;
  const bool final_out = y != nullptr;
  const Plan plan = force_plan ? *force_plan
                               : plan_for(shp, len > 0 ? len : 1, kv_splits, dc->sms, final_out, dc);
  FwdParams p;
  fill_common(p, q, k, v, shp, scale, q_st, k_st, v_st);
  p.kv_begin = int(kv_begin);
  p.kv_end = int(kv_end);
  p.err = dc->err;
  if (final_out) {
    p.y = y;
    p.ys_b = shp->y_stride[0];
    p.ys_h = shp->y_stride[1];
    p.ys_r = shp->y_stride[2];
    p.y_vec = (reinterpret_cast<uintptr_t>(y) % 16 == 0) && (p.ys_b % 4 == 0) &&
              (p.ys_h % 4 == 0) && (p.ys_r % 4 == 0);
  }
  if (plan.cluster && final_out) {
    // one launch: the splits of each query tile form a cluster and merge over DSMEM
    p.bh_begin = 0;
    p.mode = kModeFinal;
    return launch_fwd(p, shp, q_st, k_st, v_st, plan, BH, dc, strm);
  }
  if (plan.tail_s > 0 && final_out) {
    // one forward launch: whole units, then the last wave's units as key
    // pieces writing log2 partial states; K2 (PDL) merges the tail rows
    const size_t need = split_ws_bytes(shp, plan);
    if (!workspace || ws_bytes < need) return ELSA_ERR_WORKSPACE;
    const int tq = cfg_info(plan.cfg).tq, tk = cfg_info(plan.cfg).tk;
    const int64_t rows_t = tail_rows(shp, plan);
    const int64_t ntiles = ceil_div(len, tk);
    float* ws = static_cast<float*>(workspace);
    p.bh_begin = 0;
    p.mode = kModeFinal;
    p.tail_first = int(plan.tail_first);
    p.tail_splits = plan.tail_s;
    p.tail_split_keys = int(ceil_div(ntiles, plan.tail_s) * tk);
    p.tail_row0 = BH * shp->n_q - rows_t;
    p.pm = ws;
    p.pS = ws + int64_t(plan.tail_s) * rows_t;
    p.pW = ws + ((int64_t(plan.tail_s) * rows_t * 2 + 3) & ~int64_t(3));
    p.part_stride = rows_t;
    p.pw_pitch = 64;
    p.pw_vec = reinterpret_cast<uintptr_t>(p.pW) % 16 == 0;
    p.grid_units = plan.tail_first +
                   (ceil_div(shp->n_q, tq) * BH - plan.tail_first) * plan.tail_s;
    if (int st = launch_fwd(p, shp, q_st, k_st, v_st, plan, BH, dc, strm)) return st;
    MergeParams mp;
    std::memset(&mp, 0, sizeof(mp));
    mp.m = p.pm;
    mp.S = p.pS;
    mp.W = p.pW;
    mp.parts = plan.tail_s;
    mp.rows = rows_t;
    mp.dv = int(shp->dv);
    mp.w_pitch = 64;
    mp.part_stride = rows_t;
    mp.log2_domain = 1;
    mp.err = dc->err;
    mp.finalize = 1;
    mp.y = y;
    mp.H = int(shp->H);
    mp.n_q = int(shp->n_q);
    mp.bh_begin = 0;
    mp.row0 = p.tail_row0;
    mp.ys_b = shp->y_stride[0];
    mp.ys_h = shp->y_stride[1];
    mp.ys_r = shp->y_stride[2];
    return launch_merge(mp, strm, true);
  }
  if (plan.splits <= 1) {
    p.bh_begin = 0;
    if (final_out) {
      p.mode = kModeFinal;
    } else {
      p.mode = kModePartialNat;
      p.pm = m_out;
      p.pS = S_out;
      p.pW = W_out;
      p.part_stride = BH * shp->n_q;
      p.pw_pitch = int(shp->dv);
      p.pw_vec = (reinterpret_cast<uintptr_t>(W_out) % 16 == 0) && (shp->dv % 4 == 0);
    }
    return launch_fwd(p, shp, q_st, k_st, v_st, plan, BH, dc, strm);
  }
  const size_t need = split_ws_bytes(shp, plan);
  if (!workspace || ws_bytes < need) return ELSA_ERR_WORKSPACE;
  float* ws = static_cast<float*>(workspace);
  const int splits = plan.splits;
  for (int64_t bh0 = 0; bh0 < BH; bh0 += plan.heads_per_batch) {
    const int64_t cnt = BH - bh0 < plan.heads_per_batch ? BH - bh0 : plan.heads_per_batch;
    const int64_t rows = cnt * shp->n_q;
    p.bh_begin = int(bh0);
    p.mode = kModePartialLog2;
    p.pm = ws;
    p.pS = ws + int64_t(splits) * rows;
    // W starts on a 16-byte boundary (float4 stores); the pitch is a multiple of 4
    p.pW = ws + ((int64_t(splits) * rows * 2 + 3) & ~int64_t(3));
    p.part_stride = rows;
    p.pw_pitch = int(64 * dv_slices(shp->dv));
    p.pw_vec = reinterpret_cast<uintptr_t>(p.pW) % 16 == 0;
    if (int st = launch_fwd(p, shp, q_st, k_st, v_st, plan, cnt, dc, strm)) return st;
    MergeParams mp;
    std::memset(&mp, 0, sizeof(mp));
    mp.m = p.pm;
    mp.S = p.pS;
    mp.W = p.pW;
    mp.parts = splits;
    mp.rows = rows;
    mp.dv = int(shp->dv);
    mp.w_pitch = int(64 * dv_slices(shp->dv));
    mp.part_stride = rows;
    mp.log2_domain = 1;
    mp.err = dc->err;
    if (final_out) {
      mp.finalize = 1;
      mp.y = y;
      mp.H = int(shp->H);
      mp.n_q = int(shp->n_q);
      mp.bh_begin = int(bh0);
      mp.ys_b = shp->y_stride[0];
      mp.ys_h = shp->y_stride[1];
      mp.ys_r = shp->y_stride[2];
    } else {
      const int64_t off = bh0 * shp->n_q;
      mp.finalize = 0;
      mp.m_out = m_out + off;
      mp.S_out = S_out + off;
      mp.W_out = W_out + off * shp->dv;
      mp.out_pitch = int(shp->dv);
      mp.out_log2_to_nat = 1;
    }
    if (int st = launch_merge(mp, strm, true)) return st;
  }
  return ELSA_OK;
}

// ---------------------------------------------------------------------------
// Host-buffer pipeline (elsa_fwd_f32_host). The (b, h) heads are cut into up
// to kPipeMaxGroups groups; group g's Q/K/V go host -> device on one copy
// stream, its forward runs on compute stream g % kPipeStreams as soon as its
// inputs landed, and its Y goes device -> host on a second copy stream as soon
// as it is computed. Several compute streams keep CTAs of the next groups
// resident while a group drains, so the device runs the same plan (config and
// kv splits of the WHOLE problem) at the same occupancy as one launch, and the
// PCIe transfers hide under the FFMA work except for the first group's inputs
// and the last group's output.
// ---------------------------------------------------------------------------
constexpr int kPipeStreams = 4;
constexpr int kPipeMaxGroups = 16;

struct HostPipe {
  bool ready = false;
  cudaStream_t in = nullptr, out = nullptr, comp[kPipeStreams] = {};
  cudaEvent_t start = nullptr, done = nullptr;
  cudaEvent_t ev_in[kPipeMaxGroups] = {}, ev_comp[kPipeMaxGroups] = {};
  std::mutex mu;  // one enqueue sequence at a time per device (events are reused)
};
HostPipe g_pipe[kMaxDevices];

int host_pipe(HostPipe** out) {
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= kMaxDevices) return ELSA_ERR_CUDA;
  HostPipe& hp = g_pipe[dev];
  std::lock_guard<std::mutex> lk(g_mu);
  if (!hp.ready) {
    cudaError_t e = cudaStreamCreateWithFlags(&hp.in, cudaStreamNonBlocking);
    if (e == cudaSuccess) e = cudaStreamCreateWithFlags(&hp.out, cudaStreamNonBlocking);
    for (int i = 0; i < kPipeStreams && e == cudaSuccess; ++i)
      e = cudaStreamCreateWithFlags(&hp.comp[i], cudaStreamNonBlocking);
    if (e == cudaSuccess) e = cudaEventCreateWithFlags(&hp.start, cudaEventDisableTiming);
    if (e == cudaSuccess) e = cudaEventCreateWithFlags(&hp.done, cudaEventDisableTiming);
    for (int i = 0; i < kPipeMaxGroups && e == cudaSuccess; ++i) {
      e = cudaEventCreateWithFlags(&hp.ev_in[i], cudaEventDisableTiming);
      if (e == cudaSuccess) e = cudaEventCreateWithFlags(&hp.ev_comp[i], cudaEventDisableTiming);
    }
    if (e != cudaSuccess) return cuda_fail(e, "host pipeline streams/events");
    hp.ready = true;
  }
  *out = &hp;
  return ELSA_OK;
}

size_t align256(size_t x) { return (x + 255) & ~size_t(255); }

struct HostLayout {
  Plan plan;        // the whole problem's plan, applied to every group
  Plan group_plan;  // same config / splits, heads_per_batch capped at the group size
  int64_t hpg = 1;  // (b, h) heads per group
  int groups = 1;
  size_t off_k = 0, off_v = 0, off_y = 0, off_ws = 0, ws_each = 0, total = 0;
};

bool dense_shape(const elsa_shape* s) {
  const int64_t q[3] = {s->H * s->n_q * s->d, s->n_q * s->d, s->d};
  const int64_t k[3] = {s->H * s->n_kv * s->d, s->n_kv * s->d, s->d};
  const int64_t v[3] = {s->H * s->n_kv * s->dv, s->n_kv * s->dv, s->dv};
  const int64_t y[3] = {s->H * s->n_q * s->dv, s->n_q * s->dv, s->dv};
  for (int i = 0; i < 3; ++i) {
    // strides of size-1 axes are irrelevant
    const bool skip = (i == 0 && s->B == 1) || (i == 1 && s->H == 1);
    if (skip) continue;
    if (s->q_stride[i] != q[i] || s->k_stride[i] != k[i] || s->v_stride[i] != v[i] ||
        s->y_stride[i] != y[i])
      return false;
  }
  return true;
}

elsa_shape group_shape(const elsa_shape* s, int64_t cnt) {
  elsa_shape g = *s;
  g.B = 1;
  g.H = cnt;
  const int64_t qs[3] = {cnt * s->n_q * s->d, s->n_q * s->d, s->d};
  const int64_t ks[3] = {cnt * s->n_kv * s->d, s->n_kv * s->d, s->d};
  const int64_t vs[3] = {cnt * s->n_kv * s->dv, s->n_kv * s->dv, s->dv};
  const int64_t ys[3] = {cnt * s->n_q * s->dv, s->n_q * s->dv, s->dv};
  std::memcpy(g.q_stride, qs, sizeof(qs));
  std::memcpy(g.k_stride, ks, sizeof(ks));
  std::memcpy(g.v_stride, vs, sizeof(vs));
  std::memcpy(g.y_stride, ys, sizeof(ys));
  return g;
}

HostLayout host_layout(const elsa_shape* s, int kv_splits, int sms, DeviceCache* dc) {
  HostLayout L;
  const int64_t BH = s->B * s->H;
  L.plan = plan_for(s, s->n_kv, kv_splits, sms, true, dc);
  L.plan.tail_s = 0;  // groups re-plan nothing: the tail split is per whole problem
  L.plan.tail_first = 0;
  const int64_t g = BH < kPipeMaxGroups ? (BH > 0 ? BH : 1) : kPipeMaxGroups;
  L.hpg = ceil_div(BH > 0 ? BH : 1, g);
  L.groups = int(ceil_div(BH > 0 ? BH : 1, L.hpg));
  L.group_plan = L.plan;
  if (L.group_plan.heads_per_batch > L.hpg) L.group_plan.heads_per_batch = L.hpg;
  const elsa_shape gs = group_shape(s, L.hpg);
  L.ws_each = align256(split_ws_bytes(&gs, L.group_plan));
  const size_t nq = size_t(BH) * size_t(s->n_q), nkv = size_t(BH) * size_t(s->n_kv);
  L.off_k = align256(nq * size_t(s->d) * 4);
  L.off_v = L.off_k + align256(nkv * size_t(s->d) * 4);
  L.off_y = L.off_v + align256(nkv * size_t(s->dv) * 4);
  L.off_ws = L.off_y + align256(nq * size_t(s->dv) * 4);
  L.total = L.off_ws + size_t(kPipeStreams) * L.ws_each;
  return L;
}

}  // namespace

extern "C" {

int elsa_abi_version(void) { return ELSA_ABI_VERSION; }

const char* elsa_strerror(int status) {
  switch (status) {
    case ELSA_OK:
      return "ok";
    case ELSA_ERR_SHAPE:
      return "shape/config error (unsupported geometry, stride or argument)";
    case ELSA_ERR_NUMERICAL:
      return "numerical error: softmax normalizer is zero or non-finite";
    case ELSA_ERR_CUDA:
      return "CUDA runtime error";
    case ELSA_ERR_NCCL:
      return "NCCL error";
    case ELSA_ERR_WORKSPACE:
      return "workspace missing or too small";
    default:
      return "unknown elsa status";
  }
}

int elsa_scan_depth(int64_t n, int64_t block_size) {
  if (n < 1 || block_size < 1) return -1;
  auto clog2 = [](int64_t x) {
    int r = 0;
    while ((int64_t(1) << r) < x) ++r;
    return r;
  };
  const int64_t b_eff = block_size < n ? block_size : n;
  const int64_t blocks = ceil_div(n, block_size);
  return clog2(b_eff) + 2 * clog2(blocks) + 3;
}

int elsa_resolve_kv_splits(const elsa_shape* shp, int requested) {
  if (!valid_shape(shp) || requested < 0) return -ELSA_ERR_SHAPE;
  DeviceCache* dc = nullptr;
  int sms = 148;
  if (current_device_cache(&dc) == ELSA_OK) sms = dc->sms;
  return plan_for(shp, shp->n_kv, requested, sms, true, dc).splits;
}

size_t elsa_workspace_bytes(const elsa_shape* shp, int kv_splits) {
  if (!valid_shape(shp) || kv_splits < 0) return 0;
  DeviceCache* dc = nullptr;
  int sms = 148;
  if (current_device_cache(&dc) == ELSA_OK) sms = dc->sms;
  return split_ws_bytes(shp, plan_for(shp, shp->n_kv, kv_splits, sms, true, dc));
}

size_t elsa_partial_workspace_bytes(const elsa_shape* shp, int64_t kv_begin, int64_t kv_end,
                                    int kv_splits) {
  if (!valid_shape(shp) || kv_splits < 0 || kv_begin < 0 || kv_end > shp->n_kv) return 0;
  DeviceCache* dc = nullptr;
  int sms = 148;
  if (current_device_cache(&dc) == ELSA_OK) sms = dc->sms;
  const int64_t len = kv_end - kv_begin;
  // partial states never use the cluster merge (its output is Y)
  return split_ws_bytes(shp, plan_for(shp, len > 0 ? len : 1, kv_splits, sms, false, dc));
}

// Development aid: cudaOccupancyMaxActiveClusters of the cluster-merge kernel
// (cfg 0 = w4r8, 2 = w8r8) for `splits`-CTA clusters on the current device.
int elsa_dev_max_active_clusters(int cfg, int splits) {
  DeviceCache* dc = nullptr;
  if (current_device_cache(&dc) != ELSA_OK) return -1;
  return active_clusters(cfg == kCfgW8R8 ? kCfgW8R8 : kCfgW4R8, splits, dc);
}

void elsa_dev_set_cluster(int mode) { g_cluster_mode = mode < 0 ? 0 : (mode > 2 ? 2 : mode); }

// Development aid: tail-split mode (0 off, 1 measured rule, s >= 2 force s pieces).
void elsa_dev_set_tail(int mode) { g_tail_mode = mode < 0 ? 0 : mode; }

// Development aid: force a d <= 64 configuration by name ("w4r8", "w8r8",
// "w8r16", "w8r8acc"; anything else = the planner's choice).
void elsa_dev_force_config(const char* name) { g_forced_cfg = cfg_from_name(name); }

int elsa_fwd_f32(const float* q, const float* k, const float* v, float* y,
                 const elsa_shape* shp, double scale, int kv_splits, void* workspace,
                 size_t ws_bytes, void* stream) {
  t_last_launches = 0;
  if (!valid_shape(shp) || kv_splits < 0 || !std::isfinite(scale)) return ELSA_ERR_SHAPE;
  if (!q || !k || !v || !y) return ELSA_ERR_SHAPE;
  if (shp->y_stride[0] < 0 || shp->y_stride[2] < 0) return ELSA_ERR_SHAPE;
  if (shp->B * shp->H * shp->n_q == 0) return ELSA_OK;
  return run_forward(q, k, v, shp, scale, 0, shp->n_kv, kv_splits, workspace, ws_bytes,
                     static_cast<cudaStream_t>(stream), y, nullptr, nullptr, nullptr);
}

size_t elsa_host_workspace_bytes(const elsa_shape* shp, int kv_splits) {
  if (!valid_shape(shp) || kv_splits < 0) return 0;
  DeviceCache* dc = nullptr;
  int sms = 148;
  if (current_device_cache(&dc) == ELSA_OK) sms = dc->sms;
  return host_layout(shp, kv_splits, sms, dc).total;
}

int elsa_fwd_f32_host(const float* q, const float* k, const float* v, float* y,
                      const elsa_shape* shp, double scale, int kv_splits, void* dev_workspace,
                      size_t ws_bytes, void* stream) {
  t_last_launches = 0;
  if (!valid_shape(shp) || kv_splits < 0 || !std::isfinite(scale)) return ELSA_ERR_SHAPE;
  if (!q || !k || !v || !y || !dense_shape(shp)) return ELSA_ERR_SHAPE;
  if (shp->B * shp->H * shp->n_q == 0) return ELSA_OK;
  DeviceCache* dc = nullptr;
  if (int st = current_device_cache(&dc)) return st;
  const HostLayout L = host_layout(shp, kv_splits, dc->sms, dc);
  if (!dev_workspace || ws_bytes < L.total) return ELSA_ERR_WORKSPACE;
  HostPipe* hp = nullptr;
  if (int st = host_pipe(&hp)) return st;
  std::lock_guard<std::mutex> lk(hp->mu);

  char* base = static_cast<char*>(dev_workspace);
  float* dq = reinterpret_cast<float*>(base);
  float* dk = reinterpret_cast<float*>(base + L.off_k);
  float* dv = reinterpret_cast<float*>(base + L.off_v);
  float* dy = reinterpret_cast<float*>(base + L.off_y);
  const cudaStream_t caller = static_cast<cudaStream_t>(stream);
  const int64_t BH = shp->B * shp->H;
  const int64_t nq = shp->n_q, nkv = shp->n_kv, d = shp->d, dvw = shp->dv;
  int launches = 0;
  auto fail = [&](cudaError_t e, const char* where) { return cuda_fail(e, where); };

  // after the caller's prior work and after every earlier host-pipeline call
  // on this device (they share these streams and usually the workspace)
  cudaError_t e = cudaEventRecord(hp->start, caller);
  if (e == cudaSuccess) e = cudaStreamWaitEvent(hp->in, hp->start, 0);
  if (e == cudaSuccess) e = cudaStreamWaitEvent(hp->in, hp->done, 0);
  if (e != cudaSuccess) return fail(e, "host pipeline start");
  for (int g = 0; g < L.groups; ++g) {
    const int64_t bh0 = int64_t(g) * L.hpg;
    const int64_t cnt = BH - bh0 < L.hpg ? BH - bh0 : L.hpg;
    const size_t qo = size_t(bh0 * nq * d), ko = size_t(bh0 * nkv * d);
    const size_t vo = size_t(bh0 * nkv * dvw), yo = size_t(bh0 * nq * dvw);
    e = cudaMemcpyAsync(dq + qo, q + qo, size_t(cnt * nq * d) * 4, cudaMemcpyHostToDevice, hp->in);
    if (e == cudaSuccess)
      e = cudaMemcpyAsync(dk + ko, k + ko, size_t(cnt * nkv * d) * 4, cudaMemcpyHostToDevice,
                          hp->in);
    if (e == cudaSuccess)
      e = cudaMemcpyAsync(dv + vo, v + vo, size_t(cnt * nkv * dvw) * 4, cudaMemcpyHostToDevice,
                          hp->in);
    if (e == cudaSuccess) e = cudaEventRecord(hp->ev_in[g], hp->in);
    const cudaStream_t cs = hp->comp[g % kPipeStreams];
    if (e == cudaSuccess) e = cudaStreamWaitEvent(cs, hp->ev_in[g], 0);
    if (e != cudaSuccess) return fail(e, "host pipeline H2D");
    const elsa_shape gs = group_shape(shp, cnt);
    Plan gp = L.group_plan;
    if (gp.heads_per_batch > cnt) gp.heads_per_batch = cnt;
    void* ws = L.ws_each ? base + L.off_ws + size_t(g % kPipeStreams) * L.ws_each : nullptr;
    if (int st = run_forward(dq + qo, dk + ko, dv + vo, &gs, scale, 0, nkv, gp.splits, ws,
                             L.ws_each, cs, dy + yo, nullptr, nullptr, nullptr, &gp))
      return st;
    launches += t_last_launches;
    t_last_launches = 0;
    e = cudaEventRecord(hp->ev_comp[g], cs);
    if (e != cudaSuccess) return fail(e, "host pipeline record");
  }
  // D2H copies after every H2D and launch is enqueued: with pageable host
  // buffers each copy call blocks the host until its data moved, so the
  // later groups' staging and kernels must already be in flight
  for (int g = 0; g < L.groups; ++g) {
    const int64_t bh0 = int64_t(g) * L.hpg;
    const int64_t cnt = BH - bh0 < L.hpg ? BH - bh0 : L.hpg;
    const size_t yo = size_t(bh0 * nq * dvw);
    e = cudaStreamWaitEvent(hp->out, hp->ev_comp[g], 0);
    if (e == cudaSuccess)
      e = cudaMemcpyAsync(y + yo, dy + yo, size_t(cnt * nq * dvw) * 4, cudaMemcpyDeviceToHost,
                          hp->out);
    if (e != cudaSuccess) return fail(e, "host pipeline D2H");
  }
  e = cudaEventRecord(hp->done, hp->out);
  if (e == cudaSuccess) e = cudaStreamWaitEvent(caller, hp->done, 0);
  if (e != cudaSuccess) return fail(e, "host pipeline join");
  t_last_launches = launches;
  return ELSA_OK;
}

int elsa_partial_f32(const float* q, const float* k, const float* v, const elsa_shape* shp,
                     double scale, int64_t kv_begin, int64_t kv_end, float* m, float* S,
                     float* W, int kv_splits, void* workspace, size_t ws_bytes, void* stream) {
  t_last_launches = 0;
  if (!valid_shape(shp) || kv_splits < 0 || !std::isfinite(scale)) return ELSA_ERR_SHAPE;
  if (kv_begin < 0 || kv_end < kv_begin || kv_end > shp->n_kv) return ELSA_ERR_SHAPE;
  if (!q || !k || !v || !m || !S || !W) return ELSA_ERR_SHAPE;
  if (shp->B * shp->H * shp->n_q == 0) return ELSA_OK;
  return run_forward(q, k, v, shp, scale, kv_begin, kv_end, kv_splits, workspace, ws_bytes,
                     static_cast<cudaStream_t>(stream), nullptr, m, S, W);
}

int elsa_fwd_f16(const void* q, const void* k, const void* v, void* y, const elsa_shape* shp,
                 double scale, int is_bf16, void* stream) {
  t_last_launches = 0;
  if (!valid_shape(shp) || !std::isfinite(scale)) return ELSA_ERR_SHAPE;
  if (shp->d > 128 || shp->dv > 128) return ELSA_ERR_SHAPE;
  const bool wide16 = shp->d > 64 || shp->dv > 64;  // the D = 128 kernel (one query tile per CTA)
  if (!q || !k || !v || !y) return ELSA_ERR_SHAPE;
  if (shp->B * shp->H * shp->n_q == 0) return ELSA_OK;
  DeviceCache* dc = nullptr;
  if (int st = current_device_cache(&dc)) return st;
  int64_t q_st[3], k_st[3], v_st[3], y_st[3];
  std::memcpy(q_st, shp->q_stride, sizeof(q_st));
  std::memcpy(k_st, shp->k_stride, sizeof(k_st));
  std::memcpy(v_st, shp->v_stride, sizeof(v_st));
  std::memcpy(y_st, shp->y_stride, sizeof(y_st));
  sanitize(q_st, shp->n_q, shp->H, shp->B, shp->d);
  sanitize(k_st, shp->n_kv, shp->H, shp->B, shp->d);
  sanitize(v_st, shp->n_kv, shp->H, shp->B, shp->dv);
  sanitize(y_st, shp->n_q, shp->H, shp->B, shp->dv);
  // Q, K, V go through TMA (16-byte aligned bases and row strides); Y may be
  // stored element-wise
  if (!aligned16(q, q_st) || !aligned16(k, k_st) || !aligned16(v, v_st)) return ELSA_ERR_SHAPE;
  for (int i = 0; i < 3; ++i)
    if (y_st[i] < 0) return ELSA_ERR_SHAPE;
  const bool bf16 = is_bf16 != 0;
  // 64 < d <= 128: 128-key tiles with P aliased over S. ELSA_TC_TK=64 selects
  // the 64-key-tile kernel (no aliasing, S_g(t+1) overlaps the exponentials):
  // measured slower (BF16 16K 975 vs 1224, 64K 922 vs 1096; faster only at
  // n = 1K, 409 vs 350 TFLOP/s; profiles/round2_tc_d128_tk64.txt)
  // (built with -DELSA_EXPERIMENTAL_TC_TK64=1 only)
  static const int tc_tk = [] {
    const char* e = std::getenv("ELSA_TC_TK");
    return ELSA_EXPERIMENTAL_TC_TK64 && e && std::atoi(e) == 64 ? 64 : 128;
  }();
  const int kv_box = wide16 ? tc_tk : 128;
  CUtensorMap maps[3];
  if (!encode_map16(&maps[0], q, shp->d, shp->n_q, shp->H, shp->B, q_st, bf16) ||
      !encode_map16(&maps[1], k, shp->d, shp->n_kv, shp->H, shp->B, k_st, bf16, kv_box) ||
      !encode_map16(&maps[2], v, shp->dv, shp->n_kv, shp->H, shp->B, v_st, bf16, kv_box))
    return ELSA_ERR_SHAPE;
  TcParams p;
  std::memset(&p, 0, sizeof(p));
  p.y = y;
  p.B = int(shp->B);
  p.H = int(shp->H);
  p.n_q = int(shp->n_q);
  p.n_kv = int(shp->n_kv);
  p.dv = int(shp->dv);
  p.y_vec = aligned16(y, y_st) ? 1 : 0;
  p.ys_b = y_st[0];
  p.ys_h = y_st[1];
  p.ys_r = y_st[2];
  double c = std::fabs(scale) * kLog2e;
  if (c < 1e-30) c = 1e-30;
  p.c = float(c);
  p.neg = scale < 0 ? 1 : 0;
  p.err = dc->err;
  // two query tiles (two softmax warpgroups) per CTA when that still fills the
  // GPU a few times over; ELSA_TC_GROUPS forces 1 or 2
  static const int forced_groups = [] {
    const char* e = std::getenv("ELSA_TC_GROUPS");
    return e ? std::atoi(e) : 0;
  }();
  const int64_t BH = shp->B * shp->H;
  // waves of one-tile vs two-tile CTAs; a two-tile CTA takes ~1.4x a one-tile
  // CTA's time (measured: B1 H16 n = 1K one-tile 16.4 vs 20.4 us, n = 2K
  // two-tile 34.8 vs 43.0 us, BERT-base two-tile 26.6 vs 28.7 us)
  const int64_t waves1 = ceil_div(ceil_div(shp->n_q, 128) * BH, dc->sms);
  const int64_t waves2 = ceil_div(ceil_div(shp->n_q, 256) * BH, dc->sms);
  int groups = 1.4 * double(waves2) <= double(waves1) ? 2 : 1;
  if (forced_groups == 1 || forced_groups == 2) groups = forced_groups;
  auto launch = [&](auto traits, auto kern, int slot) -> int {
    using TT = decltype(traits);
    p.qtiles = int(ceil_div(shp->n_q, TT::ROWS));
    if (!dc->attr[slot]) {
      const cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                                 int(TT::SMEM_BYTES));
      if (e != cudaSuccess) return cuda_fail(e, "cudaFuncSetAttribute(tc)");
      dc->attr[slot] = true;
    }
    const int64_t gx = int64_t(p.qtiles) * BH;
    if (gx >= (int64_t(1) << 31)) return ELSA_ERR_SHAPE;
    kern<<<unsigned(gx), TT::THREADS, TT::SMEM_BYTES, static_cast<cudaStream_t>(stream)>>>(
        p, maps[0], maps[1], maps[2]);
    return ELSA_OK;
  };
  const int base = kAttrSlots - 14;  // the last fourteen slots
  // ELSA_TC_CS=2 (experiment, built with -DELSA_EXPERIMENTAL_TC_CS2=1): two
  // softmax warps per row (column split), d <= 64 two-group CTAs — measured
  // slower (BF16 16K 801 vs 905 TFLOP/s, profiles/round2_tc_cs2.txt)
  static const int tc_cs = [] {
    const char* e = std::getenv("ELSA_TC_CS");
    return ELSA_EXPERIMENTAL_TC_CS2 && e && std::atoi(e) == 2 ? 2 : 1;
  }();
  int st;
#if ELSA_EXPERIMENTAL_TC_TK64
  if (wide16 && tc_tk == 64 && groups == 2)
    st = bf16 ? launch(TcTraits<2, 128, 64>{}, fwd_tc_kernel<true, 2, 128, 64>, base + 11)
              : launch(TcTraits<2, 128, 64>{}, fwd_tc_kernel<false, 2, 128, 64>, base + 10);
  else if (wide16 && tc_tk == 64)
    st = bf16 ? launch(TcTraits<1, 128, 64>{}, fwd_tc_kernel<true, 1, 128, 64>, base + 9)
              : launch(TcTraits<1, 128, 64>{}, fwd_tc_kernel<false, 1, 128, 64>, base + 8);
  else
#endif
  if (wide16 && groups == 2)
    st = bf16 ? launch(TcTraits<2, 128>{}, fwd_tc_kernel<true, 2, 128>, base + 7)
              : launch(TcTraits<2, 128>{}, fwd_tc_kernel<false, 2, 128>, base + 6);
  else if (wide16)
    st = bf16 ? launch(TcTraits<1, 128>{}, fwd_tc_kernel<true, 1, 128>, base + 5)
              : launch(TcTraits<1, 128>{}, fwd_tc_kernel<false, 1, 128>, base + 4);
#if ELSA_EXPERIMENTAL_TC_CS2
  else if (groups == 2 && tc_cs == 2)
    st = bf16 ? launch(TcTraits<2, 64, 128, 2>{}, fwd_tc_kernel<true, 2, 64, 128, 2>, base + 13)
              : launch(TcTraits<2, 64, 128, 2>{}, fwd_tc_kernel<false, 2, 64, 128, 2>, base + 12);
#endif
  else if (groups == 2)
    st = bf16 ? launch(TcTraits<2>{}, fwd_tc_kernel<true, 2>, base + 3)
              : launch(TcTraits<2>{}, fwd_tc_kernel<false, 2>, base + 2);
  else
    st = bf16 ? launch(TcTraits<1>{}, fwd_tc_kernel<true, 1>, base + 1)
              : launch(TcTraits<1>{}, fwd_tc_kernel<false, 1>, base);
  if (st) return st;
  if (cudaPeekAtLastError() != cudaSuccess) return cuda_fail(cudaGetLastError(), "tc launch");
  ++t_last_launches;
  return ELSA_OK;
}

int elsa_merge_f32(const float* m, const float* S, const float* W, int parts, int64_t rows,
                   int dv, int64_t part_stride, int finalize, float* y, float* m_out,
                   float* S_out, float* W_out, void* stream) {
  t_last_launches = 0;
  if (parts < 1 || parts > kMergeMaxParts || rows < 0 || dv < 1 || dv > kMaxDv) return ELSA_ERR_SHAPE;
  if (part_stride < rows) return ELSA_ERR_SHAPE;
  if (!m || !S || !W) return ELSA_ERR_SHAPE;
  if (finalize ? !y : (!m_out || !S_out || !W_out)) return ELSA_ERR_SHAPE;
  if (rows == 0) return ELSA_OK;
  DeviceCache* dc = nullptr;
  if (int st = current_device_cache(&dc)) return st;
  MergeParams mp;
  std::memset(&mp, 0, sizeof(mp));
  mp.m = m;
  mp.S = S;
  mp.W = W;
  mp.parts = parts;
  mp.rows = rows;
  mp.dv = dv;
  mp.w_pitch = dv;
  mp.part_stride = part_stride;
  mp.log2_domain = 0;
  mp.finalize = finalize ? 1 : 0;
  mp.y = y;
  mp.n_q = 0;  // dense [rows][dv] output
  mp.m_out = m_out;
  mp.S_out = S_out;
  mp.W_out = W_out;
  mp.out_pitch = dv;
  mp.err = dc->err;
  return launch_merge(mp, static_cast<cudaStream_t>(stream));
}

int elsa_merge_peers_f32(const float* const* m_ptrs, const float* const* S_ptrs,
                         const float* const* W_ptrs, int ranks, int per_rank, int64_t rows_total,
                         int64_t row_lo, int64_t rows, int dv, float* y, void* stream) {
  t_last_launches = 0;
  if (!m_ptrs || !S_ptrs || !W_ptrs || !y) return ELSA_ERR_SHAPE;
  if (ranks < 1 || ranks > kMaxPeers || per_rank < 1 || ranks * per_rank > kMergeMaxParts)
    return ELSA_ERR_SHAPE;
  if (dv < 1 || dv > kMaxDv || rows < 0 || row_lo < 0 || rows_total < row_lo + rows) return ELSA_ERR_SHAPE;
  if (rows == 0) return ELSA_OK;
  DeviceCache* dc = nullptr;
  if (int st = current_device_cache(&dc)) return st;
  PeerMergeParams mp;
  std::memset(&mp, 0, sizeof(mp));
  for (int r = 0; r < ranks; ++r) {
    if (!m_ptrs[r] || !S_ptrs[r] || !W_ptrs[r]) return ELSA_ERR_SHAPE;
    mp.m[r] = m_ptrs[r];
    mp.S[r] = S_ptrs[r];
    mp.W[r] = W_ptrs[r];
  }
  mp.ranks = ranks;
  mp.per_rank = per_rank;
  mp.rows_total = rows_total;
  mp.row_lo = row_lo;
  mp.rows = rows;
  mp.dv = dv;
  mp.y = y;
  mp.err = dc->err;
  constexpr int kWarps = 8;
  const int64_t blocks = ceil_div(rows, kWarps);
  if (blocks >= (int64_t(1) << 31)) return ELSA_ERR_SHAPE;
  const int parts = ranks * per_rank;
  auto kern = parts <= 2    ? merge_peers_kernel<2>
              : parts <= 4  ? merge_peers_kernel<4>
              : parts <= 8  ? merge_peers_kernel<8>
              : parts <= 16 ? merge_peers_kernel<16>
                            : merge_peers_kernel<32>;
  const dim3 grid{unsigned(blocks), unsigned(dv_slices(dv)), 1u};
  kern<<<grid, kWarps * 32, 0, static_cast<cudaStream_t>(stream)>>>(mp);
  if (cudaPeekAtLastError() != cudaSuccess) return cuda_fail(cudaGetLastError(), "peer merge launch");
  ++t_last_launches;
  return ELSA_OK;
}

int elsa_blockwise_f32(const float* q, const float* k, const float* v, const elsa_shape* shp,
                       double scale, int64_t block_size, float* m, float* S, float* W,
                       void* stream) {
  t_last_launches = 0;
  if (!valid_shape(shp) || block_size < 1 || !std::isfinite(scale)) return ELSA_ERR_SHAPE;
  if (!q || !k || !v || !m || !S || !W) return ELSA_ERR_SHAPE;
  if (shp->B * shp->H * shp->n_q == 0) return ELSA_OK;
  DeviceCache* dc = nullptr;
  if (int st = current_device_cache(&dc)) return st;
  int64_t q_st[3], k_st[3], v_st[3];
  std::memcpy(q_st, shp->q_stride, sizeof(q_st));
  std::memcpy(k_st, shp->k_stride, sizeof(k_st));
  std::memcpy(v_st, shp->v_stride, sizeof(v_st));
  sanitize(q_st, shp->n_q, shp->H, shp->B, shp->d);
  sanitize(k_st, shp->n_kv, shp->H, shp->B, shp->d);
  sanitize(v_st, shp->n_kv, shp->H, shp->B, shp->dv);
  const int64_t BH = shp->B * shp->H;
  const int64_t nb = ceil_div(shp->n_kv, block_size);
  const int64_t bsz = block_size < shp->n_kv ? block_size : shp->n_kv;
  if (bsz >= (int64_t(1) << 30)) return ELSA_ERR_SHAPE;
  // one split per key block; the kernel's own planner picks the CTA shape for
  // a single-split problem of one block's length
  Plan plan = plan_for(shp, bsz, 1, dc->sms);
  plan.splits = 1;
  constexpr int64_t kMaxGridY = 65535;
  for (int64_t b0 = 0; b0 < nb; b0 += kMaxGridY) {
    const int64_t cnt = nb - b0 < kMaxGridY ? nb - b0 : kMaxGridY;
    FwdParams p;
    fill_common(p, q, k, v, shp, scale, q_st, k_st, v_st);
    p.kv_begin = int(b0 * block_size);
    p.kv_end = int(shp->n_kv);
    p.split_keys = int(bsz);
    p.err = dc->err;
    p.bh_begin = 0;
    p.mode = kModePartialNat;
    p.pm = m + b0;
    p.pS = S + b0;
    p.pW = W + b0 * shp->dv;
    p.part_stride = 1;
    p.row_stride = nb;
    p.pw_pitch = int(shp->dv);
    p.pw_vec = (reinterpret_cast<uintptr_t>(p.pW) % 16 == 0) && (shp->dv % 4 == 0);
    Plan pl = plan;
    pl.splits = int(cnt);
    if (int st = launch_fwd(p, shp, q_st, k_st, v_st, pl, BH, dc,
                            static_cast<cudaStream_t>(stream)))
      return st;
  }
  return ELSA_OK;
}

size_t elsa_block_scan_workspace_bytes(int64_t rows, int nblocks, int dv) {
  if (rows < 0 || nblocks < 1 || dv < 1 || dv > kMaxDv) return 0;
  int64_t kp = 1;
  while (kp < nblocks) kp <<= 1;
  return size_t(rows) * size_t(kp) * size_t(2 + dv) * sizeof(float);
}

int elsa_block_scan_f32(const float* m, const float* S, const float* W, int64_t rows, int nblocks,
                        int dv, float* total_m, float* total_S, float* total_W, float* pre_m,
                        float* pre_S, float* pre_W, void* workspace, size_t ws_bytes,
                        void* stream) {
  t_last_launches = 0;
  if (rows < 0 || nblocks < 1 || dv < 1 || dv > kMaxDv) return ELSA_ERR_SHAPE;
  if (!m || !S || !W || !total_m || !total_S || !total_W) return ELSA_ERR_SHAPE;
  const bool pre = pre_m || pre_S || pre_W;
  if (pre && !(pre_m && pre_S && pre_W)) return ELSA_ERR_SHAPE;
  if (rows == 0) return ELSA_OK;
  if (!workspace || ws_bytes < elsa_block_scan_workspace_bytes(rows, nblocks, dv))
    return ELSA_ERR_WORKSPACE;
  DeviceCache* dc = nullptr;
  if (int st = current_device_cache(&dc)) return st;
  BlockScanParams bp;
  std::memset(&bp, 0, sizeof(bp));
  bp.m = m;
  bp.S = S;
  bp.W = W;
  bp.rows = rows;
  bp.K = nblocks;
  bp.K_pad = 1;
  bp.levels = 0;
  while (bp.K_pad < nblocks) {
    bp.K_pad <<= 1;
    ++bp.levels;
  }
  bp.dv = dv;
  bp.ws = static_cast<float*>(workspace);
  bp.total_m = total_m;
  bp.total_S = total_S;
  bp.total_W = total_W;
  bp.pre_m = pre ? pre_m : nullptr;
  bp.pre_S = pre_S;
  bp.pre_W = pre_W;
  constexpr int kWarps = 8;
  const int64_t blocks = ceil_div(rows, kWarps);
  if (blocks >= (int64_t(1) << 31)) return ELSA_ERR_SHAPE;
  // per-warp slice of the padded array in shared memory when it fits (the
  // global workspace is still required by the ABI and used beyond that)
  const size_t smem = size_t(kWarps) * size_t(bp.K_pad) * size_t(2 + dv) * sizeof(float);
  if (smem <= 48 * 1024) {  // larger slices cost more occupancy than they save (measured K = 32)
    static bool attr_set[kMaxDevices] = {};
    int dev = 0;
    cudaGetDevice(&dev);
    if (dev >= 0 && dev < kMaxDevices && !attr_set[dev]) {
      const cudaError_t e = cudaFuncSetAttribute(
          block_scan_f32_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, 48 * 1024);
      if (e != cudaSuccess) return cuda_fail(e, "cudaFuncSetAttribute(block scan)");
      attr_set[dev] = true;
    }
    block_scan_f32_kernel<true><<<unsigned(blocks), kWarps * 32, smem,
                                  static_cast<cudaStream_t>(stream)>>>(bp);
  } else {
    block_scan_f32_kernel<false><<<unsigned(blocks), kWarps * 32, 0,
                                   static_cast<cudaStream_t>(stream)>>>(bp);
  }
  if (cudaPeekAtLastError() != cudaSuccess) return cuda_fail(cudaGetLastError(), "block scan launch");
  ++t_last_launches;
  return ELSA_OK;
}

int elsa_device_alloc(size_t bytes, void** ptr) {
  if (!ptr) return ELSA_ERR_SHAPE;
  *ptr = nullptr;
  if (bytes == 0) return ELSA_OK;
  const cudaError_t e = cudaMalloc(ptr, bytes);
  return e == cudaSuccess ? ELSA_OK : cuda_fail(e, "cudaMalloc");
}

int elsa_device_free(void* ptr) {
  if (!ptr) return ELSA_OK;
  const cudaError_t e = cudaFree(ptr);
  return e == cudaSuccess ? ELSA_OK : cuda_fail(e, "cudaFree");
}

int elsa_get_device_error(void* stream, int* code) {
  if (!code) return ELSA_ERR_SHAPE;
  DeviceCache* dc = nullptr;
  if (int st = current_device_cache(&dc)) return st;
  cudaStream_t strm = static_cast<cudaStream_t>(stream);
  int host = 0;
  if (cudaMemcpyAsync(&host, dc->err, sizeof(int), cudaMemcpyDeviceToHost, strm) != cudaSuccess)
    return ELSA_ERR_CUDA;
  if (cudaMemsetAsync(dc->err, 0, sizeof(int), strm) != cudaSuccess) return ELSA_ERR_CUDA;
  if (cudaStreamSynchronize(strm) != cudaSuccess) return ELSA_ERR_CUDA;
  *code = host;
  return ELSA_OK;
}

int elsa_ffma_peak(void* stream, double* tflops) {
  if (!tflops) return ELSA_ERR_SHAPE;
  DeviceCache* dc = nullptr;
  if (int st = current_device_cache(&dc)) return st;
  cudaStream_t strm = static_cast<cudaStream_t>(stream);
  float* sink = nullptr;
  if (cudaMallocAsync(reinterpret_cast<void**>(&sink), 256 * sizeof(float), strm) != cudaSuccess)
    return ELSA_ERR_CUDA;
  const int blocks = dc->sms * 4;
  const int threads = 256;
  const int iters = 4096;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  // best of: the attention-shaped 8x4 register outer product and the
  // bank-conflict-free immediate form (the FMA pipe's ceiling)
  double best = 0.0;
  int rc = ELSA_OK;
  for (int variant = 0; variant < 2 && rc == ELSA_OK; ++variant) {
    auto kern = variant == 0 ? ffma_peak_kernel : ffma_peak_imm_kernel;
    kern<<<blocks, threads, 0, strm>>>(sink, iters / 4, 0.5f);  // warm-up
    cudaEventRecord(e0, strm);
    kern<<<blocks, threads, 0, strm>>>(sink, iters, 0.5f);
    cudaEventRecord(e1, strm);
    if (cudaEventSynchronize(e1) != cudaSuccess) rc = ELSA_ERR_CUDA;
    float ms = 0.f;
    cudaEventElapsedTime(&ms, e0, e1);
    const double flops = 2.0 * double(kFfmaPerIter) * iters * double(blocks) * threads;
    const double tf = flops / (double(ms) * 1e-3) / 1e12;
    if (tf > best) best = tf;
  }
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  cudaFreeAsync(sink, strm);
  if (rc) return rc;
  *tflops = best;
  return ELSA_OK;
}

int elsa_last_launch_count(void) { return t_last_launches; }

const char* elsa_last_cuda_error(void) { return t_last_cuda_error; }

int elsa_describe_plan(const elsa_shape* shp, int kv_splits, char* buf, size_t n) {
  if (!valid_shape(shp) || kv_splits < 0 || !buf || n == 0) return ELSA_ERR_SHAPE;
  DeviceCache* dc = nullptr;
  int sms = 148;
  if (current_device_cache(&dc) == ELSA_OK) sms = dc->sms;
  const Plan pl = plan_for(shp, shp->n_kv, kv_splits, sms, true, dc);
  static const char* names[] = {"w4r8",     "w8r16",        "w8r8",    "w8r8d128",
                                "w8r8v128", "w8r8d128v128", "w8r8d96", "w8r8d96v128",
                                "w8r8d256", "w4r8d256v128", "w8r8d32v32", "w8r8d96v96",
                                "w8r8v96", "w8r8d128v96", "w4r8d256v256", "w8r8acc", "w8r4"};
  static_assert(sizeof(names) / sizeof(names[0]) == kCfgW8R4 + 1, "one name per config");
  if (pl.cfg < 0 || pl.cfg > kCfgW8R4) return ELSA_ERR_SHAPE;
  const CfgInfo ci = cfg_info(pl.cfg);
  const int64_t slices = ceil_div(shp->dv, cfg_dv(pl.cfg));
  const int64_t chain = ceil_div(ceil_div(shp->n_kv, ci.tk), pl.splits);
  std::string extra = slices > 1 ? " dv_slices=" + std::to_string(slices) : std::string();
  if (pl.cluster) extra += " cluster_merge=dsmem";
  if (pl.tail_s > 0)
    extra += " tail_split=" + std::to_string(pl.tail_s) + "x(units>=" +
             std::to_string(pl.tail_first) + ")";
  if (chain > chain_cap(pl.cfg))
    extra += " chain_tiles=" + std::to_string(chain) + " (over the " +
             std::to_string(chain_cap(pl.cfg)) + "-tile cap: > kMaxSplits x cap keys)";
  std::snprintf(buf, n, "%s tq=%d tk=%d kv_splits=%d heads_per_batch=%lld%s", names[pl.cfg],
                ci.tq, ci.tk, pl.splits, static_cast<long long>(pl.heads_per_batch),
                extra.c_str());
  return ELSA_OK;
}

// Development aid (ELSA_TC_TRACE builds only; not part of include/elsa.h):
// copies K5's per-tile clock stamps (16 slots x kTcTraceTiles x 8) to `out`.
int elsa_dev_read_tc_trace(unsigned long long* out, size_t n) {
#ifdef ELSA_TC_TRACE
  const size_t total = 16 * kTcTraceTiles * 8;
  if (n > total) n = total;
  return cudaMemcpyFromSymbol(out, g_tc_trace, n * sizeof(unsigned long long)) == cudaSuccess
             ? ELSA_OK
             : ELSA_ERR_CUDA;
#else
  (void)out;
  (void)n;
  return ELSA_ERR_SHAPE;
#endif
}

// Development aid (ELSA_TRACE builds only; not part of include/elsa.h):
// copies the phase-timestamp buffer to host memory `out` (n entries).
int elsa_dev_read_trace(unsigned long long* out, size_t n) {
#ifdef ELSA_TRACE
  if (!g_trace) return ELSA_ERR_SHAPE;
  const size_t total = kTraceWords;
  if (n > total) n = total;
  return cudaMemcpy(out, g_trace, n * sizeof(unsigned long long), cudaMemcpyDeviceToHost) ==
                 cudaSuccess
             ? ELSA_OK
             : ELSA_ERR_CUDA;
#else
  (void)out;
  (void)n;
  return ELSA_ERR_SHAPE;
#endif
}

}  // extern "C"
