/*
 * elsa.h — C-ABI of libelsa.so, the B200 (sm_100a) FP32 exact-attention
 * library that computes softmax(Q K^T * scale) V as an associative
 * (m, S, W) state reduction (ELSA, arXiv 2604.23798).
 *
 * Plain C: no CUDA, torch or C++ types cross this boundary. Device
 * pointers are raw `float*`; streams are passed as `void*` holding a
 * `cudaStream_t` (NULL = legacy default stream). All buffers are
 * caller-owned device memory; the library never allocates on the hot
 * path. Every entry point is stream-ordered and never synchronises the
 * host except `elsa_get_device_error` and `elsa_ffma_peak`.
 *
 * Reference interface each entry point replaces (the reference package
 * `scanattn` is pure Python/numpy, /root/reference/pkg/src/scanattn):
 *
 *   elsa_fwd_f32      <- engine.scan_forward(problem, cfg)        engine.py:385-427
 *                        (score-tile producer engine.py:352-358, intra-block
 *                        scan engine.py:148-176/315-339, inter-block sweep
 *                        engine.py:179-199, epilogue engine.py:375-382)
 *   elsa_fwd_f32_host <- the same call with the reference's host (numpy)
 *                        arrays in and out, copies pipelined with the kernels
 *   elsa_partial_f32  <- engine.blockwise_states(...) + inter_block_combine
 *                        engine.py:430-451 / 265-297: the (m, S, W) summary
 *                        of one contiguous key range (Proposition 1,
 *                        PAPER.md:662-666) — the per-KV-shard state
 *   elsa_merge_f32    <- monoid.merge_tree / merge_lanes_into
 *                        monoid.py:234-265 / 160-200, plus the epilogue
 *                        W / S with the normalizer check engine.py:377-382
 *   elsa_scan_depth   <- engine.scan_depth                        engine.py:47-55
 *   status codes      <- errors.py:8-54 mapped as the CLI does, cli.py:341-354
 */
#ifndef ELSA_H_
#define ELSA_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define ELSA_ABI_VERSION 1

/* Status codes. 2/3 match the reference CLI's exit codes for ShapeError /
 * NumericalError (cli.py:344-351). */
typedef enum {
  ELSA_OK = 0,
  ELSA_ERR_SHAPE = 2,      /* bad shape / stride / config  (errors.ShapeError)     */
  ELSA_ERR_NUMERICAL = 3,  /* normalizer <= 0 or non-finite (errors.NumericalError) */
  ELSA_ERR_CUDA = 5,       /* CUDA runtime / launch failure                         */
  ELSA_ERR_NCCL = 6,       /* collective failure (reported by the host layer)       */
  ELSA_ERR_WORKSPACE = 7   /* workspace missing or too small                        */
} elsa_status;

/* Problem geometry. Q:(B,H,n_q,d) K:(B,H,n_kv,d) V:(B,H,n_kv,dv) Y:(B,H,n_q,dv).
 * Strides are in ELEMENTS for the (b, h, row) axes; the last axis of every
 * tensor must be contiguous (stride 1). d <= 256, dv <= 4096 (V wider than the
 * kernel's 64 / 128 columns runs as column slices). */
typedef struct {
  int64_t B, H, n_q, n_kv, d, dv;
  int64_t q_stride[3];
  int64_t k_stride[3];
  int64_t v_stride[3];
  int64_t y_stride[3];
} elsa_shape;

/* ABI version (ELSA_ABI_VERSION of the built library). */
int elsa_abi_version(void);

/* Human-readable text for a status code (static storage). */
const char* elsa_strerror(int status);

/* The reference's depth bound L(n, B) = ceil(log2 min(B,n)) +
 * 2*ceil(log2 ceil(n/B)) + 3 (engine.py:47-55). Returns -1 for n<1 or B<1. */
int elsa_scan_depth(int64_t n, int64_t block_size);

/* kv_splits actually used by elsa_fwd_f32 for `requested` (0 = auto:
 * enough key-range splits to fill the GPU, bounded by the tile count). */
int elsa_resolve_kv_splits(const elsa_shape* shp, int requested);

/* Workspace bytes elsa_fwd_f32 needs for `kv_splits` (0 = auto). Zero when
 * the resolved split count is 1 or the splits merge inside the launch
 * (thread-block-cluster merge over distributed shared memory); non-zero for
 * an auto plan whose last partly-empty wave runs as key pieces (tail split). */
size_t elsa_workspace_bytes(const elsa_shape* shp, int kv_splits);

/* Workspace bytes elsa_partial_f32 needs for keys [kv_begin, kv_end) and
 * `kv_splits` (0 = auto): partial states always merge through the split
 * workspace (their output is a state, not Y). */
size_t elsa_partial_workspace_bytes(const elsa_shape* shp, int64_t kv_begin, int64_t kv_end,
                                    int kv_splits);

/* Y = softmax(Q K^T * scale) V, FP32 in, FP32 FFMA arithmetic, FP32 out.
 * kv_splits: 0 = auto, else the number of contiguous key-range partitions
 * whose partial states are merged by a fixed balanced tree (bitwise
 * deterministic for a given split count). Numerical failures (normalizer
 * <= 0 or non-finite) raise the device error word; read it with
 * elsa_get_device_error. */
int elsa_fwd_f32(const float* q, const float* k, const float* v, float* y,
                 const elsa_shape* shp, double scale, int kv_splits,
                 void* workspace, size_t ws_bytes, void* stream);

/* Device workspace elsa_fwd_f32_host needs: device copies of Q, K, V and Y
 * plus the kv-split workspace of each concurrently running head group. */
size_t elsa_host_workspace_bytes(const elsa_shape* shp, int kv_splits);

/* Y = softmax(Q K^T * scale) V with q, k, v, y in HOST memory (dense
 * row-major (B,H,n,d) arrays; the shape's strides must describe that dense
 * layout). The reference's entry point takes host arrays
 * (engine.scan_forward, engine.py:385-427: numpy in, a new numpy Y out); this
 * is its end-to-end counterpart: the (b, h) heads are cut into groups whose
 * host->device copies, forward kernels and device->host copies overlap on
 * internal per-device streams, all ordered after prior work on `stream`;
 * `stream` waits for the last copy, so y is complete once `stream` is.
 * Page-locked host buffers make the copies asynchronous; pageable ones work
 * but serialise the host. dev_workspace: elsa_host_workspace_bytes() bytes of
 * device memory. Same status codes and device error word as elsa_fwd_f32. */
int elsa_fwd_f32_host(const float* q, const float* k, const float* v, float* y,
                      const elsa_shape* shp, double scale, int kv_splits,
                      void* dev_workspace, size_t ws_bytes, void* stream);

/* Partial state of keys [kv_begin, kv_end) for every query row:
 * m[row] (natural-log anchor, -inf for an empty range), S[row], and
 * W[row*dv + c], rows ordered (b, h, q) densely: row = (b*H + h)*n_q + q.
 * The triple follows monoid.StateTriple (monoid.py:73-119): S = sum
 * exp(s - m), W = sum exp(s - m) v. kv_splits/workspace as for elsa_fwd_f32
 * (internal splits are merged before the state is written). */
int elsa_partial_f32(const float* q, const float* k, const float* v,
                     const elsa_shape* shp, double scale,
                     int64_t kv_begin, int64_t kv_end,
                     float* m, float* S, float* W,
                     int kv_splits, void* workspace, size_t ws_bytes,
                     void* stream);

/* FP16 / BF16 variant: the QK^T and PV contractions on the
 * tcgen05 tensor cores with FP32 accumulation in TMEM; the (m, S, W) states,
 * their combine and the epilogue in FP32. q, k, v, y are 16-bit
 * (is_bf16 ? bfloat16 : float16) with d, dv <= 128; q, k, v with 16-byte
 * aligned bases and strides (TMA); y is written in the same format (any
 * strides). */
int elsa_fwd_f16(const void* q, const void* k, const void* v, void* y,
                 const elsa_shape* shp, double scale, int is_bf16, void* stream);

/* Merge `parts` partial states per row with the reference's balanced
 * pairwise tree (adjacent pairs, odd tail passes through; monoid.py:234-265)
 * and its identity-guarded combine (monoid.py:160-200). Inputs are laid out
 * part-major: m[p*part_stride + row], S[...], W[(p*part_stride + row)*dv + c].
 * finalize != 0: y[row*dv + c] = W / S (normalizer check as engine.py:377-378).
 * finalize == 0: writes the merged state to m_out/S_out/W_out. */
int elsa_merge_f32(const float* m, const float* S, const float* W,
                   int parts, int64_t rows, int dv, int64_t part_stride,
                   int finalize, float* y, float* m_out, float* S_out,
                   float* W_out, void* stream);

/* Fused exchange + merge for the KV-sharded multi-GPU path:
 * rank r's m/S/W buffers (peer-mapped device pointers, e.g. symmetric memory
 * over NVLink) hold the natural-log states of its per_rank key chunks for all
 * rows_total query rows ([chunk][row], W [chunk][row][dv]); this merges rows
 * [row_lo, row_lo + rows) over all ranks * per_rank chunks in global chunk
 * order (chunk c = rank c / per_rank, local chunk c % per_rank) with the
 * merge_tree shape and writes y[rows][dv] = W / S. ranks <= 16,
 * ranks * per_rank <= 32. Replaces all_to_all + elsa_merge_f32. */
int elsa_merge_peers_f32(const float* const* m_ptrs, const float* const* S_ptrs,
                         const float* const* W_ptrs, int ranks, int per_rank,
                         int64_t rows_total, int64_t row_lo, int64_t rows, int dv,
                         float* y, void* stream);

/* Per-key-block partial states for every query row:
 * block j covers keys [j*block_size, min((j+1)*block_size, n_kv)); natural-log
 * anchors. Layout, nblocks = ceil(n_kv / block_size), rows = B*H*n_q in
 * (b, h, q) order: m[row*nblocks + j], S[...], W[(row*nblocks + j)*dv + c].
 * Replaces engine.blockwise_states (engine.py:430-451), which returns the same
 * per-block totals for one query and one (b, h). */
int elsa_blockwise_f32(const float* q, const float* k, const float* v,
                       const elsa_shape* shp, double scale, int64_t block_size,
                       float* m, float* S, float* W, void* stream);

/* Workspace for elsa_block_scan_f32: rows * 2^ceil(log2 nblocks) * (2 + dv)
 * floats. */
size_t elsa_block_scan_workspace_bytes(int64_t rows, int nblocks, int dv);

/* The reference's two-pass inter-block combine per row over nblocks states
 * ([rows][nblocks] layout as elsa_blockwise_f32 writes, natural anchors):
 * identity-padded up-sweep -> total (engine.py:179-199, 265-293) and, when
 * pre_m/pre_S/pre_W are non-NULL, the down-sweep's exclusive prefixes, identity
 * first (engine.py:202-231, 294-297). Same tree shape as the reference. */
int elsa_block_scan_f32(const float* m, const float* S, const float* W,
                        int64_t rows, int nblocks, int dv,
                        float* total_m, float* total_S, float* total_W,
                        float* pre_m, float* pre_S, float* pre_W,
                        void* workspace, size_t ws_bytes, void* stream);

/* Device memory for callers without a CUDA allocator of their own (e.g. a
 * numpy/ctypes binding sizing the workspace of elsa_fwd_f32_host): thin
 * cudaMalloc / cudaFree on the current device. Never used on the hot path. */
int elsa_device_alloc(size_t bytes, void** ptr);
int elsa_device_free(void* ptr);

/* Synchronises `stream`, returns the device error word (0 = none, else an
 * elsa_status) through *code, and clears it. */
int elsa_get_device_error(void* stream, int* code);

/* FFMA roofline microbenchmark (K4): dependent-chain-free FP32 FMA stream on
 * every SM at the live clock. Writes achieved TFLOP/s (2 flop per FMA). */
int elsa_ffma_peak(void* stream, double* tflops);

/* Number of kernels the last elsa_fwd_f32 / elsa_partial_f32 call on this
 * host thread launched (for the bench's gpu_launches accounting). */
int elsa_last_launch_count(void);

/* Human-readable launch plan elsa_fwd_f32 would use for this shape
 * (kernel configuration, query/key tile sizes, kv split count). */
int elsa_describe_plan(const elsa_shape* shp, int kv_splits, char* buf, size_t n);

/* Text of the last CUDA failure reported as ELSA_ERR_CUDA on this host
 * thread ("" if none). */
const char* elsa_last_cuda_error(void);

#ifdef __cplusplus
}
#endif

#endif /* ELSA_H_ */
