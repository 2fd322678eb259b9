/* mmi.h — C ABI of the B200 (sm_100a) MMInference sparse pre-fill library.
 *
 * Operation (PAPER.md, arXiv 2504.16083): modality-aware permutation sparse
 * attention for pre-fill.  Per attention head, an online sparse index is
 * estimated from the last query rows (Alg.1), the
 * tensors are permuted (Alg.1, Alg.2, Alg.3), block-sparse
 * causal FlashAttention runs over the selected key tiles (Alg.5-7),
 * and the output is scattered back to token order (Alg.6, Alg.7).
 *
 * Conventions (all entry points):
 *  - Every tensor pointer is a DEVICE pointer owned by the caller, unless the
 *    parameter name ends in _host.  Layouts are contiguous row-major:
 *      q [H, S, D] bf16, k/v [Hkv, S, D] bf16, o [H, S, D] bf16,
 *      lse [H, S] fp32 (natural log of the softmax normaliser), modality [S] u8.
 *  - GQA: query head h reads KV head h / (H / Hkv)  (reading: Qwen2 convention;
 *    the paper is silent).
 *  - All calls are asynchronous on `stream`; none synchronises the device or
 *    allocates / frees device memory, except the diagnostic calls marked so
 *    (they synchronise the stream).  The host plan of each distinct (problem,
 *    cfg_host) is built once and cached with a pinned copy of its device tables
 *    (small host allocations on first use; up to 16 plans are kept); the tables
 *    are copied into the workspace by mmi_estimate_index asynchronously.
 *  - Concurrency: calls on different workspaces may run concurrently on
 *    different streams / host threads; every piece of mutable device state of a
 *    call (index, scheduler counter, partial rows) lives in its workspace.
 *  - Scratch and the sparse index live in a caller-provided workspace of at
 *    least mmi_workspace_bytes(problem, cfg_host) bytes (256-byte aligned).  The
 *    same (problem, cfg_host) must be passed to every call of one pass.
 *  - Errors: arguments are validated on the host before any launch; a non-OK
 *    status is returned and mmi_last_error() gives a thread-local message.
 *    Launch failures return MMI_E_CUDA.  Nothing is launched on error.
 *  - Deterministic: the same inputs give a bit-identical index and output.
 */
#ifndef MMI_H_
#define MMI_H_

#include <stddef.h>
#include <stdint.h>

#if defined(__GNUC__)
#define MMI_API __attribute__((visibility("default")))
#else
#define MMI_API
#endif

#ifdef __cplusplus
extern "C" {
#endif

typedef struct CUstream_st* mmi_stream_t; /* == cudaStream_t */

typedef enum {
  MMI_OK = 0,
  MMI_E_INVALID = 1,     /* null pointer, bad enum value                          */
  MMI_E_SHAPE = 2,       /* H % Hkv != 0, D not in {64,128}, S < 1, ...            */
  MMI_E_CONFIG = 3,      /* pattern config invalid (see mmi_pattern)               */
  MMI_E_UNSUPPORTED = 4, /* n_modalities > MMI_MAX_MOD, stride > 1024, ...         */
  MMI_E_WORKSPACE = 5,   /* workspace null, misaligned or too small                */
  MMI_E_CUDA = 6         /* a CUDA launch / tensor-map creation failed             */
} mmi_status;

/* Pattern kinds ("A-shape, Vertical-Slash and Grid" + FULL / NONE) and the static
 * baseline patterns of the paper's evaluation (tab:impl_details P:685-688). */
typedef enum {
  MMI_PAT_NONE = 0, MMI_PAT_FULL = 1, MMI_PAT_ASHAPE = 2, MMI_PAT_VSLASH = 3, MMI_PAT_GRID = 4,
  MMI_PAT_TRISHAPE = 5,   /* y < sink or x - y < local or x >= S - bottom   (No/K-boundary heads only) */
  MMI_PAT_SF_FIXED = 6,   /* floor(y / local) == floor(x / local) or y = 0 (mod stride)  (reading C23) */
  MMI_PAT_SF_STRIDED = 7  /* x - y < local or (x - y) = 0 (mod stride)                   (reading C23) */
} mmi_kind;
/* Boundary types. K-boundary executes as No-boundary. */
typedef enum { MMI_BND_NONE = 0, MMI_BND_K = 1, MMI_BND_Q = 2, MMI_BND_2D = 3 } mmi_boundary;

/* One pattern (tab:search_space).
 *  ASHAPE: admits key y of query x iff y < sink or x - y < local   (local >= 1)
 *  VSLASH: n_vertical columns + n_slash diagonals chosen online from the
 *          last-64-query estimate; column 0 and offset 0 forced.
 *          Cross-modality pairs of 2D heads: verticals only (n_slash = 0).
 *  GRID:   stride > 0 = fixed frame_stride (phase searched); stride == 0 =
 *          search stride in [stride_min, stride_max] (max 1024).
 *          use_hline / use_vline / use_slash select the lines;
 *          sink / local (>= 1) add the first keys and the causal band (reading C8). */
typedef struct {
  int32_t kind;
  int32_t sink, local;
  int32_t n_vertical, n_slash;
  int32_t stride, stride_min, stride_max;   /* SF_*: stride (1..1024) of the vertical / dilated lines */
  uint8_t use_hline, use_vline, use_slash, _pad;
  int32_t bottom;                           /* TRISHAPE: dense query rows at the end (>= 0) */
} mmi_pattern;

#define MMI_MAX_MOD 4

/* Per-head configuration, the output of the offline search (Alg.4).
 *  NONE/K : intra[0] applies to all rows in original coordinates.
 *  Q      : intra[m] applies to query rows of modality m, original coordinates
 *           (Alg.2, reading C12).
 *  2D     : pair[a][b] applies to query modality a x key modality b; a == b in
 *           modality-rank coordinates, a != b in original coordinates with kinds
 *           NONE / FULL / ASHAPE / VSLASH(n_slash = 0) (Alg.3, C13).
 *           pair[a][a] must not be NONE for a present modality. */
typedef struct {
  int32_t boundary;
  mmi_pattern intra[MMI_MAX_MOD];
  mmi_pattern pair[MMI_MAX_MOD][MMI_MAX_MOD];
} mmi_head_config;

typedef struct {
  int32_t n_heads, n_kv_heads, seq_len, head_dim; /* H, Hkv, S, D (D in {64, 128})        */
  int32_t n_modalities;                           /* labels must be < n_modalities        */
  int32_t last_q;                                 /* estimation rows, 64          */
  int32_t block;                                  /* 128 (reading C19); only 128 supported */
  float scale;                                    /* 0 => 1/sqrt(D)               */
} mmi_problem;

/* Bytes of device workspace needed for (problem, cfg_host[0..H-1]).  0 on invalid input. */
MMI_API size_t mmi_workspace_bytes(const mmi_problem* problem, const mmi_head_config* cfg_host);

/* Step a1-a5: modality bookkeeping, last_q slab estimation, VS
 * top-k, grid stride/phase search and index (view + tile list) construction.
 * Reads q, k, modality; writes only the workspace. */
MMI_API mmi_status mmi_estimate_index(const mmi_problem* problem, const mmi_head_config* cfg_host,
                              const void* q, const void* k, const uint8_t* modality,
                              void* ws, size_t ws_bytes, mmi_stream_t stream);

/* Step a6: the permutation of Q / K / V into the views the index needs (
 * "dynamically loading and writing these tensors within the kernel").  Default build:
 * permuted Q blocks are gathered by mmi_sparse_prefill itself (TMA row gathers from q; outputs are
 * scattered by its epilogue), and this call materialises only K̄ / V̄, which many work items
 * re-read (pads zero-filled).  -DMMI_FUSE_KV builds gather K / V in the kernel too (no copy at
 * all); -DMMI_EXPLICIT_PERMUTE builds materialise Q̄ as well.  Requires mmi_estimate_index on the
 * same ws. */
MMI_API mmi_status mmi_permute(const mmi_problem* problem, const mmi_head_config* cfg_host, void* ws, size_t ws_bytes,
                       const void* q, const void* k, const void* v, mmi_stream_t stream);

/* Step a7: block-sparse causal attention over every work item of the index
 * (tcgen05 / TMEM / TMA kernel).  Rows owned by a single pass are written to
 * o / lse directly; rows with several passes (grid MAIN + SLASH, split-K h-line
 * chunks) leave fp16 normalised partial rows + fp32 LSEs in ws (reading C22:
 * requires |v| <= 65504, the fp16 range, since |O| <= max |v|).  lse may be NULL. */
MMI_API mmi_status mmi_sparse_prefill(const mmi_problem* problem, const mmi_head_config* cfg_host, void* ws,
                              size_t ws_bytes, const void* q, const void* k, const void* v, void* o, float* lse,
                              mmi_stream_t stream);

/* Step a8: LSE-merge the partial rows and scatter them to token order in o / lse.
 * After this call o [H,S,D] holds the complete sparse attention output. */
MMI_API mmi_status mmi_unpermute(const mmi_problem* problem, const mmi_head_config* cfg_host, void* ws, size_t ws_bytes,
                         void* o, float* lse, mmi_stream_t stream);

/* Same-build dense causal attention (the comparator), same kernel and tiles. */
MMI_API mmi_status mmi_dense_prefill(const mmi_problem* problem, const void* q, const void* k, const void* v, void* o,
                             float* lse, mmi_stream_t stream);

/* Sizes of the plan for (problem, cfg_host), host-only (no device work), for
 * reporting algorithmic traffic: out[0] = gathered Q rows (Q̄), out[1] = gathered
 * K/V rows (K̄ and V̄ each), out[2] = heads with LSE-merged rows, out[3] = estimation
 * slabs, out[4] = partial-output rows, out[5] = in-kernel permutation bits (1: permuted Q blocks
 * are gathered by mmi_sparse_prefill, no Q̄ copy; 2: the same for K / V).  Writes min(n, 6) values.  Returns
 * MMI_E_INVALID / MMI_E_SHAPE / MMI_E_CONFIG like mmi_workspace_bytes' validation. */
MMI_API mmi_status mmi_plan_stats(const mmi_problem* problem, const mmi_head_config* cfg_host, int64_t* out_host,
                                  int n);

/* REPORTING ONLY (synchronises the stream; call after mmi_estimate_index).  Rows the
 * permute step actually moves: out[0] / out[1] = Q̄ rows read / written, out[2] /
 * out[3] = K̄ (and V̄) rows read / written (padding rows are written as zeros). */
MMI_API mmi_status mmi_traffic_stats(const mmi_problem* problem, const mmi_head_config* cfg_host, const void* ws,
                                     size_t ws_bytes, int64_t* out_host, mmi_stream_t stream);

/* TEST ONLY (synchronises the stream).  Copies the estimated index of head h
 * to host_buf as int32 words: see mmi_export_layout in the Python binding.
 * Returns the number of int32 words needed when host_buf is NULL (via *words). */
MMI_API mmi_status mmi_export_index(const mmi_problem* problem, const mmi_head_config* cfg_host, const void* ws,
                            size_t ws_bytes, int32_t head, int32_t* host_buf, size_t* words, mmi_stream_t stream);

/* TEST ONLY: per-row admitted-key fingerprints (count, sum pos, sum pos^2) of
 * the sparse pass, int64 [H, S, 3] device buffer (zeroed by the caller). */
MMI_API mmi_status mmi_sparse_fingerprint(const mmi_problem* problem, const mmi_head_config* cfg_host, void* ws,
                                  size_t ws_bytes, const void* q, const void* k, const void* v, int64_t* fp,
                                  mmi_stream_t stream);

/* Permuted NATTEN / DiT neighborhood attention (App. F): tokens of a
 * T x Hh x Ww grid in raster order (pos = (t * Hh + y) * Ww + x, T * Hh * Ww = seq_len); every
 * query attends BIDIRECTIONALLY to the kt x kh x kw window around it, clamped inside the grid
 * (start = clamp(c - k/2, 0, L - k) per dimension, NATTEN semantics, reading C25).  The tokens are
 * permuted into bt x bh x bw = 128-token tiles so the windows become block-sparse tile lists run
 * by the same tcgen05 kernel.  q [H,S,D], k/v [Hkv,S,D], o [H,S,D] bf16, lse [H,S] fp32 (nullable).
 * The index depends only on (problem, config): built on the host once, cached, uploaded
 * asynchronously from pinned memory.  Errors: MMI_E_SHAPE (T*Hh*Ww != S, H % Hkv, D),
 * MMI_E_CONFIG (window > grid extent, tile != 128 tokens), MMI_E_WORKSPACE; message via
 * mmi_natten_last_error(). */
typedef struct {
  int32_t T, Hh, Ww;   /* token grid */
  int32_t kt, kh, kw;  /* window */
  int32_t bt, bh, bw;  /* permutation tile, bt * bh * bw = 128 */
} mmi_natten_config;
MMI_API size_t mmi_natten_workspace_bytes(const mmi_problem* problem, const mmi_natten_config* cfg);
MMI_API mmi_status mmi_natten_prefill(const mmi_problem* problem, const mmi_natten_config* cfg, void* ws,
                                      size_t ws_bytes, const void* q, const void* k, const void* v, void* o,
                                      float* lse, mmi_stream_t stream);
/* TEST ONLY: per-row admitted-key fingerprints (count, sum pos, sum pos^2) as the kernel applies
 * the window, int64 [H, S, 3] device buffer zeroed by the caller. */
MMI_API mmi_status mmi_natten_fingerprint(const mmi_problem* problem, const mmi_natten_config* cfg, void* ws,
                                          size_t ws_bytes, const void* q, const void* k, const void* v, int64_t* fp,
                                          mmi_stream_t stream);
MMI_API const char* mmi_natten_last_error(void);

/* ANALYSIS.  Top-k coverage: for every head h and sampled
 * query row rows[i] (device int32 positions), the smallest number of keys whose causal softmax
 * probabilities sum to at least `target` (e.g. 0.95 -> "top 5.78% of attention weights recall
 * 95%"), divided by the row's causal key count rows[i] + 1; written to frac [H, n_rows]
 * (device fp32).  Scratch (device) of mmi_topk_coverage_scratch_bytes(problem, n_rows) bytes.
 * Asynchronous; deterministic (integer fixed-point mass histograms).  Returns MMI_E_INVALID /
 * MMI_E_SHAPE / MMI_E_WORKSPACE on bad arguments, MMI_E_CUDA if a launch fails. */
MMI_API size_t mmi_topk_coverage_scratch_bytes(const mmi_problem* problem, int32_t n_rows);
MMI_API mmi_status mmi_topk_coverage(const mmi_problem* problem, const void* q, const void* k, const int32_t* rows,
                                     int32_t n_rows, float target, float* frac, void* scratch, size_t scratch_bytes,
                                     mmi_stream_t stream);

/* DIAGNOSTIC (synchronises the stream).  Device-side error flags raised by the last
 * mmi_estimate_index on this workspace (0 = none):
 *   MMI_FLAG_LABEL_RANGE  a modality label >= n_modalities: those tokens belong to no
 *                         modality group, so Q-/2D-boundary heads do not compute their rows;
 *   MMI_FLAG_SEG_OVERFLOW the index needed more tile segments than the plan's bound: the
 *                         affected work items were left empty (nothing is written out of bounds). */
#define MMI_FLAG_LABEL_RANGE 1u
#define MMI_FLAG_SEG_OVERFLOW 2u
MMI_API mmi_status mmi_workspace_flags(const mmi_problem* problem, const mmi_head_config* cfg_host, const void* ws,
                                       size_t ws_bytes, uint32_t* flags_host, mmi_stream_t stream);

/* Thread-local message for the last non-OK status of this thread. */
MMI_API const char* mmi_last_error(void);

/* Library version string. */
MMI_API const char* mmi_version(void);

#ifdef __cplusplus
}
#endif
#endif /* MMI_H_ */
