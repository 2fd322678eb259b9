// Internal device data structures shared by the index builder, the gather
// kernels and the block-sparse attention kernel.  Not part of the public ABI.
#pragma once
#include <cstdint>
#include <cuda_fp16.h>
#include <cuda_runtime.h>

namespace mmi {

constexpr int BLK = 128;          // row block / key tile (reading C19)
constexpr int MAX_MOD = 4;
constexpr int KPAD = 0x7fffffff;  // position of a pad key: never causally visible (reading C14)
// device-side error flags in the workspace (read back by mmi_workspace_flags)
constexpr unsigned FLAG_LABEL_RANGE = 1u;   // a modality label >= n_modalities
constexpr unsigned FLAG_SEG_OVERFLOW = 2u;  // the index needed more tile segments than the plan bound

// ---- segment: a run of consecutive 128-key tiles of one K-view ----
// meta bits: [0] space (0 = original K/V, 1 = gathered K̄/V̄), [2,5) role,
// [5] coordinate system of the pattern (0 = original position, 1 = modality
// rank), [8,16) instance id (index into the head's InstParam table).
// Every tile has a state per query half (the two 128-row blocks of a work
// item): DEAD (no admitted element for any row of the half: no MMA, no
// softmax), PRED (the element predicate is evaluated) or FULL (every element
// admitted).  Per half the segment's tiles read
//     DEAD^dh  PRED^ph  FULL*  PRED^pt  DEAD^dt      (st[half] = {dh, ph, pt, dt})
// and a tile is in the segment only if it is live for at least one half.
// R_NAT: 3D neighborhood window of a permuted NATTEN tile (f4), bidirectional
enum Role : uint32_t { R_TRUE = 0, R_A = 1, R_NOTA = 2, R_VSSL = 3, R_NAT = 4 };
enum TileState : uint32_t { TS_DEAD = 0, TS_PRED = 1, TS_FULL = 2 };
constexpr int SEG_MAX_TILES = 32767;   // per-half counts are int16
struct Seg {
  int32_t krow0;      // K-space row of the first key of the first tile
  int32_t ntiles;
  uint32_t meta;
  int32_t pad;
  int16_t st[2][4];   // per half: dead head, pred head, pred tail, dead tail
};
static_assert(sizeof(Seg) == 32, "Seg is two 16-byte loads");
__host__ __device__ inline uint32_t seg_meta(uint32_t space, uint32_t role, uint32_t rank, uint32_t inst) {
  return space | (role << 2) | (rank << 5) | (inst << 8);
}
__host__ __device__ inline uint32_t seg_tile_state(const Seg& s, int half, int t) {
  const int dh = s.st[half][0], ph = s.st[half][1], pt = s.st[half][2], dt = s.st[half][3];
  if (t < dh || t >= s.ntiles - dt) return TS_DEAD;
  if (t < dh + ph || t >= s.ntiles - dt - pt) return TS_PRED;
  return TS_FULL;
}

// Last key coordinate NOT in the local part of the A part of query coordinate x: the local band
// is y > x - local (local >= 1), or, in block mode (local < 0, SparseTransformer fixed, reading
// C23), the query's segment y >= floor(x / L) * L of L = -local keys.  Nondecreasing in x.
__host__ __device__ inline int a_thr(int x, int local) {
  return local >= 0 ? x - local : x - x % (-local) - 1;
}
// h-line rows of a grid with stride s and phase p: x = p (mod s) and x >= p (a static grid uses
// s = 1, p = S - bottom for the tri-shape's dense bottom rows)
__host__ __device__ inline bool hline_row(int x, int s, int p) { return x >= p && (x - p) % s == 0; }

// ---- pattern instance parameters for the kernel (after estimation) ----
struct InstParam {
  int32_t sink, local;      // A / NOTA roles
  int32_t s, p;             // grid stride / phase (informational)
  int32_t slash_word;       // VS: word offset of the slash-offset bitmap (-1 none)
  int32_t vmask_word;       // VS: word offset of the vertical-column bitmap (-1 none)
  int32_t pad0, pad1;
};

// ---- work item: one 128-row block of one Q-view, one online softmax ----
enum OutMode : int32_t { OUT_FINAL = 0, OUT_PARTIAL = 1 };
struct WorkItem {
  int32_t head;       // query head
  int32_t q_row0;     // first row in the Q space (orig: h*S + 128*b; gathered: view row)
  int32_t seg_off;    // first Seg
  int32_t n_segs;
  int32_t n_tiles;    // total tiles (0 => empty item)
  int32_t q_gathered; // 1 => rows come from the gathered Q̄ space
  int32_t out_mode;   // OUT_FINAL / OUT_PARTIAL
  int32_t out_row0;   // first row in the partial buffer (OUT_PARTIAL)
  int32_t inst_base;  // first InstParam of this head
  int32_t skip_s;     // >0: do not write rows whose coord = skip_p (mod skip_s)
  int32_t skip_p;     //     (hline rows owned by the HROW pass, reading C9)
  int32_t skip_rank;  //     coord system of the skip test
  int32_t row_mod;    // >=0: only rows of this modality are valid (Q-boundary class views)
  int32_t has_b;      // 1: the item also covers the next 128-row block (rows q_row0 + 128 ...)
  int32_t pad[2];     // [0] first row position (work-order key), [1] live (tile, half) pairs
};

struct AttnParams {
  const WorkItem* items;
  int32_t n_items;
  const Seg* segs;
  const InstParam* insts;
  const uint32_t* bits;
  const int32_t* qg_pos;    // gathered Q space: original position per row (-1 pad)
  const int32_t* qg_rank;   // gathered Q space: modality rank per row
  const int32_t* kg_pos;    // gathered K space: original position per row (KPAD pad)
  const int32_t* kg_rank;   // gathered K space: modality rank per row
  const int32_t* rank;      // modality rank by original position [S_pad]
  const uint8_t* labels;    // modality label by original position [S]
  void* o;                  // bf16 [H, S, D]
  float* lse;               // [H, S] (nullable)
  __half* part_o;           // fp16 partial rows [rows, D] (normalised O of one pass; merged in fp32)
  float* part_lse;
  int32_t S, H, Hkv, D;
  float scale_log2;         // tau * log2(e)
  int32_t dense;            // 1 => implicit dense causal items (same-build comparator)
  int32_t fingerprint;      // 1 => accumulate per-row admitted-key fingerprints instead of attention
  int64_t* fp_out;          // [H, S, 3] count, sum pos, sum pos^2 (fingerprint mode)
  long long* dbg;           // optional per-item timestamps (debug only)
  unsigned int* sched;      // work-item counter (zeroed before the launch)
  // in-kernel permutation: permuted Q / K / V blocks are gathered from the
  // original tensors by their source rows (TMA tile::gather4) instead of reading materialised
  // Q̄ / K̄ / V̄ copies
  int32_t fused;            // bit 0: gather permuted Q blocks from q; bit 1: K / V blocks from k / v
  const int32_t* qg_src;    // Q̄ row -> row of Q [H*S] (negative: padding)
  const int32_t* kg_src;    // K̄ row -> row of K / V [Hkv*S] (negative: padding)
  int32_t q_oob, kv_oob;    // out-of-range row (zero fill) of Q / of K and V
  // permuted NATTEN (f4): grid T x Hh x Ww, window kt x kh x kw, tiles bt x bh x bw (= 128 keys),
  // nat_tiles tiles per head in the permuted K̄ space
  int32_t nat_T, nat_H, nat_W, nat_kt, nat_kh, nat_kw, nat_bt, nat_bh, nat_bw, nat_tiles;
};

struct AttnLaunch {
  const void *q, *qg, *k, *kg, *v, *vg;   // original and gathered Q/K/V spaces (bf16 rows of D); fused:
                                          // qg / kg / vg unused, the gather maps cover q / k / v
  long long q_rows, qg_rows, kv_rows, kvg_rows;
  long long o_rows = 0, part_rows = 0;   // rows of the bf16 output [H*S] and of the fp16 partial buffer
};

cudaError_t launch_attn(const AttnLaunch& L, const AttnParams& P, int n_items_hint, cudaStream_t stream,
                        int* tmap_err);

// kernel-based byte copy / fill (util.cu): never queued behind the caller's copy-engine transfers
cudaError_t copy_bytes(void* dst, const void* src, size_t n, cudaStream_t s);
cudaError_t fill_bytes(void* dst, uint8_t v, size_t n, cudaStream_t s);

}  // namespace mmi
