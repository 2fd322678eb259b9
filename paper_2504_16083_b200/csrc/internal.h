// Internal device data structures shared by the index builder, the gather
// kernels and the block-sparse attention kernel.  Not part of the public ABI.
#pragma once
#include <cstdint>

namespace mmi {

constexpr int BLK = 128;          // row block / key tile (reading C19)
constexpr int MAX_MOD = 4;

// ---- tile entry: one 128-key tile of one K-view, visited by one work item ----
// meta bits: [0] space (0 = original K/V, 1 = gathered K̄/V̄), [1] PRED (evaluate
// the element predicate; else every element of the tile is admitted), [2,5) role,
// [5] coordinate system of the pattern (0 = original position, 1 = modality rank),
// [8,16) instance id (index into the head's InstParam table).
enum Role : uint32_t { R_TRUE = 0, R_A = 1, R_NOTA = 2, R_VSSL = 3 };
struct TileEnt {
  int32_t krow;   // row of the first key in the K space (== row in the V space)
  uint32_t meta;
};
__host__ __device__ inline uint32_t tile_meta(uint32_t space, uint32_t pred, uint32_t role, uint32_t rank,
                                              uint32_t inst) {
  return space | (pred << 1) | (role << 2) | (rank << 5) | (inst << 8);
}

// ---- pattern instance parameters (after estimation) ----
struct InstParam {
  int32_t sink, local;      // A / NOTA roles
  int32_t s, p;             // grid stride / phase (informational for the kernel)
  int32_t slash_word;       // VS: word offset of the slash-offset bitmap in the bit arena (-1 none)
  int32_t vmask_word;       // VS: word offset of the vertical-column bitmap (-1 none)
  int32_t pad0, pad1;
};

// ---- work item: one 128-row block of one Q-view, one online softmax ----
enum OutMode : int32_t { OUT_FINAL = 0, OUT_PARTIAL = 1 };
struct WorkItem {
  int32_t head;       // query head
  int32_t q_row0;     // first row in the Q space (orig: h*S + 128*b; gathered: view row)
  int32_t tile_off;   // first TileEnt
  int32_t n_tiles;    // number of TileEnt (0 => empty item)
  int32_t q_gathered; // 1 => rows come from the gathered Q̄ space
  int32_t out_mode;   // OUT_FINAL / OUT_PARTIAL
  int32_t out_row0;   // first row in the partial buffer (OUT_PARTIAL)
  int32_t inst_base;  // first InstParam of this head
  int32_t skip_s;     // >0: do not write FINAL rows whose coord = skip_p (mod skip_s)
  int32_t skip_p;     //     (hline rows owned by the HROW pass, reading C9)
  int32_t skip_rank;  //     coord system of the skip test
  int32_t pad;
};

struct AttnParams {
  const WorkItem* items;
  int32_t n_items;
  const TileEnt* tiles;
  const InstParam* insts;
  const uint32_t* bits;
  const int32_t* qg_pos;    // gathered Q space: original position per row (-1 pad)
  const int32_t* qg_rank;   // gathered Q space: modality rank per row
  const int32_t* kg_pos;    // gathered K space: original position per row (INT_MAX pad)
  const int32_t* kg_rank;   // gathered K space: modality rank per row
  const int32_t* rank;      // modality rank by original position [S_pad]
  void* o;                  // bf16 [H, S, D]
  float* lse;               // [H, S] (nullable)
  float* part_o;            // fp32 partial rows
  float* part_lse;
  int32_t S, H, Hkv, D;
  float scale_log2;         // tau * log2(e)
  int32_t dense;            // 1 => implicit dense causal items (same-build comparator)
  int32_t fingerprint;      // 1 => write per-row admitted-key fingerprints instead of attention
  int64_t* fp_out;          // [rows][3] count, sum pos, sum pos^2 (fingerprint mode)
};

struct AttnLaunch {
  const void *q, *qg, *k, *kg, *v, *vg;   // original and gathered Q/K/V spaces (bf16 rows of D)
  long long q_rows, qg_rows, kv_rows, kvg_rows;
};
}  // namespace mmi

#include <cuda_runtime.h>
namespace mmi {
cudaError_t launch_attn(const AttnLaunch& L, const AttnParams& P, int n_items_hint, cudaStream_t stream,
                        int* tmap_err);
}  // namespace mmi
