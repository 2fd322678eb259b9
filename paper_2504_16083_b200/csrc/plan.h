// Host-side plan: a deterministic function of (mmi_problem, mmi_head_config[H])
// that fixes the workspace layout and the device tables every kernel reads.
// Every entry point recomputes it (cheap); only mmi_estimate_index uploads the
// device tables (into the workspace header).
#pragma once
#include <cstddef>
#include <cstdint>
#include <string>
#include <vector>

#include "../../include/mmi.h"
#include "internal.h"

namespace mmi {

constexpr int MAX_INST = 16;     // pattern instances per head (2D: M*M pairs)
constexpr int FOLD_LO = 128;     // reading C6
constexpr int FOLD_GAP = 128;    // reading C6
constexpr int SLAB_ROWS = 64;    // max last_q
constexpr int SLAB_CHUNK = 1024; // keys per slab CTA (8 tiles)
#ifndef MMI_HROW_SPLIT
#define MMI_HROW_SPLIT 512
#endif
constexpr int HROW_SPLIT_TILES = MMI_HROW_SPLIT;  // split-K chunk of an h-line row pair (65536 keys)

enum PassKind : int32_t { PASS_MAIN = 0, PASS_HROW = 1, PASS_SLASH = 2 };
enum ViewKind : int32_t { VK_ORIG_CLASS = 0, VK_RANK_CLASS = 1, VK_MOD = 2, VK_VCOL = 3 };
enum GridFlags : int32_t { GF_H = 1, GF_V = 2, GF_SL = 4 };

// ---- device tables (uploaded by mmi_estimate_index) ----
struct DInst {
  int32_t kind, rank, qa, kb;          // rank: pattern in modality-rank coordinates; qa/kb modality (-1 all)
  int32_t sink, local, n_v, n_s;
  int32_t stride, smin, smax, flags;   // grid
  int32_t slab;                        // estimation slab (-1: static pattern)
  int32_t grid_id, vs_id;              // result slots (-1)
  int32_t v_cls_q, v_res_q, v_cls_k, v_res_k, v_vcol;  // view ids (-1)
  int32_t force;                       // VS: force column 0 / offset 0
  int32_t pad[2];                      // [0] slash partial-row base, [1] HROW split-K partial-row base
  // static grid (the f3 baselines): fixed (stride, stat_p), no estimation; local < 0
  // means "block mode": the A part is the query's segment of -local keys (SF fixed)
  int32_t stat, stat_p, pad2[2];
};
struct DView {
  int32_t kind;       // ViewKind
  int32_t space;      // 0 = Q̄ space, 1 = K̄ space
  int32_t row_off;    // first row in the space
  int32_t cap;        // capacity in rows (multiple of 128)
  int32_t head, inst; // owner
  int32_t mod;        // modality (RANK_CLASS / VCOL-in-rank); -1 otherwise
  int32_t classes;    // ORIG/RANK_CLASS: 0 = all classes (RES), 1 = class p only (CLS)
};
struct DSlab {
  int32_t head, kv, qmod, rank_mode;   // qmod: modality of the slab rows (-1: last rows overall)
  int32_t need_dg, n_chunks, pad1, pad2; // need_dg: a vertical-slash instance with slashes uses this slab
                                       // (slab_kernel); else the tcgen05 slab kernel; n_chunks: key chunks of
                                       // its pass-1 statistics
  int64_t c_off;                       // float offset of c[S]
  int64_t dg_off;                      // u64 offset of dg[S]
};
struct DPass {
  int32_t head, pass, inst, n_slots;   // inst: grid instance (HROW/SLASH), -1 for MAIN
  int32_t slot_base, qa, pad0, pad1;   // qa: Q-bnd HROW/SLASH modality filter (-1 none); pad0: HROW key chunks
  int32_t seg_base, seg_per_slot;      // static segment region of the pass: slot b at seg_base + b * seg_per_slot
};
struct DHrow {                         // one h-line (HROW) pass: its split-K partials are merged by hrow_merge
  int32_t head, inst, qa, n_split;
};
struct DHead {
  int32_t boundary, n_inst, inst_base, kv;
  int32_t qmod_view, kmod_view;        // -1 unless Q/2D (Q̄ modality view) / 2D (K̄ modality view)
  int32_t part_rows0, part_rows1;      // partial buffer regions (rows), -1 if no merge
  int32_t sl_inst[MAX_MOD];            // grid instance with slash per query modality group (-1)
};
struct GridRes {
  int32_t s, p, valid, pad;
  double J, T;
};

constexpr int FUSE_Q = 1, FUSE_KV = 2;

struct Region {
  size_t off = 0, bytes = 0;
};

struct Plan {
  mmi_problem pb{};
  int H = 0, Hkv = 0, S = 0, D = 0, M = 1, nb = 0;
  int S_pad = 0;                       // S rounded up to 128 (+128 guard)
  std::vector<DHead> heads;
  std::vector<DInst> insts;            // H * MAX_INST (unused entries kind = NONE)
  std::vector<DView> views;
  std::vector<DSlab> slabs;
  std::vector<DPass> passes;
  int n_grid = 0, n_vs = 0;
  std::vector<int> vs_nv, vs_ns;       // capacities per VS result
  std::vector<int64_t> vs_v_off, vs_s_off, vs_bits_v, vs_bits_s;  // int32 / word offsets
  int64_t vs_list_words = 0, bits_words = 0;
  int64_t qg_rows = 0, kg_rows = 0;
  int n_slots = 0;
  int64_t seg_cap = 0;
  int64_t seg_spill_base = 0, seg_spill_cap = 0;  // spill area after the static per-slot regions
  std::vector<int64_t> slot_seg_cap_prefix;  // not used on device
  int64_t part_rows = 0;
  int n_chunks = 0;                    // slab key chunks
  int c_rank_n = 0;                    // rank-mode c arrays
  // host-uploaded tables (one blob at the start of the workspace)
  std::vector<int> qview_ids, kview_ids, grid_inst, vs_inst;
  std::vector<int64_t> vs_off_tab;     // [n_vs][2] list offsets, then [n_vs][2] bit offsets
  size_t o_heads = 0, o_insts = 0, o_views = 0, o_slabs = 0, o_passes = 0, o_qv = 0, o_kv = 0, o_gi = 0, o_vi = 0,
         o_vsl = 0, o_vsb = 0, blob_bytes = 0;
  int max_ncand = 1;
  std::vector<int64_t> gacc_off;       // per grid instance: u64 offset of its [ncand][smax] fold accumulators
  int64_t gacc_words = 0;
  size_t o_gacc = 0;
  std::vector<int> merge_heads;        // heads with partial rows (LSE merge in mmi_unpermute)
  size_t o_mh = 0;
  std::vector<DHrow> hrows;            // HROW passes (split-K merge in mmi_unpermute)
  std::vector<int> stc_pairs;          // tcgen05 slab kernel: (slab a, slab b or -1) per packed M=128 tile
  size_t o_sp = 0;
  int n_dg_batch = 0;                  // slab_kernel batches (slabs with need_dg, per KV group / 4)
  size_t o_hr = 0;
  int hrow_rows_max = 0;
  // workspace regions
  Region blob;
  Region labels, mod_cnt, mod_off, perm, rank, modpos, modrank;
  Region slab_rows, slab_ml_part, slab_ml, cbuf, dgbuf, c_rank;
  Region gridres, grid_part, grid_acc, vs_lists, vs_cnt, bits;
  Region view_len, view_alias;
  Region qg_pos, qg_rank, qg_src, kg_pos, kg_rank, kg_src, qg, kg, vg;
  Region items, item_keys, item_vals, items_sorted, seg_cnt, seg_off, segs, inst_params, sort_tmp, scan_tmp;
  Region part_o, part_lse;
  Region sched, flags;
  // in-kernel permutation (f2), bit 0: permuted Q blocks gathered by the attention kernel (no Q̄
  // copy); bit 1: the same for K / V (no K̄ / V̄).  Default: Q only -- a K̄ / V̄ tile is re-read by
  // many work items (a grid head's vertical strip by every row block), so one coalesced
  // materialisation that stays in L2 beats re-gathering scattered rows from K / V each time
  // (measured: DESIGN.md §6.3)
  int fused = FUSE_Q;
  size_t total = 0;
};

// Builds the plan; returns MMI_OK or an error status with message in `err`.
mmi_status build_plan(const mmi_problem* pb, const mmi_head_config* cfg, Plan& plan, std::string& err);
std::vector<uint8_t> make_blob(const Plan& plan);

}  // namespace mmi
