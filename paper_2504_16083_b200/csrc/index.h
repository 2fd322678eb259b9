// Index builder context (device pointers into the workspace) and launchers.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

#include "internal.h"
#include "plan.h"

namespace mmi {

struct IndexCtx {
  int S, H, M, n_slots, n_passes;
  const DHead* heads;
  const DInst* insts;
  const DView* views;
  const DPass* passes;
  const int* info;
  const int* perm;
  const int* rank;
  const int* modpos;
  const uint8_t* labels;
  const GridRes* gridres;
  const int* vs_lists;
  const int* vs_cnt;
  const int64_t* vs_list_off;
  const int64_t* vs_bits_off;
  int* view_len;
  int* view_alias;      // K-view dedupe: canonical view of each view
  int *qg_pos, *qg_rank, *qg_src, *kg_pos, *kg_rank, *kg_src;
  InstParam* inst_params;
  int* seg_cnt;
  const int* seg_off;
  Seg* segs;
  WorkItem* items;
  WorkItem* items_sorted;
  int* sort_keys;
  int* sort_vals;
  const int* sort_vals_out;
  const __half* part_o;
  const float* part_lse;
  int64_t seg_cap;      // capacity of segs (plan bound)
  int64_t seg_spill_base, seg_spill_cap;  // spill area (slots whose static region is too small)
  unsigned* flags;      // device-side error flags (MMI_FLAG_*)
};

void launch_build_views(const IndexCtx& C, const int* qviews, int nq, const int* kviews, int nk, int64_t qrows,
                        int64_t krows, cudaStream_t st);
void launch_inst_params(const IndexCtx& C, int n_total, cudaStream_t st);
void launch_items_fill(const IndexCtx& C, cudaStream_t st);
void launch_items_gather(const IndexCtx& C, cudaStream_t st);
void launch_gather(const int* src, int64_t rows, int D, const void* a, void* a_out, const void* b, void* b_out,
                   cudaStream_t st);
void launch_hrow_merge(const IndexCtx& C, int D, const DHrow* hrows, int n_hrows, int max_rows, void* o, float* lse,
                       cudaStream_t st);
void launch_merge(const IndexCtx& C, int D, const int* heads_list, int n_heads, int n_rows, void* o, float* lse,
                  cudaStream_t st);

}  // namespace mmi
