// Estimation / index / gather kernel launchers (internal).
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

#include "internal.h"
#include "plan.h"

namespace mmi {

// layout of the modality info array (ints)
constexpr int MI_CNT = 0;      // [MAX_MOD] n_m
constexpr int MI_OFF = 4;      // [MAX_MOD+1] offsets of P_m in perm
constexpr int MI_PADOFF = 9;   // [MAX_MOD+1] offsets of the 128-padded groups in the modality view
constexpr int MI_WORDS = 16;

void launch_modality(const uint8_t* labels, int S, int M, int S_pad, int mod_cap, int* chunk_cnt, int* chunk_base,
                     int* info, int* perm, int* rank, int* modpos, unsigned* flags, cudaStream_t st);
int slab_tc_chunks(int S);
// a2: slab rows, pass 1 (tcgen05 pairs + slab_kernel dg batches), statistics combine, pass 2
cudaError_t launch_slabs(const DSlab* slabs, int n_slabs, int n_dg_batch, const int2* stc_pairs, int n_stc_pairs,
                         const void* q, const void* k, int S, int H, int Hkv, int D, int last_q, float scale_log2,
                         const int* info, const int* perm, const int* rank, const uint8_t* labels, int* rows,
                         int* rranks, int* sinfo, float2* ml_part, float2* ml, float* cbuf, unsigned long long* dgbuf,
                         int ml_stride, cudaStream_t st);
void launch_grid(const DInst* insts, const int* grid_inst, int n_grid, int max_ncand, int n_inst_total,
                 const DSlab* slabs, const int* sinfo, const int* info, const int* perm, const float* cbuf,
                 uint32_t* fx, int S, int S_pad, GridRes* res, double* part, const int64_t* acc_off,
                 uint32_t* acc, cudaStream_t st);
void launch_vs(const DInst* insts, const int* vs_inst, int n_vs, const DSlab* slabs, const int* sinfo, const int* info,
               const int* perm, const float* cbuf, const unsigned long long* dgbuf, const int64_t* list_off,
               const int64_t* bits_off, int* lists, int* counts, uint32_t* bits, cudaStream_t st);

}  // namespace mmi
