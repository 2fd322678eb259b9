// Online sparse-index estimation:
//   a1 modality bookkeeping   (Alg.2, Alg.3: permute by modality)
//   a2 last_q slab estimate    (Alg.1): A-hat rows, column mass c,
//                              diagonal mass dg (fixed-point, order-independent sums)
//   a3 grid stride/phase fold  (Alg.1, readings C4-C7)
//   a4 vertical-slash top-k    (reading C15): radix select, ties -> lowest index
// All reductions are deterministic (fixed order or integer atomics).
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <cfloat>
#include <climits>
#include <cstdint>

#include <cub/cub.cuh>

#include "estimate.h"
#include "ptx.cuh"

namespace mmi {

// =============================================================== a1: modality
constexpr int MOD_CHUNK = 4096;

__global__ void mod_count_kernel(const uint8_t* __restrict__ labels, int S, int M, int* __restrict__ chunk_cnt,
                                 unsigned* __restrict__ flags) {
  __shared__ int cnt[MAX_MOD];
  if (threadIdx.x < MAX_MOD) cnt[threadIdx.x] = 0;
  __syncthreads();
  const int c0 = blockIdx.x * MOD_CHUNK;
  int loc[MAX_MOD] = {0, 0, 0, 0};
  bool bad = false;
  for (int i = c0 + threadIdx.x; i < min(S, c0 + MOD_CHUNK); i += blockDim.x) {
    const int m = labels[i];
    bad |= m >= M;
#pragma unroll
    for (int q = 0; q < MAX_MOD; ++q) loc[q] += (m == q && q < M);
  }
#pragma unroll
  for (int q = 0; q < MAX_MOD; ++q)
    if (loc[q]) atomicAdd(&cnt[q], loc[q]);
  if (__any_sync(0xffffffffu, bad) && (threadIdx.x & 31) == 0) atomicOr(flags, FLAG_LABEL_RANGE);
  __syncthreads();
  if (threadIdx.x < MAX_MOD) chunk_cnt[blockIdx.x * MAX_MOD + threadIdx.x] = cnt[threadIdx.x];
}

// single warp: per modality sequential scan over chunks (fixed order)
__global__ void mod_scan_kernel(const int* __restrict__ chunk_cnt, int n_chunks, int M, int* __restrict__ chunk_base,
                                int* __restrict__ info) {
  const int m = threadIdx.x;
  if (m < MAX_MOD) {
    int run = 0;
    for (int c = 0; c < n_chunks; ++c) {
      chunk_base[c * MAX_MOD + m] = run;
      run += chunk_cnt[c * MAX_MOD + m];
    }
    info[MI_CNT + m] = (m < M) ? run : 0;
  }
  __syncwarp();
  if (threadIdx.x == 0) {
    int o = 0, po = 0;
    for (int q = 0; q < MAX_MOD; ++q) {
      info[MI_OFF + q] = o;
      info[MI_PADOFF + q] = po;
      o += info[MI_CNT + q];
      po += (info[MI_CNT + q] + BLK - 1) / BLK * BLK;
    }
    info[MI_OFF + MAX_MOD] = o;
    info[MI_PADOFF + MAX_MOD] = po;
  }
}

__global__ void mod_place_kernel(const uint8_t* __restrict__ labels, int S, int M, const int* __restrict__ chunk_base,
                                 const int* __restrict__ info, int* __restrict__ perm, int* __restrict__ rank,
                                 int* __restrict__ modpos) {
  // 256 threads x 16 consecutive positions = one 4096 chunk
  typedef cub::BlockScan<int, 256> Scan;
  __shared__ typename Scan::TempStorage tmp;
  const int c0 = blockIdx.x * MOD_CHUNK + threadIdx.x * 16;
  int lab[16];
  int loc[MAX_MOD] = {0, 0, 0, 0};
#pragma unroll
  for (int i = 0; i < 16; ++i) {
    lab[i] = (c0 + i < S) ? labels[c0 + i] : -1;
#pragma unroll
    for (int q = 0; q < MAX_MOD; ++q) loc[q] += (lab[i] == q && q < M);
  }
  int pre[MAX_MOD];
#pragma unroll
  for (int q = 0; q < MAX_MOD; ++q) {
    Scan(tmp).ExclusiveSum(loc[q], pre[q]);
    __syncthreads();
    pre[q] += chunk_base[blockIdx.x * MAX_MOD + q];
  }
#pragma unroll
  for (int i = 0; i < 16; ++i) {
    const int m = lab[i];
    if (m < 0) continue;
    if (m >= M) {  // out-of-range label (flagged by mod_count_kernel): in no modality group
      rank[c0 + i] = 0;
      continue;
    }
    int r = 0;
#pragma unroll
    for (int q = 0; q < MAX_MOD; ++q)
      if (q == m) r = pre[q]++;
    const int pos = c0 + i;
    rank[pos] = r;
    perm[info[MI_OFF + m] + r] = pos;
    modpos[info[MI_PADOFF + m] + r] = pos;
  }
}

__global__ void mod_pad_kernel(const int* __restrict__ info, int S, int S_pad, int mod_cap, int* __restrict__ rank,
                               int* __restrict__ modpos) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= S && i < S_pad) rank[i] = INT_MAX / 2;
  if (i < mod_cap) {
    bool pad = i >= info[MI_PADOFF + MAX_MOD];
    for (int q = 0; q < MAX_MOD; ++q)
      if (i >= info[MI_PADOFF + q] + info[MI_CNT + q] && i < info[MI_PADOFF + q + 1]) pad = true;
    if (pad) modpos[i] = -1;
  }
}

void launch_modality(const uint8_t* labels, int S, int M, int S_pad, int mod_cap, int* chunk_cnt, int* chunk_base,
                     int* info, int* perm, int* rank, int* modpos, unsigned* flags, cudaStream_t st) {
  const int nch = (S + MOD_CHUNK - 1) / MOD_CHUNK;
  mod_count_kernel<<<nch, 256, 0, st>>>(labels, S, M, chunk_cnt, flags);
  mod_scan_kernel<<<1, 32, 0, st>>>(chunk_cnt, nch, M, chunk_base, info);
  mod_place_kernel<<<nch, 256, 0, st>>>(labels, S, M, chunk_base, info, perm, rank, modpos);
  const int n = max(S_pad, mod_cap);
  mod_pad_kernel<<<(n + 255) / 256, 256, 0, st>>>(info, S, S_pad, mod_cap, rank, modpos);
}

// =============================================================== a2: slabs
// slab_info[s*4 + {0,1,2,3}] = {L, min pos, max pos, min rank}
__global__ void slab_rows_kernel(const DSlab* __restrict__ slabs, int S, int last_q, const int* __restrict__ info,
                                 const int* __restrict__ perm, const int* __restrict__ rank, int* __restrict__ rows,
                                 int* __restrict__ rranks, int* __restrict__ sinfo) {
  const int s = blockIdx.x, r = threadIdx.x;  // 64 threads
  const DSlab sl = slabs[s];
  int n, L, pos = -1;
  if (sl.qmod < 0) {
    n = S;
    L = min(last_q, n);
    if (r < L) pos = S - L + r;
  } else {
    n = info[MI_CNT + sl.qmod];
    L = min(last_q, n);
    if (r < L) pos = perm[info[MI_OFF + sl.qmod] + n - L + r];
  }
  rows[s * SLAB_ROWS + r] = pos;
  rranks[s * SLAB_ROWS + r] = pos >= 0 ? rank[pos] : -1;
  if (r == 0) {
    sinfo[s * 4 + 0] = L;
    sinfo[s * 4 + 1] = L > 0 ? ((sl.qmod < 0) ? S - L : perm[info[MI_OFF + sl.qmod] + n - L]) : 0;
  }
  if (r == L - 1) {
    sinfo[s * 4 + 2] = pos;
    sinfo[s * 4 + 3] = rank[(sl.qmod < 0) ? S - L : perm[info[MI_OFF + sl.qmod] + n - L]];
  }
  if (L == 0 && r == 0) {
    sinfo[s * 4 + 2] = -1;
    sinfo[s * 4 + 3] = 0;
  }
}

__device__ __forceinline__ void ldsm_x4(uint32_t (&r)[4], const void* p) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0,%1,%2,%3}, [%4];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3])
               : "r"((uint32_t)__cvta_generic_to_shared(p)));
}
__device__ __forceinline__ void mma16816(float (&d)[4], const uint32_t (&a)[4], uint32_t b0, uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
      "{%0,%1,%2,%3};"
      : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
      : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}

constexpr int SLAB_BATCH = 4;  // slabs resident per CTA

template <int D>
struct SlabSmem {
  static constexpr int LD = D + 8;  // padded rows: conflict-free ldmatrix
  __nv_bfloat16 q[SLAB_BATCH][SLAB_ROWS * LD];
  __nv_bfloat16 k[2][BLK * LD];     // cp.async double buffer
  float a[2][SLAB_ROWS][BLK + 1];   // A-hat tiles of the two slabs in flight (pass 2)
  int colidx[2][BLK];
  int red[2][8];
  int sl_idx[SLAB_BATCH];
  int nsb;
};

__device__ __forceinline__ void cp_async16(void* dst, const void* src, bool valid) {
  const uint32_t d = (uint32_t)__cvta_generic_to_shared(dst);
  const int sz = valid ? 16 : 0;
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(d), "l"(src), "r"(sz) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory"); }

// scores of one 16-row strip (rows of q_s) against one key tile: acc[nt][.] in mma layout
template <int D>
__device__ __forceinline__ void slab_strip_scores(const __nv_bfloat16* q_s, const __nv_bfloat16* k_s, int strip,
                                                  float (&acc)[16][4]) {
  const int lane = threadIdx.x % 32;
  constexpr int LD = D + 8;
#pragma unroll
  for (int i = 0; i < 16; ++i) acc[i][0] = acc[i][1] = acc[i][2] = acc[i][3] = 0.f;
#pragma unroll
  for (int kk = 0; kk < D / 16; ++kk) {
    uint32_t a[4];
    ldsm_x4(a, &q_s[(strip * 16 + (lane % 16)) * LD + kk * 16 + (lane / 16) * 8]);
#pragma unroll
    for (int n2 = 0; n2 < 8; ++n2) {
      uint32_t b[4];
      ldsm_x4(b, &k_s[(n2 * 16 + (lane % 8) + (lane / 16) * 8) * LD + kk * 16 + ((lane / 8) % 2) * 8]);
      mma16816(acc[2 * n2], a, b[0], b[1]);
      mma16816(acc[2 * n2 + 1], a, b[2], b[3]);
    }
  }
}

// mode 0: pass 1 (row max / sum partials per key chunk); mode 1: pass 2 (A-hat -> c, dg)
// grid (key chunk, KV group, slab batch); 8 warps: warps 0-3 / 4-7 take the two slabs of a pair.
template <int D>
__global__ void __launch_bounds__(256) slab_kernel(int mode, const DSlab* __restrict__ slabs, int n_slabs,
                                                   const __nv_bfloat16* __restrict__ q,
                                                   const __nv_bfloat16* __restrict__ k, int S, int H,
                                                   float scale_log2, const int* __restrict__ rows,
                                                   const int* __restrict__ rranks, const int* __restrict__ sinfo,
                                                   const uint8_t* __restrict__ labels, const int* __restrict__ rank,
                                                   float2* __restrict__ ml_part, const float2* __restrict__ ml,
                                                   float* __restrict__ cbuf, unsigned long long* __restrict__ dgbuf,
                                                   int n_chunks) {
  extern __shared__ __align__(16) uint8_t slab_smem_raw[];
  SlabSmem<D>& sm = *reinterpret_cast<SlabSmem<D>*>(slab_smem_raw);
  constexpr int LD = SlabSmem<D>::LD;
  const int chunk = blockIdx.x, kv = blockIdx.y, batch = blockIdx.z;
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const int g = lane / 4, t4 = lane % 4;
  const int ps = warp / 4, strip = warp % 4;
  const int j_chunk0 = chunk * SLAB_CHUNK;
  if (threadIdx.x == 0) {
    int ord = 0, n = 0;
    for (int si = 0; si < n_slabs; ++si) {
      if (slabs[si].kv != kv || !slabs[si].need_dg) continue;  // the other slabs run in slab_tc_kernel
      if (ord >= batch * SLAB_BATCH && ord < (batch + 1) * SLAB_BATCH) sm.sl_idx[n++] = si;
      ++ord;
    }
    sm.nsb = n;
  }
  __syncthreads();
  const int nsb = sm.nsb;
  if (nsb == 0) return;
  int maxpos = -1;
  for (int b = 0; b < nsb; ++b) maxpos = max(maxpos, sinfo[sm.sl_idx[b] * 4 + 2]);
  if (j_chunk0 > maxpos) {
    if (mode == 0)
      for (int b = 0; b < nsb; ++b)
        if (threadIdx.x < SLAB_ROWS)
          ml_part[((size_t)sm.sl_idx[b] * n_chunks + chunk) * SLAB_ROWS + threadIdx.x] = make_float2(-INFINITY, 0.f);
    return;
  }
  // resident query slabs
  constexpr int V = D / 8;
  for (int b = 0; b < nsb; ++b) {
    const int si = sm.sl_idx[b];
    const DSlab sl = slabs[si];
    for (int i = threadIdx.x; i < SLAB_ROWS * V; i += blockDim.x) {
      const int r = i / V, c = i % V;
      const int pos = rows[si * SLAB_ROWS + r];
      uint4 val = make_uint4(0, 0, 0, 0);
      if (pos >= 0) val = reinterpret_cast<const uint4*>(q + ((size_t)sl.head * S + pos) * D)[c];
      *reinterpret_cast<uint4*>(&sm.q[b][r * LD + c * 8]) = val;
    }
  }
  const int ntile = min(SLAB_CHUNK / BLK, (maxpos - j_chunk0) / BLK + 1);
  auto load_k = [&](int tt) {
    const int j0 = j_chunk0 + tt * BLK;
    __nv_bfloat16* dst = sm.k[tt & 1];
    for (int i = threadIdx.x; i < BLK * V; i += blockDim.x) {
      const int r = i / V, c = i % V;
      const bool ok = j0 + r < S;
      cp_async16(dst + r * LD + c * 8, k + ((size_t)kv * S + (ok ? j0 + r : 0)) * D + c * 8, ok);
    }
    cp_async_commit();
  };
  load_k(0);
  // pass-1 running statistics: [pair][row lo / hi]
  float m_run[2][2] = {{-INFINITY, -INFINITY}, {-INFINITY, -INFINITY}};
  float l_run[2][2] = {{0.f, 0.f}, {0.f, 0.f}};
  const int npair = (nsb + 1) / 2;
  const double FX = 4503599627370496.0;  // 2^52
  for (int tt = 0; tt < ntile; ++tt) {
    if (tt + 1 < ntile) {
      load_k(tt + 1);
      cp_async_wait<1>();
    } else {
      cp_async_wait<0>();
    }
    __syncthreads();
    const int j0 = j_chunk0 + tt * BLK;
    const __nv_bfloat16* k_s = sm.k[tt & 1];
#pragma unroll
    for (int pp = 0; pp < 2; ++pp) {
      if (pp >= npair) break;
      const int b = 2 * pp + ps;
      const bool have = b < nsb;
      const int si = have ? sm.sl_idx[b] : 0;
      const int* srow = rows + si * SLAB_ROWS;
      const int r_lo = strip * 16 + g, r_hi = r_lo + 8;
      float acc[16][4];
      if (have) {
        slab_strip_scores<D>(sm.q[b], k_s, strip, acc);
        const int pos_lo = srow[r_lo], pos_hi = srow[r_hi];
#pragma unroll
        for (int nt = 0; nt < 16; ++nt) {
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            const int j = j0 + nt * 8 + 2 * t4 + (e & 1);
            const int pr = (e < 2) ? pos_lo : pos_hi;
            acc[nt][e] = (pr >= 0 && j <= pr) ? acc[nt][e] * scale_log2 : -INFINITY;
          }
        }
      }
      if (mode == 0) {
        if (have) {
          float tm_lo = -INFINITY, tm_hi = -INFINITY;
#pragma unroll
          for (int nt = 0; nt < 16; ++nt) {
            tm_lo = fmaxf(tm_lo, fmaxf(acc[nt][0], acc[nt][1]));
            tm_hi = fmaxf(tm_hi, fmaxf(acc[nt][2], acc[nt][3]));
          }
          tm_lo = fmaxf(tm_lo, __shfl_xor_sync(0xffffffffu, tm_lo, 1));
          tm_lo = fmaxf(tm_lo, __shfl_xor_sync(0xffffffffu, tm_lo, 2));
          tm_hi = fmaxf(tm_hi, __shfl_xor_sync(0xffffffffu, tm_hi, 1));
          tm_hi = fmaxf(tm_hi, __shfl_xor_sync(0xffffffffu, tm_hi, 2));
          const float nm_lo = fmaxf(m_run[pp][0], tm_lo), nm_hi = fmaxf(m_run[pp][1], tm_hi);
          float s_lo = 0.f, s_hi = 0.f;
          if (nm_lo > -INFINITY) {
#pragma unroll
            for (int nt = 0; nt < 16; ++nt) s_lo += exp2f(acc[nt][0] - nm_lo) + exp2f(acc[nt][1] - nm_lo);
          }
          if (nm_hi > -INFINITY) {
#pragma unroll
            for (int nt = 0; nt < 16; ++nt) s_hi += exp2f(acc[nt][2] - nm_hi) + exp2f(acc[nt][3] - nm_hi);
          }
          s_lo += __shfl_xor_sync(0xffffffffu, s_lo, 1);
          s_lo += __shfl_xor_sync(0xffffffffu, s_lo, 2);
          s_hi += __shfl_xor_sync(0xffffffffu, s_hi, 1);
          s_hi += __shfl_xor_sync(0xffffffffu, s_hi, 2);
          l_run[pp][0] = (m_run[pp][0] > -INFINITY ? l_run[pp][0] * exp2f(m_run[pp][0] - nm_lo) : 0.f) + s_lo;
          l_run[pp][1] = (m_run[pp][1] > -INFINITY ? l_run[pp][1] * exp2f(m_run[pp][1] - nm_hi) : 0.f) + s_hi;
          m_run[pp][0] = nm_lo;
          m_run[pp][1] = nm_hi;
        }
      } else {
        // ---- pass 2: A-hat tile -> smem, then fixed-order column / diagonal sums ----
        if (have) {
          const float2 ma = ml[si * SLAB_ROWS + r_lo], mb = ml[si * SLAB_ROWS + r_hi];
          const float il_lo = ma.y > 0.f ? 1.f / ma.y : 0.f, il_hi = mb.y > 0.f ? 1.f / mb.y : 0.f;
#pragma unroll
          for (int nt = 0; nt < 16; ++nt) {
            const int c = nt * 8 + 2 * t4;
            sm.a[ps][r_lo][c] = acc[nt][0] > -INFINITY ? exp2f(acc[nt][0] - ma.x) * il_lo : 0.f;
            sm.a[ps][r_lo][c + 1] = acc[nt][1] > -INFINITY ? exp2f(acc[nt][1] - ma.x) * il_lo : 0.f;
            sm.a[ps][r_hi][c] = acc[nt][2] > -INFINITY ? exp2f(acc[nt][2] - mb.x) * il_hi : 0.f;
            sm.a[ps][r_hi][c + 1] = acc[nt][3] > -INFINITY ? exp2f(acc[nt][3] - mb.x) * il_hi : 0.f;
          }
        }
        // rank-mode slabs: compact the keys of the slab's modality (ranks are consecutive)
        const int tid = threadIdx.x % 128;  // thread within this slab's half
        const DSlab sl = slabs[si];
        bool isa = false;
        unsigned bal = 0;
        if (have && sl.rank_mode && sl.need_dg) {
          const int j = j0 + tid;
          isa = (j < S) && labels[j] == sl.qmod;
          bal = __ballot_sync(0xffffffffu, isa);
          if (lane == 0) sm.red[ps][strip] = __popc(bal);
        }
        __syncthreads();
        if (have && sl.rank_mode && sl.need_dg) {
          int base = 0;
          for (int w = 0; w < strip; ++w) base += sm.red[ps][w];
          if (isa) sm.colidx[ps][base + __popc(bal & ((1u << lane) - 1u))] = tid;
        }
        __syncthreads();
        if (have) {
          const int L = sinfo[si * 4 + 0];
          // column mass
          {
            const int j = j0 + tid;
            float sum = 0.f;
            for (int r = 0; r < SLAB_ROWS; ++r) sum += sm.a[ps][r][tid];
            if (j < S) cbuf[sl.c_off + j] = sum;
          }
          if (!sl.need_dg) {
            // no slash selection reads this slab's diagonal mass
          } else if (!sl.rank_mode) {
            int r0 = 0;
            while (r0 < L) {
              int r1 = r0 + 1;
              while (r1 < L && srow[r1] == srow[r1 - 1] + 1) ++r1;
              const int pb = srow[r0] - r0;
              const int width = 127 + (r1 - r0);
              for (int i = tid; i < width; i += 128) {
                const int o = pb + r0 - (j0 + 127) + i;
                if (o < 0) continue;
                float sum = 0.f;
                for (int r = r0; r < r1; ++r) {
                  const int c = pb + r - o - j0;
                  if (c >= 0 && c < BLK) sum += sm.a[ps][r][c];
                }
                if (sum > 0.f) atomicAdd(dgbuf + sl.dg_off + o, (unsigned long long)((double)sum * FX));
              }
              r0 = r1;
            }
          } else {
            const int Ka = sm.red[ps][0] + sm.red[ps][1] + sm.red[ps][2] + sm.red[ps][3];
            if (Ka > 0) {
              const int rank_lo = rank[j0 + sm.colidx[ps][0]];
              const int rho0 = rranks[si * SLAB_ROWS];
              const int width = L + Ka - 1;
              for (int i = tid; i < width; i += 128) {
                const int o = rho0 - (rank_lo + Ka - 1) + i;
                if (o < 0) continue;
                float sum = 0.f;
                for (int r = 0; r < L; ++r) {
                  const int kr = rho0 + r - o - rank_lo;
                  if (kr >= 0 && kr < Ka) sum += sm.a[ps][r][sm.colidx[ps][kr]];
                }
                if (sum > 0.f) atomicAdd(dgbuf + sl.dg_off + o, (unsigned long long)((double)sum * FX));
              }
            }
          }
        }
        __syncthreads();
      }
    }
    __syncthreads();  // all warps done with this K buffer before it is refilled
  }
  if (mode == 0 && t4 == 0) {
#pragma unroll
    for (int pp = 0; pp < 2; ++pp) {
      const int b = 2 * pp + ps;
      if (pp < npair && b < nsb) {
        const int si = sm.sl_idx[b];
        const int r_lo = strip * 16 + g, r_hi = r_lo + 8;
        ml_part[((size_t)si * n_chunks + chunk) * SLAB_ROWS + r_lo] = make_float2(m_run[pp][0], l_run[pp][0]);
        ml_part[((size_t)si * n_chunks + chunk) * SLAB_ROWS + r_hi] = make_float2(m_run[pp][1], l_run[pp][1]);
      }
    }
  }
}

__global__ void slab_combine_kernel(const DSlab* __restrict__ slabs, const float2* __restrict__ ml_part,
                                    int ml_stride, float2* __restrict__ ml) {
  const int si = blockIdx.x, r = threadIdx.x;
  const int n_chunks = slabs[si].n_chunks;  // key chunks of the kernel that ran this slab's pass 1
  float m = -INFINITY;
  for (int c = 0; c < n_chunks; ++c) m = fmaxf(m, ml_part[((size_t)si * ml_stride + c) * SLAB_ROWS + r].x);
  float l = 0.f;
  if (m > -INFINITY)
    for (int c = 0; c < n_chunks; ++c) {
      const float2 p = ml_part[((size_t)si * ml_stride + c) * SLAB_ROWS + r];
      if (p.x > -INFINITY) l += p.y * exp2f(p.x - m);
    }
  ml[si * SLAB_ROWS + r] = make_float2(m, l);
}

cudaError_t launch_slab_tc(int mode, const int2* pairs, int n_pairs, const DSlab* slabs, const void* q, const void* k,
                           int S, int Hkv, int D, float scale_log2, const int* rows, const int* sinfo, float2* ml_part,
                           const float2* ml, float* cbuf, int ml_stride, cudaStream_t st);

template <int D>
static cudaError_t launch_slab_dg(int mode, dim3 grid, const DSlab* slabs, int n_slabs, const void* q, const void* k,
                                  int S, int H, float scale_log2, int* rows, int* rranks, int* sinfo,
                                  const uint8_t* labels, const int* rank, float2* ml_part, float2* ml, float* cbuf,
                                  unsigned long long* dgbuf, int n_chunks, cudaStream_t st) {
  const int smem = sizeof(SlabSmem<D>);
  const cudaError_t e = cudaFuncSetAttribute(slab_kernel<D>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  if (e != cudaSuccess) return e;
  slab_kernel<D><<<grid, 256, smem, st>>>(mode, slabs, n_slabs, (const __nv_bfloat16*)q, (const __nv_bfloat16*)k, S,
                                          H, scale_log2, rows, rranks, sinfo, labels, rank, ml_part, ml, cbuf, dgbuf,
                                          n_chunks);
  return cudaGetLastError();
}

cudaError_t launch_slabs(const DSlab* slabs, int n_slabs, int n_dg_batch, const int2* stc_pairs, int n_stc_pairs,
                         const void* q, const void* k, int S, int H, int Hkv, int D, int last_q, float scale_log2,
                         const int* info, const int* perm, const int* rank, const uint8_t* labels, int* rows,
                         int* rranks, int* sinfo, float2* ml_part, float2* ml, float* cbuf, unsigned long long* dgbuf,
                         int ml_stride, cudaStream_t st) {
  if (n_slabs == 0) return cudaSuccess;
  slab_rows_kernel<<<n_slabs, SLAB_ROWS, 0, st>>>(slabs, S, last_q, info, perm, rank, rows, rranks, sinfo);
  const dim3 grid(ml_stride, Hkv, n_dg_batch);  // slab_kernel: 1024-key chunks (ml_stride of them)
  cudaError_t e = cudaSuccess;
  for (int mode = 0; mode < 2 && e == cudaSuccess; ++mode) {
    if (mode == 1) slab_combine_kernel<<<n_slabs, SLAB_ROWS, 0, st>>>(slabs, ml_part, ml_stride, ml);
    e = launch_slab_tc(mode, stc_pairs, n_stc_pairs, slabs, q, k, S, Hkv, D, scale_log2, rows, sinfo, ml_part, ml,
                       cbuf, ml_stride, st);
    if (e == cudaSuccess && n_dg_batch > 0)
      e = (D == 128) ? launch_slab_dg<128>(mode, grid, slabs, n_slabs, q, k, S, H, scale_log2, rows, rranks, sinfo,
                                           labels, rank, ml_part, ml, cbuf, dgbuf, ml_stride, st)
                     : launch_slab_dg<64>(mode, grid, slabs, n_slabs, q, k, S, H, scale_log2, rows, rranks, sinfo,
                                          labels, rank, ml_part, ml, cbuf, dgbuf, ml_stride, st);
  }
  return e;
}

// =============================================================== a3: grid
// fx[g][j] = round(c[j] * 2^25) in the pattern's coordinate system (rank-coordinate instances:
// c[P_a[rho]]), for every estimated grid instance: the fold reads exact integers (see below)
constexpr float FX25 = 33554432.0f;  // 2^25
__global__ void grid_prep_kernel(const DInst* __restrict__ insts, int n_inst_total, const DSlab* __restrict__ slabs,
                                 const int* __restrict__ info, const int* __restrict__ perm,
                                 const float* __restrict__ cbuf, uint32_t* __restrict__ fx, int S, int S_pad) {
  const int ii = blockIdx.y;
  const DInst x = insts[ii];
  if (x.kind != MMI_PAT_GRID || x.stat) return;
  const DSlab sl = slabs[x.slab];
  const float* c = cbuf + sl.c_off;
  uint32_t* out = fx + (size_t)x.grid_id * S_pad;
  if (x.rank) {
    const int na = info[MI_CNT + x.qa];
    const int off = info[MI_OFF + x.qa];
    for (int r = blockIdx.x * blockDim.x + threadIdx.x; r < na; r += gridDim.x * blockDim.x)
      out[r] = __float2uint_rn(c[perm[off + r]] * FX25);
  } else {
    for (int j = blockIdx.x * blockDim.x + threadIdx.x; j < S; j += gridDim.x * blockDim.x)
      out[j] = __float2uint_rn(c[j] * FX25);
  }
}

struct JP {
  double J;
  int p;
};
__device__ __forceinline__ JP jp_best(JP a, JP b) {
  if (b.J > a.J || (b.J == a.J && b.p < a.p)) return b;
  return a;
}

struct JPMax {
  __device__ __forceinline__ JP operator()(const JP& a, const JP& b) const { return jp_best(a, b); }
};

__device__ __forceinline__ void grid_window(const DInst& x, const int* sinfo, const int* info, int S, int& lo, int& hi,
                                            int& n) {
  n = x.rank ? info[MI_CNT + x.qa] : S;
  const int wmin = x.rank ? sinfo[x.slab * 4 + 3] : sinfo[x.slab * 4 + 1];
  lo = FOLD_LO;
  hi = min(wmin - FOLD_GAP, n);
}

// Fold (reading C4-C6): m_s[p] = sum_{j in W, j = p mod s} c[j] for every candidate stride.
// c >= 0 is a column mass of at most L <= 64 softmax rows, so sum_j c[j] <= 64 and c is taken to
// 2^-25 fixed point (round to nearest, grid_prep_kernel) with every partial and total sum inside
// uint32: the fold is exact integer arithmetic, hence order-independent and deterministic.
// One CTA owns FOLD_SPC consecutive strides s > smax / 2 (the others are derived exactly from a
// multiple, grid_derive_kernel) and streams the window W through shared memory (double-buffered
// bulk copies); thread (group g, phase p) of stride s <= 256 sums the chunk elements of phase p at
// g*s + k*G*s (G = 256 / s groups), threads of larger strides own up to FOLD_MAXW phases each.
// Every stride's sums stay in registers across chunks and are written once (no atomics); the chunk
// phase offset advances incrementally (no divisions in the loop).
#ifndef MMI_FOLD_CHUNK
#define MMI_FOLD_CHUNK 8192
#endif
constexpr int FOLD_CHUNK = MMI_FOLD_CHUNK;   // u32 keys per shared-memory chunk (32 KB)
#ifndef MMI_FOLD_SPC
#define MMI_FOLD_SPC 2
#endif
constexpr int FOLD_SPC = MMI_FOLD_SPC;       // candidate strides per CTA
constexpr int FOLD_THREADS = 256;
constexpr int FOLD_MAXW = 4;                 // phases per thread for strides in (256, 1024]

// sum of ptr[0], ptr[step], ... below end (4 independent chains)
__device__ __forceinline__ uint32_t strided_sum(const uint32_t* ptr, const uint32_t* end, int step) {
  uint32_t a0 = 0, a1 = 0, a2 = 0, a3 = 0;
  const int s4 = 4 * step;
  for (; ptr + 3 * step < end; ptr += s4) {
    a0 += ptr[0];
    a1 += ptr[step];
    a2 += ptr[2 * step];
    a3 += ptr[3 * step];
  }
  for (; ptr < end; ptr += step) a0 += *ptr;
  return (a0 + a1) + (a2 + a3);
}

__global__ void __launch_bounds__(FOLD_THREADS) grid_acc_kernel(const DInst* __restrict__ insts,
                                                                const int* __restrict__ grid_inst,
                                                                const int* __restrict__ sinfo,
                                                                const int* __restrict__ info,
                                                                const uint32_t* __restrict__ fx, int S, int S_pad,
                                                                const int64_t* __restrict__ acc_off,
                                                                uint32_t* __restrict__ acc) {
  extern __shared__ __align__(16) uint32_t fold_buf[];  // [2][FOLD_CHUNK]
  __shared__ uint32_t part[FOLD_THREADS];
  __shared__ __align__(8) uint64_t bar[2];
  const int gi = blockIdx.y;
  const DInst x = insts[grid_inst[gi]];
  if (x.stat) return;  // static grid: nothing to fold
  // only the strides without a candidate multiple are folded directly (s > smax / 2); the others
  // are derived exactly from a power-of-two multiple by grid_derive_kernel
  const int s_dir = max(x.smin, x.smax / 2 + 1);
  const int s0 = s_dir + blockIdx.x * FOLD_SPC;
  if (s0 > x.smax) return;
  const int ns = min(FOLD_SPC, x.smax - s0 + 1);
  int lo, hi, n;
  grid_window(x, sinfo, info, S, lo, hi, n);
  const uint32_t* c = fx + (size_t)gi * S_pad;
  const int tid = threadIdx.x;
  uint32_t accr[FOLD_SPC][FOLD_MAXW];
  int rr[FOLD_SPC], cm[FOLD_SPC], pq[FOLD_SPC];
#pragma unroll
  for (int q = 0; q < FOLD_SPC; ++q) {
    const int s = s0 + q;
#pragma unroll
    for (int w = 0; w < FOLD_MAXW; ++w) accr[q][w] = 0u;
    rr[q] = q < ns ? lo % s : 0;                     // phase of the chunk's first key
    cm[q] = q < ns ? FOLD_CHUNK % s : 0;             // phase advance per chunk
    pq[q] = q < ns && s <= FOLD_THREADS ? tid % s : 0;
  }
  // W is read with 16-byte bulk copies from a 16-byte aligned start (lo is a multiple of 128)
  const int nchunk = hi > lo ? (hi - lo + FOLD_CHUNK - 1) / FOLD_CHUNK : 0;
  if (tid == 0) {
    mbar_init(&bar[0], 1);
    mbar_init(&bar[1], 1);
    fence_barrier_init();
  }
  __syncthreads();
  auto load = [&](int ch) {
    const int j0 = lo + ch * FOLD_CHUNK;
    const int len = min(FOLD_CHUNK, hi - j0);
    const uint32_t bytes = (uint32_t)((len + 3) & ~3) * 4u;  // reads <= 3 keys past hi, inside S_pad
    mbar_arrive_expect_tx(&bar[ch & 1], bytes);
    bulk_load(fold_buf + (ch & 1) * FOLD_CHUNK, c + j0, bytes, &bar[ch & 1]);
  };
  if (tid == 0 && nchunk > 0) load(0);
  for (int ch = 0; ch < nchunk; ++ch) {
    const int len = min(FOLD_CHUNK, hi - lo - ch * FOLD_CHUNK);
    if (tid == 0 && ch + 1 < nchunk) load(ch + 1);  // buffer (ch+1)&1 was released by the last __syncthreads
    mbar_wait(&bar[ch & 1], (ch >> 1) & 1);
    const uint32_t* cb = fold_buf + (ch & 1) * FOLD_CHUNK;
    const uint32_t* end = cb + len;
#pragma unroll
    for (int q = 0; q < FOLD_SPC; ++q) {
      if (q >= ns) break;
      const int s = s0 + q, r = rr[q];
      if (s <= FOLD_THREADS) {
        const int G = FOLD_THREADS / s;
        if (tid < G * s) {
          // tid = g * s + p: elements of phase p start at (p - r) mod s + g * s = tid - r (+ s)
          const int i0 = tid - r + (pq[q] < r ? s : 0);
          accr[q][0] += strided_sum(cb + i0, end, G * s);
        }
      } else {
#pragma unroll
        for (int w = 0; w < FOLD_MAXW; ++w) {
          const int p = tid + w * FOLD_THREADS;
          if (p < s) accr[q][w] += strided_sum(cb + (p >= r ? p - r : p - r + s), end, s);
        }
      }
      const int rn = r + cm[q];
      rr[q] = rn >= s ? rn - s : rn;
    }
    __syncthreads();  // every thread is done with buffer ch & 1 before it is refilled
  }
  // combine the G groups of small strides; write m_s[p]
  uint32_t* g = acc + acc_off[gi];
#pragma unroll
  for (int q = 0; q < FOLD_SPC; ++q) {
    const int s = s0 + q;
    if (q >= ns) break;
    uint32_t* gs = g + (size_t)(s - x.smin) * x.smax;
    if (s <= FOLD_THREADS) {
      const int G = FOLD_THREADS / s;
      part[tid] = (tid < G * s) ? accr[q][0] : 0u;
      __syncthreads();
      if (tid < s) {
        uint32_t tot = 0;
        for (int grp = 0; grp < G; ++grp) tot += part[grp * s + tid];
        gs[tid] = tot;
      }
      __syncthreads();
    } else {
#pragma unroll
      for (int w = 0; w < FOLD_MAXW; ++w) {
        const int p = tid + w * FOLD_THREADS;
        if (p < s) gs[p] = accr[q][w];
      }
    }
  }
}

// m_s[p] for s < s_dir from the direct fold of its multiple L = s * 2^k in (smax / 2, smax]:
// j = p (mod s)  <=>  j mod L in {p, p + s, ..., p + (2^k - 1) s}, so m_s[p] = sum_i m_L[p + i s]
// (exact integer sums, fixed order)
__global__ void __launch_bounds__(256) grid_derive_kernel(const DInst* __restrict__ insts,
                                                          const int* __restrict__ grid_inst,
                                                          const int64_t* __restrict__ acc_off,
                                                          uint32_t* __restrict__ acc) {
  const int gi = blockIdx.y;
  const DInst x = insts[grid_inst[gi]];
  if (x.stat) return;
  const int s_dir = max(x.smin, x.smax / 2 + 1);
  const int s = x.smin + blockIdx.x;
  if (s >= s_dir) return;
  int L = s;
  while (2 * L <= x.smax) L *= 2;
  uint32_t* g = acc + acc_off[gi];
  const uint32_t* mL = g + (size_t)(L - x.smin) * x.smax;
  uint32_t* ms = g + (size_t)(s - x.smin) * x.smax;
  for (int p = threadIdx.x; p < s; p += blockDim.x) {
    uint32_t t = 0;
    for (int q = p; q < L; q += s) t += mL[q];
    ms[p] = t;
  }
}

// J(s, p) = m_s[p] - n_s[p] * T / N for one candidate stride; best phase (ties -> smaller p)
__global__ void __launch_bounds__(256) grid_eval_kernel(const DInst* __restrict__ insts, const int* __restrict__ grid_inst,
                                                        const int* __restrict__ sinfo, const int* __restrict__ info, int S,
                                                        const int64_t* __restrict__ acc_off,
                                                        const uint32_t* __restrict__ acc,
                                                        double* __restrict__ part, GridRes* __restrict__ res) {
  const int gi = blockIdx.y;
  const DInst x = insts[grid_inst[gi]];
  const int s = x.smin + blockIdx.x;
  double* out = part + ((size_t)gi * 1025 + blockIdx.x) * 2;
  if (s > x.smax || x.stat) return;
  int lo, hi, n;
  grid_window(x, sinfo, info, S, lo, hi, n);
  const int N = hi - lo;
  const uint32_t* g = acc + acc_off[gi];
  // T = sum over all phases of the smallest candidate stride (= sum of c over W, exact)
  typedef cub::BlockReduce<unsigned long long, 256> RU;
  __shared__ typename RU::TempStorage tmpu;
  unsigned long long tl = 0;
  for (int p = threadIdx.x; p < x.smin; p += blockDim.x) tl += g[p];
  const unsigned long long Tfx = RU(tmpu).Sum(tl);
  __shared__ double T_s;
  if (threadIdx.x == 0) {
    T_s = (double)Tfx / (double)FX25;
    if (blockIdx.x == 0) res[gi].T = T_s;
  }
  __syncthreads();
  if (N < s || s < 1) {
    if (threadIdx.x == 0) {
      out[0] = -INFINITY;
      out[1] = 0;
    }
    return;
  }
  const double T = T_s;
  typedef cub::BlockReduce<JP, 256> R;
  __shared__ typename R::TempStorage tmp;
  JP best;
  best.J = -INFINITY;
  best.p = INT_MAX;
  for (int p = threadIdx.x; p < s; p += blockDim.x) {
    const double m = (double)g[(size_t)(s - x.smin) * x.smax + p] / (double)FX25;
    const int j0 = lo + (((p - lo) % s) + s) % s;
    const int np = j0 < hi ? (hi - 1 - j0) / s + 1 : 0;
    JP cand;
    cand.J = m - (double)np * T / (double)N;
    cand.p = p;
    best = jp_best(best, cand);
  }
  const JP b = R(tmp).Reduce(best, JPMax());
  if (threadIdx.x == 0) {
    out[0] = b.J;
    out[1] = (double)b.p;
  }
}

struct JS {
  double J;
  int s, p;
};
struct JSMax {
  __device__ __forceinline__ JS operator()(const JS& a, const JS& b) const {
    if (b.J > a.J || (b.J == a.J && b.s < a.s)) return b;
    return a;
  }
};

// argmax over strides: larger J, ties -> smaller stride
__global__ void __launch_bounds__(1024) grid_pick_kernel(const DInst* __restrict__ insts, const int* __restrict__ grid_inst,
                                                         const double* __restrict__ part, GridRes* __restrict__ res) {
  const int gi = blockIdx.x;
  const DInst x = insts[grid_inst[gi]];
  if (x.stat) {  // static grid (f3 baselines): fixed stride and phase
    if (threadIdx.x == 0) {
      res[gi].s = x.stride;
      res[gi].p = x.stat_p;
      res[gi].J = 0.0;
      res[gi].T = 0.0;
      res[gi].valid = 1;
    }
    return;
  }
  JS best;
  best.J = -INFINITY;
  best.s = INT_MAX;
  best.p = 0;
  for (int s = x.smin + threadIdx.x; s <= x.smax; s += blockDim.x) {
    const double J = part[((size_t)gi * 1025 + (s - x.smin)) * 2];
    if (J == -INFINITY) continue;
    JS c;
    c.J = J;
    c.s = s;
    c.p = (int)part[((size_t)gi * 1025 + (s - x.smin)) * 2 + 1];
    best = JSMax()(best, c);
  }
  typedef cub::BlockReduce<JS, 1024> R;
  __shared__ typename R::TempStorage tmp;
  const JS b = R(tmp).Reduce(best, JSMax());
  if (threadIdx.x == 0) {
    const bool valid = b.s != INT_MAX;
    res[gi].s = valid ? b.s : x.smin;
    res[gi].p = valid ? b.p : 0;
    res[gi].J = valid ? b.J : 0.0;
    res[gi].valid = valid;
  }
}

void launch_grid(const DInst* insts, const int* grid_inst, int n_grid, int max_ncand, int n_inst_total,
                 const DSlab* slabs, const int* sinfo, const int* info, const int* perm, const float* cbuf,
                 uint32_t* fx, int S, int S_pad, GridRes* res, double* part, const int64_t* acc_off,
                 uint32_t* acc, cudaStream_t st) {
  if (n_grid == 0) return;
  grid_prep_kernel<<<dim3(64, n_inst_total), 256, 0, st>>>(insts, n_inst_total, slabs, info, perm, cbuf, fx, S, S_pad);
  const int n_sg = (max_ncand + FOLD_SPC - 1) / FOLD_SPC;
  const int fold_smem = 2 * FOLD_CHUNK * (int)sizeof(uint32_t);
  cudaFuncSetAttribute(grid_acc_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, fold_smem);
  grid_acc_kernel<<<dim3(n_sg, n_grid), FOLD_THREADS, fold_smem, st>>>(insts, grid_inst, sinfo, info, fx, S, S_pad,
                                                                       acc_off, acc);
  grid_derive_kernel<<<dim3(max_ncand, n_grid), 256, 0, st>>>(insts, grid_inst, acc_off, acc);
  grid_eval_kernel<<<dim3(max_ncand, n_grid), 256, 0, st>>>(insts, grid_inst, sinfo, info, S, acc_off, acc, part, res);
  grid_pick_kernel<<<n_grid, 1024, 0, st>>>(insts, grid_inst, part, res);
}

// =============================================================== a4: VS top-k
// Candidates i in [0, n_cand); key(i) = float bits of the score (>= 0).  Selects
// the top `need` by (score desc, index asc) and writes their coordinates in
// ascending order after an optional forced 0.
struct VSCtx {
  int mode;        // 0: columns POS, 1: columns RANK (modality a), 2: columns cross (modality b), 3: offsets
  const float* c;
  const unsigned long long* dg;
  const int* perm;
  int off;         // perm offset of the modality
};
__device__ __forceinline__ uint32_t vs_key(const VSCtx& x, int i) {
  float v;
  if (x.mode == 0)
    v = x.c[i];
  else if (x.mode == 1 || x.mode == 2)
    v = x.c[x.perm[x.off + i]];
  else
    v = (float)((double)x.dg[i] * (1.0 / 4503599627370496.0));
  return __float_as_uint(fmaxf(v, 0.f));
}

__global__ void __launch_bounds__(1024) vs_select_kernel(const DInst* __restrict__ insts, const int* __restrict__ vs_inst,
                                                         const DSlab* __restrict__ slabs, const int* __restrict__ sinfo,
                                                         const int* __restrict__ info, const int* __restrict__ perm,
                                                         const float* __restrict__ cbuf,
                                                         const unsigned long long* __restrict__ dgbuf,
                                                         const int64_t* __restrict__ list_off,
                                                         const int64_t* __restrict__ bits_off, int* __restrict__ lists,
                                                         int* __restrict__ counts, uint32_t* __restrict__ bits) {
  const int vi = blockIdx.x, which = blockIdx.y;  // which 0: verticals, 1: slashes
  const DInst x = insts[vs_inst[vi]];
  const DSlab sl = slabs[x.slab];
  const bool cross = (x.kb >= 0 && x.kb != x.qa);
  const int n_req = which == 0 ? x.n_v : x.n_s;
  int* out = lists + list_off[vi * 2 + which];
  uint32_t* obits = bits + bits_off[vi * 2 + which];
  if (which == 1 && (cross || n_req <= 0)) {
    if (threadIdx.x == 0) counts[vi * 2 + 1] = 0;
    return;
  }
  VSCtx ctx;
  ctx.c = cbuf + sl.c_off;
  ctx.dg = dgbuf + sl.dg_off;
  ctx.perm = perm;
  ctx.off = 0;
  int n_cand;
  const int maxpos = sinfo[x.slab * 4 + 2];
  const int L = sinfo[x.slab * 4 + 0];
  const int maxrank = sinfo[x.slab * 4 + 3] + L - 1;
  if (which == 0) {
    if (cross) {
      ctx.mode = 2;
      ctx.off = info[MI_OFF + x.kb];
      // number of keys of modality kb with position <= maxpos
      const int nb_ = info[MI_CNT + x.kb];
      int lo = 0, hi = nb_;
      while (lo < hi) {
        const int mid = (lo + hi) / 2;
        if (perm[ctx.off + mid] <= maxpos)
          lo = mid + 1;
        else
          hi = mid;
      }
      n_cand = lo;
    } else if (x.rank) {
      ctx.mode = 1;
      ctx.off = info[MI_OFF + x.qa];
      n_cand = maxrank + 1;
    } else {
      ctx.mode = 0;
      n_cand = maxpos + 1;
    }
  } else {
    ctx.mode = 3;
    n_cand = (x.rank ? maxrank : maxpos) + 1;
  }
  const int force = x.force ? 1 : 0;
  const int lo_i = force;  // candidate indices [lo_i, n_cand)
  const int N = max(0, n_cand - lo_i);
  const int need = min(max(n_req - force, 0), N);

  __shared__ int hist[256];
  __shared__ uint32_t s_prefix;
  __shared__ int s_k;
  typedef cub::BlockScan<int, 1024> Scan;
  __shared__ typename Scan::TempStorage stmp;
  __shared__ int s_carry_eq, s_carry_out;

  uint32_t prefix = 0, pmask = 0;
  int k = need;  // rank (1-based) of the threshold among remaining
  const bool take_all = (need >= N);
  if (!take_all && need > 0) {
    for (int shift = 24; shift >= 0; shift -= 8) {
      for (int i = threadIdx.x; i < 256; i += blockDim.x) hist[i] = 0;
      __syncthreads();
      for (int i = lo_i + threadIdx.x; i < n_cand; i += blockDim.x) {
        const uint32_t key = vs_key(ctx, i);
        if ((key & pmask) == prefix) atomicAdd(&hist[(key >> shift) & 255], 1);
      }
      __syncthreads();
      if (threadIdx.x == 0) {
        int kk = k, b = 255;
        for (; b >= 0; --b) {
          if (hist[b] >= kk) break;
          kk -= hist[b];
        }
        s_prefix = prefix | ((uint32_t)b << shift);
        s_k = kk;
      }
      __syncthreads();
      prefix = s_prefix;
      k = s_k;
      pmask |= 255u << shift;
      __syncthreads();
    }
  }
  const uint32_t T = prefix;  // threshold key; take all > T and the first k == T (index order)
  if (threadIdx.x == 0) {
    s_carry_eq = 0;
    s_carry_out = force;
    if (force) out[0] = 0;
  }
  __syncthreads();
  if (need > 0) {
    for (int base = lo_i; base < n_cand; base += blockDim.x) {
      const int i = base + threadIdx.x;
      int gt = 0, eq = 0;
      if (i < n_cand) {
        if (take_all) {
          gt = 1;
        } else {
          const uint32_t key = vs_key(ctx, i);
          gt = key > T;
          eq = key == T;
        }
      }
      int eq_pre;
      Scan(stmp).ExclusiveSum(eq, eq_pre);
      __syncthreads();
      const int sel = gt || (eq && (s_carry_eq + eq_pre) < k);
      int sel_pre, sel_tot;
      Scan(stmp).ExclusiveSum(sel, sel_pre, sel_tot);
      __syncthreads();
      int eq_tot = 0;
      if (threadIdx.x == blockDim.x - 1) eq_tot = eq_pre + eq;
      if (sel) {
        const int coord = (ctx.mode == 2) ? perm[ctx.off + i] : i;
        out[s_carry_out + sel_pre] = coord;
      }
      __syncthreads();
      if (threadIdx.x == blockDim.x - 1) {
        s_carry_eq += eq_tot;
        s_carry_out += sel_tot;
      }
      __syncthreads();
    }
  }
  __syncthreads();
  const int total = s_carry_out;
  if (threadIdx.x == 0) counts[vi * 2 + which] = total;
  for (int i = threadIdx.x; i < total; i += blockDim.x) {
    const int cdn = out[i];
    atomicOr(obits + (cdn >> 5), 1u << (cdn & 31));
  }
}

void launch_vs(const DInst* insts, const int* vs_inst, int n_vs, const DSlab* slabs, const int* sinfo, const int* info,
               const int* perm, const float* cbuf, const unsigned long long* dgbuf, const int64_t* list_off,
               const int64_t* bits_off, int* lists, int* counts, uint32_t* bits, cudaStream_t st) {
  if (n_vs == 0) return;
  vs_select_kernel<<<dim3(n_vs, 2), 1024, 0, st>>>(insts, vs_inst, slabs, sinfo, info, perm, cbuf, dgbuf, list_off,
                                                    bits_off, lists, counts, bits);
}

}  // namespace mmi
