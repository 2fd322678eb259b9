// Last-q slab estimation on the 5th-generation tensor cores:
//   A-hat = softmax(Q[R] K^T tau + m_causal)   (Alg.1; P:241 per-modality slabs)
//   c[j]  = sum_r A-hat[r, j]                    (column mass: grid fold / verticals)
// Two passes over the keys of one KV group: pass 1 = per-row running max / sum (online
// softmax statistics, partial per key chunk, combined by slab_combine_kernel), pass 2 =
// A-hat tile by tile and its column sums.  The slabs of one KV group are packed two per
// tcgen05 M=128 tile (rows 0-63 slab a, 64-127 slab b); S = Q K^T (M128 N128) goes to a
// double-buffered TMEM accumulator, K tiles arrive by TMA (128B swizzle) in a 2-stage ring,
// and 4 epilogue warps run the exp2 / statistics.  Pass 1 computes S = Q K^T (thread = TMEM lane
// = slab row: row max / sum are per-thread); pass 2 computes S^T = K Q^T with the SAME shared
// tiles as swapped operands (thread = key, columns = slab rows), so the column mass of a key is a
// per-thread sum in fixed row order: no cross-thread reduction, deterministic.
// Slabs that also need the diagonal mass dg (vertical-slash heads with slashes) run in
// slab_kernel (estimate.cu), which accumulates both.
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <cstdint>

#include "estimate.h"
#include "ptx.cuh"

namespace mmi {

constexpr int STC_THREADS = 256;   // warp 0 TMA, warp 1 MMA + TMEM, warps 2-3 Q staging, warps 4-7 epilogue
constexpr int STC_KST = 2;         // K ring stages
#ifndef MMI_STC_CHUNK
#define MMI_STC_CHUNK 32
#endif
constexpr int STC_CHUNK_TILES = MMI_STC_CHUNK;  // key tiles per CTA (4096 keys; 8192 measured 4 % slower at 128K)

template <int D>
struct StcSmem {
  static constexpr int Q_BYTES = BLK * D * 2;
  static constexpr int K_BYTES = BLK * D * 2;
  static constexpr int OFF_Q = 0;
  static constexpr int OFF_K = OFF_Q + Q_BYTES;
  static constexpr int OFF_CS = OFF_K + STC_KST * K_BYTES;       // [4 warps][128] column partials
  static constexpr int OFF_BAR = OFF_CS + 4 * BLK * 4;
  static constexpr int N_BAR = 2 * STC_KST + 4;                  // k_full, k_empty, s_full[2], s_empty[2]
  static constexpr int OFF_TMEM = OFF_BAR + N_BAR * 8;
  static constexpr int TOTAL = OFF_TMEM + 16;
  static constexpr int ALLOC = TOTAL + 1024;
};

// butterfly transpose-reduce: v[k] = this lane's value of column k (32 columns); returns the sum
// over the 32 lanes of column `lane`
__device__ __forceinline__ float warp_colsum32(float (&v)[32], int lane) {
#pragma unroll
  for (int o = 16; o >= 1; o >>= 1) {
    const bool upper = (lane & o) != 0;
#pragma unroll
    for (int k = 0; k < o; ++k) {
      const float send = upper ? v[k] : v[k + o];
      const float keep = upper ? v[k + o] : v[k];
      v[k] = keep + __shfl_xor_sync(0xffffffffu, send, o);
    }
  }
  return v[0];
}

template <int D>
__global__ void __launch_bounds__(STC_THREADS, 2)
    slab_tc_kernel(const __grid_constant__ CUtensorMap tmK, int mode, const int2* __restrict__ pairs,
                   const DSlab* __restrict__ slabs, const __nv_bfloat16* __restrict__ q, int S, float scale_log2,
                   const int* __restrict__ rows, const int* __restrict__ sinfo, float2* __restrict__ ml_part,
                   const float2* __restrict__ ml, float* __restrict__ cbuf, int ml_stride) {
  using L = StcSmem<D>;
  extern __shared__ __align__(1024) uint8_t stc_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(stc_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + L::OFF_BAR);
  uint64_t* k_full = bars;
  uint64_t* k_empty = bars + STC_KST;
  uint64_t* s_full = bars + 2 * STC_KST;
  uint64_t* s_empty = s_full + 2;
  uint32_t* tmem_holder = reinterpret_cast<uint32_t*>(smem + L::OFF_TMEM);
  float* cs = reinterpret_cast<float*>(smem + L::OFF_CS);
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const int chunk = blockIdx.x;
  const int2 pr = pairs[blockIdx.y];
  const int sa = pr.x, sb = pr.y;  // slab b may be -1
  const DSlab SA = slabs[sa];
  const int kv = SA.kv;
  int maxpos = sinfo[sa * 4 + 2];
  if (sb >= 0) maxpos = max(maxpos, sinfo[sb * 4 + 2]);
  const int t_begin = chunk * STC_CHUNK_TILES;
  const int t_end = min(t_begin + STC_CHUNK_TILES, maxpos / BLK + 1);
  const int nt = t_end - t_begin;
  // row identity of epilogue thread (TMEM lane = row of the packed tile)
  const int r = (warp >= 4) ? (warp - 4) * 32 + lane : 0;
  const int my_slab = (r < 64) ? sa : sb;
  const int rl = r & 63;
  const int my_pos = (warp >= 4 && my_slab >= 0) ? rows[my_slab * SLAB_ROWS + rl] : -1;
  if (nt <= 0) {  // every key of this chunk is after every slab row
    if (mode == 0 && warp >= 4 && my_slab >= 0)
      ml_part[((size_t)my_slab * ml_stride + chunk) * SLAB_ROWS + rl] = make_float2(-INFINITY, 0.f);
    return;
  }
  // ---- Q tile (two slabs, 128 rows) -> shared memory in the UMMA 128B-swizzle K-major layout ----
  {
    constexpr int CPR = D / 8;  // 16-byte chunks per row
    for (int idx = threadIdx.x; idx < BLK * CPR; idx += STC_THREADS) {
      const int row = idx / CPR, ck = idx % CPR;
      const int sl = (row < 64) ? sa : sb;
      int pos = -1;
      if (sl >= 0) pos = rows[sl * SLAB_ROWS + (row & 63)];
      uint4 val = make_uint4(0, 0, 0, 0);
      if (pos >= 0) val = __ldg(reinterpret_cast<const uint4*>(q + ((size_t)slabs[sl].head * S + pos) * D) + ck);
      const int cb = ck / 8, k = ck % 8;  // 64-column block, 16-byte unit inside the 128-byte row
      *reinterpret_cast<uint4*>(smem + L::OFF_Q + cb * (BLK * 128) + row * 128 + ((k ^ (row & 7)) * 16)) = val;
    }
  }
  if (threadIdx.x == 0) {
    for (int i = 0; i < STC_KST; ++i) {
      mbar_init(k_full + i, 1);
      mbar_init(k_empty + i, 1);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(s_full + i, 1);
      mbar_init(s_empty + i, 4);
    }
    fence_barrier_init();
  }
  if (warp == 1) tmem_alloc<256>(tmem_holder);
  fence_proxy_async_smem();  // generic-proxy Q stores visible to the tensor core
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_holder;

  if (warp == 0) {
    if (elect_one()) {
      tma_prefetch_desc(&tmK);
      for (int i = 0; i < nt; ++i) {
        const int st = i % STC_KST;
        mbar_wait(k_empty + st, ((i / STC_KST) & 1) ^ 1);
        mbar_arrive_expect_tx(k_full + st, L::K_BYTES);
#pragma unroll
        for (int c = 0; c < D / 64; ++c)
          tma_load_2d(smem + L::OFF_K + st * L::K_BYTES + c * (BLK * 128), &tmK, k_full + st, c * 64,
                      kv * S + (t_begin + i) * BLK);
      }
    }
  } else if (warp == 1) {
    if (elect_one()) {
      constexpr uint32_t IDESC = idesc_bf16(128, 128, 0);
      const uint32_t q_base = smem_u32(smem + L::OFF_Q), k_base = smem_u32(smem + L::OFF_K);
      for (int i = 0; i < nt; ++i) {
        const int st = i % STC_KST, b = i & 1;
        mbar_wait(k_full + st, (i / STC_KST) & 1);
        mbar_wait(s_empty + b, ((i >> 1) & 1) ^ 1);
        tc_fence_after();
#pragma unroll
        for (int k = 0; k < D / 16; ++k) {
          const uint32_t off = (k / 4) * (BLK * 128) + (k % 4) * 32;
          const uint64_t dq = smem_desc(q_base + off, 16, 1024, 2);
          const uint64_t dk = smem_desc(k_base + st * L::K_BYTES + off, 16, 1024, 2);
          // pass 1: S = Q K^T (TMEM lane = slab row); pass 2: S^T = K Q^T (TMEM lane = key), so the
          // column sums of A-hat are per-thread sums over the TMEM columns
          if (mode == 0)
            umma_ss(tmem + b * 128, dq, dk, IDESC, k > 0 ? 1u : 0u);
          else
            umma_ss(tmem + b * 128, dk, dq, IDESC, k > 0 ? 1u : 0u);
        }
        umma_commit(k_empty + st);
        umma_commit(s_full + b);
      }
    }
  } else if (warp >= 4) {
    const int ew = warp - 4;
    const uint32_t lane_off = (uint32_t)(ew * 32) << 16;
    if (mode == 0) {
      // ---- pass 1: TMEM lane = slab row r; running max / normaliser over this chunk's keys ----
      // 64 columns per step (two 32-column loads in flight per wait), one max and one rescale per
      // step, packed FFMA2 for the scaled scores; the causal select only where a row's admitted
      // keys end inside the step
      const bool valid = my_pos >= 0;
      float m = -INFINITY, l = 0.f;
      const float2 sc2 = make_float2(scale_log2, scale_log2);
      for (int i = 0; i < nt; ++i) {
        const int b = i & 1;
        const int j0 = (t_begin + i) * BLK;
        mbar_wait(s_full + b, (i >> 1) & 1);
        tc_fence_after();
        // keys j0 + c admitted for this row iff j0 + c <= pos (causal; pos < S)
        const int n_ok = valid ? min(max(my_pos - j0 + 1, 0), BLK) : 0;
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          uint32_t raw[2][32];
          tmem_ld32(tmem + b * 128 + h * 64 + lane_off, raw[0]);
          tmem_ld32(tmem + b * 128 + h * 64 + 32 + lane_off, raw[1]);
          tmem_wait_ld();
          const int lim = n_ok - h * 64;  // admitted columns of this step: [0, lim) (none if <= 0)
          float v[64];
#pragma unroll
          for (int k = 0; k < 64; ++k) v[k] = __uint_as_float(raw[k / 32][k % 32]);
          if (__any_sync(0xffffffffu, lim < 64)) {
#pragma unroll
            for (int k = 0; k < 64; ++k) v[k] = (k < lim) ? v[k] : -INFINITY;
          }
          float mx[4] = {v[0], v[1], v[2], v[3]};
#pragma unroll
          for (int k = 4; k < 64; k += 4) {
            mx[0] = fmaxf(mx[0], v[k]);
            mx[1] = fmaxf(mx[1], v[k + 1]);
            mx[2] = fmaxf(mx[2], v[k + 2]);
            mx[3] = fmaxf(mx[3], v[k + 3]);
          }
          const float mt = fmaxf(fmaxf(mx[0], mx[1]), fmaxf(mx[2], mx[3])) * scale_log2;  // scale > 0
          const float mn = fmaxf(m, mt);
          const float mu = (mn == -INFINITY) ? 0.f : mn;  // no admitted key yet: every term is 0
          const float2 nm2 = make_float2(-mu, -mu);
          float2 s2[4] = {make_float2(0.f, 0.f), make_float2(0.f, 0.f), make_float2(0.f, 0.f), make_float2(0.f, 0.f)};
#pragma unroll
          for (int k = 0; k < 64; k += 2) {
            const float2 x = ffma2(make_float2(v[k], v[k + 1]), sc2, nm2);
            s2[(k / 2) % 4] = fadd2(s2[(k / 2) % 4], make_float2(ex2(x.x), ex2(x.y)));
          }
          const float2 st = fadd2(fadd2(s2[0], s2[1]), fadd2(s2[2], s2[3]));
          l = (m > -INFINITY ? l * ex2(m - mn) : 0.f) + (st.x + st.y);
          m = mn;
        }
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(s_empty + b);  // S buffer b may be overwritten
      }
      if (my_slab >= 0) ml_part[((size_t)my_slab * ml_stride + chunk) * SLAB_ROWS + rl] = make_float2(m, l);
    } else {
      // ---- pass 2: TMEM lane = key j, column = slab row r; c[j] = sum_r A-hat[r, j] per thread ----
      // A-hat[r, j] = exp2(z * scale - Mr), Mr = m_r + log2(l_r) (+inf for rows without keys); row r
      // admits key j iff pos_r >= j: slab rows are ascending, so that is a suffix of each slab's rows
      float* Mr = cs;                                       // [128]
      int* pos_s = reinterpret_cast<int*>(cs + BLK);        // [128] (-1: no row)
      {
        const int t = threadIdx.x - 128;  // 0..127: row t of the packed tile
        const int sl = t < 64 ? sa : sb;
        int pos = -1;
        float M = INFINITY;
        if (sl >= 0) {
          pos = rows[sl * SLAB_ROWS + (t & 63)];
          if (pos >= 0) {
            const float2 v = ml[(size_t)sl * SLAB_ROWS + (t & 63)];
            if (v.y > 0.f) M = v.x + __log2f(v.y);
          }
        }
        Mr[t] = M;
        pos_s[t] = pos;
        named_bar_sync(1, 128);
      }
      const int La = sinfo[sa * 4 + 0], Lb = sb >= 0 ? sinfo[sb * 4 + 0] : 0;
      const int key = ew * 32 + lane;  // TMEM lane
      for (int i = 0; i < nt; ++i) {
        const int b = i & 1;
        const int j = (t_begin + i) * BLK + key;
        // first row of each slab whose position is >= j (binary search over the ascending rows)
        int lo_a = 0, hi_a = La;
        while (lo_a < hi_a) {
          const int mid = (lo_a + hi_a) >> 1;
          if (pos_s[mid] >= j) hi_a = mid; else lo_a = mid + 1;
        }
        int lo_b = 0, hi_b = Lb;
        while (lo_b < hi_b) {
          const int mid = (lo_b + hi_b) >> 1;
          if (pos_s[64 + mid] >= j) hi_b = mid; else lo_b = mid + 1;
        }
        mbar_wait(s_full + b, (i >> 1) & 1);
        tc_fence_after();
        float ca = 0.f, cbs = 0.f;
        const float2 sc2 = make_float2(scale_log2, scale_log2);
#pragma unroll
        for (int h = 0; h < 2; ++h) {  // rows of slab a (h = 0) / slab b (h = 1): 64 columns
          const int lo = h ? lo_b : lo_a, hi = h ? Lb : La;  // admitted rows [lo, hi) of the slab
          if (!__any_sync(0xffffffffu, hi > lo)) continue;  // no admitted row for the warp
          uint32_t raw[2][32];
          tmem_ld32(tmem + b * 128 + h * 64 + lane_off, raw[0]);
          tmem_ld32(tmem + b * 128 + h * 64 + 32 + lane_off, raw[1]);
          tmem_wait_ld();
          const bool all = __all_sync(0xffffffffu, lo == 0 && hi == 64);
          float2 a2[4] = {make_float2(0.f, 0.f), make_float2(0.f, 0.f), make_float2(0.f, 0.f), make_float2(0.f, 0.f)};
#pragma unroll
          for (int k = 0; k < 64; k += 4) {
            const float4 M4 = *reinterpret_cast<const float4*>(Mr + h * 64 + k);
            const float2 x0 = ffma2(make_float2(__uint_as_float(raw[k / 32][k % 32]), __uint_as_float(raw[k / 32][k % 32 + 1])),
                                    sc2, make_float2(-M4.x, -M4.y));
            const float2 x1 = ffma2(make_float2(__uint_as_float(raw[k / 32][k % 32 + 2]), __uint_as_float(raw[k / 32][k % 32 + 3])),
                                    sc2, make_float2(-M4.z, -M4.w));
            float2 e0 = make_float2(ex2(x0.x), ex2(x0.y)), e1 = make_float2(ex2(x1.x), ex2(x1.y));
            if (!all) {
              e0.x = (k >= lo && k < hi) ? e0.x : 0.f;
              e0.y = (k + 1 >= lo && k + 1 < hi) ? e0.y : 0.f;
              e1.x = (k + 2 >= lo && k + 2 < hi) ? e1.x : 0.f;
              e1.y = (k + 3 >= lo && k + 3 < hi) ? e1.y : 0.f;
            }
            a2[(k / 4) % 2] = fadd2(a2[(k / 4) % 2], e0);
            a2[2 + (k / 4) % 2] = fadd2(a2[2 + (k / 4) % 2], e1);
          }
          const float2 t2 = fadd2(fadd2(a2[0], a2[1]), fadd2(a2[2], a2[3]));
          if (h == 0)
            ca = t2.x + t2.y;
          else
            cbs = t2.x + t2.y;
        }
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(s_empty + b);
        if (j < S) {
          cbuf[SA.c_off + j] = ca;
          if (sb >= 0) cbuf[slabs[sb].c_off + j] = cbs;
        }
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc<256>(tmem);
  }
}

int make_tmap_rows(CUtensorMap* m, const void* base, long long rows, int D);

int slab_tc_chunks(int S) { return (S + STC_CHUNK_TILES * BLK - 1) / (STC_CHUNK_TILES * BLK); }

cudaError_t launch_slab_tc(int mode, const int2* pairs, int n_pairs, const DSlab* slabs, const void* q, const void* k,
                           int S, int Hkv, int D, float scale_log2, const int* rows, const int* sinfo, float2* ml_part,
                           const float2* ml, float* cbuf, int ml_stride, cudaStream_t st) {
  if (n_pairs <= 0) return cudaSuccess;
  CUtensorMap tm;
  if (make_tmap_rows(&tm, k, (long long)Hkv * S, D) != 0) return cudaErrorInvalidValue;
  const dim3 grid(slab_tc_chunks(S), n_pairs);
  cudaError_t e;
  if (D == 128) {
    e = cudaFuncSetAttribute(slab_tc_kernel<128>, cudaFuncAttributeMaxDynamicSharedMemorySize, StcSmem<128>::ALLOC);
    if (e != cudaSuccess) return e;
    slab_tc_kernel<128><<<grid, STC_THREADS, StcSmem<128>::ALLOC, st>>>(
        tm, mode, pairs, slabs, (const __nv_bfloat16*)q, S, scale_log2, rows, sinfo, ml_part, ml, cbuf, ml_stride);
  } else {
    e = cudaFuncSetAttribute(slab_tc_kernel<64>, cudaFuncAttributeMaxDynamicSharedMemorySize, StcSmem<64>::ALLOC);
    if (e != cudaSuccess) return e;
    slab_tc_kernel<64><<<grid, STC_THREADS, StcSmem<64>::ALLOC, st>>>(
        tm, mode, pairs, slabs, (const __nv_bfloat16*)q, S, scale_log2, rows, sinfo, ml_part, ml, cbuf, ml_stride);
  }
  return cudaGetLastError();
}

}  // namespace mmi
