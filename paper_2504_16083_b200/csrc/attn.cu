// Block-sparse causal FlashAttention for sm_100a (tcgen05 + TMEM + TMA).
//
// Implements the online-softmax recurrence of Alg.5/6/7 (PAPER.md P:920-983,
// P:1015-1034): per 128-row query block, loop over the listed key
// tiles, S = tau Q K^T, S <- mask(S), m_new = max(m, rowmax S), P = exp(S - m_new),
// l = alpha l + rowsum P (reading C10: rowsum of P), O = alpha O + P V, and finally
// O <- diag(l)^-1 O.  The tile list (which key tiles of which K-view) and the
// element predicate come from the index (mmi_estimate_index), so one kernel
// executes every pattern / boundary type ("sparse loading with dense
// computation").
//
// Warp roles (one CTA per SM, persistent, static round-robin over LPT-ordered
// work items):
//   warp 0     TMA producer: Q tile, K/V tiles (+ key positions for PRED tiles)
//   warp 1     MMA issuer: S = Q K^T into TMEM (double buffered), O += P V
//   warp 2     TMEM allocator
//   warps 4-7  softmax / correction / epilogue, thread t owns query row t
//              (TMEM lane t): tcgen05.ld S, predicate, exp2, P -> smem (bf16,
//              128B-swizzled K-major UMMA layout), lazy O rescale in TMEM.
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <climits>
#include <cstdint>
#include <cstdio>

#include "internal.h"
#include "ptx.cuh"

namespace mmi {

constexpr int NST = 2;             // K/V pipeline stages
constexpr int NTHREADS = 256;
constexpr float RESCALE_THRESH = 8.0f;  // lazy rescale: P <= 2^8 (log2 domain)

template <int D>
struct Smem {
  static constexpr int Q_BYTES = BLK * D * 2;
  static constexpr int KV_BYTES = BLK * D * 2;
  static constexpr int P_BYTES = BLK * BLK * 2;
  static constexpr int OFF_Q = 0;
  static constexpr int OFF_P = OFF_Q + Q_BYTES;
  static constexpr int OFF_K = OFF_P + P_BYTES;
  static constexpr int OFF_V = OFF_K + NST * KV_BYTES;
  static constexpr int OFF_KPOS = OFF_V + NST * KV_BYTES;
  static constexpr int OFF_KRANK = OFF_KPOS + NST * BLK * 4;
  static constexpr int OFF_BAR = OFF_KRANK + NST * BLK * 4;
  static constexpr int N_BAR = 2 + 2 * NST + 4 + 4;
  static constexpr int OFF_TMEM = OFF_BAR + N_BAR * 8;
  static constexpr int TOTAL = OFF_TMEM + 16;
  static constexpr int ALLOC = TOTAL + 1024;  // alignment slack
};

struct ItemView {
  int head, q_row0, seg_off, n_segs, n_tiles, q_gathered, out_mode, out_row0, inst_base, skip_s, skip_p, skip_rank,
      row_mod, rb;
};

__device__ __forceinline__ ItemView load_item(const AttnParams& P, int idx) {
  ItemView v;
  if (P.dense) {
    const int nb = (P.S + BLK - 1) / BLK;
    const int rb = nb - 1 - idx / P.H;  // longest rows first (LPT)
    v.head = idx % P.H;
    v.q_row0 = v.head * P.S + rb * BLK;
    v.rb = rb;
    v.seg_off = 0;
    v.n_segs = 1;
    v.n_tiles = rb + 1;
    v.q_gathered = 0;
    v.out_mode = OUT_FINAL;
    v.out_row0 = 0;
    v.inst_base = 0;
    v.skip_s = 0;
    v.skip_p = 0;
    v.skip_rank = 0;
    v.row_mod = -1;
    return v;
  }
  const WorkItem w = P.items[idx];
  v.head = w.head;
  v.q_row0 = w.q_row0;
  v.seg_off = w.seg_off;
  v.n_segs = w.n_segs;
  v.n_tiles = w.n_tiles;
  v.q_gathered = w.q_gathered;
  v.out_mode = w.out_mode;
  v.out_row0 = w.out_row0;
  v.inst_base = w.inst_base;
  v.skip_s = w.skip_s;
  v.skip_p = w.skip_p;
  v.skip_rank = w.skip_rank;
  v.row_mod = w.row_mod;
  v.rb = 0;
  return v;
}

struct TileInfo {
  int krow;
  uint32_t space, pred, role, rmode, inst;
};

// walks the item's segments tile by tile (every warp role keeps its own cursor)
struct SegIter {
  Seg cur;
  int seg_i, t;
  __device__ __forceinline__ void init(const AttnParams& P, const ItemView& it) {
    seg_i = 0;
    t = 0;
    if (P.dense) {
      cur.krow0 = (it.head / (P.H / P.Hkv)) * P.S;
      cur.ntiles = it.rb + 1;
      cur.meta = seg_meta(0, R_TRUE, 0, 0);
      cur.pred_head = 0;
      cur.pred_tail = 1;
    } else {
      cur.ntiles = 0;
      seg_i = -1;
    }
  }
  __device__ __forceinline__ TileInfo next(const AttnParams& P, const ItemView& it) {
    while (t >= cur.ntiles) {
      ++seg_i;
      cur = P.segs[it.seg_off + seg_i];
      t = 0;
    }
    TileInfo ti;
    ti.krow = cur.krow0 + t * BLK;
    ti.space = cur.meta & 1u;
    ti.role = (cur.meta >> 2) & 7u;
    ti.rmode = (cur.meta >> 5) & 1u;
    ti.inst = (cur.meta >> 8) & 0xffu;
    ti.pred = (t < cur.pred_head || t >= cur.ntiles - cur.pred_tail) ? 1u : 0u;
    ++t;
    return ti;
  }
};

template <int D>
__global__ void __launch_bounds__(NTHREADS, 1)
    attn_kernel(const __grid_constant__ CUtensorMap tmQo, const __grid_constant__ CUtensorMap tmQg,
                const __grid_constant__ CUtensorMap tmKo, const __grid_constant__ CUtensorMap tmKg,
                const __grid_constant__ CUtensorMap tmVo, const __grid_constant__ CUtensorMap tmVg,
                const AttnParams P) {
  using L = Smem<D>;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + L::OFF_BAR);
  uint64_t* q_full = bars + 0;
  uint64_t* q_empty = bars + 1;
  uint64_t* kv_full = bars + 2;
  uint64_t* kv_empty = bars + 2 + NST;
  uint64_t* s_full = bars + 2 + 2 * NST;   // [2]
  uint64_t* s_empty = s_full + 2;          // [2]
  uint64_t* p_full = s_empty + 2;
  uint64_t* p_empty = p_full + 1;
  uint64_t* o_full = p_empty + 1;
  uint64_t* o_empty = o_full + 1;
  uint32_t* tmem_holder = reinterpret_cast<uint32_t*>(smem + L::OFF_TMEM);
  int32_t* kpos_s = reinterpret_cast<int32_t*>(smem + L::OFF_KPOS);
  int32_t* krank_s = reinterpret_cast<int32_t*>(smem + L::OFF_KRANK);

  const int warp = threadIdx.x / 32;
  const int lane = threadIdx.x % 32;

  if (threadIdx.x == 0) {
    mbar_init(q_full, 1);
    mbar_init(q_empty, 1);
    for (int i = 0; i < NST; ++i) {
      mbar_init(kv_full + i, 1);
      mbar_init(kv_empty + i, 1);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(s_full + i, 1);
      mbar_init(s_empty + i, 128);
    }
    mbar_init(p_full, 128);
    mbar_init(p_empty, 1);
    mbar_init(o_full, 1);
    mbar_init(o_empty, 128);
    fence_barrier_init();
  }
  if (warp == 2) tmem_alloc<512>(tmem_holder);
  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&tmQo);
    tma_prefetch_desc(&tmQg);
    tma_prefetch_desc(&tmKo);
    tma_prefetch_desc(&tmKg);
    tma_prefetch_desc(&tmVo);
    tma_prefetch_desc(&tmVg);
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_holder;
  const uint32_t tS[2] = {tmem, tmem + 128};
  const uint32_t tO = tmem + 256;

  const int n_items = P.dense ? P.H * ((P.S + BLK - 1) / BLK) : P.n_items;

  if (warp == 0) {
    // ======================= TMA producer =======================
    if (elect_one()) {
      int stage = 0;
      uint32_t kv_phase = 0, q_phase = 0;
      for (int idx = blockIdx.x; idx < n_items; idx += gridDim.x) {
        const ItemView it = load_item(P, idx);
        if (it.n_tiles <= 0) continue;
        mbar_wait(q_empty, q_phase ^ 1);
        q_phase ^= 1;
        mbar_arrive_expect_tx(q_full, L::Q_BYTES);
        const CUtensorMap* tq = it.q_gathered ? &tmQg : &tmQo;
#pragma unroll
        for (int c = 0; c < D / 64; ++c)
          tma_load_2d(smem + L::OFF_Q + c * (BLK * 128), tq, q_full, c * 64, it.q_row0);
        SegIter si;
        si.init(P, it);
        for (int t = 0; t < it.n_tiles; ++t) {
          const TileInfo e = si.next(P, it);
          const uint32_t space = e.space, pred = e.pred, rank = e.rmode;
          mbar_wait(kv_empty + stage, kv_phase ^ 1);
          uint32_t bytes = 2 * L::KV_BYTES;
          const bool cp_pos = (pred || P.fingerprint) && space;
          const bool cp_rank = pred && space && rank;
          if (cp_pos) bytes += BLK * 4;
          if (cp_rank) bytes += BLK * 4;
          mbar_arrive_expect_tx(kv_full + stage, bytes);
          const CUtensorMap* tk = space ? &tmKg : &tmKo;
          const CUtensorMap* tv = space ? &tmVg : &tmVo;
          uint8_t* ks = smem + L::OFF_K + stage * L::KV_BYTES;
          uint8_t* vs = smem + L::OFF_V + stage * L::KV_BYTES;
#pragma unroll
          for (int c = 0; c < D / 64; ++c) {
            tma_load_2d(ks + c * (BLK * 128), tk, kv_full + stage, c * 64, e.krow);
            tma_load_2d(vs + c * (BLK * 128), tv, kv_full + stage, c * 64, e.krow);
          }
          if (cp_pos) bulk_load(kpos_s + stage * BLK, P.kg_pos + e.krow, BLK * 4, kv_full + stage);
          if (cp_rank) bulk_load(krank_s + stage * BLK, P.kg_rank + e.krow, BLK * 4, kv_full + stage);
          if (++stage == NST) {
            stage = 0;
            kv_phase ^= 1;
          }
        }
      }
    }
  } else if (warp == 1) {
    // ======================= MMA issuer =======================
    constexpr uint32_t IDESC_S = idesc_bf16(128, 128, 0);
    constexpr uint32_t IDESC_O = idesc_bf16(128, D, 1);
    const uint32_t q_base = smem_u32(smem + L::OFF_Q);
    const uint32_t p_base = smem_u32(smem + L::OFF_P);
    const uint32_t k_base = smem_u32(smem + L::OFF_K);
    const uint32_t v_base = smem_u32(smem + L::OFF_V);
    int stage = 0;
    uint32_t kv_phase = 0, q_phase = 0, p_phase = 0, o_phase = 0;
    uint32_t s_phase[2] = {0, 0};
    int sbuf = 0;
    const bool leader = elect_one();
    for (int idx = blockIdx.x; idx < n_items; idx += gridDim.x) {
      const ItemView it = load_item(P, idx);
      if (it.n_tiles <= 0) continue;
      mbar_wait(q_full, q_phase);
      q_phase ^= 1;
      tc_fence_after();
      int prev_stage = -1;
      for (int t = 0; t <= it.n_tiles; ++t) {
        int cur_stage = stage;
        if (t < it.n_tiles) {
          // S[sbuf] = Q K_t^T
          mbar_wait(kv_full + stage, kv_phase);
          mbar_wait(s_empty + sbuf, s_phase[sbuf] ^ 1);
          tc_fence_after();
          if (leader) {
#pragma unroll
            for (int k = 0; k < D / 16; ++k) {
              const uint32_t off = (k / 4) * (BLK * 128) + (k % 4) * 32;
              const uint64_t ad = smem_desc(q_base + off, 16, 1024, 2);
              const uint64_t bd = smem_desc(k_base + stage * L::KV_BYTES + off, 16, 1024, 2);
              umma_ss(tS[sbuf], ad, bd, IDESC_S, k > 0 ? 1u : 0u);
            }
            umma_commit(s_full + sbuf);
            if (t == it.n_tiles - 1) umma_commit(q_empty);
          }
          __syncwarp();
          s_phase[sbuf] ^= 1;
          sbuf ^= 1;
          if (++stage == NST) {
            stage = 0;
            kv_phase ^= 1;
          }
        }
        if (t >= 1) {
          // O += P_{t-1} V_{t-1}
          mbar_wait(p_full, p_phase);
          p_phase ^= 1;
          if (t == 1) {
            mbar_wait(o_empty, o_phase ^ 1);  // previous item's epilogue has read O
          }
          tc_fence_after();
          if (leader) {
#pragma unroll
            for (int k = 0; k < BLK / 16; ++k) {
              const uint32_t aoff = (k / 4) * (BLK * 128) + (k % 4) * 32;
              const uint64_t ad = smem_desc(p_base + aoff, 16, 1024, 2);
              const uint64_t bd = smem_desc(v_base + prev_stage * L::KV_BYTES + k * 2048, BLK * 128, 1024, 2);
              umma_ss(tO, ad, bd, IDESC_O, (t > 1 || k > 0) ? 1u : 0u);
            }
            umma_commit(kv_empty + prev_stage);
            umma_commit(p_empty);
            if (t == it.n_tiles) umma_commit(o_full);
          }
          __syncwarp();
        }
        prev_stage = cur_stage;
      }
      o_phase ^= 1;
    }
  } else if (warp >= 4) {
    // ======================= softmax / epilogue =======================
    const int row = threadIdx.x - 128;                 // TMEM lane == query row
    const uint32_t lane_off = (uint32_t)((warp - 4) * 32) << 16;
    const uint32_t p_base = smem_u32(smem + L::OFF_P);
    int stage = 0;
    uint32_t kv_phase = 0, p_phase = 0, o_phase = 0;
    uint32_t s_phase[2] = {0, 0};
    int sbuf = 0;
    const int G = P.H / P.Hkv;
    for (int idx = blockIdx.x; idx < n_items; idx += gridDim.x) {
      const ItemView it = load_item(P, idx);
      if (it.n_tiles <= 0) continue;  // empty slot: nothing to compute or write
      // row identity
      int xpos, xrank;
      if (it.q_gathered) {
        xpos = P.qg_pos[it.q_row0 + row];
        xrank = P.qg_rank[it.q_row0 + row];
      } else {
        xpos = it.q_row0 - it.head * P.S + row;
        xrank = (xpos < P.S && P.rank) ? P.rank[xpos] : xpos;
      }
      bool valid = xpos >= 0 && xpos < P.S;
      if (valid && it.row_mod >= 0) valid = (P.labels[xpos] == it.row_mod);
      bool write = valid;
      if (it.skip_s > 0 && valid) {
        const int c = it.skip_rank ? xrank : xpos;
        if (c % it.skip_s == it.skip_p) write = false;
      }
      float m_used = -INFINITY, l_sum = 0.f;
      long long fp_cnt = 0, fp_s1 = 0, fp_s2 = 0;
      const int kv = it.head / G;
      SegIter si;
      si.init(P, it);
      for (int t = 0; t < it.n_tiles; ++t) {
        const TileInfo e = si.next(P, it);
        const uint32_t space = e.space, pred = e.pred, role = e.role, rmode = e.rmode, inst = e.inst;
        mbar_wait(s_full + sbuf, s_phase[sbuf]);
        s_phase[sbuf] ^= 1;
        tc_fence_after();
        float s[BLK];
#pragma unroll
        for (int c = 0; c < BLK / 32; ++c) {
          uint32_t r[32];
          tmem_ld32(tS[sbuf] + lane_off + c * 32, r);
          tmem_wait_ld();
#pragma unroll
          for (int j = 0; j < 32; ++j) s[c * 32 + j] = __uint_as_float(r[j]) * P.scale_log2;
        }
        tc_fence_before();
        mbar_arrive(s_empty + sbuf);
        sbuf ^= 1;
        if (pred || (P.fingerprint && space)) mbar_wait(kv_full + stage, kv_phase);
        if (pred) {
          // key coordinates for this tile
          int sink = 0, local = 0;
          const uint32_t* sl_bits = nullptr;
          const uint32_t* vm_bits = nullptr;
          if (!P.dense) {
            const InstParam ip = P.insts[it.inst_base + inst];
            sink = ip.sink;
            local = ip.local;
            if (ip.slash_word >= 0) sl_bits = P.bits + ip.slash_word;
            if (ip.vmask_word >= 0) vm_bits = P.bits + ip.vmask_word;
          }
          const int x = rmode ? xrank : xpos;
          const int kbase = e.krow - kv * P.S;
#pragma unroll
          for (int c = 0; c < BLK; ++c) {
            int ypos, y;
            if (space) {
              ypos = kpos_s[stage * BLK + c];
              y = rmode ? krank_s[stage * BLK + c] : ypos;
            } else {
              ypos = kbase + c;
              y = ypos;
            }
            bool ok = valid && (ypos <= xpos);
            if (role == R_A) {
              ok = ok && ((y < sink) || (x - y < local));
            } else if (role == R_NOTA) {
              ok = ok && !((y < sink) || (x - y < local));
            } else if (role == R_VSSL) {
              if (ok) {
                const int o = x - y;
                const bool in_sl = (sl_bits[o >> 5] >> (o & 31)) & 1u;
                const bool in_v = (vm_bits[y >> 5] >> (y & 31)) & 1u;
                ok = in_sl && !in_v;
              }
            }
            if (!ok) s[c] = -INFINITY;
            if (P.fingerprint && ok) {
              fp_cnt += 1;
              fp_s1 += ypos;
              fp_s2 += (long long)ypos * ypos;
            }
          }
        } else if (P.fingerprint && valid) {
          const int kbase = e.krow - kv * P.S;
          for (int c = 0; c < BLK; ++c) {
            const int ypos = space ? kpos_s[stage * BLK + c] : kbase + c;
            fp_cnt += 1;
            fp_s1 += ypos;
            fp_s2 += (long long)ypos * ypos;
          }
        }
        if (++stage == NST) {
          stage = 0;
          kv_phase ^= 1;
        }
        // ---- online softmax (log2 domain) ----
        float mt = -INFINITY;
#pragma unroll
        for (int c = 0; c < BLK; ++c) mt = fmaxf(mt, s[c]);
        float alpha = 1.f;
        bool rescale = false;
        if (mt > m_used + RESCALE_THRESH || (m_used == -INFINITY && mt > -INFINITY)) {
          alpha = (m_used == -INFINITY) ? 0.f : ex2(m_used - mt);
          rescale = (m_used != -INFINITY);
          m_used = mt;
        }
        const float mu = (m_used == -INFINITY) ? 0.f : m_used;
        float ls = 0.f;
        uint32_t pk[BLK / 2];
#pragma unroll
        for (int c = 0; c < BLK; c += 2) {
          const float p0 = ex2(s[c] - mu);
          const float p1 = ex2(s[c + 1] - mu);
          ls += p0 + p1;
          pk[c / 2] = pack_bf16(p0, p1);
        }
        l_sum = l_sum * alpha + ls;
        // P buffer and O are free once the previous P V has completed
        mbar_wait(p_empty, p_phase ^ 1);
        p_phase ^= 1;
        tc_fence_after();
        if (t > 0 && __any_sync(0xffffffffu, rescale)) {
#pragma unroll
          for (int c = 0; c < D / 32; ++c) {
            uint32_t r[32];
            tmem_ld32(tO + lane_off + c * 32, r);
            tmem_wait_ld();
#pragma unroll
            for (int j = 0; j < 32; ++j) r[j] = __float_as_uint(__uint_as_float(r[j]) * alpha);
            tmem_st32(tO + lane_off + c * 32, r);
          }
          tmem_wait_st();
        }
        // P row -> smem, K-major SW128: chunk = key/64, 16B unit u at (u ^ (row & 7))
#pragma unroll
        for (int u = 0; u < BLK / 8; ++u) {
          const int chunk = u / 8, uu = u % 8;
          const uint32_t addr = p_base + chunk * (BLK * 128) + row * 128 + ((uu ^ (row & 7)) << 4);
          st_shared_v4(addr, pk[u * 4 + 0], pk[u * 4 + 1], pk[u * 4 + 2], pk[u * 4 + 3]);
        }
        fence_proxy_async_smem();
        tc_fence_before();
        mbar_arrive(p_full);
      }
      // ---- epilogue ----
      if (it.n_tiles > 0) {
        mbar_wait(o_full, o_phase);
        o_phase ^= 1;
        tc_fence_after();
      }
      const float inv_l = l_sum > 0.f ? 1.f / l_sum : 0.f;
      const float lse_v = l_sum > 0.f ? (m_used + __log2f(l_sum)) * 0.6931471805599453f : -INFINITY;
      if (P.fingerprint) {
        if (it.n_tiles > 0) {
          tc_fence_before();
          mbar_arrive(o_empty);
        }
        if (write) {
          long long* f = reinterpret_cast<long long*>(P.fp_out) + 3ll * ((long long)it.head * P.S + xpos);
          atomicAdd(reinterpret_cast<unsigned long long*>(f + 0), (unsigned long long)fp_cnt);
          atomicAdd(reinterpret_cast<unsigned long long*>(f + 1), (unsigned long long)fp_s1);
          atomicAdd(reinterpret_cast<unsigned long long*>(f + 2), (unsigned long long)fp_s2);
        }
        continue;
      }
      if (it.out_mode == OUT_FINAL) {
        __nv_bfloat16* orow = reinterpret_cast<__nv_bfloat16*>(P.o) + ((size_t)it.head * P.S + xpos) * D;
#pragma unroll
        for (int c = 0; c < D / 32; ++c) {
          uint32_t r[32];
          if (it.n_tiles > 0) {
            tmem_ld32(tO + lane_off + c * 32, r);
            tmem_wait_ld();
          } else {
#pragma unroll
            for (int j = 0; j < 32; ++j) r[j] = 0u;
          }
          if (write) {
            uint4* dst = reinterpret_cast<uint4*>(orow + c * 32);
#pragma unroll
            for (int j = 0; j < 4; ++j) {
              uint4 w;
              w.x = pack_bf16(__uint_as_float(r[8 * j + 0]) * inv_l, __uint_as_float(r[8 * j + 1]) * inv_l);
              w.y = pack_bf16(__uint_as_float(r[8 * j + 2]) * inv_l, __uint_as_float(r[8 * j + 3]) * inv_l);
              w.z = pack_bf16(__uint_as_float(r[8 * j + 4]) * inv_l, __uint_as_float(r[8 * j + 5]) * inv_l);
              w.w = pack_bf16(__uint_as_float(r[8 * j + 6]) * inv_l, __uint_as_float(r[8 * j + 7]) * inv_l);
              dst[j] = w;
            }
          }
        }
        if (write && P.lse) P.lse[(size_t)it.head * P.S + xpos] = lse_v;
      } else {
        float* prow = P.part_o + (size_t)(it.out_row0 + row) * D;
#pragma unroll
        for (int c = 0; c < D / 32; ++c) {
          uint32_t r[32];
          if (it.n_tiles > 0) {
            tmem_ld32(tO + lane_off + c * 32, r);
            tmem_wait_ld();
          } else {
#pragma unroll
            for (int j = 0; j < 32; ++j) r[j] = 0u;
          }
          float4* dst = reinterpret_cast<float4*>(prow + c * 32);
#pragma unroll
          for (int j = 0; j < 8; ++j)
            dst[j] = make_float4(__uint_as_float(r[4 * j]) * inv_l, __uint_as_float(r[4 * j + 1]) * inv_l,
                                 __uint_as_float(r[4 * j + 2]) * inv_l, __uint_as_float(r[4 * j + 3]) * inv_l);
        }
        P.part_lse[it.out_row0 + row] = valid ? lse_v : -INFINITY;
      }
      if (it.n_tiles > 0) {
        tc_fence_before();
        mbar_arrive(o_empty);
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 2) {
    tc_fence_after();
    tmem_dealloc<512>(tmem);
  }
}

// ------------------------------------------------------------------ host side
typedef CUresult (*PFN_encodeTiled)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                    const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                    CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

static PFN_encodeTiled get_encode() {
  static PFN_encodeTiled fn = nullptr;
  if (!fn) {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_encodeTiled>(p);
  }
  return fn;
}

// rows x D bf16 row-major tensor; box = 128 rows x 64 columns, 128B swizzle
int make_tmap_rows(CUtensorMap* m, const void* base, long long rows, int D) {
  PFN_encodeTiled enc = get_encode();
  if (!enc) return -1;
  if (rows <= 0) rows = 1;
  cuuint64_t dims[2] = {(cuuint64_t)D, (cuuint64_t)rows};
  cuuint64_t strides[1] = {(cuuint64_t)D * 2};
  cuuint32_t box[2] = {64, (cuuint32_t)BLK};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = enc(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(base), dims, strides, box, estr,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS ? 0 : (int)r;
}

static int g_num_sms = 0;

cudaError_t launch_attn(const AttnLaunch& L, const AttnParams& P, int n_items_hint, cudaStream_t stream,
                        int* tmap_err) {
  CUtensorMap m[6];
  int e = 0;
  e |= make_tmap_rows(&m[0], L.q, L.q_rows, P.D);
  e |= make_tmap_rows(&m[1], L.qg ? L.qg : L.q, L.qg ? L.qg_rows : L.q_rows, P.D);
  e |= make_tmap_rows(&m[2], L.k, L.kv_rows, P.D);
  e |= make_tmap_rows(&m[3], L.kg ? L.kg : L.k, L.kg ? L.kvg_rows : L.kv_rows, P.D);
  e |= make_tmap_rows(&m[4], L.v, L.kv_rows, P.D);
  e |= make_tmap_rows(&m[5], L.vg ? L.vg : L.v, L.vg ? L.kvg_rows : L.kv_rows, P.D);
  if (tmap_err) *tmap_err = e;
  if (e) return cudaErrorInvalidValue;
  if (!g_num_sms) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&g_num_sms, cudaDevAttrMultiProcessorCount, dev);
  }
  int grid = g_num_sms;
  if (n_items_hint > 0 && n_items_hint < grid) grid = n_items_hint;
  if (grid <= 0) return cudaSuccess;
  if (P.D == 128) {
    auto kfn = attn_kernel<128>;
    cudaFuncSetAttribute(kfn, cudaFuncAttributeMaxDynamicSharedMemorySize, Smem<128>::ALLOC);
    kfn<<<grid, NTHREADS, Smem<128>::ALLOC, stream>>>(m[0], m[1], m[2], m[3], m[4], m[5], P);
  } else {
    auto kfn = attn_kernel<64>;
    cudaFuncSetAttribute(kfn, cudaFuncAttributeMaxDynamicSharedMemorySize, Smem<64>::ALLOC);
    kfn<<<grid, NTHREADS, Smem<64>::ALLOC, stream>>>(m[0], m[1], m[2], m[3], m[4], m[5], P);
  }
  return cudaGetLastError();
}

}  // namespace mmi
