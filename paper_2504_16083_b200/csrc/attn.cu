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
//   warp 0     TMA Q loader (one Q tile per work item)
//   warp 1     MMA issuer: S = Q K^T into TMEM (double buffered), O += P V; TMEM alloc
//   warp 2     TMA K loader (K ring, + key positions / ranks for PRED tiles)
//   warp 3     TMA V loader (V ring, decoupled from K so K runs ahead)
//   warps 4-7  softmax / correction / epilogue, thread t owns query row t
//              (TMEM lane t): tcgen05.ld S, predicate mask, exp2, P (bf16) -> TMEM
//              aliasing S (A operand of the P V tcgen05.mma), lazy O rescale in TMEM.
// Work items are fetched dynamically (atomic counter) by warp 0 and broadcast to
// the other roles through a 4-deep shared-memory ring.
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <climits>
#include <cstdint>
#include <cstdio>

#include "internal.h"
#include "ptx.cuh"

namespace mmi {

constexpr float RESCALE_THRESH = 8.0f;  // lazy rescale: P <= 2^8 (log2 domain)

// Work items cover two 128-row query blocks (halves A and B); each half has its
// own softmax warpgroup, TMEM S/P buffer (128 columns) and O accumulator (128
// columns): 512 columns total.  K/V tiles are shared by both halves.
template <int D>
struct Cfg {
  static constexpr int KST = (D == 128) ? 2 : 3;  // K ring stages
  static constexpr int VST = (D == 128) ? 2 : 3;  // V ring stages
};
constexpr int SCHED_RING = 4;
constexpr int NWARP_CTRL = 4;                     // scheduler+Q, MMA, K loader, V loader
constexpr int NTHREADS = 32 * (NWARP_CTRL + 8);  // + two softmax warpgroups
constexpr int LAUNCH_REGS = 168;                  // ptxas allocation at __launch_bounds__(384, 1)
#ifndef MMI_CTRL_REGS
#define MMI_CTRL_REGS 56
#define MMI_SOFT_REGS 224
#endif
constexpr int CTRL_REGS = MMI_CTRL_REGS;                    // setmaxnreg budgets: .inc only draws on what .dec released
constexpr int SOFT_REGS = MMI_SOFT_REGS;                    // inside the CTA's launch allocation (384*168), else it blocks forever
static_assert(128 * CTRL_REGS + 256 * SOFT_REGS <= NTHREADS * LAUNCH_REGS, "setmaxnreg budget exceeds launch allocation");

template <int D>
struct Smem {
  static constexpr int KST = Cfg<D>::KST, VST = Cfg<D>::VST;
  static constexpr int Q_BYTES = BLK * D * 2;  // one 128-row half
  static constexpr int KV_BYTES = BLK * D * 2;
  static constexpr int OFF_Q = 0;
  static constexpr int OFF_K = OFF_Q + 2 * Q_BYTES;
  static constexpr int OFF_V = OFF_K + KST * KV_BYTES;
  static constexpr int OFF_KPOS = OFF_V + VST * KV_BYTES;
  static constexpr int OFF_KRANK = OFF_KPOS + KST * BLK * 4;
  static constexpr int OFF_SCHED = OFF_KRANK + KST * BLK * 4;
  static constexpr int OFF_BAR = OFF_SCHED + 64;
  // q_full q_empty k_full[KST] k_empty[KST] v_full[VST] v_empty[VST] s_full[2] p_full[2] o_full[2] o_empty[2]
  // sched_full[R] sched_empty[R]
  static constexpr int N_BAR = 2 + 2 * KST + 2 * VST + 8 + 2 * SCHED_RING;
  static constexpr int OFF_TMEM = OFF_BAR + N_BAR * 8;
  static constexpr int TOTAL = OFF_TMEM + 16;
  static constexpr int ALLOC = TOTAL + 1024;  // alignment slack
};

struct ItemView {
  int head, q_row0, seg_off, n_segs, n_tiles, q_gathered, out_mode, out_row0, inst_base, skip_s, skip_p, skip_rank,
      row_mod, rb, has_b;
};

__device__ __forceinline__ ItemView load_item(const AttnParams& P, int idx) {
  ItemView v;
  if (P.dense) {
    const int nb = (P.S + BLK - 1) / BLK;
    const int npair = (nb + 1) / 2;
    const int pk = npair - 1 - idx / P.H;  // longest rows first (LPT)
    v.head = idx % P.H;
    v.q_row0 = v.head * P.S + 2 * pk * BLK;
    v.has_b = (2 * pk + 1 < nb) ? 1 : 0;
    v.rb = 2 * pk + v.has_b;  // last row block of the pair
    v.seg_off = 0;
    v.n_segs = 1;
    v.n_tiles = v.rb + 1;
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
  v.has_b = w.has_b;
  v.rb = 0;
  return v;
}

// sets bits [lo, hi] (clipped to [0, 127]) of a 128-bit mask
__device__ __forceinline__ void range_mask(uint32_t (&mw)[4], int lo, int hi) {
  lo = max(lo, 0);
  hi = min(hi, BLK - 1);
  if (hi < lo) return;
#pragma unroll
  for (int w = 0; w < 4; ++w) {
    const int a = max(lo - 32 * w, 0), b = min(hi - 32 * w, 31);
    if (b >= a) {
      const uint32_t hiMask = (b == 31) ? 0xffffffffu : ((1u << (b + 1)) - 1u);
      const uint32_t loMask = (1u << a) - 1u;
      mw[w] |= hiMask & ~loMask;
    }
  }
}

// number of entries <= v in an ascending int array of 128 (shared memory)
__device__ __forceinline__ int count_le(const int* a, int v) {
  int i = 0;
#pragma unroll
  for (int step = 64; step > 0; step >>= 1)
    if (a[i + step - 1] <= v) i += step;
  return i + ((i == BLK - 1 && a[BLK - 1] <= v) ? 1 : 0);
}

// 128 bits of a bitmap starting at bit `lo` (bits below 0 read as 0): out[w] bit i = bit(lo + 32w + i)
__device__ __forceinline__ void bit_window(const uint32_t* bits, int lo, uint32_t (&out)[4]) {
  const int wb = (lo >= 0) ? (lo >> 5) : -((-lo + 31) >> 5);
  const int sh = lo - wb * 32;
  uint32_t w[5];
#pragma unroll
  for (int i = 0; i < 5; ++i) w[i] = (wb + i >= 0) ? __ldg(bits + wb + i) : 0u;
#pragma unroll
  for (int i = 0; i < 4; ++i) out[i] = __funnelshift_r(w[i], w[i + 1], sh);
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
      cur.pred_tail = it.has_b ? 2 : 1;  // diagonal tiles of both halves
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
  constexpr int KST = L::KST, VST = L::VST;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + L::OFF_BAR);
  uint64_t* q_full = bars + 0;
  uint64_t* q_empty = bars + 1;
  uint64_t* k_full = bars + 2;
  uint64_t* k_empty = k_full + KST;
  uint64_t* v_full = k_empty + KST;
  uint64_t* v_empty = v_full + VST;
  uint64_t* s_full = v_empty + VST;  // [2] per half: S written by the MMA
  uint64_t* p_full = s_full + 2;     // [2] per half: P (bf16, aliasing S in TMEM) written by the softmax
  uint64_t* o_full = p_full + 2;     // [2] per half
  uint64_t* o_empty = o_full + 2;    // [2] per half
  uint64_t* sched_full = o_empty + 2;
  uint64_t* sched_empty = sched_full + SCHED_RING;
  uint32_t* tmem_holder = reinterpret_cast<uint32_t*>(smem + L::OFF_TMEM);
  int32_t* kpos_s = reinterpret_cast<int32_t*>(smem + L::OFF_KPOS);
  int32_t* krank_s = reinterpret_cast<int32_t*>(smem + L::OFF_KRANK);
  volatile int32_t* sched_ring = reinterpret_cast<volatile int32_t*>(smem + L::OFF_SCHED);

  const int warp = threadIdx.x / 32;
  const int lane = threadIdx.x % 32;

  if (threadIdx.x == 0) {
    mbar_init(q_full, 1);
    mbar_init(q_empty, 1);
    for (int i = 0; i < KST; ++i) {
      mbar_init(k_full + i, 1);
      mbar_init(k_empty + i, 1 + 8);  // last S-MMA commit + one arrival per softmax warp (key coords consumed)
    }
    for (int i = 0; i < VST; ++i) {
      mbar_init(v_full + i, 1);
      mbar_init(v_empty + i, 1);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(s_full + i, 1);
      mbar_init(p_full + i, 128);
      mbar_init(o_full + i, 1);
      mbar_init(o_empty + i, 128);
    }
    for (int i = 0; i < SCHED_RING; ++i) {
      mbar_init(sched_full + i, 1);
      mbar_init(sched_empty + i, 3 + 8);  // K loader, V loader, MMA, 8 softmax warps
    }
    fence_barrier_init();
  }
  if (warp == 1) tmem_alloc<512>(tmem_holder);
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
  // TMEM columns: S/P of half h at 128 h, O of half h at 256 + 128 h
  const int n_items = P.dense ? P.H * ((((P.S + BLK - 1) / BLK) + 1) / 2) : P.n_items;
  auto fetch = [&](int i) -> int {
    const int slot = i % SCHED_RING;
    mbar_wait(sched_full + slot, (i / SCHED_RING) & 1);
    return sched_ring[slot];
  };

  if (warp < NWARP_CTRL) {
    asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;\n" ::"n"(CTRL_REGS));
    if (warp == 0) {
      // ======================= scheduler + Q loader =======================
      if (elect_one()) {
        uint32_t q_phase = 0;
        for (int i = 0;; ++i) {
          const int slot = i % SCHED_RING;
          mbar_wait(sched_empty + slot, ((i / SCHED_RING) & 1) ^ 1);
          int idx = (i == 0) ? (int)blockIdx.x : (int)gridDim.x + (int)atomicAdd(P.sched, 1u);
          if (idx >= n_items) idx = -1;
          sched_ring[slot] = idx;
          mbar_arrive(sched_full + slot);
          if (idx < 0) break;
          const ItemView it = load_item(P, idx);
          if (it.n_tiles <= 0) continue;
          if (P.dbg) P.dbg[idx * 8 + 0] = gtimer();
          mbar_wait(q_empty, q_phase ^ 1);
          q_phase ^= 1;
          mbar_arrive_expect_tx(q_full, (it.has_b ? 2 : 1) * L::Q_BYTES);
          const CUtensorMap* tq = it.q_gathered ? &tmQg : &tmQo;
          for (int hf = 0; hf < (it.has_b ? 2 : 1); ++hf) {
#pragma unroll
            for (int c = 0; c < D / 64; ++c)
              tma_load_2d(smem + L::OFF_Q + hf * L::Q_BYTES + c * (BLK * 128), tq, q_full, c * 64,
                          it.q_row0 + hf * BLK);
          }
        }
      }
    } else if (warp == 2 || warp == 3) {
      // ======================= K loader (warp 2) / V loader (warp 3) =======================
      const bool is_k = (warp == 2);
      if (elect_one()) {
        int stage = 0;
        uint32_t phase = 0;
        const int NS = is_k ? KST : VST;
        uint64_t* full = is_k ? k_full : v_full;
        uint64_t* empty = is_k ? k_empty : v_empty;
        for (int i = 0;; ++i) {
          const int idx = fetch(i);
          mbar_arrive(sched_empty + i % SCHED_RING);
          if (idx < 0) break;
          const ItemView it = load_item(P, idx);
          if (it.n_tiles <= 0) continue;
          SegIter si;
          si.init(P, it);
          for (int t = 0; t < it.n_tiles; ++t) {
            const TileInfo e = si.next(P, it);
            mbar_wait(empty + stage, phase ^ 1);
            uint32_t bytes = L::KV_BYTES;
            const bool cp_pos = is_k && (e.pred || P.fingerprint) && e.space;
            const bool cp_rank = is_k && e.pred && e.space && e.rmode;
            if (cp_pos) bytes += BLK * 4;
            if (cp_rank) bytes += BLK * 4;
            mbar_arrive_expect_tx(full + stage, bytes);
            const CUtensorMap* tm = is_k ? (e.space ? &tmKg : &tmKo) : (e.space ? &tmVg : &tmVo);
            uint8_t* dst = smem + (is_k ? L::OFF_K : L::OFF_V) + stage * L::KV_BYTES;
#pragma unroll
            for (int c = 0; c < D / 64; ++c) tma_load_2d(dst + c * (BLK * 128), tm, full + stage, c * 64, e.krow);
            if (cp_pos) bulk_load(kpos_s + stage * BLK, P.kg_pos + e.krow, BLK * 4, full + stage);
            if (cp_rank) bulk_load(krank_s + stage * BLK, P.kg_rank + e.krow, BLK * 4, full + stage);
            if (++stage == NS) {
              stage = 0;
              phase ^= 1;
            }
          }
        }
      }
    } else {
      // ======================= MMA issuer (one thread) =======================
      if (elect_one()) {
        constexpr uint32_t IDESC_S = idesc_bf16(128, 128, 0);
        constexpr uint32_t IDESC_O = idesc_bf16(128, D, 1);
        const uint32_t q_base = smem_u32(smem + L::OFF_Q);
        const uint32_t k_base = smem_u32(smem + L::OFF_K);
        const uint32_t v_base = smem_u32(smem + L::OFF_V);
        int ks = 0, vs = 0;
        uint32_t k_phase = 0, v_phase = 0, q_phase = 0;
        uint32_t p_phase[2] = {0, 0}, o_phase[2] = {0, 0};
        for (int i = 0;; ++i) {
          const int idx = fetch(i);
          mbar_arrive(sched_empty + i % SCHED_RING);
          if (idx < 0) break;
          const ItemView it = load_item(P, idx);
          const int n = it.n_tiles;
          if (n <= 0) continue;
          const int nh = it.has_b ? 2 : 1;
          mbar_wait(q_full, q_phase);
          q_phase ^= 1;
          tc_fence_after();
          // S_h(t) = Q_h K_t^T into the half's S buffer (its previous P was consumed by
          // a P V issued earlier; tcgen05.mma executes in issue order)
          auto issue_s = [&](int hf, int t) {
#pragma unroll
            for (int k = 0; k < D / 16; ++k) {
              const uint32_t off = (k / 4) * (BLK * 128) + (k % 4) * 32;
              const uint64_t ad = smem_desc(q_base + hf * L::Q_BYTES + off, 16, 1024, 2);
              const uint64_t bd = smem_desc(k_base + ks * L::KV_BYTES + off, 16, 1024, 2);
              umma_ss(tmem + 128 * hf, ad, bd, IDESC_S, k > 0 ? 1u : 0u);
            }
            umma_commit(s_full + hf);
            if (hf == nh - 1) {
              umma_commit(k_empty + ks);  // K(t) consumed by every half
              if (t == n - 1) umma_commit(q_empty);
            }
          };
          // O_h += P_h(t) V_t, P read from TMEM (A operand)
          auto issue_pv = [&](int hf, int t) {
            mbar_wait(p_full + hf, p_phase[hf]);
            p_phase[hf] ^= 1;
            if (t == 0) mbar_wait(o_empty + hf, o_phase[hf] ^ 1);  // previous item's epilogue read O_h
            tc_fence_after();
#pragma unroll
            for (int k = 0; k < BLK / 16; ++k) {
              const uint64_t bd = smem_desc(v_base + vs * L::KV_BYTES + k * 2048, BLK * 128, 1024, 2);
              umma_ts(tmem + 256 + 128 * hf, tmem + 128 * hf + k * 8, bd, IDESC_O, (t > 0 || k > 0) ? 1u : 0u);
            }
            if (t == n - 1) {
              umma_commit(o_full + hf);
              o_phase[hf] ^= 1;
            }
          };
          // prologue: S of tile 0 for every half
          mbar_wait(k_full + ks, k_phase);
          tc_fence_after();
          for (int hf = 0; hf < nh; ++hf) issue_s(hf, 0);
          if (++ks == KST) {
            ks = 0;
            k_phase ^= 1;
          }
          for (int t = 0; t < n; ++t) {
            mbar_wait(v_full + vs, v_phase);
            const bool more = (t + 1 < n);
            // half A: P V(t), then S(t+1) while half B's softmax still runs
            issue_pv(0, t);
            if (more) {
              mbar_wait(k_full + ks, k_phase);
              tc_fence_after();
              issue_s(0, t + 1);
            }
            if (nh == 2) {
              issue_pv(1, t);
              if (more) issue_s(1, t + 1);
            }
            umma_commit(v_empty + vs);
            if (++vs == VST) {
              vs = 0;
              v_phase ^= 1;
            }
            if (more && ++ks == KST) {
              ks = 0;
              k_phase ^= 1;
            }
          }
        }
      }
    }
  } else {
    asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;\n" ::"n"(SOFT_REGS));
    // ======================= softmax / correction / epilogue (one warpgroup per half) =======================
    const int hf = (warp - NWARP_CTRL) / 4;          // half of the item this warpgroup owns
    const int row = (threadIdx.x - 32 * NWARP_CTRL) % 128;  // TMEM lane == row of the half
    const uint32_t lane_off = (uint32_t)((warp % 4) * 32) << 16;
    const uint32_t tS = tmem + 128 * hf + lane_off;
    const uint32_t tO = tmem + 256 + 128 * hf + lane_off;
    int stage = 0;  // K ring stage (key coordinates)
    uint32_t kv_phase = 0, s_phase = 0, o_phase = 0;
    const int G = P.H / P.Hkv;
    for (int i = 0;; ++i) {
      const int idx = fetch(i);
      __syncwarp();
      if (lane == 0) mbar_arrive(sched_empty + i % SCHED_RING);
      if (idx < 0) break;
      const ItemView it = load_item(P, idx);
      if (it.n_tiles <= 0) continue;  // empty slot: nothing to compute or write
      if (hf == 1 && !it.has_b) {
        // absent half: only release the key-coordinate stages
        for (int t = 0; t < it.n_tiles; ++t) {
          mbar_wait(k_full + stage, kv_phase);
          __syncwarp();
          if (lane == 0) mbar_arrive(k_empty + stage);
          if (++stage == KST) {
            stage = 0;
            kv_phase ^= 1;
          }
        }
        continue;
      }
      if (P.dbg && row == 0 && hf == 0) P.dbg[idx * 8 + 3] = gtimer();
      // row identity
      const int qrow = it.q_row0 + hf * BLK + row;
      int xpos, xrank;
      if (it.q_gathered) {
        xpos = P.qg_pos[qrow];
        xrank = P.qg_rank[qrow];
      } else {
        xpos = qrow - it.head * P.S;
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
        mbar_wait(s_full + hf, s_phase);
        s_phase ^= 1;
        tc_fence_after();
        float s[BLK];
#pragma unroll
        for (int c = 0; c < BLK / 32; ++c) {
          uint32_t r[32];
          tmem_ld32(tS + c * 32, r);
          tmem_wait_ld();
#pragma unroll
          for (int j = 0; j < 32; ++j) s[c * 32 + j] = __uint_as_float(r[j]);  // raw scores
        }
        if (pred || (P.fingerprint && space)) mbar_wait(k_full + stage, kv_phase);
        if (pred || P.fingerprint) {
          // admitted-key bit mask of this tile (bit c <-> key c), then one unrolled select
          uint32_t mw[4] = {0u, 0u, 0u, 0u};
          if (valid) {
            const int kbase = e.krow - kv * P.S;
            if (!pred) {
              range_mask(mw, 0, BLK - 1);
            } else {
              int sink = 0, local = 0;
              const uint32_t* sl_bits = nullptr;
              const uint32_t* vm_bits = nullptr;
              if (!P.dense && role != R_TRUE) {
                const InstParam ip = P.insts[it.inst_base + inst];
                sink = ip.sink;
                local = ip.local;
                if (ip.slash_word >= 0) sl_bits = P.bits + ip.slash_word;
                if (ip.vmask_word >= 0) vm_bits = P.bits + ip.vmask_word;
              }
              const int x = rmode ? xrank : xpos;
              // Keys of every view are ascending inside a tile, so each role is at most two
              // index ranges: [0, n_causal) intersected with the pattern's coordinate ranges.
              int n_causal, n_sink, n_lt_local, ybase;
              if (!space) {
                n_causal = min(max(xpos - kbase + 1, 0), BLK);
                n_sink = min(max(sink - kbase, 0), BLK);
                n_lt_local = min(max(x - local - kbase + 1, 0), BLK);  // keys with y <= x - local
                ybase = kbase;
              } else {
                const int* kp = kpos_s + stage * BLK;
                const int* yc = rmode ? (krank_s + stage * BLK) : kp;
                n_causal = count_le(kp, xpos);
                n_sink = (role == R_A || role == R_NOTA) ? count_le(yc, sink - 1) : 0;
                n_lt_local = (role == R_A || role == R_NOTA) ? count_le(yc, x - local) : 0;
                ybase = yc[0];
              }
              if (role == R_TRUE) {
                range_mask(mw, 0, n_causal - 1);
              } else if (role == R_A) {
                range_mask(mw, 0, min(n_sink, n_causal) - 1);
                range_mask(mw, n_lt_local, n_causal - 1);
              } else if (role == R_NOTA) {
                range_mask(mw, n_sink, min(n_lt_local, n_causal) - 1);
              } else {
                // vertical-slash: coordinates contiguous in the tile (original K, or a modality's
                // rank-ordered keys); slash bits of offsets x - ybase - c, bit-reversed window
                range_mask(mw, 0, n_causal - 1);
                uint32_t ws[4], wv[4];
                bit_window(sl_bits, x - ybase - (BLK - 1), ws);
                bit_window(vm_bits, ybase, wv);
#pragma unroll
                for (int w = 0; w < 4; ++w) mw[w] &= __brev(ws[3 - w]) & ~wv[w];
              }
            }
            if (P.fingerprint) {
#pragma unroll
              for (int w = 0; w < 4; ++w) {
                uint32_t bitsw = mw[w];
                while (bitsw) {
                  const int c = w * 32 + __ffs(bitsw) - 1;
                  bitsw &= bitsw - 1;
                  const long long ypos = space ? kpos_s[stage * BLK + c] : kbase + c;
                  fp_cnt += 1;
                  fp_s1 += ypos;
                  fp_s2 += ypos * ypos;
                }
              }
            }
          }
#pragma unroll
          for (int c = 0; c < BLK; ++c)
            if (!((mw[c >> 5] >> (c & 31)) & 1u)) s[c] = -INFINITY;
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(k_empty + stage);  // key coordinates of this stage consumed
        if (++stage == KST) {
          stage = 0;
          kv_phase ^= 1;
        }
        // ---- online softmax (log2 domain), lazy rescale ----
        float mt = -INFINITY;
#pragma unroll
        for (int c = 0; c < BLK; ++c) mt = fmaxf(mt, s[c]);
        if (mt > -INFINITY) mt *= P.scale_log2;  // tau * log2(e) > 0 commutes with max
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
          const float p0 = ex2(fmaf(s[c], P.scale_log2, -mu));
          const float p1 = ex2(fmaf(s[c + 1], P.scale_log2, -mu));
          ls += p0 + p1;
          pk[c / 2] = pack_bf16(p0, p1);
        }
        l_sum = l_sum * alpha + ls;
        // O correction only when the running max moved; O_h is quiescent: P V_h(t-1) was
        // issued before S_h(t), which has completed.
        if (t > 0 && __any_sync(0xffffffffu, rescale)) {
#pragma unroll
          for (int c = 0; c < D / 32; ++c) {
            uint32_t r[32];
            tmem_ld32(tO + c * 32, r);
            tmem_wait_ld();
#pragma unroll
            for (int j = 0; j < 32; ++j) r[j] = __float_as_uint(__uint_as_float(r[j]) * alpha);
            tmem_st32(tO + c * 32, r);
          }
        }
        // P (bf16 pairs) -> TMEM columns [0, 64) of this half's S buffer
        tmem_st32(tS, *reinterpret_cast<uint32_t(*)[32]>(&pk[0]));
        tmem_st32(tS + 32, *reinterpret_cast<uint32_t(*)[32]>(&pk[32]));
        tmem_wait_st();
        tc_fence_before();
        mbar_arrive(p_full + hf);
      }
      // ---- epilogue ----
      mbar_wait(o_full + hf, o_phase);
      o_phase ^= 1;
      tc_fence_after();
      const float inv_l = l_sum > 0.f ? 1.f / l_sum : 0.f;
      const float lse_v = l_sum > 0.f ? (m_used + __log2f(l_sum)) * 0.6931471805599453f : -INFINITY;
      if (P.fingerprint) {
        tc_fence_before();
        mbar_arrive(o_empty + hf);
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
          tmem_ld32(tO + c * 32, r);
          tmem_wait_ld();
          if (c == D / 32 - 1) {
            tc_fence_before();
            mbar_arrive(o_empty + hf);  // O in registers: the next item's first P V may start
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
        float* prow = P.part_o + (size_t)(it.out_row0 + hf * BLK + row) * D;
#pragma unroll
        for (int c = 0; c < D / 32; ++c) {
          uint32_t r[32];
          tmem_ld32(tO + c * 32, r);
          tmem_wait_ld();
          if (c == D / 32 - 1) {
            tc_fence_before();
            mbar_arrive(o_empty + hf);
          }
          float4* dst = reinterpret_cast<float4*>(prow + c * 32);
#pragma unroll
          for (int j = 0; j < 8; ++j)
            dst[j] = make_float4(__uint_as_float(r[4 * j]) * inv_l, __uint_as_float(r[4 * j + 1]) * inv_l,
                                 __uint_as_float(r[4 * j + 2]) * inv_l, __uint_as_float(r[4 * j + 3]) * inv_l);
        }
        P.part_lse[it.out_row0 + hf * BLK + row] = valid ? lse_v : -INFINITY;
      }
      if (P.dbg && row == 0 && hf == 0) P.dbg[idx * 8 + 6] = gtimer();
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
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
// work-item counters for launches without a workspace (dense comparator); rotating slots
__device__ unsigned int g_sched_counters[64];
static unsigned g_sched_slot = 0;

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
  if (n_items_hint > 0 && (n_items_hint + 1) / 2 < grid) grid = (n_items_hint + 1) / 2;
  if (grid <= 0) return cudaSuccess;
  AttnParams Pl = P;
  if (!Pl.sched) {
    unsigned int* base = nullptr;
    cudaGetSymbolAddress(reinterpret_cast<void**>(&base), g_sched_counters);
    Pl.sched = base + (g_sched_slot++ % 64);
  }
  cudaMemsetAsync(Pl.sched, 0, sizeof(unsigned int), stream);
  if (P.D == 128) {
    auto kfn = attn_kernel<128>;
    cudaFuncSetAttribute(kfn, cudaFuncAttributeMaxDynamicSharedMemorySize, Smem<128>::ALLOC);
    kfn<<<grid, NTHREADS, Smem<128>::ALLOC, stream>>>(m[0], m[1], m[2], m[3], m[4], m[5], Pl);
  } else {
    auto kfn = attn_kernel<64>;
    cudaFuncSetAttribute(kfn, cudaFuncAttributeMaxDynamicSharedMemorySize, Smem<64>::ALLOC);
    kfn<<<grid, NTHREADS, Smem<64>::ALLOC, stream>>>(m[0], m[1], m[2], m[3], m[4], m[5], Pl);
  }
  return cudaGetLastError();
}

}  // namespace mmi
