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
// Work item = two 128-row query blocks (halves A and B) sharing one list of key-tile segments
// with per-half DEAD / PRED / FULL tile states.  One persistent CTA per SM; items are fetched
// dynamically from the workspace counter (locality / longest-first order) and broadcast to the
// roles through a 4-deep shared-memory ring.  Warp roles:
//   warp 0      scheduler + Q loader (permuted Q rows gathered with TMA tile::gather4)
//   warp 1      MMA issuer (one elected thread): per key tile P_A(t,0)V, P_B(t,0)V, P_A(t,1)V,
//               S_A(t+1), P_B(t,1)V, S_B(t+1) (S = one M128 N128 group per half); TMEM alloc
//   warp 2      K TMA ring (+ key positions / ranks of gathered tiles that are masked)
//   warp 3      V TMA ring (decoupled from K so K runs ahead)
//   warps 4-11  softmax / correction / epilogue, one warpgroup per half; thread t owns query row
//               t (TMEM lane t): tcgen05.ld S, predicate mask, exp2, P (bf16) -> TMEM aliasing S
//               (A operand of the P V tcgen05.mma), lazy O rescale, O -> bf16 / fp16 stores.
// Measured alternatives and the per-event timeline: DESIGN.md 6.1-6.2, profiles/r2_ab_attention.md.
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <climits>
#include <cstdint>
#include <cstdio>

#include "internal.h"
#include "ptx.cuh"

namespace mmi {

#ifndef MMI_RESCALE_THRESH
#define MMI_RESCALE_THRESH 8.0f
#endif
constexpr float RESCALE_THRESH = MMI_RESCALE_THRESH;  // lazy rescale: P <= 2^8 (log2 domain)
// column pairs (bit i of each group of 8 pairs) whose exp2 runs as a polynomial on the FMA pipe
// instead of MUFU.EX2 (MUFU is 4 lanes/clk per SM sub-partition).  Same-box A/B on the final
// pipeline: 2/8 -> 1/8 -> 0/8 emulated = 3.706 -> 3.670 -> 3.663 ms (128K), 193.6 -> 171.2 ->
// 169.7 ms (256K), 67.4 -> 66.0 -> 65.0 ms (1M): the softmax is issue-bound, not MUFU-bound, so
// every exp2 stays on MUFU (the polynomial remains for experiments)
#ifndef MMI_EMU_MASK
#define MMI_EMU_MASK 0x00u
#endif
constexpr uint32_t EMU_MASK = MMI_EMU_MASK;

// Work items cover two 128-row query blocks (halves A and B); each half has its
// own softmax warpgroup, TMEM S/P buffer (128 columns = two 64-key sub-tile
// slots) and O accumulator (128 columns): 512 columns total.  K/V tiles are
// shared by both halves.
template <int D>
struct Cfg {
  static constexpr int KST = (D == 128) ? 2 : 3;  // K ring stages
  static constexpr int VST = (D == 128) ? 2 : 3;  // V ring stages
};
constexpr int SCHED_RING = 4;
constexpr int SCHED_ENTRY = 128;  // bytes per ring entry: item index + staged WorkItem
static_assert(16 + sizeof(WorkItem) <= SCHED_ENTRY, "WorkItem does not fit the scheduler ring entry");
constexpr int NWARP_CTRL = 4;                      // scheduler+Q, MMA, K loader, V loader
#ifndef MMI_HPW
#define MMI_HPW 1
#endif
constexpr int HPW = MMI_HPW;                       // query halves per softmax warpgroup (1 or 2)
static_assert(HPW == 1 || HPW == 2, "HPW must be 1 or 2");
constexpr int NWARP_SOFT = 8 / HPW;                // softmax warpgroups: one per half, or one for both
constexpr int NTHREADS = 32 * (NWARP_CTRL + NWARP_SOFT);
constexpr int LAUNCH_REGS = (HPW == 1) ? 168 : 255;  // ptxas allocation at __launch_bounds__(NTHREADS, 1)
#ifndef MMI_CTRL_REGS
#if MMI_HPW == 1
#define MMI_CTRL_REGS 88
#define MMI_SOFT_REGS 208
#else
#define MMI_CTRL_REGS 0  // 256 threads: every warp keeps the launch allocation
#define MMI_SOFT_REGS 0
#endif
#endif
constexpr int CTRL_REGS = MMI_CTRL_REGS;  // setmaxnreg budgets: .inc only draws on what .dec released
constexpr int SOFT_REGS = MMI_SOFT_REGS;  // inside the CTA's launch allocation, else it blocks forever
static_assert(32 * NWARP_CTRL * CTRL_REGS + 32 * NWARP_SOFT * SOFT_REGS <= NTHREADS * LAUNCH_REGS,
              "setmaxnreg budget exceeds launch allocation");
constexpr int NKP = 4;
// epilogue staging row: 64 B of output (32 16-bit columns) + 16 B pad, so that 8 consecutive rows
// written by 8 lanes (one 16 B vector each) fall in distinct bank groups
constexpr int EPI_STRIDE = 80;
static_assert((32 * EPI_STRIDE) % 512 == 0, "staging buffers must stay 512 B aligned");  // key-coordinate ring (positions / ranks of gathered key tiles that need them)

// MMI_PROF builds (scratch/variants.sh only) accumulate per-phase SM clocks into g_prof
#ifdef MMI_PROF
__device__ unsigned long long g_prof[32];
#define PROF_DECL(n) long long prof_##n = 0
#define PROF_T() clock64()
#define PROF_ADD(n, t0) prof_##n += clock64() - (t0)
#define PROF_FLUSH(i, n) atomicAdd(&g_prof[i], (unsigned long long)prof_##n)
#else
#define PROF_DECL(n)
#define PROF_T() 0ll
#define PROF_ADD(n, t0)
#define PROF_FLUSH(i, n)
#endif
// MMI_TRACE builds (scratch only): per-event SM clock stamps of CTA 0 -- region 0 the MMA issuer,
// 1 / 2 lane 0 of the first softmax warp of half A / B; event = (clock - t0) << 8 | code << 4 | arg
#ifdef MMI_TRACE
constexpr int TRACE_N = 16384;
__device__ unsigned long long g_trace[3][TRACE_N];
__device__ int g_trace_n[3];
#define TRACE(reg, code, arg)                                                                          \
  do {                                                                                                 \
    if (blockIdx.x == 0 && tr_n < TRACE_N)                                                             \
      g_trace[reg][tr_n++] = ((unsigned long long)(clock64() - tr_t0) << 8) | ((code) << 4) | (arg);   \
  } while (0)
#else
#define TRACE(reg, code, arg)
#endif

template <int D>
struct Smem {
  static constexpr int KST = Cfg<D>::KST, VST = Cfg<D>::VST;
  static constexpr int Q_BYTES = BLK * D * 2;  // one 128-row half
  static constexpr int KV_BYTES = BLK * D * 2;
  static constexpr int OFF_Q = 0;
  static constexpr int OFF_K = OFF_Q + 2 * Q_BYTES;
  static constexpr int OFF_V = OFF_K + KST * KV_BYTES;
  static constexpr int OFF_KPOS = OFF_V + VST * KV_BYTES;
  static constexpr int OFF_KRANK = OFF_KPOS + NKP * BLK * 4;
  static constexpr int OFF_SCHED = OFF_KRANK + NKP * BLK * 4;  // [SCHED_RING] x {idx, pad, WorkItem}: 128 B
  static constexpr int OFF_RI = OFF_SCHED + SCHED_RING * SCHED_ENTRY;     // [2] x {pos[256], rank[256]} of the item's rows
  // [softmax warp] epilogue staging, 32 rows x EPI_STRIDE each (two 1 KB TMA buffers), 512 B aligned
  static constexpr int OFF_EPI = (OFF_RI + 2 * 2 * 2 * BLK * 4 + 1023) & ~1023;
  static constexpr int OFF_BAR = OFF_EPI + NWARP_SOFT * 32 * EPI_STRIDE;
  // q_full q_empty k_full[KST] k_empty[KST] v_full[VST] v_empty[VST] s_full[2][2] p_full[2][2] o_full[2]
  // o_empty[2] pv_done[2] sched_full[R] sched_empty[R] kp_full[NKP] kp_empty[NKP]
  static constexpr int N_BAR = 2 + 2 * KST + 2 * VST + 14 + 2 * SCHED_RING + 2 * NKP + 4;
  static constexpr int OFF_TMEM = OFF_BAR + N_BAR * 8;
  static constexpr int OFF_LIVE = OFF_TMEM + 16;  // [KST] live-half bits of the tile in each K stage
  static constexpr int TOTAL = OFF_LIVE + 16;
  static constexpr int ALLOC = TOTAL + 1024;  // alignment slack
};

struct ItemView {
  int head, q_row0, seg_off, n_segs, n_tiles, q_gathered, out_mode, out_row0, inst_base, skip_s, skip_p, skip_rank,
      row_mod, rb, has_b;
};

__device__ __forceinline__ ItemView load_item(const AttnParams& P, int idx, const WorkItem* staged) {
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
  const WorkItem w = *staged;  // copied to shared memory by the scheduler
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

// three count_le searches in lockstep (independent shared-memory probes overlap their latency):
// a1 = #{a <= v1}, b2 = #{b <= v2}, b3 = #{b <= v3}
__device__ __forceinline__ void count_le3(const int* a, int v1, const int* b, int v2, int v3, int& a1, int& b2,
                                          int& b3) {
  int i = 0, j = 0, k = 0;
#pragma unroll
  for (int step = 64; step > 0; step >>= 1) {
    const int x = a[i + step - 1], y = b[j + step - 1], z = b[k + step - 1];
    if (x <= v1) i += step;
    if (y <= v2) j += step;
    if (z <= v3) k += step;
  }
  a1 = i + ((i == BLK - 1 && a[BLK - 1] <= v1) ? 1 : 0);
  b2 = j + ((j == BLK - 1 && b[BLK - 1] <= v2) ? 1 : 0);
  b3 = k + ((k == BLK - 1 && b[BLK - 1] <= v3) ? 1 : 0);
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

// 128-bit admitted-key mask of a permuted NATTEN key tile for the query at raster position xpos:
// per dimension the window [start, start + k) with start = clamp(c - k/2, 0, L - k) (reading C25),
// intersected with the tile's local coordinates; key bit (lt * bh + ly) * bw + lx.
__device__ __forceinline__ void natten_mask(const AttnParams& P, int xpos, int krow, uint32_t (&mw)[4]) {
  const int HW = P.nat_H * P.nat_W;
  const int qt = xpos / HW, qy = (xpos / P.nat_W) % P.nat_H, qx = xpos % P.nat_W;
  const int st = min(max(qt - P.nat_kt / 2, 0), P.nat_T - P.nat_kt);
  const int sy = min(max(qy - P.nat_kh / 2, 0), P.nat_H - P.nat_kh);
  const int sx = min(max(qx - P.nat_kw / 2, 0), P.nat_W - P.nat_kw);
  const int tile = (krow / BLK) % P.nat_tiles;
  const int nX = (P.nat_W + P.nat_bw - 1) / P.nat_bw, nY = (P.nat_H + P.nat_bh - 1) / P.nat_bh;
  const int TX = tile % nX, TY = (tile / nX) % nY, TT = tile / (nX * nY);
  // local admitted ranges [lo, hi) per dimension
  const int t0 = max(st - TT * P.nat_bt, 0), t1 = min(st + P.nat_kt - TT * P.nat_bt, P.nat_bt);
  const int y0 = max(sy - TY * P.nat_bh, 0), y1 = min(sy + P.nat_kh - TY * P.nat_bh, P.nat_bh);
  const int x0 = max(sx - TX * P.nat_bw, 0), x1 = min(sx + P.nat_kw - TX * P.nat_bw, P.nat_bw);
  if (t1 <= t0 || y1 <= y0 || x1 <= x0) return;
  for (int lt = t0; lt < t1; ++lt)
    for (int ly = y0; ly < y1; ++ly) {
      const int b = (lt * P.nat_bh + ly) * P.nat_bw;
      range_mask(mw, b + x0, b + x1 - 1);
    }
}

struct TileInfo {
  int krow;
  uint32_t space, role, rmode, inst;
  uint32_t st0, st1;  // TileState of half A / half B
  __device__ __forceinline__ uint32_t st(int hf) const { return hf ? st1 : st0; }
  __device__ __forceinline__ bool pred_any() const { return st0 == TS_PRED || st1 == TS_PRED; }
  __device__ __forceinline__ uint32_t live() const { return (st0 != TS_DEAD ? 1u : 0u) | (st1 != TS_DEAD ? 2u : 0u); }
};

// walks the item's segments tile by tile (every warp role keeps its own cursor)
struct SegIter {
  Seg cur;
  int seg_i, t;
  __device__ __forceinline__ void init(const AttnParams& P, const ItemView& it) {
    seg_i = 0;
    t = 0;
    if (P.dense) {
      // implicit dense causal pair of row blocks (2k, 2k+1): keys 0 .. rb; half A's diagonal is tile
      // 2k (tile 2k+1 dead for it), half B's diagonal is tile 2k+1
      cur.krow0 = (it.head / (P.H / P.Hkv)) * P.S;
      cur.ntiles = it.rb + 1;
      cur.meta = seg_meta(0, R_TRUE, 0, 0);
      cur.st[0][0] = 0;
      cur.st[0][1] = 0;
      cur.st[0][2] = 1;
      cur.st[0][3] = it.has_b ? 1 : 0;
      cur.st[1][0] = it.has_b ? 0 : (int16_t)cur.ntiles;
      cur.st[1][1] = 0;
      cur.st[1][2] = it.has_b ? 1 : 0;
      cur.st[1][3] = 0;
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
    ti.st0 = seg_tile_state(cur, 0, t);
    ti.st1 = seg_tile_state(cur, 1, t);
    ++t;
    return ti;
  }
};

// Warp-collective row gather of one 128-row block into the 128B-swizzled tile layout of TMA box
// {64 columns, 128 rows}: lane l gathers rows 4l .. 4l+3 (source rows src[4l .. 4l+3]; negative =
// padding -> the out-of-range row `oob`, zero-filled) for every 64-column block.
template <int D>
__device__ __forceinline__ void gather_rows_tma(uint8_t* dst, const CUtensorMap* tm, uint64_t* bar,
                                                const int32_t* src, int oob, int lane) {
  int4 r = __ldg(reinterpret_cast<const int4*>(src) + lane);
  r.x = r.x < 0 ? oob : r.x;
  r.y = r.y < 0 ? oob : r.y;
  r.z = r.z < 0 ? oob : r.z;
  r.w = r.w < 0 ? oob : r.w;
#pragma unroll
  for (int c = 0; c < D / 64; ++c) tma_gather4(dst + c * (BLK * 128) + lane * 4 * 128, tm, bar, c * 64, r.x, r.y, r.z, r.w);
}

template <int D>
__global__ void __launch_bounds__(NTHREADS, 1)
    attn_kernel(const __grid_constant__ CUtensorMap tmQo, const __grid_constant__ CUtensorMap tmQg,
                const __grid_constant__ CUtensorMap tmKo, const __grid_constant__ CUtensorMap tmKg,
                const __grid_constant__ CUtensorMap tmVo, const __grid_constant__ CUtensorMap tmVg,
                const __grid_constant__ CUtensorMap tmO, const __grid_constant__ CUtensorMap tmPart,
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
  uint64_t* s_full = v_empty + VST;  // [half][slot]: S of a 64-key sub-tile written by the MMA
  uint64_t* p_full = s_full + 4;     // [half][slot]: P (bf16, aliasing S in TMEM) written by the softmax
  uint64_t* o_full = p_full + 4;     // [half]
  uint64_t* o_empty = o_full + 2;    // [half]
  uint64_t* pv_done = o_empty + 2;   // [half]: one commit per P V (completion counter)
  uint64_t* sched_full = pv_done + 2;
  uint64_t* sched_empty = sched_full + SCHED_RING;
  uint64_t* kp_full = sched_empty + SCHED_RING;
  uint64_t* ri_full = kp_full + 2 * NKP;  // [2] row identities (positions / ranks) of an item staged
  uint64_t* ri_empty = ri_full + 2;     // [2]
  uint64_t* kp_empty = kp_full + NKP;
  uint32_t* tmem_holder = reinterpret_cast<uint32_t*>(smem + L::OFF_TMEM);
  int32_t* kpos_s = reinterpret_cast<int32_t*>(smem + L::OFF_KPOS);
  int32_t* krank_s = reinterpret_cast<int32_t*>(smem + L::OFF_KRANK);
  volatile int32_t* sched_ring = reinterpret_cast<volatile int32_t*>(smem + L::OFF_SCHED);  // stride SCHED_ENTRY
  int32_t* ri_s = reinterpret_cast<int32_t*>(smem + L::OFF_RI);
  volatile int32_t* live_s = reinterpret_cast<volatile int32_t*>(smem + L::OFF_LIVE);

  const int warp = threadIdx.x / 32;
  const int lane = threadIdx.x % 32;

  if (threadIdx.x == 0) {
    mbar_init(q_full, 1);
    mbar_init(q_empty, 1);
    for (int i = 0; i < KST; ++i) {
      mbar_init(k_full + i, 1);
      mbar_init(k_empty + i, 1);  // last S-MMA commit
    }
    for (int i = 0; i < VST; ++i) {
      mbar_init(v_full + i, 1);
      mbar_init(v_empty + i, 1);
    }
    for (int i = 0; i < 4; ++i) {
      mbar_init(s_full + i, 1);
      mbar_init(p_full + i, 128);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(o_full + i, 1);
      mbar_init(o_empty + i, 128);
      mbar_init(pv_done + i, 1);
    }
    for (int i = 0; i < SCHED_RING; ++i) {
      mbar_init(sched_full + i, 1);
      mbar_init(sched_empty + i, 3 + NWARP_SOFT);  // K loader, V loader, MMA, softmax warps
    }
    for (int i = 0; i < NKP; ++i) {
      mbar_init(kp_full + i, 1);
      mbar_init(kp_empty + i, NWARP_SOFT);  // one arrival per softmax warp
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(ri_full + i, 1);
      mbar_init(ri_empty + i, NWARP_SOFT);
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
#ifdef MMI_TRACE
  const long long tr_t0 = clock64();
  int tr_n = 0;
  const int tr_reg = (warp == 1 && lane == 0) ? 0 : (warp == NWARP_CTRL && lane == 0) ? 1 : (warp == NWARP_CTRL + 4 && lane == 0) ? 2 : -1;
#define TR(code, arg) do { if (tr_reg >= 0) TRACE(tr_reg, code, arg); } while (0)
#else
#define TR(code, arg)
#endif
  // TMEM columns: S/P of half h at 128 h, O of half h at 256 + 128 h
  const int n_items = P.dense ? P.H * ((((P.S + BLK - 1) / BLK) + 1) / 2) : P.n_items;
  auto fetch = [&](int i) -> int {
    const int slot = i % SCHED_RING;
    mbar_wait(sched_full + slot, (i / SCHED_RING) & 1);
    return sched_ring[slot * (SCHED_ENTRY / 4)];
  };
  // the item of ring entry i (the scheduler staged its WorkItem next to the index)
  auto item_of = [&](int i, int idx) -> ItemView {
    return load_item(P, idx, reinterpret_cast<const WorkItem*>(smem + L::OFF_SCHED + (i % SCHED_RING) * SCHED_ENTRY + 16));
  };

  if (warp < NWARP_CTRL) {
    if (CTRL_REGS > 0) asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;\n" ::"n"(CTRL_REGS > 0 ? CTRL_REGS : 256));
    if (warp == 0) {
      // ======================= scheduler + Q loader =======================
      // lane 0 schedules and stages; the whole warp issues the row gathers of permuted Q blocks
      const bool leader = (lane == 0);
      uint32_t q_phase = 0, rs_phase = 0;
      int rs = 0;
      for (int i = 0;; ++i) {
        const int slot = i % SCHED_RING;
        int idx = 0;
        if (leader) {
          mbar_wait(sched_empty + slot, ((i / SCHED_RING) & 1) ^ 1);
          // dynamic fetch from the workspace counter; static round-robin without one (dense
          // comparator: its implicit items are already in longest-first order)
          idx = (i == 0) ? (int)blockIdx.x
                         : (P.sched ? (int)gridDim.x + (int)atomicAdd(P.sched, 1u) : (int)blockIdx.x + i * (int)gridDim.x);
          if (idx >= n_items) idx = -1;
          sched_ring[slot * (SCHED_ENTRY / 4)] = idx;
          if (idx >= 0 && !P.dense) {
            const int4* src = reinterpret_cast<const int4*>(P.items + idx);
            int4* dst = reinterpret_cast<int4*>(smem + L::OFF_SCHED + slot * SCHED_ENTRY + 16);
#pragma unroll
            for (int w = 0; w < (int)(sizeof(WorkItem) / 16); ++w) dst[w] = src[w];
          }
          mbar_arrive(sched_full + slot);
        }
        idx = __shfl_sync(0xffffffffu, idx, 0);
        __syncwarp();
        if (idx < 0) break;
        const ItemView it = item_of(i, idx);
        if (it.n_tiles <= 0) continue;
        if (leader) {
          if (P.dbg) P.dbg[idx * 8 + 0] = gtimer();
          if (!P.dense) {
            // stage the rows' positions / ranks (contiguous slices) for the softmax warps
            mbar_wait(ri_empty + rs, rs_phase ^ 1);
            const int nrows = it.has_b ? 2 * BLK : BLK;
            int32_t* rip = ri_s + rs * 4 * BLK;
            if (it.q_gathered) {
              mbar_arrive_expect_tx(ri_full + rs, 2 * nrows * 4);
              bulk_load(rip, P.qg_pos + it.q_row0, nrows * 4, ri_full + rs);
              bulk_load(rip + 2 * BLK, P.qg_rank + it.q_row0, nrows * 4, ri_full + rs);
            } else {
              const int x0 = it.q_row0 - it.head * P.S;
              const int n4 = P.rank ? (min(nrows, P.S - x0) & ~3) : 0;  // whole 16-byte groups
              mbar_arrive_expect_tx(ri_full + rs, n4 * 4);
              if (n4 > 0) bulk_load(rip + 2 * BLK, P.rank + x0, n4 * 4, ri_full + rs);
            }
          }
          mbar_wait(q_empty, q_phase ^ 1);
          mbar_arrive_expect_tx(q_full, (it.has_b ? 2 : 1) * L::Q_BYTES);
        }
        if (!P.dense && ++rs == 2) {
          rs = 0;
          rs_phase ^= 1;
        }
        q_phase ^= 1;
        __syncwarp();
        if (it.q_gathered && (P.fused & 1)) {
          // in-kernel permutation: the rows of a permuted Q block are gathered straight
          // from Q (tile::gather4, 4 rows per lane and 64-column block)
          for (int hf = 0; hf < (it.has_b ? 2 : 1); ++hf)
            gather_rows_tma<D>(smem + L::OFF_Q + hf * L::Q_BYTES, &tmQg, q_full,
                               P.qg_src + it.q_row0 + hf * BLK, P.q_oob, lane);
        } else if (leader) {
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
      const bool leader = (lane == 0);
      int stage = 0, kps = 0;
      uint32_t phase = 0, kp_phase = 0;
      const int NS = is_k ? KST : VST;
      uint64_t* full = is_k ? k_full : v_full;
      uint64_t* empty = is_k ? k_empty : v_empty;
      for (int i = 0;; ++i) {
        const int idx = fetch(i);
        __syncwarp();
        if (leader) mbar_arrive(sched_empty + i % SCHED_RING);
        if (idx < 0) break;
        const ItemView it = item_of(i, idx);
        if (it.n_tiles <= 0) continue;
        SegIter si;
        si.init(P, it);
        for (int t = 0; t < it.n_tiles; ++t) {
          const TileInfo e = si.next(P, it);
          uint8_t* dst = smem + (is_k ? L::OFF_K : L::OFF_V) + stage * L::KV_BYTES;
          if (leader) {
            mbar_wait(empty + stage, phase ^ 1);
            if (is_k) live_s[stage] = (int)e.live();  // read by the MMA issuer after k_full (release: the arrive below)
            mbar_arrive_expect_tx(full + stage, L::KV_BYTES);
          }
          __syncwarp();
          if (e.space && (P.fused & 2)) {
            // in-kernel permutation (Alg.6 "Load index I_chip"): the tile's rows are
            // gathered from the original K / V by their source rows (tile::gather4)
            gather_rows_tma<D>(dst, is_k ? &tmKg : &tmVg, full + stage, P.kg_src + e.krow, P.kv_oob, lane);
          } else if (leader) {
            const CUtensorMap* tm = is_k ? (e.space ? &tmKg : &tmKo) : (e.space ? &tmVg : &tmVo);
#pragma unroll
            for (int c = 0; c < D / 64; ++c) tma_load_2d(dst + c * (BLK * 128), tm, full + stage, c * 64, e.krow);
          }
          // key coordinates of gathered tiles the softmax masks or fingerprints (same predicate there)
          const bool cp_pos = is_k && (e.pred_any() || P.fingerprint) && e.space;
          if (cp_pos) {
            if (leader) {
              const bool cp_rank = e.pred_any() && e.rmode;
              mbar_wait(kp_empty + kps, kp_phase ^ 1);
              mbar_arrive_expect_tx(kp_full + kps, (cp_rank ? 2 : 1) * BLK * 4);
              bulk_load(kpos_s + kps * BLK, P.kg_pos + e.krow, BLK * 4, kp_full + kps);
              if (cp_rank) bulk_load(krank_s + kps * BLK, P.kg_rank + e.krow, BLK * 4, kp_full + kps);
            }
            if (++kps == NKP) {
              kps = 0;
              kp_phase ^= 1;
            }
          }
          if (++stage == NS) {
            stage = 0;
            phase ^= 1;
          }
        }
      }
    } else {
      // ======================= MMA issuer (one thread) =======================
      // Per key tile t: P_A(t, 0) V, P_B(t, 0) V, P_A(t, 1) V, S_A(t + 1), P_B(t, 1) V, S_B(t + 1)
      // (last tile: P_A V pair, O_A complete, P_B V pair, O_B complete),
      // where sub-tile (t, u) = keys [64u, 64u + 64) of the tile, S_h(t) is one M128 N128 group
      // into both 64-column slots of half h's S buffer and P_h(t, u) overwrites the first 32 columns
      // of slot u.  (Measured alternatives, tests/issuer_sim.py: a dynamic issuer advancing each
      // half independently with N=64 scores one tile ahead was 1.6x slower -- with 2-stage K/V
      // rings the halves drift apart and stall on each other's stage releases.)
#ifdef MMI_WARP_ISSUER
      {
        const bool leader = elect_one();
#else
      if (elect_one()) {
        constexpr bool leader = true;
#endif
        constexpr uint32_t IDESC_S128 = idesc_bf16(128, 128, 0);
        [[maybe_unused]] constexpr uint32_t IDESC_S64 = idesc_bf16(128, 64, 0);
        constexpr uint32_t IDESC_O = idesc_bf16(128, D, 1);
        const uint32_t q_base = smem_u32(smem + L::OFF_Q);
        const uint32_t k_base = smem_u32(smem + L::OFF_K);
        const uint32_t v_base = smem_u32(smem + L::OFF_V);
        // operand descriptors: base descriptor + (byte offset >> 4) in the start-address field
        const uint64_t dq0 = smem_desc(q_base, 16, 1024, 2), dk0 = smem_desc(k_base, 16, 1024, 2);
        const uint64_t dv0 = smem_desc(v_base, BLK * 128, 1024, 2);
        int ks = 0, vs = 0;
        uint32_t k_phase = 0, v_phase = 0, q_phase = 0;
        uint32_t p_bits = 0, o_bits = 0;  // phase bits: P per (half, slot), O per half (no indexed arrays: they would live in local memory)
        PROF_DECL(wp); PROF_DECL(wk); PROF_DECL(wv); PROF_DECL(wq); PROF_DECL(wo); PROF_DECL(tot); PROF_DECL(nt);
        [[maybe_unused]] const long long prof_start = PROF_T();
        for (int i = 0;; ++i) {
          const int idx = fetch(i);
          if (leader) mbar_arrive(sched_empty + i % SCHED_RING);
          if (idx < 0) break;
          const ItemView it = item_of(i, idx);
          const int n = it.n_tiles;
          if (n <= 0) continue;
          const int nh = it.has_b ? 2 : 1;
          long long t0 = PROF_T();
          mbar_wait(q_full, q_phase);
          PROF_ADD(wq, t0);
          TR(3, 0);
          q_phase ^= 1;
          tc_fence_after();
          // O_h += P_h(j) V(j), P read from TMEM (A operand), V stage vs; `started` bit hf: O_h
          // already holds a P V of this item
          uint32_t started = 0;
          auto issue_pv = [&](int hf, int j) {
            const int u = j & 1;
            long long t0 = PROF_T();
            mbar_wait(p_full + 2 * hf + u, (p_bits >> (2 * hf + u)) & 1u);
            PROF_ADD(wp, t0);
            p_bits ^= 1u << (2 * hf + u);
            t0 = PROF_T();
            const bool first = !((started >> hf) & 1u);
            if (first) mbar_wait(o_empty + hf, ((o_bits >> hf) & 1u) ^ 1u);  // previous item's epilogue read O_h
            PROF_ADD(wo, t0);
            tc_fence_after();
            TR(1, 2 * hf + u);
#pragma unroll
            for (int k = 0; k < 4; ++k) {
              const uint64_t bd = dv0 + (uint64_t)((vs * L::KV_BYTES + (4 * u + k) * 2048) >> 4);
              if (leader) umma_ts(tmem + 256 + 128 * hf, tmem + 128 * hf + 64 * u + k * 8, bd, IDESC_O,
                      (!first || k > 0) ? 1u : 0u);
            }
            started |= 1u << hf;
            if (leader) umma_commit(pv_done + hf);  // completion count of the half's P V (softmax rescale)
          };
          // Tiles dead for a half (no admitted element for its rows, per the index's per-half tile
          // states) issue neither its S nor its P V; the K loader passes each stage's live-half bits.
          // S of a whole 128-key tile is ONE M128 N128 MMA group into both 64-column slots of the
          // half (full tensor rate: A 4 KB + B 4 KB of shared memory per 64 clk; two N=64 groups
          // cost 2 x 48 clk, bound by the 128 B/clk operand bandwidth).  S_h(t+1) overwrites P_h(t),
          // so it is issued right after P_h(t, u=1) V: the other half's work fills the MMA pipe while
          // this half's softmax runs.
          auto issue_s128 = [&](int hf, int kst) {
            TR(2, 2 * hf);
#pragma unroll
            for (int k = 0; k < D / 16; ++k) {
              const uint32_t off = (k / 4) * (BLK * 128) + (k % 4) * 32;
              const uint64_t ad = dq0 + (uint64_t)((hf * L::Q_BYTES + off) >> 4);
              const uint64_t bd = dk0 + (uint64_t)((kst * L::KV_BYTES + off) >> 4);
              if (leader) umma_ss(tmem + 128 * hf, ad, bd, IDESC_S128, k > 0 ? 1u : 0u);
            }
            if (leader) umma_commit(s_full + 2 * hf);  // both 64-key slots: one phase per tile
          };
#ifdef MMI_S64
          // (experiment) S of one 64-key slot, issued right after the P V that freed the slot
          auto issue_s64 = [&](int hf, int kst, int u) {
            TR(2, 2 * hf + u);
#pragma unroll
            for (int k = 0; k < D / 16; ++k) {
              const uint32_t off = (k / 4) * (BLK * 128) + (k % 4) * 32;
              const uint64_t ad = dq0 + (uint64_t)((hf * L::Q_BYTES + off) >> 4);
              const uint64_t bd = dk0 + (uint64_t)((kst * L::KV_BYTES + u * 64 * 128 + off) >> 4);
              if (leader) umma_ss(tmem + 128 * hf + 64 * u, ad, bd, IDESC_S64, k > 0 ? 1u : 0u);
            }
            if (leader) umma_commit(s_full + 2 * hf + u);
          };
#endif
          t0 = PROF_T();
          mbar_wait(k_full + ks, k_phase);
          PROF_ADD(wk, t0);
          tc_fence_after();
          uint32_t live_cur = (uint32_t)live_s[ks], live_next = 0;
          for (int hf = 0; hf < nh; ++hf)
            if ((live_cur >> hf) & 1u) {
#ifdef MMI_S64
              issue_s64(hf, ks, 0);
              issue_s64(hf, ks, 1);
#else
              issue_s128(hf, ks);
#endif
            }
          if (n == 1 && leader) umma_commit(q_empty);  // last S of the item issued
          if (leader) umma_commit(k_empty + ks);
          if (++ks == KST) {
            ks = 0;
            k_phase ^= 1;
          }
          for (int t = 0; t < n; ++t) {
            const bool ahead = (t + 1 < n);
            t0 = PROF_T();
            mbar_wait(v_full + vs, v_phase);
            PROF_ADD(wv, t0);
            if (ahead) {
              t0 = PROF_T();
              mbar_wait(k_full + ks, k_phase);
              PROF_ADD(wk, t0);
              tc_fence_after();
              live_next = (uint32_t)live_s[ks];
            }
#ifdef MMI_PROF
            prof_nt += 2 * nh;
#endif
            if (ahead) {
#ifdef MMI_S64
              for (int u = 0; u < 2; ++u)
                for (int hf = 0; hf < nh; ++hf) {
                  if ((live_cur >> hf) & 1u) issue_pv(hf, 2 * t + u);
                  if ((live_next >> hf) & 1u) issue_s64(hf, ks, u);
                }
#else
              for (int hf = 0; hf < nh; ++hf)
                if ((live_cur >> hf) & 1u) issue_pv(hf, 2 * t);
              for (int hf = 0; hf < nh; ++hf) {
                if ((live_cur >> hf) & 1u) issue_pv(hf, 2 * t + 1);
                if ((live_next >> hf) & 1u) issue_s128(hf, ks);
              }
#endif
            } else {
              // last tile: each half's P V pair, then its O is complete -- half A's epilogue does
              // not wait for half B's last softmax
              for (int hf = 0; hf < nh; ++hf) {
                if ((live_cur >> hf) & 1u) {
                  issue_pv(hf, 2 * t);
                  issue_pv(hf, 2 * t + 1);
                }
                if ((started >> hf) & 1u) {  // a half with no live tile in the item has no O
                  if (leader) umma_commit(o_full + hf);
                  o_bits ^= 1u << hf;
                }
              }
            }
            if (t + 1 == n - 1 && leader) umma_commit(q_empty);  // last S of the item issued
            if (leader) umma_commit(v_empty + vs);
            if (++vs == VST) {
              vs = 0;
              v_phase ^= 1;
            }
            if (ahead) {
              if (leader) umma_commit(k_empty + ks);
              if (++ks == KST) {
                ks = 0;
                k_phase ^= 1;
              }
            }
            live_cur = live_next;
          }
        }
        PROF_ADD(tot, prof_start);
#ifdef MMI_TRACE
        if (blockIdx.x == 0) g_trace_n[0] = tr_n;
#endif
        if (leader) {
          PROF_FLUSH(0, tot); PROF_FLUSH(1, wp); PROF_FLUSH(2, wk); PROF_FLUSH(3, wv); PROF_FLUSH(4, wq);
          PROF_FLUSH(5, wo); PROF_FLUSH(6, nt);
        }
      }
    }
  } else {
    if (SOFT_REGS > 0) asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;\n" ::"n"(SOFT_REGS > 0 ? SOFT_REGS : 256));
    // ======================= softmax / correction / epilogue =======================
    // HPW = 1: one warpgroup per half (8 warps); HPW = 2: one warpgroup does both halves, half A's
    // sub-tiles then half B's (4 warps; the two halves never contend for MUFU on a sub-partition).
    // Thread t owns TMEM lane t = row t of each of its halves.
    const int h0 = (HPW == 1) ? (warp - NWARP_CTRL) / 4 : 0;  // first half this warpgroup owns
    const int row = (threadIdx.x - 32 * NWARP_CTRL) % 128;     // TMEM lane == row of the half
    const uint32_t lane_off = (uint32_t)((warp % 4) * 32) << 16;
    int kps = 0;  // key-coordinate ring
    uint32_t kp_phase = 0;
    int rs = 0;  // row-identity stage
    uint32_t rs_phase = 0;
    // per-half pipeline phases (persist across items)
    // pv_done[hf] completes one phase per P V of the half: a completion counter.  A rescale at the
    // half's sub-tile number n (counted over all items) needs P V number n - 1 to have landed and
    // waits for the phase of parity (n - 1) & 1.  That parity wait is unambiguous: S_h(t) is issued
    // after P_h(t - 1, 1) V, so when sub-tile n = 2t + u is processed every P V before n - 1 has
    // completed and P V n is not issued yet (its P is this sub-tile's output) -- the completed
    // count is n - 1 or n.  Phases nobody waits for are expected (a rescale is rare); compute-
    // sanitizer synccheck reports them as "missing wait", which is benign for this use.
    uint32_t s_phase[HPW], o_phase[HPW], n_sub[HPW];
#pragma unroll
    for (int j = 0; j < HPW; ++j) {
      s_phase[j] = 0;
      o_phase[j] = n_sub[j] = 0;
    }
    const int G = P.H / P.Hkv;
    PROF_DECL(stot); PROF_DECL(sws); PROF_DECL(sld); PROF_DECL(smask); PROF_DECL(ssm); PROF_DECL(sresc);
    PROF_DECL(spst); PROF_DECL(sepi); PROF_DECL(snt); PROF_DECL(snr); PROF_DECL(sfetch); PROF_DECL(sitem); PROF_DECL(smword); PROF_DECL(sepw); PROF_DECL(sepl);
    [[maybe_unused]] const long long sprof_start = PROF_T();
    for (int i = 0;; ++i) {
      long long t0 = PROF_T();
      const int idx = fetch(i);
      PROF_ADD(sfetch, t0);
      __syncwarp();
      if (lane == 0) mbar_arrive(sched_empty + i % SCHED_RING);
      if (idx < 0) break;
      const ItemView it = item_of(i, idx);
      if (it.n_tiles <= 0) continue;  // empty slot: nothing to compute or write
      const int nh_mine = (HPW == 1) ? ((h0 == 0 || it.has_b) ? 1 : 0) : (it.has_b ? 2 : 1);
      // row identity (positions / ranks staged in shared memory by warp 0)
      int xpos[HPW], xrank[HPW];
#pragma unroll
      for (int j = 0; j < HPW; ++j) {
        xpos[j] = it.q_row0 + (h0 + j) * BLK + row - it.head * P.S;
        xrank[j] = xpos[j];
      }
      if (!P.dense) {
        mbar_wait(ri_full + rs, rs_phase);
        const int32_t* rip = ri_s + rs * 4 * BLK;
#pragma unroll
        for (int j = 0; j < HPW; ++j) {
          const int li = (h0 + j) * BLK + row;
          if (it.q_gathered) {
            xpos[j] = rip[li];
            xrank[j] = rip[2 * BLK + li];
          } else if (P.rank) {
            const int x0 = it.q_row0 - it.head * P.S;
            const int n4 = min((it.has_b ? 2 : 1) * BLK, P.S - x0) & ~3;
            xrank[j] = li < n4 ? rip[2 * BLK + li] : (xpos[j] < P.S ? P.rank[xpos[j]] : xpos[j]);
          }
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(ri_empty + rs);
        if (++rs == 2) {
          rs = 0;
          rs_phase ^= 1;
        }
      }
      if (nh_mine == 0) {
        // absent half: only release the key-coordinate stages
        SegIter si;
        si.init(P, it);
        for (int t = 0; t < it.n_tiles; ++t) {
          const TileInfo e = si.next(P, it);
          if (e.space && (e.pred_any() || P.fingerprint)) {
            mbar_wait(kp_full + kps, kp_phase);
            __syncwarp();
            if (lane == 0) mbar_arrive(kp_empty + kps);
            if (++kps == NKP) {
              kps = 0;
              kp_phase ^= 1;
            }
          }
        }
        continue;
      }
      if (P.dbg && row == 0 && h0 == 0) P.dbg[idx * 8 + 3] = gtimer();
      TR(9, 0);
      t0 = PROF_T();
      bool valid[HPW], write[HPW];
      float m_used[HPW], l_sum[HPW];
      long long fp_cnt[HPW], fp_s1[HPW], fp_s2[HPW];
      int n_live[HPW];  // tiles of this item live for the half (= P V MMAs into O_h / 2)
#pragma unroll
      for (int j = 0; j < HPW; ++j) {
        valid[j] = xpos[j] >= 0 && xpos[j] < P.S;
        if (valid[j] && it.row_mod >= 0) valid[j] = (P.labels[xpos[j]] == it.row_mod);
        write[j] = valid[j];
        if (it.skip_s > 0 && valid[j]) {
          const int c = it.skip_rank ? xrank[j] : xpos[j];
          if (hline_row(c, it.skip_s, it.skip_p)) write[j] = false;  // owned by the HROW pass
        }
        m_used[j] = -INFINITY;
        l_sum[j] = 0.f;
        fp_cnt[j] = fp_s1[j] = fp_s2[j] = 0;
        n_live[j] = 0;
      }
      const int kv = it.head / G;
      SegIter si;
      si.init(P, it);
      int c_inst = -1, c_sink = 0, c_local = 0;  // cached pattern parameters of the current instance
      const uint32_t* c_sl = nullptr;
      const uint32_t* c_vm = nullptr;
      PROF_ADD(sitem, t0);
      for (int t = 0; t < it.n_tiles; ++t) {
        const TileInfo e = si.next(P, it);
        // the K loader staged this tile's key coordinates for whichever half masks it
        const bool kp_stage = e.space && (e.pred_any() || P.fingerprint);
        const uint32_t space = e.space, role = e.role, rmode = e.rmode, inst = e.inst;
        uint32_t mw[HPW][4];  // admitted-key mask of the tile per half (bit c <-> key c)
        t0 = PROF_T();
        if (kp_stage) mbar_wait(kp_full + kps, kp_phase);
        const int* kp = kpos_s + kps * BLK;
#pragma unroll
        for (int j = 0; j < HPW; ++j) {
          mw[j][0] = mw[j][1] = mw[j][2] = mw[j][3] = 0u;
          const int hf = h0 + j;
          if (j >= nh_mine) continue;
          const uint32_t my_st = e.st(hf);
          if (my_st == TS_DEAD) continue;
          const uint32_t pred = (my_st == TS_PRED) ? 1u : 0u;
          if (!(pred || P.fingerprint) || !valid[j]) continue;
          const int kbase = e.krow - kv * P.S;
          if (!pred) {
            range_mask(mw[j], 0, BLK - 1);
          } else if (role == R_NAT) {
            natten_mask(P, xpos[j], e.krow, mw[j]);
          } else {
            if (!P.dense && role != R_TRUE && (int)inst != c_inst) {
              // pattern parameters of the tile's instance: reloaded only when the instance changes
              const InstParam ip = P.insts[it.inst_base + inst];
              c_inst = (int)inst;
              c_sink = ip.sink;
              c_local = ip.local;
              c_sl = ip.slash_word >= 0 ? P.bits + ip.slash_word : nullptr;
              c_vm = ip.vmask_word >= 0 ? P.bits + ip.vmask_word : nullptr;
            }
            const int sink = c_sink, local = c_local;
            const int x = rmode ? xrank[j] : xpos[j];
            // Keys of every view are ascending inside a tile, so each role is at most two
            // index ranges: [0, n_causal) intersected with the pattern's coordinate ranges.
            int n_causal, n_sink, n_lt_local, ybase;
            const int thr = a_thr(x, local);  // keys y <= thr are outside the local part
            if (!space) {
              n_causal = min(max(xpos[j] - kbase + 1, 0), BLK);
              n_sink = min(max(sink - kbase, 0), BLK);
              n_lt_local = min(max(thr - kbase + 1, 0), BLK);
              ybase = kbase;
            } else {
              const int* yc = rmode ? (krank_s + kps * BLK) : kp;
              if (role == R_A || role == R_NOTA) {
                count_le3(kp, xpos[j], yc, sink - 1, thr, n_causal, n_sink, n_lt_local);
              } else {
                n_causal = count_le(kp, xpos[j]);
                n_sink = n_lt_local = 0;
              }
              ybase = yc[0];
            }
            if (role == R_TRUE) {
              range_mask(mw[j], 0, n_causal - 1);
            } else if (role == R_A) {
              range_mask(mw[j], 0, min(n_sink, n_causal) - 1);
              range_mask(mw[j], n_lt_local, n_causal - 1);
            } else if (role == R_NOTA) {
              range_mask(mw[j], n_sink, min(n_lt_local, n_causal) - 1);
            } else {
              // vertical-slash: coordinates contiguous in the tile (original K, or a modality's
              // rank-ordered keys); slash bits of offsets x - ybase - c, bit-reversed window.  A
              // slash range's first tile may start below key 0 (ybase < 0): those keys are masked.
              range_mask(mw[j], -ybase, n_causal - 1);
              uint32_t ws[4], wv[4];
              bit_window(c_sl, x - ybase - (BLK - 1), ws);
              bit_window(c_vm, ybase, wv);
#pragma unroll
              for (int w = 0; w < 4; ++w) mw[j][w] &= __brev(ws[3 - w]) & ~wv[w];
            }
          }
          if (P.fingerprint) {
#pragma unroll
            for (int w = 0; w < 4; ++w) {
              uint32_t bitsw = mw[j][w];
              while (bitsw) {
                const int c = w * 32 + __ffs(bitsw) - 1;
                bitsw &= bitsw - 1;
                const long long ypos = space ? kp[c] : kbase + c;
                fp_cnt[j] += 1;
                fp_s1[j] += ypos;
                fp_s2[j] += ypos * ypos;
              }
            }
          }
        }
        if (kp_stage) {
          __syncwarp();
          if (lane == 0) mbar_arrive(kp_empty + kps);  // key coordinates of this stage consumed
          if (++kps == NKP) {
            kps = 0;
            kp_phase ^= 1;
          }
        }
        PROF_ADD(smword, t0);
#pragma unroll
        for (int j = 0; j < HPW; ++j) {
          const int hf = h0 + j;
          if (j >= nh_mine) continue;
          const uint32_t my_st = e.st(hf);
          if (my_st == TS_DEAD) continue;  // no admitted element for these rows: no S, no P V for this half
          ++n_live[j];
          const bool masked = (my_st == TS_PRED) || P.fingerprint;
          const uint32_t tS = tmem + 128 * hf + lane_off;
          const uint32_t tO = tmem + 256 + 128 * hf + lane_off;
#pragma unroll
          for (int u = 0; u < 2; ++u) {
            t0 = PROF_T();
#ifdef MMI_S64
            mbar_wait(s_full + 2 * hf + u, (s_phase[j] >> u) & 1u);  // per-slot S
            s_phase[j] ^= 1u << u;
#else
            if (u == 0) {  // S of both 64-key slots landed together (one M128 N128 group)
              mbar_wait(s_full + 2 * hf, s_phase[j]);
              s_phase[j] ^= 1;
            }
#endif
            PROF_ADD(sws, t0);
            TR(4, u);
            t0 = PROF_T();
            tc_fence_after();
#ifdef MMI_NOSOFT
            // pipeline ceiling experiment (scratch builds only): no softmax work at all
            tc_fence_before();
            mbar_arrive(p_full + 2 * hf + u);
            ++n_sub[j];
            continue;
#endif
            float s[64];
#pragma unroll
            for (int c = 0; c < 2; ++c) {
              uint32_t r[32];
              tmem_ld32(tS + 64 * u + c * 32, r);
              tmem_wait_ld();
#pragma unroll
              for (int q = 0; q < 32; ++q) s[c * 32 + q] = __uint_as_float(r[q]);  // raw scores
            }
            PROF_ADD(sld, t0);
            t0 = PROF_T();
            // (sub-tiles every row of the warp fully admits skip the select: diagonal / sink / local
            // tiles are mostly all-or-nothing per 64 keys)
            if (masked && !__all_sync(0xffffffffu, (mw[j][2 * u] & mw[j][2 * u + 1]) == 0xffffffffu)) {
#pragma unroll
              for (int c = 0; c < 64; ++c)
                if (!((mw[j][2 * u + (c >> 5)] >> (c & 31)) & 1u)) s[c] = -INFINITY;
            }
            PROF_ADD(smask, t0);
            t0 = PROF_T();
            // ---- online softmax (log2 domain), lazy rescale ----
            float mx[8];
#pragma unroll
            for (int q = 0; q < 8; ++q) mx[q] = fmaxf(s[q], s[q + 8]);
#pragma unroll
            for (int c = 16; c < 64; c += 16)
#pragma unroll
              for (int q = 0; q < 8; ++q) mx[q] = fmaxf(mx[q], fmaxf(s[c + q], s[c + 8 + q]));
            float mt = fmaxf(fmaxf(fmaxf(mx[0], mx[1]), fmaxf(mx[2], mx[3])),
                             fmaxf(fmaxf(mx[4], mx[5]), fmaxf(mx[6], mx[7])));
            if (mt > -INFINITY) mt *= P.scale_log2;  // tau * log2(e) > 0 commutes with max
            float alpha = 1.f;
            bool rescale = false;
            if (mt > m_used[j] + RESCALE_THRESH || (m_used[j] == -INFINITY && mt > -INFINITY)) {
              alpha = (m_used[j] == -INFINITY) ? 0.f : ex2(m_used[j] - mt);
              rescale = (m_used[j] != -INFINITY);
              m_used[j] = mt;
            }
            const float mu = (m_used[j] == -INFINITY) ? 0.f : m_used[j];
            const float2 sc2 = make_float2(P.scale_log2, P.scale_log2), nmu2 = make_float2(-mu, -mu);
            float2 ls2[4] = {make_float2(0.f, 0.f), make_float2(0.f, 0.f), make_float2(0.f, 0.f),
                             make_float2(0.f, 0.f)};
            uint32_t pk[32];
#pragma unroll
            for (int c = 0; c < 64; c += 2) {
              const float2 x = ffma2(make_float2(s[c], s[c + 1]), sc2, nmu2);
              float2 pr;
              if ((EMU_MASK >> ((c / 2) % 8)) & 1u) {
                pr = exp2_poly2(x);
              } else {
                pr.x = ex2(x.x);
                pr.y = ex2(x.y);
              }
              ls2[(c / 2) % 4] = fadd2(ls2[(c / 2) % 4], pr);
              pk[c / 2] = pack_bf16(pr.x, pr.y);
            }
            const float2 lsa = fadd2(fadd2(ls2[0], ls2[1]), fadd2(ls2[2], ls2[3]));
            l_sum[j] = l_sum[j] * alpha + (lsa.x + lsa.y);
            PROF_ADD(ssm, t0);
            TR(5, u);
            t0 = PROF_T();
            // O correction only when the running max moved (rare): P(j - 1) V may still be in flight
            const bool any_rescale = __any_sync(0xffffffffu, rescale);
            if (any_rescale && n_sub[j] > 0) mbar_wait(pv_done + hf, (n_sub[j] - 1) & 1u);
            if (any_rescale) {
              tc_fence_after();
#pragma unroll
              for (int c = 0; c < D / 32; ++c) {
                uint32_t r[32];
                tmem_ld32(tO + c * 32, r);
                tmem_wait_ld();
#pragma unroll
                for (int q = 0; q < 32; ++q) r[q] = __float_as_uint(__uint_as_float(r[q]) * alpha);
                tmem_st32(tO + c * 32, r);
              }
#ifdef MMI_PROF
              prof_snr += 1;
#endif
            }
            PROF_ADD(sresc, t0);
            t0 = PROF_T();
            // P (bf16 pairs) -> TMEM columns [64u, 64u + 32) of this half's S buffer
            tmem_st32(tS + 64 * u, pk);  // (two 16-column stores, the first issued mid-loop: 2 % slower)
            tmem_wait_st();
            tc_fence_before();
            mbar_arrive(p_full + 2 * hf + u);
            ++n_sub[j];  // P V number n_sub - 1 will complete a phase of pv_done[hf]
            PROF_ADD(spst, t0);
            TR(6, u);
#ifdef MMI_PROF
            prof_snt += 1;
#endif
          }
        }
      }
      // ---- epilogue ----  (a half with no live tile in this item has no O: it writes zeros / -inf)
#pragma unroll
      for (int j = 0; j < HPW; ++j) {
        const int hf = h0 + j;
        if (j >= nh_mine) continue;
        const uint32_t tO = tmem + 256 + 128 * hf + lane_off;
        t0 = PROF_T();
        const bool has_o = n_live[j] > 0;
        TR(7, 0);
        if (has_o) {
          mbar_wait(o_full + hf, o_phase[j]);
          o_phase[j] ^= 1;
          tc_fence_after();
        }
        PROF_ADD(sepw, t0);
        TR(10, 0);
        // no admitted key in this item <=> the running max never left -inf (the polynomial exp2
        // maps masked scores to 2^-125, so l_sum alone does not tell)
        const float lsum = (m_used[j] == -INFINITY) ? 0.f : l_sum[j];
        const float inv_l = lsum > 0.f ? 1.f / lsum : 0.f;
        const float lse_v = lsum > 0.f ? (m_used[j] + __log2f(lsum)) * 0.6931471805599453f : -INFINITY;
        if (P.fingerprint) {
          if (has_o) {
            tc_fence_before();
            mbar_arrive(o_empty + hf);
          }
          if (write[j]) {
            long long* f = reinterpret_cast<long long*>(P.fp_out) + 3ll * ((long long)it.head * P.S + xpos[j]);
            atomicAdd(reinterpret_cast<unsigned long long*>(f + 0), (unsigned long long)fp_cnt[j]);
            atomicAdd(reinterpret_cast<unsigned long long*>(f + 1), (unsigned long long)fp_s1[j]);
            atomicAdd(reinterpret_cast<unsigned long long*>(f + 2), (unsigned long long)fp_s2[j]);
          }
          continue;
        }
        // O (fp32, TMEM) -> 16-bit registers: bf16 for final rows, fp16 for partial rows (merged in
        // fp32 by merge_kernel).  O is released as soon as it is in registers.
        const bool fin = (it.out_mode == OUT_FINAL);
        uint32_t ov[D / 2];
#pragma unroll
        for (int c = 0; c < D / 32; c += 2) {  // two 32-column loads in flight per wait
          uint32_t r[2][32];
          if (has_o) {
            tmem_ld32(tO + c * 32, r[0]);
            tmem_ld32(tO + c * 32 + 32, r[1]);
            tmem_wait_ld();
          } else {
#pragma unroll
            for (int q = 0; q < 32; ++q) r[0][q] = r[1][q] = 0u;
          }
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            if (fin) {
#pragma unroll
              for (int q = 0; q < 16; ++q)
                ov[(c + h) * 16 + q] =
                    pack_bf16(__uint_as_float(r[h][2 * q]) * inv_l, __uint_as_float(r[h][2 * q + 1]) * inv_l);
            } else {
#pragma unroll
              for (int q = 0; q < 16; ++q)
                ov[(c + h) * 16 + q] =
                    pack_f16(__uint_as_float(r[h][2 * q]) * inv_l, __uint_as_float(r[h][2 * q + 1]) * inv_l);
            }
          }
        }
        if (has_o) {
          tc_fence_before();
          mbar_arrive(o_empty + hf);  // the next item's first P V of this half may start
        }
        PROF_ADD(sepl, t0);
        TR(11, fin ? (it.q_gathered ? 1 : 0) : 2);
        t0 = PROF_T();
#ifdef MMI_NOEPI
        continue;  // pipeline ceiling experiment (scratch builds only): no output stores
#endif
        // destination row (0: not written).  Partial rows are always written (zeros for invalid
        // rows: the merge weights them by exp(-inf) = 0, which must not meet a NaN).
        unsigned long long dst = 0;
        if (fin) {
          if (write[j]) dst = reinterpret_cast<unsigned long long>(reinterpret_cast<__nv_bfloat16*>(P.o) +
                                                                   ((size_t)it.head * P.S + xpos[j]) * D);
        } else {
          dst = reinterpret_cast<unsigned long long>(P.part_o + (size_t)(it.out_row0 + hf * BLK + row) * D);
        }
        const uint32_t ebuf = smem_u32(smem + L::OFF_EPI + (warp - NWARP_CTRL) * 32 * EPI_STRIDE);
        const int wrow0 = (warp % 4) * 32;  // first row of this warp in the half (its TMEM lane base)
#if defined(MMI_EPI_NOTMA)
        if (false) {
#else
        if (!fin || (!it.q_gathered && __all_sync(0xffffffffu, write[j]))) {
#endif
          // The warp's 32 rows are contiguous in the destination (partial rows, or final rows of an
          // original-order block that are all written): each 16-column chunk (32 rows x 32 B) is
          // staged in the TMA 32B-swizzle layout (16 B half q of row r at q ^ ((r >> 2) & 1):
          // conflict-free) in one of two 1 KB buffers and written by one asynchronous TMA tensor
          // store; a buffer is refilled once the store two chunks back has read it.
          const CUtensorMap* tm = fin ? &tmO : &tmPart;
          const int grow = (fin ? it.q_row0 : it.out_row0) + hf * BLK + wrow0;
#pragma unroll
          for (int c = 0; c < D / 16; ++c) {
            const uint32_t buf = ebuf + (c & 1) * 1024;
            if (c >= 2) {
              if (lane == 0) bulk_wait_read1();
              __syncwarp();
            }
#pragma unroll
            for (int q = 0; q < 2; ++q)
              st_shared_v4(buf + lane * 32 + ((q ^ ((lane >> 2) & 1)) * 16), ov[c * 8 + 4 * q],
                           ov[c * 8 + 4 * q + 1], ov[c * 8 + 4 * q + 2], ov[c * 8 + 4 * q + 3]);
            fence_proxy_async_smem();
            __syncwarp();
            if (lane == 0) {
              tma_store_2d(tm, buf, c * 16, grow);
              bulk_commit();
            }
          }
          if (lane == 0) bulk_wait_read0();  // staging buffers free for the next item / half
          __syncwarp();
        } else {
          // scattered rows: thread-per-row stores would touch 32 rows (32 L1 wavefronts) per
          // instruction; instead each 64-byte column chunk of the warp's 32 rows is transposed
          // through shared memory so that one 16-byte store instruction writes 8 rows x 64 B.
          unsigned long long dsts[4];
#pragma unroll
          for (int k = 0; k < 4; ++k) dsts[k] = __shfl_sync(0xffffffffu, dst, k * 8 + (lane >> 2));
#pragma unroll
          for (int c = 0; c < D / 32; ++c) {
#pragma unroll
            for (int q = 0; q < 4; ++q)
              st_shared_v4(ebuf + lane * EPI_STRIDE + q * 16, ov[c * 16 + 4 * q], ov[c * 16 + 4 * q + 1],
                           ov[c * 16 + 4 * q + 2], ov[c * 16 + 4 * q + 3]);
            __syncwarp();
#pragma unroll
            for (int k = 0; k < 4; ++k) {
              const uint4 w = ld_shared_v4(ebuf + (k * 8 + (lane >> 2)) * EPI_STRIDE + (lane & 3) * 16);
              if (dsts[k]) *reinterpret_cast<uint4*>(dsts[k] + c * 64 + (lane & 3) * 16) = w;
            }
            __syncwarp();
          }
        }
        if (fin) {
          if (write[j] && P.lse) P.lse[(size_t)it.head * P.S + xpos[j]] = lse_v;
        } else {
          P.part_lse[it.out_row0 + hf * BLK + row] = valid[j] ? lse_v : -INFINITY;
        }
        if (P.dbg && row == 0 && hf == 0) P.dbg[idx * 8 + 6] = gtimer();
        PROF_ADD(sepi, t0);
        TR(8, 0);
      }
    }
    if (lane == 0) bulk_wait0();  // this warp's TMA output stores are complete
#ifdef MMI_TRACE
    if (blockIdx.x == 0 && tr_reg > 0) g_trace_n[tr_reg] = tr_n;
#endif
    PROF_ADD(stot, sprof_start);
    if (lane == 0) {
      PROF_FLUSH(8, stot); PROF_FLUSH(9, sws); PROF_FLUSH(10, sld); PROF_FLUSH(11, smask); PROF_FLUSH(12, ssm);
      PROF_FLUSH(13, sresc); PROF_FLUSH(14, spst); PROF_FLUSH(15, sepi); PROF_FLUSH(16, snt); PROF_FLUSH(17, snr);
      PROF_FLUSH(18, sfetch); PROF_FLUSH(19, sitem); PROF_FLUSH(20, smword); PROF_FLUSH(21, sepw); PROF_FLUSH(22, sepl);
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
#ifdef MMI_TRACE
extern "C" __attribute__((visibility("default"))) int mmi_debug_trace(unsigned long long* out, int* n) {
  cudaDeviceSynchronize();
  cudaMemcpyFromSymbol(out, g_trace, sizeof(g_trace));
  cudaMemcpyFromSymbol(n, g_trace_n, sizeof(g_trace_n));
  return 0;
}
#endif
#ifdef MMI_PROF
extern "C" __attribute__((visibility("default"))) int mmi_debug_prof(unsigned long long* out, int reset) {
  cudaDeviceSynchronize();
  cudaMemcpyFromSymbol(out, g_prof, sizeof(g_prof));
  if (reset) {
    unsigned long long z[32] = {0};
    cudaMemcpyToSymbol(g_prof, z, sizeof(z));
  }
  return 0;
}
#endif
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

// rows x D bf16 row-major tensor for tile::gather4: box = 64 columns x 1 row, 128B swizzle (each
// gather4 lands 4 rows of 128 B; the swizzle follows the shared-memory address, so 32 gathers build
// the same tile as one {64, 128} box load)
static int make_tmap_gather(CUtensorMap* m, const void* base, long long rows, int D) {
  PFN_encodeTiled enc = get_encode();
  if (!enc) return -1;
  if (rows <= 0) rows = 1;
  cuuint64_t dims[2] = {(cuuint64_t)D, (cuuint64_t)rows};
  cuuint64_t strides[1] = {(cuuint64_t)D * 2};
  cuuint32_t box[2] = {64, 1};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = enc(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(base), dims, strides, box, estr,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS ? 0 : (int)r;
}

// rows x D 16-bit row-major output; box = 32 rows x 16 columns (32 B), 32B swizzle (epilogue staging)
static int make_tmap_out(CUtensorMap* m, const void* base, long long rows, int D, CUtensorMapDataType dt) {
  PFN_encodeTiled enc = get_encode();
  if (!enc) return -1;
  if (rows <= 0) rows = 1;
  cuuint64_t dims[2] = {(cuuint64_t)D, (cuuint64_t)rows};
  cuuint64_t strides[1] = {(cuuint64_t)D * 2};
  cuuint32_t box[2] = {16, 32};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = enc(m, dt, 2, const_cast<void*>(base), dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                   CU_TENSOR_MAP_SWIZZLE_32B, CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS ? 0 : (int)r;
}

static int g_num_sms = 0;

cudaError_t launch_attn(const AttnLaunch& L, const AttnParams& P, int n_items_hint, cudaStream_t stream,
                        int* tmap_err) {
  CUtensorMap m[8];
  int e = 0;
  e |= make_tmap_rows(&m[0], L.q, L.q_rows, P.D);
  e |= make_tmap_rows(&m[2], L.k, L.kv_rows, P.D);
  e |= make_tmap_rows(&m[4], L.v, L.kv_rows, P.D);
  // permuted blocks: row-gather maps over the ORIGINAL tensors (in-kernel permutation, P.fused) or
  // tile maps over the materialised Q̄ / K̄ / V̄
  if (P.fused & 1)
    e |= make_tmap_gather(&m[1], L.q, L.q_rows, P.D);
  else
    e |= make_tmap_rows(&m[1], L.qg ? L.qg : L.q, L.qg ? L.qg_rows : L.q_rows, P.D);
  if (P.fused & 2) {
    e |= make_tmap_gather(&m[3], L.k, L.kv_rows, P.D);
    e |= make_tmap_gather(&m[5], L.v, L.kv_rows, P.D);
  } else {
    e |= make_tmap_rows(&m[3], L.kg ? L.kg : L.k, L.kg ? L.kvg_rows : L.kv_rows, P.D);
    e |= make_tmap_rows(&m[5], L.vg ? L.vg : L.v, L.vg ? L.kvg_rows : L.kv_rows, P.D);
  }
  // output maps (epilogue TMA stores): bf16 O [H*S, D] and fp16 partial rows [part_rows, D]
  e |= make_tmap_out(&m[6], P.o ? P.o : L.q, P.o ? L.o_rows : L.q_rows, P.D, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16);
  e |= make_tmap_out(&m[7], L.part_rows > 0 ? (const void*)P.part_o : L.q, L.part_rows > 0 ? L.part_rows : L.q_rows,
                     P.D, CU_TENSOR_MAP_DATA_TYPE_FLOAT16);
  if (tmap_err) *tmap_err = e;
  if (e) return cudaErrorInvalidValue;
  if (!g_num_sms) {
    int dev = 0;
    cudaError_t ce = cudaGetDevice(&dev);
    if (ce == cudaSuccess) ce = cudaDeviceGetAttribute(&g_num_sms, cudaDevAttrMultiProcessorCount, dev);
    if (ce != cudaSuccess) return ce;
  }
  int grid = g_num_sms;
  if (n_items_hint > 0 && (n_items_hint + 1) / 2 < grid) grid = (n_items_hint + 1) / 2;
  if (grid <= 0) return cudaSuccess;
  const AttnParams& Pl = P;
  if (Pl.sched) {  // the caller's workspace counter, zeroed in stream order before the launch
    const cudaError_t ce = fill_bytes(Pl.sched, 0, sizeof(unsigned int), stream);
    if (ce != cudaSuccess) return ce;
  }
  if (P.D == 128) {
    auto kfn = attn_kernel<128>;
    const cudaError_t ce = cudaFuncSetAttribute(kfn, cudaFuncAttributeMaxDynamicSharedMemorySize, Smem<128>::ALLOC);
    if (ce != cudaSuccess) return ce;
    kfn<<<grid, NTHREADS, Smem<128>::ALLOC, stream>>>(m[0], m[1], m[2], m[3], m[4], m[5], m[6], m[7], Pl);
  } else {
    auto kfn = attn_kernel<64>;
    const cudaError_t ce = cudaFuncSetAttribute(kfn, cudaFuncAttributeMaxDynamicSharedMemorySize, Smem<64>::ALLOC);
    if (ce != cudaSuccess) return ce;
    kfn<<<grid, NTHREADS, Smem<64>::ALLOC, stream>>>(m[0], m[1], m[2], m[3], m[4], m[5], m[6], m[7], Pl);
  }
  return cudaGetLastError();
}

}  // namespace mmi
