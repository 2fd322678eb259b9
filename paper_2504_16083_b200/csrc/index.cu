// Index construction, permutation gathers (a6) and the
// inverse-permute LSE merge (a8).
//
// Views are position lists in the gathered Q̄ / K̄ spaces (Alg.1 P:213 row- and
// column-wise grid permutation, Alg.2/3 P:254/P:340 modality permutation,
// P:708 "convert them into a sparse format i_vs").  Work items are 128-row
// blocks of a Q-view with a list of segments (runs of key tiles of a K-view)
// and an element role; their union per row is exactly the paper's mask, each
// admitted element owned by exactly one pass (reading C9).
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <climits>
#include <cstdint>
#include <type_traits>

#include "estimate.h"
#include "index.h"

namespace mmi {


__device__ __forceinline__ int pad128d(int x) { return (x + BLK - 1) / BLK * BLK; }
__device__ __forceinline__ int cdiv(int a, int b) { return (a + b - 1) / b; }

// class geometry of an arithmetic residue view over base coords [0, n)
struct ClassGeo {
  int n, s, q, rem, padq1, padq;
  __device__ __forceinline__ void init(int n_, int s_) {
    n = n_;
    s = s_;
    q = n / s;
    rem = n % s;
    padq1 = pad128d(q + 1);
    padq = pad128d(q);
  }
  __device__ __forceinline__ int nr(int r) const { return q + (r < rem ? 1 : 0); }
  __device__ __forceinline__ int classoff(int r) const {
    return min(r, rem) * padq1 + max(0, r - rem) * padq;
  }
  __device__ __forceinline__ int total() const { return rem * padq1 + (s - rem) * padq; }
  // RES view row -> (r, t); false if beyond the view
  __device__ __forceinline__ bool locate(int row, int& r, int& t) const {
    const int a = rem * padq1;
    if (row < a) {
      r = row / padq1;
      t = row % padq1;
      return true;
    }
    if (padq == 0) return false;
    const int b = row - a;
    r = rem + b / padq;
    t = b % padq;
    return r < s;
  }
};

__device__ __forceinline__ int lower_bound_i(const int* a, int n, int v) {
  int lo = 0, hi = n;
  while (lo < hi) {
    const int mid = (lo + hi) >> 1;
    if (a[mid] < v)
      lo = mid + 1;
    else
      hi = mid;
  }
  return lo;
}
__device__ __forceinline__ int upper_bound_i(const int* a, int n, int v) {
  int lo = 0, hi = n;
  while (lo < hi) {
    const int mid = (lo + hi) >> 1;
    if (a[mid] <= v)
      lo = mid + 1;
    else
      hi = mid;
  }
  return lo;
}

// ================================================================ K-view dedupe
// The gathered K̄ / V̄ view of a pattern depends only on (KV group, view kind, classes, modality,
// stride, phase) -- not on the query head -- so the heads of a KV group whose estimated grids agree
// share one copy (SURVEY §7 hard part (g)): alias[v] = the first K-space view with the same key.
// Modality views (2D heads) of a group are identical; VS column views stay per head.
__global__ void view_alias_kernel(IndexCtx C, int n_views) {
  const int v = blockIdx.x * blockDim.x + threadIdx.x;
  if (v >= n_views) return;
  const DView a = C.views[v];
  int canon = v;
  if (a.space == 1 && a.kind != VK_VCOL) {
    const int kva = C.heads[a.head].kv;
    int sa = 0, pa = 0;
    if (a.kind == VK_ORIG_CLASS || a.kind == VK_RANK_CLASS) {
      const GridRes g = C.gridres[C.insts[a.head * MAX_INST + a.inst].grid_id];
      sa = g.s;
      pa = a.classes ? g.p : 0;
    }
    for (int u = 0; u < v; ++u) {
      const DView b = C.views[u];
      if (b.space != 1 || b.kind != a.kind || b.classes != a.classes || b.mod != a.mod) continue;
      if (C.heads[b.head].kv != kva) continue;
      if (a.kind == VK_ORIG_CLASS || a.kind == VK_RANK_CLASS) {
        const GridRes g = C.gridres[C.insts[b.head * MAX_INST + b.inst].grid_id];
        if (g.s != sa || (a.classes ? g.p : 0) != pa) continue;
      }
      canon = u;
      break;
    }
  }
  C.view_alias[v] = canon;
}

__device__ __forceinline__ int kview_row0(const IndexCtx& C, int v) { return C.views[C.view_alias[v]].row_off; }

// ================================================================ views
__global__ void build_views_kernel(IndexCtx C, int space, const int* __restrict__ view_ids, int n_view_ids,
                                   int64_t rows_total) {
  const int64_t row = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (row >= rows_total) return;
  // find the view containing this row
  int lo = 0, hi = n_view_ids - 1, v = -1;
  while (lo <= hi) {
    const int mid = (lo + hi) >> 1;
    const DView& dv = C.views[view_ids[mid]];
    if (row < dv.row_off)
      hi = mid - 1;
    else if (row >= (int64_t)dv.row_off + dv.cap)
      lo = mid + 1;
    else {
      v = view_ids[mid];
      break;
    }
  }
  int* pos_a = space ? C.kg_pos : C.qg_pos;
  int* rank_a = space ? C.kg_rank : C.qg_rank;
  int* src_a = space ? C.kg_src : C.qg_src;
  const int PADPOS = space ? KPAD : -1;
  if (v < 0) {
    pos_a[row] = PADPOS;
    rank_a[row] = PADPOS;
    src_a[row] = -2;
    return;
  }
  if (space && C.view_alias[v] != v) {  // deduplicated K view: its canonical copy is gathered instead
    pos_a[row] = PADPOS;
    rank_a[row] = PADPOS;
    src_a[row] = -2;
    if (row == C.views[v].row_off) C.view_len[v] = 0;
    return;
  }
  const DView dv = C.views[v];
  const int i = (int)(row - dv.row_off);
  const int h = dv.head;
  const int srcbase = space ? (C.heads[h].kv * C.S) : (h * C.S);
  int pos = -1, rk = -1, len = 0;
  bool valid = false;
  if (dv.kind == VK_MOD) {
    len = C.info[MI_PADOFF + MAX_MOD];
    if (i < len) {
      pos = C.modpos[i];
      valid = pos >= 0;
      if (valid) rk = C.rank[pos];
    }
  } else if (dv.kind == VK_ORIG_CLASS || dv.kind == VK_RANK_CLASS) {
    const DInst x = C.insts[h * MAX_INST + dv.inst];
    const GridRes g = C.gridres[x.grid_id];
    const bool rnk = dv.kind == VK_RANK_CLASS;
    const int n = rnk ? C.info[MI_CNT + dv.mod] : C.S;
    int coord = -1;
    if (dv.classes == 1) {
      const int np = g.p < n ? (n - g.p + g.s - 1) / g.s : 0;
      len = pad128d(np);
      if (i < np) coord = g.p + g.s * i;
    } else {
      ClassGeo cg;
      cg.init(n, g.s);
      len = cg.total();
      int r, t;
      if (i < len && cg.locate(i, r, t) && t < cg.nr(r)) coord = r + g.s * t;
    }
    if (coord >= 0) {
      valid = true;
      if (rnk) {
        pos = C.perm[C.info[MI_OFF + dv.mod] + coord];
        rk = coord;
      } else {
        pos = coord;
        rk = C.rank[pos];
      }
    }
  } else if (dv.kind == VK_VCOL) {
    const DInst x = C.insts[h * MAX_INST + dv.inst];
    const int cnt = C.vs_cnt[x.vs_id * 2];
    len = pad128d(cnt);
    if (i < cnt) {
      const int coord = C.vs_lists[C.vs_list_off[x.vs_id * 2] + i];
      valid = true;
      if (x.rank) {
        pos = C.perm[C.info[MI_OFF + x.qa] + coord];
        rk = coord;
      } else {
        pos = coord;
        rk = C.rank[pos];
      }
    }
  }
  if (i == 0) C.view_len[v] = len;
  if (valid) {
    pos_a[row] = pos;
    rank_a[row] = rk;
    src_a[row] = srcbase + pos;
  } else {
    pos_a[row] = PADPOS;
    rank_a[row] = PADPOS;
    src_a[row] = (i < len) ? -1 : -2;
  }
}

// ================================================================ instance params
__global__ void inst_params_kernel(IndexCtx C, int n_total) {
  const int ii = blockIdx.x * blockDim.x + threadIdx.x;
  if (ii >= n_total) return;
  const DInst x = C.insts[ii];
  InstParam ip;
  ip.sink = x.sink;
  ip.local = x.local;
  ip.s = ip.p = 0;
  ip.slash_word = ip.vmask_word = -1;
  ip.pad0 = ip.pad1 = 0;
  if (x.kind == MMI_PAT_GRID) {
    const GridRes g = C.gridres[x.grid_id];
    ip.s = g.s;
    ip.p = g.p;
  }
  if (x.kind == MMI_PAT_VSLASH) {
    ip.vmask_word = (int)C.vs_bits_off[x.vs_id * 2];
    ip.slash_word = (int)C.vs_bits_off[x.vs_id * 2 + 1];
  }
  C.inst_params[ii] = ip;
}

// ================================================================ items / segments
struct RowsInfo {
  int xp_lo, xp_hi;   // positions of first / last valid row
  int xr_lo, xr_hi;   // modality ranks (rank-coordinate views)
};
// rows of a work item: the pair (both halves, which fixes the key-tile ranges) and each half
// (which fixes the per-half tile states)
struct Rows {
  RowsInfo R;
  RowsInfo H[2];
  int nh;
};

struct Emitter {
  Seg* out;        // nullptr => count only
  int cap;         // segments `out` holds (further ones are counted, not written)
  int n_segs, n_tiles, n_live;  // n_live: live (tile, half) pairs
  __device__ __forceinline__ void add(int krow0, int ntiles, uint32_t meta, const int (&c)[2][5]) {
    if (ntiles <= 0) return;
    if (out && n_segs < cap) {
      Seg s;
      s.krow0 = krow0;
      s.ntiles = ntiles;
      s.meta = meta;
      s.pad = 0;
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        s.st[h][0] = (int16_t)c[h][0];
        s.st[h][1] = (int16_t)c[h][1];
        s.st[h][2] = (int16_t)c[h][3];
        s.st[h][3] = (int16_t)c[h][4];
      }
      out[n_segs] = s;
    }
    ++n_segs;
    n_tiles += ntiles;
    n_live += 2 * ntiles - c[0][0] - c[0][4] - c[1][0] - c[1][4];
  }
};

// Builds segments tile by tile: per half a phase automaton DEAD-head -> PRED-head -> FULL ->
// PRED-tail -> DEAD-tail (phases 0..4); a tile that would move a half backwards starts a new
// segment; a tile dead for both halves is dropped.
struct SegBuilder {
  int krow_t0, start, n;
  uint32_t meta;
  int ph[2];
  int c[2][5];
  bool open;
  __device__ __forceinline__ static int adv(int p, uint32_t st) {
    if (st == TS_DEAD) return p <= 0 ? 0 : 4;
    if (st == TS_PRED) return p <= 1 ? 1 : (p <= 3 ? 3 : -1);
    return p <= 2 ? 2 : -1;
  }
  __device__ __forceinline__ void flush(Emitter& E) {
    if (open && n > 0) E.add(krow_t0 + start * BLK, n, meta, c);
    open = false;
  }
  __device__ __forceinline__ void push(Emitter& E, int t, uint32_t s0, uint32_t s1) {
    if (s0 == TS_DEAD && s1 == TS_DEAD) {
      flush(E);
      return;
    }
    int n0 = -1, n1 = -1;
    if (open && n < SEG_MAX_TILES) {
      n0 = adv(ph[0], s0);
      n1 = adv(ph[1], s1);
    }
    if (n0 < 0 || n1 < 0) {
      flush(E);
      open = true;
      start = t;
      n = 0;
      ph[0] = ph[1] = 0;
#pragma unroll
      for (int h = 0; h < 2; ++h)
#pragma unroll
        for (int k = 0; k < 5; ++k) c[h][k] = 0;
      n0 = adv(0, s0);
      n1 = adv(0, s1);
    }
    ph[0] = n0;
    ph[1] = n1;
    c[0][n0]++;
    c[1][n1]++;
    ++n;
  }
};

// A K-view for emission: maps tile t -> coords / positions, krow.
struct KView {
  int kind;          // 0 ORIG K, 1 MOD region (rank coords), 2 class view (CLS / one RES class), 3 VCOL
  int space;
  int row0;          // K-space row of tile 0
  int base;          // ORIG: key position of index 0 (slash ranges start anywhere, even below 0)
  int n;             // valid keys
  int kv_base;       // ORIG: kv*S
  // class views
  int cls_r, cls_s;
  const int* pos_of_rank;  // MOD / rank-class: P_b (positions by rank), else nullptr
  const int* list;         // VCOL coords
  int list_rank;           // VCOL coords are ranks (use pos_of_rank)
  __device__ __forceinline__ int coord_at(int i) const {
    if (kind == 0) return base + i;
    if (kind == 1) return i;
    if (kind == 2) return cls_r + cls_s * i;
    return list[i];
  }
  __device__ __forceinline__ int pos_at(int i) const {
    const int c = coord_at(i);
    if (kind == 0) return c;  // (may be < 0 for a slash range: such keys are masked)
    if (kind == 1) return pos_of_rank[c];
    if (kind == 2) return pos_of_rank ? pos_of_rank[c] : c;
    return list_rank ? pos_of_rank[c] : c;
  }
};

// state of tile t of a K-view for the rows of one half (rows info R; `exists` false for an absent half)
__device__ __forceinline__ uint32_t tile_state(const KView& kv, int t, uint32_t role, int rmode, const RowsInfo& R,
                                               bool exists, int sink, int local, const int* sl = nullptr,
                                               int ns = 0) {
  if (!exists) return TS_DEAD;
  const int i0 = t * BLK, i1 = min(t * BLK + BLK - 1, kv.n - 1);
  const int yp_lo = kv.pos_at(i0), yp_hi = kv.pos_at(i1);
  if (yp_lo > R.xp_hi) return TS_DEAD;          // every key after every row of the half
  const int y_lo = rmode ? (kv.kind == 0 ? i0 : kv.coord_at(i0)) : yp_lo;
  const int y_hi = rmode ? (kv.kind == 0 ? i1 : kv.coord_at(i1)) : yp_hi;
  const int x_lo = rmode ? R.xr_lo : R.xp_lo;
  const int x_hi = rmode ? R.xr_hi : R.xp_hi;
  // the A part of a row x is y < sink or y > thr(x) (thr nondecreasing in x; a_thr, internal.h)
  if (role == R_A && y_lo >= sink && y_hi <= a_thr(x_lo, local)) return TS_DEAD;   // neither sink nor band
  if (role == R_NOTA && (y_hi < sink || y_lo > a_thr(x_hi, local))) return TS_DEAD;  // all inside the A part
  if (role == R_VSSL && sl) {
    // slash tile: live for the half iff some slash offset o = x - y joins one of its rows to one of
    // the tile's keys (the index keeps the offsets ascending)
    const int o_lo = max(x_lo - y_hi, 0), o_hi = x_hi - y_lo;
    const int q = lower_bound_i(sl, ns, o_lo);
    if (q >= ns || sl[q] > o_hi) return TS_DEAD;
  }
  const bool pads = (t * BLK + BLK - 1 >= kv.n);
  if (pads || yp_hi > R.xp_lo) return TS_PRED;  // pad keys / not causally full
  if (role == R_TRUE) return TS_FULL;
  if (role == R_VSSL) return TS_PRED;
  if (role == R_A) return ((y_hi < sink) || (y_lo > a_thr(x_hi, local))) ? TS_FULL : TS_PRED;
  return ((y_lo >= sink) && (y_hi <= a_thr(x_lo, local))) ? TS_FULL : TS_PRED;  // R_NOTA
}

// emit tiles [t0, t1) of a K-view (segments of per-half DEAD / PRED / FULL runs)
__device__ void emit_range(Emitter& E, const KView& kv, int t0, int t1, uint32_t role, int rmode, uint32_t inst,
                           const RowsInfo (&RH)[2], int nh, int sink, int local, const int* sl = nullptr,
                           int ns = 0) {
  SegBuilder b;
  b.open = false;
  b.krow_t0 = kv.row0;
  b.meta = seg_meta(kv.space, role, rmode, inst);
  for (int t = t0; t < t1; ++t)
    b.push(E, t, tile_state(kv, t, role, rmode, RH[0], true, sink, local, sl, ns),
           tile_state(kv, t, role, rmode, RH[1], nh > 1, sink, local, sl, ns));
  b.flush(E);
}

// tiles of a K-view whose key coordinate range intersects [c_lo, c_hi] (coords ascending)
__device__ __forceinline__ void coord_tiles(const KView& kv, int c_lo, int c_hi, int& t0, int& t1) {
  if (c_hi < c_lo || kv.n == 0) {
    t0 = t1 = 0;
    return;
  }
  int i_lo, i_hi;
  if (kv.kind == 0 || kv.kind == 1) {
    i_lo = max(c_lo, 0);
    i_hi = min(c_hi, kv.n - 1);
  } else if (kv.kind == 2) {
    i_lo = c_lo <= kv.cls_r ? 0 : cdiv(c_lo - kv.cls_r, kv.cls_s);
    i_hi = c_hi < kv.cls_r ? -1 : min((c_hi - kv.cls_r) / kv.cls_s, kv.n - 1);
  } else {
    i_lo = lower_bound_i(kv.list, kv.n, c_lo);
    i_hi = upper_bound_i(kv.list, kv.n, c_hi) - 1;
  }
  if (i_hi < i_lo) {
    t0 = t1 = 0;
    return;
  }
  t0 = i_lo / BLK;
  t1 = i_hi / BLK + 1;
}

// MOD region of modality b in POS coordinates (cross pairs): keys with position in [p_lo, p_hi]
__device__ __forceinline__ void pos_tiles_mod(const int* Pb, int nb_, int p_lo, int p_hi, int& t0, int& t1) {
  const int i_lo = lower_bound_i(Pb, nb_, p_lo);
  const int i_hi = upper_bound_i(Pb, nb_, p_hi) - 1;
  if (i_hi < i_lo) {
    t0 = t1 = 0;
    return;
  }
  t0 = i_lo / BLK;
  t1 = i_hi / BLK + 1;
}

struct ItemCtx {
  int h, kv;
  const DHead* hd;
};

// K-view of the pattern's key base (No/Q: original K; 2D: modality region kb)
__device__ KView base_kview(const IndexCtx& C, const ItemCtx& I, const DInst& x) {
  KView k;
  k.base = 0;
  k.cls_r = 0;
  k.cls_s = 1;
  k.list = nullptr;
  k.list_rank = 0;
  if (I.hd->boundary == MMI_BND_2D) {
    const int b = x.kb;
    k.kind = 1;
    k.space = 1;
    k.row0 = kview_row0(C, I.hd->kmod_view) + C.info[MI_PADOFF + b];
    k.n = C.info[MI_CNT + b];
    k.kv_base = 0;
    k.pos_of_rank = C.perm + C.info[MI_OFF + b];
  } else {
    k.kind = 0;
    k.space = 0;
    k.row0 = I.kv * C.S;
    k.n = C.S;
    k.kv_base = I.kv * C.S;
    k.pos_of_rank = nullptr;
  }
  return k;
}

// segments of one pattern instance for MAIN-type rows (and 2D cross pairs of HROW rows)
__device__ void emit_main(const IndexCtx& C, const ItemCtx& I, int ii, Emitter& E, const Rows& RW) {
  const RowsInfo& R = RW.R;
  const DInst x = C.insts[I.h * MAX_INST + ii];
  if (x.kind == MMI_PAT_NONE) return;
  KView kb = base_kview(C, I, x);
  const int rmode = x.rank;
  const bool cross_pos = (I.hd->boundary == MMI_BND_2D) && !x.rank;  // keys of modality kb, POS coords
  const int x_lo = rmode ? R.xr_lo : R.xp_lo;
  const int x_hi = rmode ? R.xr_hi : R.xp_hi;
  auto range_coords = [&](int c_lo, int c_hi, int& t0, int& t1) {
    if (cross_pos)
      pos_tiles_mod(kb.pos_of_rank, kb.n, c_lo, c_hi, t0, t1);
    else
      coord_tiles(kb, c_lo, c_hi, t0, t1);
  };
  if (x.kind == MMI_PAT_FULL) {
    int t0, t1;
    range_coords(0, x_hi, t0, t1);
    emit_range(E, kb, 0, t1, R_TRUE, rmode, ii, RW.H, RW.nh, 0, 0);
    return;
  }
  if (x.kind == MMI_PAT_ASHAPE || x.kind == MMI_PAT_GRID) {
    int a0, a1, b0, b1;
    range_coords(0, min(x.sink - 1, x_hi), a0, a1);
    range_coords(max(0, a_thr(x_lo, x.local) + 1), x_hi, b0, b1);
    if (a1 > a0 && b1 > b0 && b0 <= a1) {  // overlapping / adjacent -> one range
      emit_range(E, kb, min(a0, b0), max(a1, b1), R_A, rmode, ii, RW.H, RW.nh, x.sink, x.local);
    } else {
      if (a1 > a0) emit_range(E, kb, a0, a1, R_A, rmode, ii, RW.H, RW.nh, x.sink, x.local);
      if (b1 > b0) emit_range(E, kb, b0, b1, R_A, rmode, ii, RW.H, RW.nh, x.sink, x.local);
    }
    if (x.kind == MMI_PAT_GRID && (x.flags & GF_V)) {
      const GridRes g = C.gridres[x.grid_id];
      KView kc;
      kc.base = 0;
      kc.kind = 2;
      kc.space = 1;
      kc.row0 = kview_row0(C, x.v_cls_k);
      const int n = rmode ? C.info[MI_CNT + x.qa] : C.S;
      kc.n = g.p < n ? (n - g.p + g.s - 1) / g.s : 0;
      kc.cls_r = g.p;
      kc.cls_s = g.s;
      kc.pos_of_rank = rmode ? C.perm + C.info[MI_OFF + x.qa] : nullptr;
      kc.list = nullptr;
      kc.list_rank = 0;
      int t0, t1;
      coord_tiles(kc, 0, x_hi, t0, t1);
      emit_range(E, kc, 0, t1, R_NOTA, rmode, ii, RW.H, RW.nh, x.sink, x.local);
    }
    return;
  }
  if (x.kind == MMI_PAT_VSLASH) {
    const DView vv = C.views[x.v_vcol];
    KView kc;
    kc.base = 0;
    kc.kind = 3;
    kc.space = 1;
    kc.row0 = vv.row_off;
    kc.n = C.vs_cnt[x.vs_id * 2];
    kc.cls_r = 0;
    kc.cls_s = 1;
    kc.list = C.vs_lists + C.vs_list_off[x.vs_id * 2];
    kc.list_rank = rmode;
    kc.pos_of_rank = rmode ? C.perm + C.info[MI_OFF + x.qa] : nullptr;
    {
      // vertical columns: coords of the list (positions, or ranks in rank mode) <= x_hi
      int t0, t1;
      coord_tiles(kc, 0, cross_pos ? R.xp_hi : x_hi, t0, t1);
      emit_range(E, kc, 0, t1, R_TRUE, rmode, ii, RW.H, RW.nh, 0, 0);
    }
    if (!cross_pos) {
      // slash offsets: key coords [x_lo - o, x_hi - o]; the windows move left as o grows
      const int ns = C.vs_cnt[x.vs_id * 2 + 1];
      const int* sl = C.vs_lists + C.vs_list_off[x.vs_id * 2 + 1];
      if (kb.kind == 0) {
        // original K: tiles are anchored at the right end of each merged window range, so an
        // isolated offset costs one tile per half (its window, exactly) instead of two or three
        // 128-aligned tiles; a range's leftmost tile may start below key 0 (those keys are masked).
        // Ranges are disjoint: a window that reaches into the current range's tile span joins it.
        int rh = 0, rl = 0, qs = 0, qe = 0;  // current range: coords [rl, rh], offsets sl[qs..qe]
        bool have = false;
        auto flush = [&]() {
          const int nt = (rh - rl + BLK) / BLK;
          KView kt = kb;
          kt.base = rh - nt * BLK + 1;
          kt.row0 = kb.row0 + kt.base;
          kt.n = kb.n - kt.base;
          // the per-half states only need the range's own offsets (a short list)
          emit_range(E, kt, 0, nt, R_VSSL, rmode, ii, RW.H, RW.nh, 0, 0, sl + qs, qe - qs + 1);
        };
        for (int q = 0; q < ns; ++q) {
          const int o = sl[q];
          const int wh = x_hi - o;
          if (wh < 0) break;
          const int wl = x_lo - o;
          if (have) {
            const int tl = rh - ((rh - rl + BLK) / BLK) * BLK + 1;  // current leftmost tile start
            if (wh >= tl - 1) {
              rl = min(rl, wl);
              qe = q;
              continue;
            }
            flush();
          }
          rh = wh;
          rl = wl;
          qs = qe = q;
          have = true;
        }
        if (have) flush();
      } else {
        int cl = 0, ch = -1, qs = 0, qe = -1;
        for (int q = 0; q < ns; ++q) {
          const int o = sl[q];
          const int c_hi = x_hi - o;
          if (c_hi < 0) break;
          const int c_lo = max(0, x_lo - o);
          int t0, t1;
          coord_tiles(kb, c_lo, c_hi, t0, t1);
          if (t1 <= t0) continue;
          if (ch < cl) {
            cl = t0;
            ch = t1 - 1;
            qs = qe = q;
          } else if (t1 - 1 >= cl - 1) {
            cl = min(cl, t0);
            qe = q;
          } else {
            emit_range(E, kb, cl, ch + 1, R_VSSL, rmode, ii, RW.H, RW.nh, 0, 0, sl + qs, qe - qs + 1);
            cl = t0;
            ch = t1 - 1;
            qs = qe = q;
          }
        }
        if (ch >= cl) emit_range(E, kb, cl, ch + 1, R_VSSL, rmode, ii, RW.H, RW.nh, 0, 0, sl + qs, qe - qs + 1);
      }
    }
    return;
  }
}

// builds (or counts) one work-item slot
// Work order (ascending 32-bit key, stable): the L2 reuse of key tiles decides the kernel's DRAM
// traffic at 1M tokens, so items that read the same keys run at the same time:
//   class 0  very long items (>= LONG_LIVE live tile-halves), longest first (load balance);
//   class 1  h-row split-K chunks by (key chunk, KV group, row pair, head): every pair and every
//            h-line head of a group reads the same 65536 keys of a chunk;
//   class 2  MAIN items by (row position, head): the heads of a KV group share the band / sink tiles;
//   class 3  SLASH items by (head, residue class, pair): the pairs of a class share its K̄ tiles.
constexpr int LONG_LIVE = 4096;
__device__ __forceinline__ uint32_t order_key(uint32_t cls, uint32_t v) { return (cls << 30) | (v & 0x3FFFFFFFu); }

__device__ __forceinline__ int slot_pass(const IndexCtx& C, int slot) {
  int lo = 0, hi = C.n_passes - 1;
  while (lo < hi) {
    const int mid = (lo + hi + 1) >> 1;
    if (C.passes[mid].slot_base <= slot)
      lo = mid;
    else
      hi = mid - 1;
  }
  return lo;
}

__device__ void build_slot(const IndexCtx& C, int slot, Emitter& E, WorkItem& W, uint32_t& okey) {
  const DPass ps = C.passes[slot_pass(C, slot)];
  const int b = slot - ps.slot_base;
  ItemCtx I;
  I.h = ps.head;
  I.hd = &C.heads[ps.head];
  I.kv = I.hd->kv;
  const DHead& hd = *I.hd;
  W.head = I.h;
  W.q_row0 = 0;
  W.seg_off = 0;
  W.n_segs = 0;
  W.n_tiles = 0;
  W.q_gathered = 0;
  W.out_mode = OUT_FINAL;
  W.out_row0 = 0;
  W.inst_base = I.h * MAX_INST;
  W.skip_s = W.skip_p = W.skip_rank = 0;
  W.row_mod = -1;
  W.has_b = 0;
  W.pad[0] = W.pad[1] = 0;
  Rows RW;
  RowsInfo& R = RW.R;
  if (ps.pass == PASS_MAIN) {
    int grp;
    int row_in_view;  // first row of block A in the MAIN view (partial-buffer row)
    if (hd.qmod_view < 0) {
      const int p0 = 2 * b * BLK;
      if (p0 >= C.S) return;
      W.q_row0 = I.h * C.S + p0;
      W.has_b = (p0 + BLK < C.S) ? 1 : 0;
      for (int hf = 0; hf < 2; ++hf) {
        RW.H[hf].xp_lo = min(p0 + hf * BLK, C.S - 1);
        RW.H[hf].xp_hi = min(C.S, p0 + (hf + 1) * BLK) - 1;
        RW.H[hf].xr_lo = RW.H[hf].xr_hi = 0;
      }
      row_in_view = p0;
      grp = 0;
    } else {
      // pair b inside modality group m (blocks of a group never pair across groups)
      int k = b, a = -1, kk = 0, nblk = 0;
      for (int m = 0; m < MAX_MOD; ++m) {
        nblk = (C.info[MI_CNT + m] + BLK - 1) / BLK;
        const int pairs = (nblk + 1) / 2;
        if (k < pairs) {
          a = m;
          kk = k;
          break;
        }
        k -= pairs;
      }
      if (a < 0) return;
      const int i0 = C.info[MI_PADOFF + a] + 2 * kk * BLK;
      const int iend = C.info[MI_PADOFF + a] + C.info[MI_CNT + a] - 1;  // last valid row of the group
      W.q_row0 = C.views[hd.qmod_view].row_off + i0;
      W.q_gathered = 1;
      W.has_b = (2 * kk + 1 < nblk) ? 1 : 0;
      for (int hf = 0; hf < 2; ++hf) {
        const int lo = min(i0 + hf * BLK, iend), hi = min(i0 + (hf + 1) * BLK - 1, iend);
        RW.H[hf].xp_lo = C.modpos[lo];
        RW.H[hf].xp_hi = C.modpos[hi];
        RW.H[hf].xr_lo = C.rank[RW.H[hf].xp_lo];
        RW.H[hf].xr_hi = C.rank[RW.H[hf].xp_hi];
      }
      row_in_view = i0;
      grp = a;
    }
    RW.nh = W.has_b ? 2 : 1;
    R.xp_lo = RW.H[0].xp_lo;
    R.xr_lo = RW.H[0].xr_lo;
    R.xp_hi = RW.H[RW.nh - 1].xp_hi;
    R.xr_hi = RW.H[RW.nh - 1].xr_hi;
    // skip rows owned by the HROW pass; partial output when the group has a slash pass
    for (int ii = 0; ii < hd.n_inst; ++ii) {
      const DInst x = C.insts[I.h * MAX_INST + ii];
      const bool mine = (x.qa < 0) || (x.qa == grp && (x.kb < 0 || x.kb == grp));
      if (!mine || x.kind != MMI_PAT_GRID) continue;
      const GridRes g = C.gridres[x.grid_id];
      if (x.flags & GF_H) {
        W.skip_s = g.s;
        W.skip_p = g.p;
        W.skip_rank = x.rank;
      }
    }
    if (hd.sl_inst[grp] >= 0) {
      W.out_mode = OUT_PARTIAL;
      W.out_row0 = hd.part_rows0 + row_in_view;
    }
    W.pad[0] = R.xp_lo;
    okey = order_key(2, (uint32_t)(R.xp_lo / BLK) * 64u + (uint32_t)(I.h & 63));
    for (int ii = 0; ii < hd.n_inst; ++ii) {
      const DInst x = C.insts[I.h * MAX_INST + ii];
      if (x.qa >= 0 && x.qa != grp) continue;
      emit_main(C, I, ii, E, RW);
    }
  } else {
    const int ii = ps.inst;
    const DInst x = C.insts[I.h * MAX_INST + ii];
    const GridRes g = C.gridres[x.grid_id];
    const int n = x.rank ? C.info[MI_CNT + x.qa] : C.S;
    const int* P_a = x.rank ? C.perm + C.info[MI_OFF + x.qa] : nullptr;
    int r, t0, nr, chunk = 0;
    if (ps.pass == PASS_HROW) {
      // split-K (FlashDecoding-style, Alg.5 P:920-947 "sparse load in Q"): slot = (row pair, key chunk)
      const int n_split = ps.pad0;
      chunk = b % n_split;
      r = g.p;
      nr = r < n ? (n - r + g.s - 1) / g.s : 0;
      t0 = 2 * (b / n_split) * BLK;
      const DView qv = C.views[x.v_cls_q];
      W.q_row0 = qv.row_off + t0;
      W.out_mode = OUT_PARTIAL;
      W.out_row0 = x.pad[1] + chunk * qv.cap + t0;
      okey = order_key(1, ((uint32_t)min(chunk, 127) << 23) | ((uint32_t)(I.kv & 31) << 18) |
                              ((uint32_t)min(b / n_split, 4095) << 6) | (uint32_t)(I.h & 63));
    } else {
      // pair b inside residue class r: classes r < rem hold q+1 keys, the others q
      ClassGeo cg;
      cg.init(n, g.s);
      const int pa = ((cg.q + 1 + BLK - 1) / BLK + 1) / 2, pb = ((cg.q + BLK - 1) / BLK + 1) / 2;
      int kk;
      if (b < cg.rem * pa) {
        r = b / pa;
        kk = b % pa;
      } else {
        if (pb == 0) return;
        r = cg.rem + (b - cg.rem * pa) / pb;
        kk = (b - cg.rem * pa) % pb;
        if (r >= g.s) return;
      }
      if (r == g.p && (x.flags & (GF_H | GF_V))) return;  // class p owned by H / V passes (C9)
      nr = cg.nr(r);
      t0 = 2 * kk * BLK;
      okey = order_key(3, ((uint32_t)(I.h & 63) << 22) | ((uint32_t)min(r, 1023) << 12) | (uint32_t)min(kk, 4095));
      const int res_row = cg.classoff(r) + t0;
      const DView qv = C.views[x.v_res_q];
      W.q_row0 = qv.row_off + res_row;
      W.out_mode = OUT_PARTIAL;
      W.out_row0 = x.pad[0] + res_row;
    }
    if (t0 >= nr) return;
    W.has_b = (t0 + BLK < nr) ? 1 : 0;
    RW.nh = W.has_b ? 2 : 1;
    W.q_gathered = 1;
    W.row_mod = ps.qa;
    for (int hf = 0; hf < 2; ++hf) {
      const int ta = min(t0 + hf * BLK, nr - 1), tb = min(t0 + (hf + 1) * BLK - 1, nr - 1);
      const int ca = r + g.s * ta, cb = r + g.s * tb;
      if (x.rank) {
        RW.H[hf].xr_lo = ca;
        RW.H[hf].xr_hi = cb;
        RW.H[hf].xp_lo = P_a[ca];
        RW.H[hf].xp_hi = P_a[cb];
      } else {
        RW.H[hf].xp_lo = ca;
        RW.H[hf].xp_hi = cb;
        RW.H[hf].xr_lo = RW.H[hf].xr_hi = 0;
      }
    }
    R.xp_lo = RW.H[0].xp_lo;
    R.xr_lo = RW.H[0].xr_lo;
    R.xp_hi = RW.H[RW.nh - 1].xp_hi;
    R.xr_hi = RW.H[RW.nh - 1].xr_hi;
    const int c_hi = x.rank ? R.xr_hi : R.xp_hi;
    W.pad[0] = R.xp_lo;
    if (ps.pass == PASS_HROW) {
      // the whole causal row of the pattern's key base (role TRUE), key chunk `chunk`
      DInst xf = x;
      xf.kind = MMI_PAT_FULL;
      KView kb = base_kview(C, I, xf);
      int tt0, tt1;
      coord_tiles(kb, 0, c_hi, tt0, tt1);
      const int k0 = chunk * HROW_SPLIT_TILES, k1 = min(tt1, k0 + HROW_SPLIT_TILES);
      if (k0 >= k1) return;   // the rows of this pair are shorter than the chunk start
      emit_range(E, kb, k0, k1, R_TRUE, x.rank, ii, RW.H, RW.nh, 0, 0);
      if (hd.boundary == MMI_BND_2D && chunk == 0) {
        for (int jj = 0; jj < hd.n_inst; ++jj) {
          const DInst y = C.insts[I.h * MAX_INST + jj];
          if (y.qa == x.qa && y.kb != x.qa) emit_main(C, I, jj, E, RW);
        }
      }
    } else {
      // same residue class of the key base, causal, minus the A-part (role NOTA)
      ClassGeo cg;
      cg.init(n, g.s);
      KView kc;
      kc.base = 0;
      kc.kind = 2;
      kc.space = 1;
      kc.row0 = kview_row0(C, x.v_res_k) + cg.classoff(r);
      kc.n = nr;
      kc.cls_r = r;
      kc.cls_s = g.s;
      kc.pos_of_rank = P_a;
      kc.list = nullptr;
      kc.list_rank = 0;
      int tt0, tt1;
      coord_tiles(kc, 0, c_hi, tt0, tt1);
      emit_range(E, kc, 0, tt1, R_NOTA, x.rank, ii, RW.H, RW.nh, x.sink, x.local);
    }
  }
}

// One pass over the slots: a slot writes its segments straight into its static region of the pass
// (seg_base + b * seg_per_slot, the plan's analytic per-slot bound), so no count pass and no scan.
// A slot whose bound is short (counted while writing) is rebuilt into the spill area; only if
// that is full too is the item left empty and FLAG_SEG_OVERFLOW raised.
__global__ void items_fill_kernel(IndexCtx C) {
  const int slot = blockIdx.x * blockDim.x + threadIdx.x;
  if (slot >= C.n_slots) return;
  const DPass ps = C.passes[slot_pass(C, slot)];
  int off = ps.seg_base + (slot - ps.slot_base) * ps.seg_per_slot;
  Emitter E;
  E.out = C.segs + off;
  E.cap = ps.seg_per_slot;
  E.n_segs = E.n_tiles = E.n_live = 0;
  WorkItem W;
  uint32_t okey = 0;
  build_slot(C, slot, E, W, okey);
  if (E.n_segs > E.cap) {
    const int need = E.n_segs;
    const unsigned long long sp = atomicAdd(reinterpret_cast<unsigned long long*>(C.seg_cnt), (unsigned long long)need);
    if ((long long)sp + need <= C.seg_spill_cap) {
      off = (int)(C.seg_spill_base + (long long)sp);
      E.out = C.segs + off;
      E.cap = need;
      E.n_segs = E.n_tiles = E.n_live = 0;
      okey = 0;
      build_slot(C, slot, E, W, okey);
    }
  }
  if (E.n_segs > E.cap) {
    // static region and spill area both short: the item stays empty (its rows are not computed)
    // and mmi_workspace_flags reports it
    atomicOr(C.flags, FLAG_SEG_OVERFLOW);
    W.seg_off = off;
    W.n_segs = W.n_tiles = 0;
    W.pad[1] = 0;
    C.items[slot] = W;
    C.sort_keys[slot] = (int)0xFFFFFFFFu;
    C.sort_vals[slot] = slot;
    return;
  }
  W.seg_off = off;
  W.n_segs = E.n_segs;
  W.n_tiles = E.n_tiles;
  W.pad[1] = E.n_live;
  C.items[slot] = W;
  // work order (see order_key); empty items last (the kernel stops at the first one)
  uint32_t key = 0xFFFFFFFFu;
#ifdef MMI_ORDER_LPT  // round-1 order (A/B experiments): long items by length, others by position
  if (E.n_live >= 96)
    key = ~(uint32_t)(0x40000000 + E.n_live);
  else if (E.n_tiles > 0)
    key = ~(uint32_t)(0x3FFFFFFF - ((W.pad[0] / BLK) * 64 + (W.head & 63)));
#else
  if (E.n_live >= LONG_LIVE)
    key = order_key(0, 0x3FFFFFFFu - (uint32_t)E.n_live);
  else if (E.n_tiles > 0)
    key = okey;
#endif
  C.sort_keys[slot] = (int)key;
  C.sort_vals[slot] = slot;
}

__global__ void items_gather_kernel(IndexCtx C) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= C.n_slots) return;
  C.items_sorted[i] = C.items[C.sort_vals_out[i]];
}

// ================================================================ permute (a6)
template <int D>
__global__ void gather_rows_kernel(const int* __restrict__ src, int64_t rows, const __nv_bfloat16* __restrict__ a,
                                   __nv_bfloat16* __restrict__ a_out, const __nv_bfloat16* __restrict__ b,
                                   __nv_bfloat16* __restrict__ b_out) {
  constexpr int V = D / 8;  // uint4 per row
  const int64_t gid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t row = gid / V;
  const int c = (int)(gid % V);
  if (row >= rows) return;
  const int s = src[row];
  if (s == -2) return;  // beyond the view's length: never read
  uint4 va = make_uint4(0, 0, 0, 0), vb = make_uint4(0, 0, 0, 0);
  if (s >= 0) {
    va = __ldg(reinterpret_cast<const uint4*>(a + (size_t)s * D) + c);
    if (b) vb = __ldg(reinterpret_cast<const uint4*>(b + (size_t)s * D) + c);
  }
  reinterpret_cast<uint4*>(a_out + (size_t)row * D)[c] = va;
  if (b) reinterpret_cast<uint4*>(b_out + (size_t)row * D)[c] = vb;
}

// ================================================================ merge (a8)
// One warp merges MERGE_R = 32 rows: lane r resolves row r's metadata (a chain of dependent
// loads: modality position, instance, grid result, residue-class offset), then the rows' data
// move in batches of MERGE_B rows whose partial-row loads are all issued before any use; each
// lane owns CPL contiguous columns (D = 32 CPL), so a row is one 32-lane vector access.
constexpr int MERGE_R = 32;
constexpr int MERGE_B = 8;
template <int CPL>
__global__ void merge_kernel(IndexCtx C, const int* __restrict__ heads_list, int n_rows,
                             __nv_bfloat16* __restrict__ o, float* __restrict__ lse) {
  constexpr int D = 32 * CPL;
  const int warp_g = (blockIdx.x * blockDim.x + threadIdx.x) / 32;
  const int lane = threadIdx.x % 32;
  const int i_base = warp_g * MERGE_R;
  if (i_base >= n_rows) return;
  const int h = heads_list[blockIdx.y];
  const DHead hd = C.heads[h];
  int pos = -1;
  long long j0 = -1, j1 = -1;
  float w0 = 0.f, w1 = 0.f, inv = 0.f, lsev = -INFINITY;
  if (lane < MERGE_R && i_base + lane < n_rows) {
    const int i = i_base + lane;
    int grp = 0;
    bool ok = true;
    if (hd.qmod_view < 0) {
      pos = i;
      ok = pos < C.S;
    } else {
      ok = i < C.info[MI_PADOFF + MAX_MOD];
      pos = ok ? C.modpos[i] : -1;
      ok = ok && pos >= 0;
      if (ok) grp = C.labels[pos];
    }
    const int gi = ok ? hd.sl_inst[grp] : -1;
    if (gi >= 0) {
      const DInst x = C.insts[h * MAX_INST + gi];
      const GridRes g = C.gridres[x.grid_id];
      const int coord = x.rank ? C.rank[pos] : pos;
      const int r = coord % g.s;
      if ((x.flags & GF_H) && hline_row(coord, g.s, g.p)) {
        pos = -1;  // written by the HROW pass
      } else {
        // a partial row whose work item had no live tile was never written: its LSE is the NaN
        // fill of mmi_sparse_prefill and it contributes nothing (its O row is not read)
        j0 = hd.part_rows0 + i;
        float l0 = C.part_lse[j0];
        if (!(l0 > -INFINITY)) {
          l0 = -INFINITY;
          j0 = -1;
        }
        float l1 = -INFINITY;
        if (!(r == g.p && (x.flags & (GF_H | GF_V)))) {
          ClassGeo cg;
          cg.init(x.rank ? C.info[MI_CNT + x.qa] : C.S, g.s);
          j1 = x.pad[0] + cg.classoff(r) + coord / g.s;
          l1 = C.part_lse[j1];
          if (!(l1 > -INFINITY)) {
            l1 = -INFINITY;
            j1 = -1;
          }
        }
        const float m = fmaxf(l0, l1);
        w0 = (l0 == -INFINITY) ? 0.f : __expf(l0 - m);
        w1 = (l1 == -INFINITY) ? 0.f : __expf(l1 - m);
        const float tot = w0 + w1;
        inv = tot > 0.f ? 1.f / tot : 0.f;
        lsev = tot > 0.f ? m + __logf(tot) : -INFINITY;
      }
    } else {
      pos = -1;
    }
  }
  using VH = typename std::conditional<CPL == 4, uint2, uint32_t>::type;  // CPL fp16 / bf16 values
#pragma unroll 1
  for (int r0 = 0; r0 < MERGE_R; r0 += MERGE_B) {
    VH a[MERGE_B], b[MERGE_B];
#pragma unroll
    for (int r = 0; r < MERGE_B; ++r) {
      const int p = __shfl_sync(0xffffffffu, pos, r0 + r);
      const long long q0 = __shfl_sync(0xffffffffu, j0, r0 + r), q1 = __shfl_sync(0xffffffffu, j1, r0 + r);
      a[r] = VH{};
      b[r] = VH{};
      if (p >= 0) {
        if (q0 >= 0) a[r] = *reinterpret_cast<const VH*>(C.part_o + q0 * D + CPL * lane);
        if (q1 >= 0) b[r] = *reinterpret_cast<const VH*>(C.part_o + q1 * D + CPL * lane);
      }
    }
#pragma unroll
    for (int r = 0; r < MERGE_B; ++r) {
      const int p = __shfl_sync(0xffffffffu, pos, r0 + r);
      const float x0 = __shfl_sync(0xffffffffu, w0, r0 + r), x1 = __shfl_sync(0xffffffffu, w1, r0 + r);
      const float xi = __shfl_sync(0xffffffffu, inv, r0 + r);
      if (p < 0) continue;
      const __half2* ha = reinterpret_cast<const __half2*>(&a[r]);
      const __half2* hb = reinterpret_cast<const __half2*>(&b[r]);
      VH out;
      __nv_bfloat162* ob = reinterpret_cast<__nv_bfloat162*>(&out);
#pragma unroll
      for (int c = 0; c < CPL / 2; ++c) {
        const float2 fa = __half22float2(ha[c]), fb = __half22float2(hb[c]);
        ob[c] = __floats2bfloat162_rn((fa.x * x0 + fb.x * x1) * xi, (fa.y * x0 + fb.y * x1) * xi);
      }
      *reinterpret_cast<VH*>(o + ((size_t)h * C.S + p) * D + CPL * lane) = out;
    }
  }
  if (lane < MERGE_R && pos >= 0 && lse) lse[(size_t)h * C.S + pos] = lsev;
}

// ================================================================ split-K merge of h-line rows (a8)
// One warp per h-line row: the row's key chunks c = 0 .. x_tile / HROW_SPLIT_TILES (every chunk that
// holds one of its causal keys; later chunks hold none) are LSE-merged (Alg.5 P:940-942 rescaling,
// generalised to n partials) in fp32 and written to token order.
template <int CPL>
__global__ void hrow_merge_kernel(IndexCtx C, const DHrow* __restrict__ hrows, int max_rows,
                                  __nv_bfloat16* __restrict__ o, float* __restrict__ lse) {
  constexpr int D = 32 * CPL;
  const DHrow hr = hrows[blockIdx.y];
  const int i = (blockIdx.x * blockDim.x + threadIdx.x) / 32;
  const int lane = threadIdx.x % 32;
  const DInst x = C.insts[hr.head * MAX_INST + hr.inst];
  const DView qv = C.views[x.v_cls_q];
  if (i >= max_rows || i >= qv.cap) return;
  const int pos = C.qg_pos[qv.row_off + i];
  if (pos < 0 || pos >= C.S) return;
  if (hr.qa >= 0 && C.labels[pos] != hr.qa) return;   // Q-boundary: a row of another modality
  const GridRes g = C.gridres[x.grid_id];
  const int coord = g.p + g.s * i;                      // key-base coordinate (position or rank)
  const int nc = min(coord / BLK / HROW_SPLIT_TILES + 1, hr.n_split);
  const long long base = x.pad[1] + i;
  float m = -INFINITY;
  for (int c = lane; c < nc; c += 32) {
    const float l = C.part_lse[base + (long long)c * qv.cap];
    if (l > -INFINITY) m = fmaxf(m, l);
  }
#pragma unroll
  for (int off = 16; off; off >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, off));
  float acc[CPL];
#pragma unroll
  for (int k = 0; k < CPL; ++k) acc[k] = 0.f;
  float wsum = 0.f;
  for (int c = 0; c < nc; ++c) {
    const long long row = base + (long long)c * qv.cap;
    const float l = C.part_lse[row];
    if (!(l > -INFINITY)) continue;  // empty chunk for this row (or never written: NaN fill)
    const float w = __expf(l - m);
    wsum += w;
    const __half* src = C.part_o + row * D + CPL * lane;
#pragma unroll
    for (int k = 0; k < CPL; k += 2) {
      const float2 f = __half22float2(*reinterpret_cast<const __half2*>(src + k));
      acc[k] += w * f.x;
      acc[k + 1] += w * f.y;
    }
  }
  const float inv = wsum > 0.f ? 1.f / wsum : 0.f;
  __nv_bfloat16* dst = o + ((size_t)hr.head * C.S + pos) * D + CPL * lane;
#pragma unroll
  for (int k = 0; k < CPL; k += 2)
    *reinterpret_cast<__nv_bfloat162*>(dst + k) = __floats2bfloat162_rn(acc[k] * inv, acc[k + 1] * inv);
  if (lse && lane == 0) lse[(size_t)hr.head * C.S + pos] = wsum > 0.f ? m + __logf(wsum) : -INFINITY;
}

// ================================================================ launchers
void launch_hrow_merge(const IndexCtx& C, int D, const DHrow* hrows, int n_hrows, int max_rows, void* o, float* lse,
                       cudaStream_t st) {
  if (n_hrows <= 0 || max_rows <= 0) return;
  const dim3 grid((unsigned)((max_rows * 32 + 255) / 256), n_hrows);
  if (D == 128)
    hrow_merge_kernel<4><<<grid, 256, 0, st>>>(C, hrows, max_rows, (__nv_bfloat16*)o, lse);
  else
    hrow_merge_kernel<2><<<grid, 256, 0, st>>>(C, hrows, max_rows, (__nv_bfloat16*)o, lse);
}
void launch_build_views(const IndexCtx& C, const int* qviews, int nq, const int* kviews, int nk, int64_t qrows,
                        int64_t krows, cudaStream_t st) {
  const int nv = nq + nk;
  if (nv > 0) view_alias_kernel<<<(nv + 127) / 128, 128, 0, st>>>(C, nv);
  if (qrows > 0) build_views_kernel<<<(unsigned)((qrows + 255) / 256), 256, 0, st>>>(C, 0, qviews, nq, qrows);
  if (krows > 0) build_views_kernel<<<(unsigned)((krows + 255) / 256), 256, 0, st>>>(C, 1, kviews, nk, krows);
}
void launch_inst_params(const IndexCtx& C, int n_total, cudaStream_t st) {
  inst_params_kernel<<<(n_total + 127) / 128, 128, 0, st>>>(C, n_total);
}
void launch_items_fill(const IndexCtx& C, cudaStream_t st) {
  items_fill_kernel<<<(C.n_slots + 127) / 128, 128, 0, st>>>(C);
}
void launch_items_gather(const IndexCtx& C, cudaStream_t st) {
  items_gather_kernel<<<(C.n_slots + 127) / 128, 128, 0, st>>>(C);
}
void launch_gather(const int* src, int64_t rows, int D, const void* a, void* a_out, const void* b, void* b_out,
                   cudaStream_t st) {
  if (rows <= 0) return;
  const int64_t threads = rows * (D / 8);
  const unsigned grid = (unsigned)((threads + 255) / 256);
  if (D == 128)
    gather_rows_kernel<128><<<grid, 256, 0, st>>>(src, rows, (const __nv_bfloat16*)a, (__nv_bfloat16*)a_out,
                                                  (const __nv_bfloat16*)b, (__nv_bfloat16*)b_out);
  else
    gather_rows_kernel<64><<<grid, 256, 0, st>>>(src, rows, (const __nv_bfloat16*)a, (__nv_bfloat16*)a_out,
                                                 (const __nv_bfloat16*)b, (__nv_bfloat16*)b_out);
}
void launch_merge(const IndexCtx& C, int D, const int* heads_list, int n_heads, int n_rows, void* o, float* lse,
                  cudaStream_t st) {
  if (n_rows <= 0 || n_heads <= 0) return;
  const long long threads = (long long)((n_rows + MERGE_R - 1) / MERGE_R) * 32;
  const dim3 grid((unsigned)((threads + 255) / 256), n_heads);
  if (D == 128)
    merge_kernel<4><<<grid, 256, 0, st>>>(C, heads_list, n_rows, (__nv_bfloat16*)o, lse);
  else
    merge_kernel<2><<<grid, 256, 0, st>>>(C, heads_list, n_rows, (__nv_bfloat16*)o, lse);
}

}  // namespace mmi
