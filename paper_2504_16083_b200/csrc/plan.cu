// Host planner: validation of the per-head configs and the workspace layout.
#include <algorithm>
#include <cstdio>
#include <climits>
#include <cstring>

#include "plan.h"
#include "sort.h"
#include "estimate.h"

namespace mmi {

static inline int64_t pad128(int64_t x) { return (x + 127) / 128 * 128; }
static inline size_t align256(size_t x) { return (x + 255) / 256 * 256; }

static bool needs_est(const mmi_pattern& p) { return p.kind == MMI_PAT_VSLASH || p.kind == MMI_PAT_GRID; }

static mmi_status check_pattern(const mmi_pattern& p, bool cross, int h, const char* where, std::string& err) {
  char buf[256];
  auto bad = [&](mmi_status st, const char* msg) {
    snprintf(buf, sizeof(buf), "head %d %s: %s", h, where, msg);
    err = buf;
    return st;
  };
  switch (p.kind) {
    case MMI_PAT_NONE:
    case MMI_PAT_FULL:
      return MMI_OK;
    case MMI_PAT_ASHAPE:
      if (p.local < 1 || p.sink < 0) return bad(MMI_E_CONFIG, "A-shape needs local >= 1, sink >= 0");
      return MMI_OK;
    case MMI_PAT_VSLASH:
      if (p.n_vertical < 1) return bad(MMI_E_CONFIG, "vertical-slash needs n_vertical >= 1");
      if (cross && p.n_slash != 0) return bad(MMI_E_CONFIG, "cross-modality vertical-slash must have n_slash = 0");
      if (!cross && p.n_slash < 1) return bad(MMI_E_CONFIG, "vertical-slash needs n_slash >= 1");
      return MMI_OK;
    case MMI_PAT_GRID:
      if (cross) return bad(MMI_E_CONFIG, "grid pattern on a cross-modality pair");
      if (p.local < 1 || p.sink < 0) return bad(MMI_E_CONFIG, "grid needs local >= 1, sink >= 0");
      if (p.stride < 0) return bad(MMI_E_CONFIG, "grid stride < 0");
      if (p.stride > 1024) return bad(MMI_E_UNSUPPORTED, "grid stride > 1024");
      if (p.stride == 0 && (p.stride_min < 1 || p.stride_max < p.stride_min || p.stride_max > 1024))
        return bad(MMI_E_CONFIG, "searched grid needs 1 <= stride_min <= stride_max <= 1024");
      return MMI_OK;
    case MMI_PAT_TRISHAPE:
      if (cross) return bad(MMI_E_CONFIG, "tri-shape on a cross-modality pair");
      if (p.local < 1 || p.sink < 0 || p.bottom < 0) return bad(MMI_E_CONFIG, "tri-shape needs local >= 1, sink >= 0, bottom >= 0");
      return MMI_OK;
    case MMI_PAT_SF_FIXED:
    case MMI_PAT_SF_STRIDED:
      if (cross) return bad(MMI_E_CONFIG, "SparseTransformer pattern on a cross-modality pair");
      if (p.local < 1) return bad(MMI_E_CONFIG, "SparseTransformer pattern needs local >= 1");
      if (p.stride < 1 || p.stride > 1024) return bad(MMI_E_UNSUPPORTED, "SparseTransformer stride not in [1, 1024]");
      return MMI_OK;
    default:
      return bad(MMI_E_INVALID, "unknown pattern kind");
  }
}

// the static baselines execute as grids with a fixed (stride, phase) and no estimation:
//   TRISHAPE(sink, local, bottom) -> h-lines on the rows x >= S - bottom (stride 1, phase S - bottom)
//   SF_FIXED(l, stride)           -> v-lines y = 0 (mod stride), A part = the query's l-key segment
//   SF_STRIDED(l, stride)         -> slash lines (x - y) = 0 (mod stride), A part = local window l
static mmi_pattern as_grid(const mmi_pattern& p, int S, int& stat, int& stat_p) {
  stat = 0;
  stat_p = 0;
  if (p.kind < MMI_PAT_TRISHAPE) return p;
  mmi_pattern g = p;
  g.kind = MMI_PAT_GRID;
  g.use_hline = g.use_vline = g.use_slash = 0;
  stat = 1;
  if (p.kind == MMI_PAT_TRISHAPE) {
    g.stride = 1;
    g.use_hline = 1;
    stat_p = std::max(0, S - p.bottom);
  } else {
    g.sink = 0;
    if (p.kind == MMI_PAT_SF_FIXED) {
      g.use_vline = 1;
      g.local = -p.local;  // block mode
    } else {
      g.use_slash = 1;
    }
  }
  g.stride_min = g.stride_max = g.stride;
  return g;
}

mmi_status build_plan(const mmi_problem* pb, const mmi_head_config* cfg, Plan& P, std::string& err) {
  if (!cfg) {
    err = "cfg_host is NULL";
    return MMI_E_INVALID;
  }
  P = Plan();
  P.pb = *pb;
  P.H = pb->n_heads;
  P.Hkv = pb->n_kv_heads;
  P.S = pb->seq_len;
  P.D = pb->head_dim;
  P.M = pb->n_modalities;
  P.nb = (P.S + BLK - 1) / BLK;
  P.S_pad = (int)pad128(P.S) + BLK;
  const int H = P.H, S = P.S, M = P.M;
  const int G = P.H / P.Hkv;
  const int64_t mod_cap = pad128((int64_t)S + (int64_t)M * BLK);  // padded modality-grouped view
  const int nbk_max = (int)(mod_cap / BLK);

  // ---------------- validation ----------------
  for (int h = 0; h < H; ++h) {
    const mmi_head_config& c = cfg[h];
    mmi_status st;
    if (c.boundary == MMI_BND_NONE || c.boundary == MMI_BND_K) {
      if (c.intra[0].kind == MMI_PAT_NONE) {
        err = "head " + std::to_string(h) + ": intra[0] is NONE (rows would have no keys)";
        return MMI_E_CONFIG;
      }
      if ((st = check_pattern(c.intra[0], false, h, "intra[0]", err)) != MMI_OK) return st;
    } else if (c.boundary == MMI_BND_Q || c.boundary == MMI_BND_2D) {
      for (int a = 0; a < M; ++a)
        for (int b = 0; b < M; ++b)
          if ((c.boundary == MMI_BND_Q ? (b == 0 ? c.intra[a].kind : 0) : c.pair[a][b].kind) == MMI_PAT_TRISHAPE) {
            err = "head " + std::to_string(h) + ": tri-shape is supported on No/K-boundary heads only";
            return MMI_E_CONFIG;
          }
    }
    if (c.boundary == MMI_BND_NONE || c.boundary == MMI_BND_K) {
    } else if (c.boundary == MMI_BND_Q) {
      for (int m = 0; m < M; ++m) {
        if (c.intra[m].kind == MMI_PAT_NONE) {
          err = "head " + std::to_string(h) + ": Q-boundary intra[" + std::to_string(m) + "] is NONE";
          return MMI_E_CONFIG;
        }
        if ((st = check_pattern(c.intra[m], false, h, "intra", err)) != MMI_OK) return st;
      }
    } else if (c.boundary == MMI_BND_2D) {
      for (int a = 0; a < M; ++a)
        for (int b = 0; b < M; ++b) {
          if (a == b && c.pair[a][a].kind == MMI_PAT_NONE) {
            err = "head " + std::to_string(h) + ": 2D pair[a][a] is NONE";
            return MMI_E_CONFIG;
          }
          if ((st = check_pattern(c.pair[a][b], a != b, h, "pair", err)) != MMI_OK) return st;
        }
    } else {
      err = "head " + std::to_string(h) + ": unknown boundary";
      return MMI_E_INVALID;
    }
  }

  // ---------------- instances, slabs, views ----------------
  P.heads.resize(H);
  P.insts.assign((size_t)H * MAX_INST, DInst{});
  for (auto& x : P.insts) {
    x.kind = MMI_PAT_NONE;
    x.slab = x.grid_id = x.vs_id = -1;
    x.v_cls_q = x.v_res_q = x.v_cls_k = x.v_res_k = x.v_vcol = -1;
    x.qa = x.kb = -1;
  }
  int64_t qrow = 0, krow = 0;
  auto add_view = [&](int kind, int space, int64_t cap, int head, int inst, int mod, int classes) {
    DView v;
    v.kind = kind;
    v.space = space;
    v.cap = (int32_t)std::min<int64_t>(pad128(cap), INT32_MAX / 2);
    v.row_off = (int32_t)std::min<int64_t>(space == 0 ? qrow : krow, INT32_MAX / 2);
    v.head = head;
    v.inst = inst;
    v.mod = mod;
    v.classes = classes;
    if (space == 0)
      qrow += v.cap;
    else
      krow += v.cap;
    P.views.push_back(v);
    return (int)P.views.size() - 1;
  };
  int64_t part_rows = 0;
  for (int h = 0; h < H; ++h) {
    const mmi_head_config& c = cfg[h];
    DHead& hd = P.heads[h];
    memset(&hd, 0, sizeof(hd));
    hd.boundary = c.boundary;
    hd.inst_base = h * MAX_INST;
    hd.kv = h / G;
    hd.qmod_view = hd.kmod_view = -1;
    hd.part_rows0 = hd.part_rows1 = -1;
    for (int a = 0; a < MAX_MOD; ++a) hd.sl_inst[a] = -1;
    const bool modq = (c.boundary == MMI_BND_Q || c.boundary == MMI_BND_2D);
    if (modq) hd.qmod_view = add_view(VK_MOD, 0, mod_cap, h, -1, -1, 0);
    if (c.boundary == MMI_BND_2D) hd.kmod_view = add_view(VK_MOD, 1, mod_cap, h, -1, -1, 0);
    int slab_of_group[MAX_MOD] = {-1, -1, -1, -1};
    int n = 0;
    auto add_inst = [&](const mmi_pattern& p_in, int qa, int kb, int rank) {
      int stat = 0, stat_p = 0;
      const mmi_pattern p = as_grid(p_in, S, stat, stat_p);
      DInst& x = P.insts[(size_t)h * MAX_INST + n];
      x.stat = stat;
      x.stat_p = stat_p;
      x.kind = p.kind;
      x.rank = rank;
      x.qa = qa;
      x.kb = kb;
      x.sink = p.sink;
      x.local = p.local;
      x.n_v = p.n_vertical;
      x.n_s = p.n_slash;
      x.stride = p.stride;
      x.smin = p.stride > 0 ? p.stride : p.stride_min;
      x.smax = p.stride > 0 ? p.stride : p.stride_max;
      x.flags = (p.use_hline ? GF_H : 0) | (p.use_vline ? GF_V : 0) | (p.use_slash ? GF_SL : 0);
      x.force = (kb < 0 || qa == kb) ? 1 : 0;
      const int grp = qa < 0 ? 0 : qa;
      if (needs_est(p) && !stat) {
        if (slab_of_group[grp] < 0) {
          DSlab sl;
          memset(&sl, 0, sizeof(sl));
          sl.head = h;
          sl.kv = h / G;
          sl.qmod = qa;
          sl.rank_mode = (c.boundary == MMI_BND_2D) ? 1 : 0;
          P.slabs.push_back(sl);
          slab_of_group[grp] = (int)P.slabs.size() - 1;
        }
        x.slab = slab_of_group[grp];
        if (p.kind == MMI_PAT_VSLASH && p.n_slash > 0) P.slabs[x.slab].need_dg = 1;
      }
      // base size of the class views: S (original coordinates) or S (upper bound of n_a, rank coordinates)
      const int64_t nbase = S;
      if (p.kind == MMI_PAT_GRID) {
        x.grid_id = P.n_grid++;
        const int vk = rank ? VK_RANK_CLASS : VK_ORIG_CLASS;
        // class-p views: every (S - p) / s rows; a static grid knows its phase (tri-shape: the
        // bottom rows only)
        const int64_t cls_n = stat ? std::max<int64_t>(0, (nbase - stat_p + x.smin - 1) / x.smin)
                                   : (nbase + x.smin - 1) / x.smin;
        const int64_t cls_cap = pad128(cls_n) + BLK;
        const int64_t res_cap = pad128(nbase + (int64_t)x.smax * BLK) + BLK;
        if (p.use_hline) x.v_cls_q = add_view(vk, 0, cls_cap, h, n, rank ? qa : -1, 1);
        if (p.use_slash) x.v_res_q = add_view(vk, 0, res_cap, h, n, rank ? qa : -1, 0);
        if (p.use_vline) x.v_cls_k = add_view(vk, 1, cls_cap, h, n, rank ? qa : -1, 1);
        if (p.use_slash) x.v_res_k = add_view(vk, 1, res_cap, h, n, rank ? qa : -1, 0);
        if (p.use_slash) {
          hd.sl_inst[grp] = n;
          x.pad[0] = (int32_t)part_rows;  // partial slot-1 rows (RES_Q layout)
          part_rows += P.views[x.v_res_q].cap;
        }
      } else if (p.kind == MMI_PAT_VSLASH) {
        x.vs_id = P.n_vs++;
        P.vs_nv.push_back(p.n_vertical);
        P.vs_ns.push_back(p.n_slash);
        x.v_vcol = add_view(VK_VCOL, 1, pad128(p.n_vertical) + BLK, h, n, rank ? qa : -1, 0);
      }
      ++n;
    };
    if (c.boundary == MMI_BND_NONE || c.boundary == MMI_BND_K) {
      add_inst(c.intra[0], -1, -1, 0);
    } else if (c.boundary == MMI_BND_Q) {
      for (int m = 0; m < M; ++m) add_inst(c.intra[m], m, -1, 0);
    } else {
      for (int a = 0; a < M; ++a)
        for (int b = 0; b < M; ++b)
          if (c.pair[a][b].kind != MMI_PAT_NONE) add_inst(c.pair[a][b], a, b, a == b ? 1 : 0);
    }
    hd.n_inst = n;
    bool any_sl = false;
    for (int a = 0; a < MAX_MOD; ++a) any_sl |= hd.sl_inst[a] >= 0;
    if (any_sl) {
      hd.part_rows0 = (int32_t)part_rows;
      part_rows += modq ? mod_cap : (int64_t)P.nb * BLK;
    }
  }
  P.part_rows = part_rows;
  for (size_t i = 0; i < P.slabs.size(); ++i) {
    P.slabs[i].c_off = (int64_t)i * P.S_pad;
    P.slabs[i].dg_off = (int64_t)i * P.S_pad;
  }
  // slab kernels: slabs whose diagonal mass is needed run in slab_kernel (batches of 4 per KV
  // group); the others are packed two per tcgen05 M=128 tile (same KV group)
  {
    std::vector<int> dg_per_kv(P.Hkv, 0);
    for (int kv = 0; kv < P.Hkv; ++kv) {
      int pending = -1;
      for (size_t i = 0; i < P.slabs.size(); ++i) {
        if (P.slabs[i].kv != kv) continue;
        if (P.slabs[i].need_dg) {
          dg_per_kv[kv]++;
          continue;
        }
        if (pending < 0) {
          pending = (int)i;
        } else {
          P.stc_pairs.push_back(pending);
          P.stc_pairs.push_back((int)i);
          pending = -1;
        }
      }
      if (pending >= 0) {
        P.stc_pairs.push_back(pending);
        P.stc_pairs.push_back(-1);
      }
    }
    for (int c : dg_per_kv) P.n_dg_batch = std::max(P.n_dg_batch, (c + 3) / 4);
    const int n_old = (S + SLAB_CHUNK - 1) / SLAB_CHUNK;
    const int n_tc = slab_tc_chunks(S);
    for (auto& sl : P.slabs) sl.n_chunks = sl.need_dg ? n_old : n_tc;
  }
  P.qg_rows = qrow + BLK;
  P.kg_rows = krow + BLK;

  // ---------------- passes and segment capacity ----------------
  auto segbound = [&](const DInst& x) -> int64_t {
    switch (x.kind) {
      case MMI_PAT_FULL: return 1;
      case MMI_PAT_ASHAPE: return 2;
      case MMI_PAT_GRID: return 3;
      case MMI_PAT_VSLASH: return 1 + std::min<int64_t>(2 * (int64_t)x.n_s + 2, nbk_max / 2 + 2);
      default: return 0;
    }
  };
  int slot = 0;
  int64_t segcap = 0;
  int64_t part_rows_hrow_cursor = P.part_rows;  // HROW split-K partial rows follow the MAIN / SLASH ones
  for (int h = 0; h < H; ++h) {
    const DHead& hd = P.heads[h];
    const bool modq = hd.qmod_view >= 0;
    // MAIN
    DPass mp;
    memset(&mp, 0, sizeof(mp));
    mp.head = h;
    mp.pass = PASS_MAIN;
    mp.inst = -1;
    mp.qa = -1;
    // work items are pairs of 128-row blocks of one group (modality / residue class)
    mp.n_slots = modq ? (int)((mod_cap / BLK + 1) / 2 + M) : (P.nb + 1) / 2;
    mp.slot_base = slot;
    slot += mp.n_slots;
    P.passes.push_back(mp);
    const size_t mp_idx = P.passes.size() - 1;
    int64_t per_main = 0;
    for (int a = 0; a < MAX_MOD; ++a) {
      int64_t s = 0;
      for (int i = 0; i < hd.n_inst; ++i) {
        const DInst& x = P.insts[(size_t)h * MAX_INST + i];
        if (x.qa < 0 || x.qa == a) s += segbound(x);
      }
      per_main = std::max(per_main, s);
    }
    P.passes[mp_idx].seg_base = (int32_t)segcap;  // (the total is checked against 2^31 below)
    P.passes[mp_idx].seg_per_slot = (int32_t)(3 * per_main + 2);
    segcap += (3 * per_main + 2) * mp.n_slots;
    for (int i = 0; i < hd.n_inst; ++i) {
      const DInst& x = P.insts[(size_t)h * MAX_INST + i];
      if (x.kind != MMI_PAT_GRID) continue;
      int64_t cross = 0;
      if (hd.boundary == MMI_BND_2D)
        for (int j = 0; j < hd.n_inst; ++j) {
          const DInst& y = P.insts[(size_t)h * MAX_INST + j];
          if (y.qa == x.qa && y.kb != x.qa) cross += segbound(y);
        }
      if (x.v_cls_q >= 0) {
        // split-K: (row pair, key chunk of HROW_SPLIT_TILES tiles of the key base)
        const int64_t base_keys = (hd.boundary == MMI_BND_2D) ? S : (int64_t)S;  // upper bound of n_a too
        const int n_split = (int)std::max<int64_t>(1, (base_keys + (int64_t)HROW_SPLIT_TILES * BLK - 1) /
                                                           ((int64_t)HROW_SPLIT_TILES * BLK));
        const int n_pairs = (P.views[x.v_cls_q].cap / BLK + 1) / 2 + 1;
        DPass p2;
        memset(&p2, 0, sizeof(p2));
        p2.head = h;
        p2.pass = PASS_HROW;
        p2.inst = i;
        p2.qa = (hd.boundary == MMI_BND_Q) ? x.qa : -1;
        p2.pad0 = n_split;
        p2.n_slots = n_pairs * n_split;
        p2.slot_base = slot;
        p2.seg_base = (int32_t)segcap;
        p2.seg_per_slot = (int32_t)(3 + 3 * cross);
        slot += p2.n_slots;
        P.passes.push_back(p2);
        segcap += (3 + 3 * cross) * p2.n_slots;
        P.insts[(size_t)h * MAX_INST + i].pad[1] = (int32_t)part_rows_hrow_cursor;
        part_rows_hrow_cursor += (int64_t)n_split * P.views[x.v_cls_q].cap;
        DHrow hr;
        hr.head = h;
        hr.inst = i;
        hr.qa = p2.qa;
        hr.n_split = n_split;
        P.hrows.push_back(hr);
        P.hrow_rows_max = std::max(P.hrow_rows_max, P.views[x.v_cls_q].cap);
      }
      if (x.v_res_q >= 0) {
        DPass p3;
        memset(&p3, 0, sizeof(p3));
        p3.head = h;
        p3.pass = PASS_SLASH;
        p3.inst = i;
        p3.qa = (hd.boundary == MMI_BND_Q) ? x.qa : -1;
        p3.n_slots = (P.views[x.v_res_q].cap / BLK + 1) / 2 + x.smax + 1;
        p3.slot_base = slot;
        p3.seg_base = (int32_t)segcap;
        p3.seg_per_slot = 3;
        slot += p3.n_slots;
        P.passes.push_back(p3);
        segcap += 3 * p3.n_slots;
      }
    }
  }
  P.n_slots = slot;
  // static per-slot regions, then a spill area for a slot whose analytic bound is short
  P.seg_spill_base = segcap;
  P.seg_spill_cap = std::max<int64_t>(segcap / 8, 4096);
  P.seg_cap = segcap + P.seg_spill_cap + 16;
  P.part_rows = part_rows_hrow_cursor;

  // VS lists / bitmaps
  const int64_t bitw = (int64_t)S / 32 + 8;  // slack: 128-bit windows may read past S
  for (int i = 0; i < P.n_vs; ++i) {
    P.vs_v_off.push_back(P.vs_list_words);
    P.vs_list_words += pad128(P.vs_nv[i]);
    P.vs_s_off.push_back(P.vs_list_words);
    P.vs_list_words += pad128(std::max(P.vs_ns[i], 1));
    P.vs_bits_v.push_back(P.bits_words);
    P.bits_words += bitw;
    P.vs_bits_s.push_back(P.bits_words);
    P.bits_words += bitw;
  }
  P.n_chunks = (S + SLAB_CHUNK - 1) / SLAB_CHUNK;

  // ---------------- workspace layout ----------------
  size_t off = 0;
  auto reg = [&](Region& r, size_t bytes) {
    r.off = off;
    r.bytes = bytes;
    off = align256(off + std::max<size_t>(bytes, 16));
  };
  const size_t nS = (size_t)P.S_pad;
  // table lists
  for (int v = 0; v < (int)P.views.size(); ++v) (P.views[v].space == 0 ? P.qview_ids : P.kview_ids).push_back(v);
  P.grid_inst.assign(std::max(P.n_grid, 1), 0);
  P.vs_inst.assign(std::max(P.n_vs, 1), 0);
  for (int i = 0; i < (int)P.insts.size(); ++i) {
    if (P.insts[i].grid_id >= 0) {
      P.grid_inst[P.insts[i].grid_id] = i;
      P.max_ncand = std::max(P.max_ncand, P.insts[i].smax - P.insts[i].smin + 1);
    }
    if (P.insts[i].vs_id >= 0) P.vs_inst[P.insts[i].vs_id] = i;
  }
  P.gacc_off.assign(std::max(P.n_grid, 1), 0);
  for (int g = 0; g < P.n_grid; ++g) {
    const DInst& x = P.insts[P.grid_inst[g]];
    P.gacc_off[g] = P.gacc_words;
    P.gacc_words += (int64_t)(x.smax - x.smin + 1) * x.smax;
  }
  P.vs_off_tab.assign((size_t)4 * std::max(P.n_vs, 1), 0);
  for (int i = 0; i < P.n_vs; ++i) {
    P.vs_off_tab[2 * i] = P.vs_v_off[i];
    P.vs_off_tab[2 * i + 1] = P.vs_s_off[i];
    P.vs_off_tab[(size_t)2 * std::max(P.n_vs, 1) + 2 * i] = P.vs_bits_v[i];
    P.vs_off_tab[(size_t)2 * std::max(P.n_vs, 1) + 2 * i + 1] = P.vs_bits_s[i];
  }
  {
    size_t b = 0;
    auto sub = [&](size_t& o, size_t bytes) {
      o = b;
      b = align256(b + std::max<size_t>(bytes, 16));
    };
    sub(P.o_heads, sizeof(DHead) * H);
    sub(P.o_insts, sizeof(DInst) * P.insts.size());
    sub(P.o_views, sizeof(DView) * P.views.size());
    sub(P.o_slabs, sizeof(DSlab) * P.slabs.size());
    sub(P.o_passes, sizeof(DPass) * P.passes.size());
    sub(P.o_qv, sizeof(int) * P.qview_ids.size());
    sub(P.o_kv, sizeof(int) * P.kview_ids.size());
    sub(P.o_gi, sizeof(int) * P.grid_inst.size());
    sub(P.o_vi, sizeof(int) * P.vs_inst.size());
    sub(P.o_vsl, sizeof(int64_t) * 2 * std::max(P.n_vs, 1));
    sub(P.o_vsb, sizeof(int64_t) * 2 * std::max(P.n_vs, 1));
    sub(P.o_gacc, sizeof(int64_t) * P.gacc_off.size());
    for (int h = 0; h < H; ++h)
      if (P.heads[h].part_rows0 >= 0) P.merge_heads.push_back(h);
    sub(P.o_mh, sizeof(int) * std::max<size_t>(P.merge_heads.size(), 1));
    sub(P.o_hr, sizeof(DHrow) * std::max<size_t>(P.hrows.size(), 1));
    sub(P.o_sp, sizeof(int) * std::max<size_t>(P.stc_pairs.size(), 2));
    P.blob_bytes = b;
  }
  reg(P.blob, P.blob_bytes);
  reg(P.labels, nS);
  reg(P.mod_cnt, sizeof(int) * (3 * MAX_MOD + 4));  // counts, offsets, padded offsets
  reg(P.mod_off, sizeof(int) * ((size_t)((S + 4095) / 4096) + 1) * MAX_MOD * 2);  // chunk counts / bases
  reg(P.perm, sizeof(int) * nS);
  reg(P.rank, sizeof(int) * nS);
  reg(P.modpos, sizeof(int) * (size_t)mod_cap);
  const size_t ns = std::max<size_t>(P.slabs.size(), 1);
  reg(P.slab_rows, sizeof(int) * ns * SLAB_ROWS * 2 + sizeof(int) * ns * 4);
  reg(P.slab_ml_part, sizeof(float) * 2 * ns * (size_t)P.n_chunks * SLAB_ROWS);
  reg(P.slab_ml, sizeof(float) * 2 * ns * SLAB_ROWS);
  reg(P.cbuf, sizeof(float) * ns * nS);
  reg(P.dgbuf, sizeof(unsigned long long) * ns * nS);
  reg(P.c_rank, sizeof(uint32_t) * std::max(P.n_grid, 1) * nS);  // 2^-25 fixed-point c per grid instance
  reg(P.gridres, sizeof(GridRes) * std::max(P.n_grid, 1));
  reg(P.grid_part, sizeof(double) * 2 * std::max(P.n_grid, 1) * 1025);
  reg(P.grid_acc, sizeof(unsigned long long) * std::max<int64_t>(P.gacc_words, 1));
  reg(P.vs_lists, sizeof(int) * std::max<int64_t>(P.vs_list_words, 1));
  reg(P.vs_cnt, sizeof(int) * 2 * std::max(P.n_vs, 1));
  reg(P.bits, sizeof(uint32_t) * std::max<int64_t>(P.bits_words, 1));
  reg(P.view_len, sizeof(int) * std::max<size_t>(P.views.size(), 1));
  reg(P.view_alias, sizeof(int) * std::max<size_t>(P.views.size(), 1));
  reg(P.qg_pos, sizeof(int) * P.qg_rows);
  reg(P.qg_rank, sizeof(int) * P.qg_rows);
  reg(P.qg_src, sizeof(int) * P.qg_rows);
  reg(P.kg_pos, sizeof(int) * P.kg_rows);
  reg(P.kg_rank, sizeof(int) * P.kg_rows);
  reg(P.kg_src, sizeof(int) * P.kg_rows);
#if defined(MMI_EXPLICIT_PERMUTE)
  P.fused = 0;  // mmi_permute materialises Q̄ / K̄ / V̄ (the round-1 path, kept for A/B measurement)
#elif defined(MMI_FUSE_KV)
  P.fused = FUSE_Q | FUSE_KV;
#endif
  reg(P.qg, (P.fused & FUSE_Q) ? 0 : (size_t)P.qg_rows * P.D * 2);
  reg(P.kg, (P.fused & FUSE_KV) ? 0 : (size_t)P.kg_rows * P.D * 2);
  reg(P.vg, (P.fused & FUSE_KV) ? 0 : (size_t)P.kg_rows * P.D * 2);
  reg(P.items, sizeof(WorkItem) * P.n_slots);
  reg(P.items_sorted, sizeof(WorkItem) * P.n_slots);
  reg(P.item_keys, sizeof(int) * 2 * (size_t)P.n_slots);
  reg(P.item_vals, sizeof(int) * 2 * (size_t)P.n_slots);
  reg(P.sort_tmp, sizeof(int) * sort_hist_ints(P.n_slots));
  reg(P.seg_cnt, sizeof(int) * (P.n_slots + 1));
  reg(P.seg_off, sizeof(int) * (P.n_slots + 1));
  reg(P.segs, sizeof(Seg) * P.seg_cap);
  reg(P.inst_params, sizeof(InstParam) * P.insts.size());
  reg(P.scan_tmp, sizeof(int) * scan_tmp_ints(P.n_slots + 1));
  reg(P.sched, 256);   // attention work-item counter (zeroed on the call's stream before each launch)
  reg(P.flags, 256);   // device-side error flags (mmi_workspace_flags)
  reg(P.part_o, sizeof(uint16_t) * (size_t)std::max<int64_t>(P.part_rows, 1) * P.D);  // fp16
  reg(P.part_lse, sizeof(float) * (size_t)std::max<int64_t>(P.part_rows, 1));
  P.total = off;
  // 32-bit row / segment indexing inside the kernels (WorkItem.q_row0, DView.row_off, Seg.krow0)
  const int64_t lim = (int64_t)1 << 31;
  int64_t worst = std::max<int64_t>({P.qg_rows, P.kg_rows, P.part_rows, P.seg_cap, (int64_t)P.n_slots + 1,
                                     (int64_t)P.Hkv * P.S + BLK, (int64_t)P.H * P.S + BLK});
  for (const DView& v : P.views) worst = std::max<int64_t>(worst, (int64_t)v.row_off + v.cap);
  if (worst >= lim) {
    err = "plan needs " + std::to_string(worst) + " rows / segments: exceeds 32-bit indexing";
    return MMI_E_UNSUPPORTED;
  }
  return MMI_OK;
}

std::vector<uint8_t> make_blob(const Plan& P) {
  std::vector<uint8_t> b(P.blob_bytes, 0);
  auto put = [&](size_t off, const void* src, size_t bytes) {
    if (bytes) memcpy(b.data() + off, src, bytes);
  };
  put(P.o_heads, P.heads.data(), sizeof(DHead) * P.heads.size());
  put(P.o_insts, P.insts.data(), sizeof(DInst) * P.insts.size());
  put(P.o_views, P.views.data(), sizeof(DView) * P.views.size());
  put(P.o_slabs, P.slabs.data(), sizeof(DSlab) * P.slabs.size());
  put(P.o_passes, P.passes.data(), sizeof(DPass) * P.passes.size());
  put(P.o_qv, P.qview_ids.data(), sizeof(int) * P.qview_ids.size());
  put(P.o_kv, P.kview_ids.data(), sizeof(int) * P.kview_ids.size());
  put(P.o_gi, P.grid_inst.data(), sizeof(int) * P.grid_inst.size());
  put(P.o_vi, P.vs_inst.data(), sizeof(int) * P.vs_inst.size());
  const size_t nv = (size_t)std::max(P.n_vs, 1);
  put(P.o_vsl, P.vs_off_tab.data(), sizeof(int64_t) * 2 * nv);
  put(P.o_vsb, P.vs_off_tab.data() + 2 * nv, sizeof(int64_t) * 2 * nv);
  put(P.o_gacc, P.gacc_off.data(), sizeof(int64_t) * P.gacc_off.size());
  put(P.o_mh, P.merge_heads.data(), sizeof(int) * P.merge_heads.size());
  put(P.o_hr, P.hrows.data(), sizeof(DHrow) * P.hrows.size());
  put(P.o_sp, P.stc_pairs.data(), sizeof(int) * P.stc_pairs.size());
  return b;
}

}  // namespace mmi
