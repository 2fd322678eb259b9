// Permuted NATTEN / DiT neighborhood attention (App. F: "the
// 2D/3D sliding window attention in NATTEN can be converted into dense tensor core computation
// via permutation").  Tokens of a T x Hh x Ww grid (raster order) are permuted into 3D tiles of
// bt x bh x bw = 128 tokens; the window of a query tile then covers a small box of key tiles, so
// the same block-sparse tcgen05 kernel runs it: permuted Q blocks gathered in-kernel (TMA row
// gathers), K̄ / V̄ materialised once per call, the window predicate (role R_NAT, bidirectional)
// evaluated only on border tiles, outputs scattered back to raster order by the epilogue.
// The index depends only on the geometry: it is built on the host once per (problem, config) and
// uploaded from pinned memory.
#include <cuda_runtime.h>
#include <algorithm>
#include <climits>
#include <cstring>
#include <memory>
#include <mutex>
#include <string>
#include <vector>

#include "../../include/mmi.h"
#include "index.h"
#include "internal.h"

namespace mmi {

namespace {

struct NatPlan {
  std::string key;
  mmi_problem pb{};
  mmi_natten_config nc{};
  int nT = 0, nY = 0, nX = 0, n_tiles = 0;
  int64_t q_rows = 0, k_rows = 0;
  std::vector<WorkItem> items;
  std::vector<Seg> segs;
  size_t o_items = 0, o_segs = 0, blob_bytes = 0;
  size_t off_blob = 0, off_qpos = 0, off_qsrc = 0, off_kpos = 0, off_ksrc = 0, off_kg = 0, off_vg = 0, off_sched = 0;
  size_t total = 0;
  uint8_t* blob_pinned = nullptr;
  cudaEvent_t ev = nullptr;
  ~NatPlan() {
    if (ev) {
      cudaEventSynchronize(ev);
      cudaEventDestroy(ev);
    }
    if (blob_pinned) cudaFreeHost(blob_pinned);
  }
};

std::mutex g_nat_mu;
std::vector<std::shared_ptr<NatPlan>> g_nat_cache;

inline size_t a256(size_t x) { return (x + 255) / 256 * 256; }
inline int wstart(int c, int k, int L) { return std::min(std::max(c - k / 2, 0), L - k); }

// per-half state of key tile (tt, ty, tx) for the queries of tile (qt, qy, qx)
uint32_t nat_state(const mmi_natten_config& c, int qT, int qY, int qX, int kT, int kY, int kX) {
  const int L[3] = {c.T, c.Hh, c.Ww}, k[3] = {c.kt, c.kh, c.kw}, b[3] = {c.bt, c.bh, c.bw};
  const int qtile[3] = {qT, qY, qX}, ktile[3] = {kT, kY, kX};
  bool full = true;
  for (int d = 0; d < 3; ++d) {
    const int q_lo = qtile[d] * b[d], q_hi = std::min(L[d], q_lo + b[d]) - 1;
    if (q_lo > q_hi) return TS_DEAD;
    const int k_lo = ktile[d] * b[d], k_hi_raw = k_lo + b[d] - 1, k_hi = std::min(L[d] - 1, k_hi_raw);
    const int any_lo = wstart(q_lo, k[d], L[d]), any_hi = wstart(q_hi, k[d], L[d]) + k[d] - 1;  // union of windows
    if (k_hi < any_lo || k_lo > any_hi) return TS_DEAD;
    const int all_lo = wstart(q_hi, k[d], L[d]), all_hi = wstart(q_lo, k[d], L[d]) + k[d] - 1;  // intersection
    if (k_hi_raw != k_hi || k_lo < all_lo || k_hi > all_hi) full = false;
  }
  return full ? TS_FULL : TS_PRED;
}

struct HostSegBuilder {
  std::vector<Seg>* out;
  int krow_t0 = 0, start = 0, n = 0, ph[2] = {0, 0}, c[2][5];
  bool open = false;
  uint32_t meta = 0;
  static int adv(int p, uint32_t st) {
    if (st == TS_DEAD) return p <= 0 ? 0 : 4;
    if (st == TS_PRED) return p <= 1 ? 1 : (p <= 3 ? 3 : -1);
    return p <= 2 ? 2 : -1;
  }
  void flush() {
    if (open && n > 0) {
      Seg s;
      s.krow0 = krow_t0 + start * BLK;
      s.ntiles = n;
      s.meta = meta;
      s.pad = 0;
      for (int h = 0; h < 2; ++h) {
        s.st[h][0] = (int16_t)c[h][0];
        s.st[h][1] = (int16_t)c[h][1];
        s.st[h][2] = (int16_t)c[h][3];
        s.st[h][3] = (int16_t)c[h][4];
      }
      out->push_back(s);
    }
    open = false;
  }
  void push(int t, uint32_t s0, uint32_t s1) {
    if (s0 == TS_DEAD && s1 == TS_DEAD) {
      flush();
      return;
    }
    int n0 = -1, n1 = -1;
    if (open && n < SEG_MAX_TILES) {
      n0 = adv(ph[0], s0);
      n1 = adv(ph[1], s1);
    }
    if (n0 < 0 || n1 < 0) {
      flush();
      open = true;
      start = t;
      n = 0;
      memset(c, 0, sizeof(c));
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

mmi_status check_nat(const mmi_problem* pb, const mmi_natten_config* c, std::string& err) {
  if (!pb || !c) {
    err = "null problem / config";
    return MMI_E_INVALID;
  }
  if (pb->n_heads < 1 || pb->n_kv_heads < 1 || pb->n_heads % pb->n_kv_heads) {
    err = "n_heads must be a positive multiple of n_kv_heads";
    return MMI_E_SHAPE;
  }
  if (pb->head_dim != 64 && pb->head_dim != 128) {
    err = "head_dim not in {64,128}";
    return MMI_E_SHAPE;
  }
  if (c->T < 1 || c->Hh < 1 || c->Ww < 1 || (long long)c->T * c->Hh * c->Ww != pb->seq_len) {
    err = "T * Hh * Ww must equal seq_len";
    return MMI_E_SHAPE;
  }
  if (c->kt < 1 || c->kh < 1 || c->kw < 1 || c->kt > c->T || c->kh > c->Hh || c->kw > c->Ww) {
    err = "window sizes must be in [1, grid extent]";
    return MMI_E_CONFIG;
  }
  if (c->bt < 1 || c->bh < 1 || c->bw < 1 || c->bt * c->bh * c->bw != BLK) {
    err = "tile bt * bh * bw must be 128";
    return MMI_E_CONFIG;
  }
  if ((long long)pb->n_heads * (pb->seq_len + 4LL * BLK) * 8 > (1LL << 31)) {
    err = "problem too large for 32-bit permuted-row indexing";
    return MMI_E_UNSUPPORTED;
  }
  return MMI_OK;
}

mmi_status nat_plan(const mmi_problem* pb, const mmi_natten_config* c, std::shared_ptr<NatPlan>& out, std::string& err,
                    bool need_blob) {
  mmi_status st = check_nat(pb, c, err);
  if (st != MMI_OK) return st;
  std::string key(reinterpret_cast<const char*>(pb), sizeof(*pb));
  key.append(reinterpret_cast<const char*>(c), sizeof(*c));
  std::lock_guard<std::mutex> lk(g_nat_mu);
  for (auto& e : g_nat_cache)
    if (e->key == key) {
      out = e;
      break;
    }
  if (!out) {
    auto P = std::make_shared<NatPlan>();
    P->key = key;
    P->pb = *pb;
    P->nc = *c;
    P->nT = (c->T + c->bt - 1) / c->bt;
    P->nY = (c->Hh + c->bh - 1) / c->bh;
    P->nX = (c->Ww + c->bw - 1) / c->bw;
    P->n_tiles = P->nT * P->nY * P->nX;
    const int H = pb->n_heads, Hkv = pb->n_kv_heads, G = H / Hkv;
    P->q_rows = (int64_t)H * P->n_tiles * BLK;
    P->k_rows = (int64_t)Hkv * P->n_tiles * BLK;
    const int npair = (P->n_tiles + 1) / 2;
    // items ordered (pair, head): the heads of a KV group read the same key tiles back to back (L2)
    for (int pr = 0; pr < npair; ++pr)
      for (int h = 0; h < H; ++h) {
        WorkItem W;
        memset(&W, 0, sizeof(W));
        const int kv = h / G;
        const int ta = 2 * pr, tb = 2 * pr + 1;
        const int has_b = tb < P->n_tiles;
        W.head = h;
        W.q_row0 = (int)((int64_t)h * P->n_tiles * BLK + (int64_t)ta * BLK);
        W.seg_off = (int)P->segs.size();
        W.q_gathered = 1;
        W.out_mode = OUT_FINAL;
        W.row_mod = -1;
        W.has_b = has_b;
        W.pad[0] = ta * BLK;
        int qc[2][3];
        for (int hf = 0; hf < 2; ++hf) {
          const int t = hf ? (has_b ? tb : ta) : ta;
          qc[hf][0] = t / (P->nX * P->nY);
          qc[hf][1] = (t / P->nX) % P->nY;
          qc[hf][2] = t % P->nX;
        }
        // key tile box: union of the two query tiles' window boxes
        int lo[3], hi[3];
        const int L[3] = {c->T, c->Hh, c->Ww}, k[3] = {c->kt, c->kh, c->kw}, b[3] = {c->bt, c->bh, c->bw};
        for (int d = 0; d < 3; ++d) {
          lo[d] = INT_MAX;
          hi[d] = -1;
          for (int hf = 0; hf < (has_b ? 2 : 1); ++hf) {
            const int q_lo = qc[hf][d] * b[d], q_hi = std::min(L[d], q_lo + b[d]) - 1;
            lo[d] = std::min(lo[d], wstart(q_lo, k[d], L[d]) / b[d]);
            hi[d] = std::max(hi[d], (wstart(q_hi, k[d], L[d]) + k[d] - 1) / b[d]);
          }
        }
        HostSegBuilder sb;
        sb.out = &P->segs;
        sb.meta = seg_meta(1, R_NAT, 0, 0);
        const int nseg0 = (int)P->segs.size();
        for (int tt = lo[0]; tt <= hi[0]; ++tt)
          for (int ty = lo[1]; ty <= hi[1]; ++ty) {
            sb.krow_t0 = (int)((int64_t)kv * P->n_tiles * BLK + (int64_t)((tt * P->nY + ty) * P->nX) * BLK);
            sb.open = false;
            for (int tx = lo[2]; tx <= hi[2]; ++tx) {
              const uint32_t s0 = nat_state(*c, qc[0][0], qc[0][1], qc[0][2], tt, ty, tx);
              const uint32_t s1 = has_b ? nat_state(*c, qc[1][0], qc[1][1], qc[1][2], tt, ty, tx) : TS_DEAD;
              sb.push(tx, s0, s1);
            }
            sb.flush();
          }
        W.n_segs = (int)P->segs.size() - nseg0;
        int nt = 0, live = 0;
        for (int i = nseg0; i < (int)P->segs.size(); ++i) {
          const Seg& s = P->segs[i];
          nt += s.ntiles;
          live += 2 * s.ntiles - s.st[0][0] - s.st[0][3] - s.st[1][0] - s.st[1][3];
        }
        W.n_tiles = nt;
        W.pad[1] = live;
        P->items.push_back(W);
      }
    size_t off = 0;
    auto reg = [&](size_t& o, size_t bytes) {
      o = off;
      off = a256(off + std::max<size_t>(bytes, 16));
    };
    P->o_items = 0;
    P->o_segs = a256(sizeof(WorkItem) * P->items.size());
    P->blob_bytes = P->o_segs + sizeof(Seg) * std::max<size_t>(P->segs.size(), 1);
    reg(P->off_blob, P->blob_bytes);
    reg(P->off_qpos, sizeof(int) * P->q_rows);
    reg(P->off_qsrc, sizeof(int) * P->q_rows);
    reg(P->off_kpos, sizeof(int) * P->k_rows);
    reg(P->off_ksrc, sizeof(int) * P->k_rows);
    reg(P->off_kg, (size_t)P->k_rows * pb->head_dim * 2);
    reg(P->off_vg, (size_t)P->k_rows * pb->head_dim * 2);
    reg(P->off_sched, 256);
    P->total = off;
    if (g_nat_cache.size() >= 8) g_nat_cache.erase(g_nat_cache.begin());
    g_nat_cache.push_back(P);
    out = P;
  }
  if (need_blob && !out->blob_pinned) {
    uint8_t* pin = nullptr;
    if (cudaHostAlloc(reinterpret_cast<void**>(&pin), out->blob_bytes, cudaHostAllocDefault) != cudaSuccess) {
      err = "cudaHostAlloc of the NATTEN index failed";
      return MMI_E_CUDA;
    }
    memset(pin, 0, out->blob_bytes);
    memcpy(pin + out->o_items, out->items.data(), sizeof(WorkItem) * out->items.size());
    memcpy(pin + out->o_segs, out->segs.data(), sizeof(Seg) * out->segs.size());
    if (cudaEventCreateWithFlags(&out->ev, cudaEventDisableTiming) != cudaSuccess) {
      cudaFreeHost(pin);
      err = "cudaEventCreate failed";
      return MMI_E_CUDA;
    }
    out->blob_pinned = pin;
  }
  return MMI_OK;
}

// permuted row r (Q̄: r over H heads, K̄: over Hkv heads) -> raster position / source row / pad
__global__ void natten_views_kernel(int64_t rows, int n_tiles, int S, int T, int Hh, int Ww, int bt, int bh, int bw,
                                    int nY, int nX, int pad_pos, int* __restrict__ pos_out, int* __restrict__ src_out) {
  const int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= rows) return;
  const int per_head = n_tiles * BLK;
  const int head = (int)(r / per_head), local = (int)(r % per_head);
  const int tile = local / BLK, l = local % BLK;
  const int TX = tile % nX, TY = (tile / nX) % nY, TT = tile / (nX * nY);
  const int lx = l % bw, ly = (l / bw) % bh, lt = l / (bw * bh);
  const int t = TT * bt + lt, y = TY * bh + ly, x = TX * bw + lx;
  if (t < T && y < Hh && x < Ww) {
    const int pos = (t * Hh + y) * Ww + x;
    pos_out[r] = pos;
    src_out[r] = head * S + pos;
  } else {
    pos_out[r] = pad_pos;
    src_out[r] = -1;
  }
}

}  // namespace

int nat_tiles_of(const mmi_natten_config* c) {
  return ((c->T + c->bt - 1) / c->bt) * ((c->Hh + c->bh - 1) / c->bh) * ((c->Ww + c->bw - 1) / c->bw);
}

}  // namespace mmi

using namespace mmi;

static thread_local char g_nat_err[512];

extern "C" MMI_API const char* mmi_natten_last_error(void) { return g_nat_err; }

extern "C" MMI_API size_t mmi_natten_workspace_bytes(const mmi_problem* pb, const mmi_natten_config* cfg) {
  std::shared_ptr<NatPlan> P;
  std::string err;
  if (nat_plan(pb, cfg, P, err, false) != MMI_OK) {
    snprintf(g_nat_err, sizeof(g_nat_err), "%s", err.c_str());
    return 0;
  }
  return P->total;
}

static mmi_status nat_run(const mmi_problem* pb, const mmi_natten_config* cfg, void* ws, size_t ws_bytes,
                          const void* q, const void* k, const void* v, void* o, float* lse, int64_t* fp,
                          mmi_stream_t stream) {
  std::shared_ptr<NatPlan> P;
  std::string err;
  mmi_status st = nat_plan(pb, cfg, P, err, false);
  if (st == MMI_OK && (!ws || reinterpret_cast<uintptr_t>(ws) % 256 || ws_bytes < P->total)) {
    err = "workspace NULL, misaligned or too small";
    st = MMI_E_WORKSPACE;
  }
  if (st == MMI_OK && (!q || !k || !v || (!o && !fp))) {
    err = "null tensor pointer";
    st = MMI_E_INVALID;
  }
  if (st == MMI_OK) st = nat_plan(pb, cfg, P, err, true);
  if (st != MMI_OK) {
    snprintf(g_nat_err, sizeof(g_nat_err), "%s", err.c_str());
    return st;
  }
  cudaStream_t s = (cudaStream_t)stream;
  char* w = reinterpret_cast<char*>(ws);
  const mmi_natten_config& c = P->nc;
  const int S = pb->seq_len, D = pb->head_dim;
  if (cudaMemcpyAsync(w + P->off_blob, P->blob_pinned, P->blob_bytes, cudaMemcpyHostToDevice, s) != cudaSuccess ||
      cudaEventRecord(P->ev, s) != cudaSuccess)
    return MMI_E_CUDA;
  int* qpos = reinterpret_cast<int*>(w + P->off_qpos);
  int* qsrc = reinterpret_cast<int*>(w + P->off_qsrc);
  int* kpos = reinterpret_cast<int*>(w + P->off_kpos);
  int* ksrc = reinterpret_cast<int*>(w + P->off_ksrc);
  natten_views_kernel<<<(unsigned)((P->q_rows + 255) / 256), 256, 0, s>>>(P->q_rows, P->n_tiles, S, c.T, c.Hh, c.Ww, c.bt,
                                                                         c.bh, c.bw, P->nY, P->nX, -1, qpos, qsrc);
  natten_views_kernel<<<(unsigned)((P->k_rows + 255) / 256), 256, 0, s>>>(P->k_rows, P->n_tiles, S, c.T, c.Hh, c.Ww, c.bt,
                                                                         c.bh, c.bw, P->nY, P->nX, KPAD, kpos, ksrc);
  // K̄ / V̄: one coalesced materialisation per call (every key tile is re-read by the ~ window / tile
  // query tiles around it); Q blocks are gathered by the attention kernel itself
  launch_gather(ksrc, P->k_rows, D, k, w + P->off_kg, v, w + P->off_vg, s);
  AttnParams A;
  memset(&A, 0, sizeof(A));
  A.items = reinterpret_cast<const WorkItem*>(w + P->off_blob + P->o_items);
  A.n_items = (int)P->items.size();
  A.segs = reinterpret_cast<const Seg*>(w + P->off_blob + P->o_segs);
  A.qg_pos = qpos;
  A.qg_rank = qpos;
  A.kg_pos = kpos;
  A.kg_rank = kpos;
  A.o = o;
  A.lse = lse;
  A.S = S;
  A.H = pb->n_heads;
  A.Hkv = pb->n_kv_heads;
  A.D = D;
  A.scale_log2 = (pb->scale > 0.f ? pb->scale : 1.0f / sqrtf((float)D)) * 1.4426950408889634f;
  A.sched = reinterpret_cast<unsigned int*>(w + P->off_sched);
  A.fused = 1;  // Q blocks gathered in-kernel
  A.qg_src = qsrc;
  A.kg_src = ksrc;
  A.nat_T = c.T;
  A.nat_H = c.Hh;
  A.nat_W = c.Ww;
  A.nat_kt = c.kt;
  A.nat_kh = c.kh;
  A.nat_kw = c.kw;
  A.nat_bt = c.bt;
  A.nat_bh = c.bh;
  A.nat_bw = c.bw;
  A.nat_tiles = P->n_tiles;
  A.fingerprint = fp ? 1 : 0;
  A.fp_out = fp;
  AttnLaunch L;
  memset(&L, 0, sizeof(L));
  L.q = q;
  L.k = k;
  L.kg = w + P->off_kg;
  L.v = v;
  L.vg = w + P->off_vg;
  L.q_rows = (long long)pb->n_heads * S;
  L.kv_rows = (long long)pb->n_kv_heads * S;
  L.kvg_rows = P->k_rows;
  L.qg_rows = P->q_rows;
  L.o_rows = (long long)pb->n_heads * S;
  int te = 0;
  const cudaError_t e = launch_attn(L, A, A.n_items, s, &te);
  if (te || e != cudaSuccess) {
    snprintf(g_nat_err, sizeof(g_nat_err), "attention launch: %s", te ? "tensor map" : cudaGetErrorString(e));
    return MMI_E_CUDA;
  }
  return MMI_OK;
}

extern "C" MMI_API mmi_status mmi_natten_prefill(const mmi_problem* pb, const mmi_natten_config* cfg, void* ws,
                                                 size_t ws_bytes, const void* q, const void* k, const void* v, void* o,
                                                 float* lse, mmi_stream_t stream) {
  return nat_run(pb, cfg, ws, ws_bytes, q, k, v, o, lse, nullptr, stream);
}

/* TEST ONLY: per-row admitted-key fingerprints (count, sum pos, sum pos^2) of the NATTEN mask as the
 * kernel evaluates it, int64 [H, S, 3] device buffer (zeroed by the caller). */
extern "C" MMI_API mmi_status mmi_natten_fingerprint(const mmi_problem* pb, const mmi_natten_config* cfg, void* ws,
                                                     size_t ws_bytes, const void* q, const void* k, const void* v,
                                                     int64_t* fp, mmi_stream_t stream) {
  if (!fp) return MMI_E_INVALID;
  return nat_run(pb, cfg, ws, ws_bytes, q, k, v, nullptr, nullptr, fp, stream);
}
