// C ABI entry points (include/mmi.h): host-side validation, workspace layout,
// launch sequencing.  All compute runs in the kernels of this directory.
#include <cuda_runtime.h>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <memory>
#include <mutex>
#include <string>
#include <vector>

#include "../../include/mmi.h"
#include "estimate.h"
#include "index.h"
#include "internal.h"
#include "plan.h"
#include "sort.h"

using namespace mmi;


static thread_local char g_err[1024];
static long long* g_dbg = nullptr;  // debug-only per-item timestamps (mmi_debug_set_timestamps)
extern "C" MMI_API void mmi_debug_set_timestamps(long long* p) { g_dbg = p; }

static mmi_status fail(mmi_status st, const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof(g_err), fmt, ap);
  va_end(ap);
  return st;
}

extern "C" const char* mmi_last_error(void) { return g_err; }
extern "C" const char* mmi_version(void) { return "mmi-b200 0.2 (sm_100a)"; }

static mmi_status check_problem(const mmi_problem* pb) {
  if (!pb) return fail(MMI_E_INVALID, "problem is NULL");
  if (pb->n_heads < 1 || pb->n_kv_heads < 1 || pb->n_heads % pb->n_kv_heads)
    return fail(MMI_E_SHAPE, "n_heads (%d) must be a positive multiple of n_kv_heads (%d)", pb->n_heads,
                pb->n_kv_heads);
  if (pb->head_dim != 64 && pb->head_dim != 128) return fail(MMI_E_SHAPE, "head_dim %d not in {64,128}", pb->head_dim);
  if (pb->seq_len < 1) return fail(MMI_E_SHAPE, "seq_len %d < 1", pb->seq_len);
  if ((long long)(pb->seq_len + 4 * 128) * pb->n_heads > (1ll << 30))
    return fail(MMI_E_UNSUPPORTED, "H*S too large for 32-bit row indexing");
  if (pb->block != 128) return fail(MMI_E_UNSUPPORTED, "block must be 128");
  if (pb->n_modalities < 1 || pb->n_modalities > MMI_MAX_MOD)
    return fail(MMI_E_UNSUPPORTED, "n_modalities %d not in [1,%d]", pb->n_modalities, MMI_MAX_MOD);
  if (pb->last_q < 1 || pb->last_q > 64) return fail(MMI_E_UNSUPPORTED, "last_q must be in [1,64]");
  return MMI_OK;
}

static float tau_of(const mmi_problem* pb) {
  return pb->scale > 0.f ? pb->scale : 1.0f / sqrtf((float)pb->head_dim);
}

// ---------------------------------------------------------------- plan cache
// The plan (workspace layout + device tables) is a pure function of (problem, cfg[H]).  It is built
// once per distinct (problem, cfg) and kept, together with a PINNED host copy of the device-table
// blob, so that the four calls of a step neither rebuild it nor upload from pageable memory
// (pageable cudaMemcpyAsync may block the host and is not capturable in a CUDA graph).
struct CachedPlan {
  std::string key;
  Plan P;
  uint8_t* blob_pinned = nullptr;
  cudaEvent_t last_upload = nullptr;  // recorded after every upload from blob_pinned
  uint64_t stamp = 0;
  ~CachedPlan() {
    if (last_upload) {
      cudaEventSynchronize(last_upload);  // the last async copy from blob_pinned has finished
      cudaEventDestroy(last_upload);
    }
    if (blob_pinned) cudaFreeHost(blob_pinned);
  }
};
static std::mutex g_cache_mu;
static std::vector<std::shared_ptr<CachedPlan>> g_cache;
static uint64_t g_cache_clock = 0;
constexpr size_t PLAN_CACHE_CAP = 16;

static std::string plan_key(const mmi_problem* pb, const mmi_head_config* cfg) {
  std::string k(reinterpret_cast<const char*>(pb), sizeof(mmi_problem));
  k.append(reinterpret_cast<const char*>(cfg), sizeof(mmi_head_config) * (size_t)pb->n_heads);
  return k;
}

static mmi_status get_plan(const mmi_problem* pb, const mmi_head_config* cfg, std::shared_ptr<CachedPlan>& out,
                           bool need_blob) {
  mmi_status st = check_problem(pb);
  if (st != MMI_OK) return st;
  if (!cfg) return fail(MMI_E_INVALID, "cfg_host is NULL");
  const std::string key = plan_key(pb, cfg);
  {
    std::lock_guard<std::mutex> lk(g_cache_mu);
    for (auto& e : g_cache)
      if (e->key == key) {
        e->stamp = ++g_cache_clock;
        out = e;
        if (!need_blob || e->blob_pinned) return MMI_OK;
        break;
      }
  }
  if (!out) {
    auto e = std::make_shared<CachedPlan>();
    std::string err;
    st = build_plan(pb, cfg, e->P, err);
    if (st != MMI_OK) return fail(st, "%s", err.c_str());
    e->key = key;
    out = e;
  }
  std::lock_guard<std::mutex> lk(g_cache_mu);
  if (need_blob && !out->blob_pinned) {
    const std::vector<uint8_t> blob = make_blob(out->P);
    uint8_t* pin = nullptr;
    // mapped: the estimate call's copy kernel reads it over PCIe (no copy-engine transfer, which
    // would queue behind the caller's large host <-> device copies on other streams)
    cudaError_t ce = cudaHostAlloc(reinterpret_cast<void**>(&pin), std::max<size_t>(blob.size(), 16),
                                   cudaHostAllocMapped | cudaHostAllocPortable);
    if (ce != cudaSuccess) return fail(MMI_E_CUDA, "cudaHostAlloc(device tables): %s", cudaGetErrorString(ce));
    memcpy(pin, blob.data(), blob.size());
    ce = cudaEventCreateWithFlags(&out->last_upload, cudaEventDisableTiming);
    if (ce != cudaSuccess) {
      cudaFreeHost(pin);
      return fail(MMI_E_CUDA, "cudaEventCreate: %s", cudaGetErrorString(ce));
    }
    out->blob_pinned = pin;
  }
  bool present = false;
  for (auto& e : g_cache) present |= (e.get() == out.get());
  if (!present) {
    if (g_cache.size() >= PLAN_CACHE_CAP) {  // evict the least recently used entry
      size_t lru = 0;
      for (size_t i = 1; i < g_cache.size(); ++i)
        if (g_cache[i]->stamp < g_cache[lru]->stamp) lru = i;
      g_cache.erase(g_cache.begin() + lru);  // freed when its last user drops it
    }
    out->stamp = ++g_cache_clock;
    g_cache.push_back(out);
  }
  return MMI_OK;
}

static mmi_status check_ws(const Plan& P, const void* ws, size_t ws_bytes) {
  if (!ws) return fail(MMI_E_WORKSPACE, "workspace is NULL");
  if (reinterpret_cast<uintptr_t>(ws) % 256) return fail(MMI_E_WORKSPACE, "workspace not 256-byte aligned");
  if (ws_bytes < P.total) return fail(MMI_E_WORKSPACE, "workspace too small: %zu < %zu bytes", ws_bytes, P.total);
  return MMI_OK;
}

static mmi_status prepare(const mmi_problem* pb, const mmi_head_config* cfg, const void* ws, size_t ws_bytes,
                          std::shared_ptr<CachedPlan>& cp, bool need_ws = true, bool need_blob = false) {
  mmi_status st = get_plan(pb, cfg, cp, false);
  if (st != MMI_OK) return st;
  if (need_ws && (st = check_ws(cp->P, ws, ws_bytes)) != MMI_OK) return st;
  return need_blob ? get_plan(pb, cfg, cp, true) : MMI_OK;
}

template <typename T>
static T* at(void* ws, const Region& r) {
  return reinterpret_cast<T*>(reinterpret_cast<char*>(ws) + r.off);
}
template <typename T>
static T* blob_at(void* ws, const Plan& P, size_t sub) {
  return reinterpret_cast<T*>(reinterpret_cast<char*>(ws) + P.blob.off + sub);
}

static IndexCtx make_ctx(const Plan& P, void* ws) {
  IndexCtx C;
  memset(&C, 0, sizeof(C));
  C.S = P.S;
  C.H = P.H;
  C.M = P.M;
  C.n_slots = P.n_slots;
  C.n_passes = (int)P.passes.size();
  C.heads = blob_at<DHead>(ws, P, P.o_heads);
  C.insts = blob_at<DInst>(ws, P, P.o_insts);
  C.views = blob_at<DView>(ws, P, P.o_views);
  C.passes = blob_at<DPass>(ws, P, P.o_passes);
  C.info = at<int>(ws, P.mod_cnt);
  C.perm = at<int>(ws, P.perm);
  C.rank = at<int>(ws, P.rank);
  C.modpos = at<int>(ws, P.modpos);
  C.labels = at<uint8_t>(ws, P.labels);
  C.gridres = at<GridRes>(ws, P.gridres);
  C.vs_lists = at<int>(ws, P.vs_lists);
  C.vs_cnt = at<int>(ws, P.vs_cnt);
  C.vs_list_off = blob_at<int64_t>(ws, P, P.o_vsl);
  C.vs_bits_off = blob_at<int64_t>(ws, P, P.o_vsb);
  C.view_len = at<int>(ws, P.view_len);
  C.view_alias = at<int>(ws, P.view_alias);
  C.qg_pos = at<int>(ws, P.qg_pos);
  C.qg_rank = at<int>(ws, P.qg_rank);
  C.qg_src = at<int>(ws, P.qg_src);
  C.kg_pos = at<int>(ws, P.kg_pos);
  C.kg_rank = at<int>(ws, P.kg_rank);
  C.kg_src = at<int>(ws, P.kg_src);
  C.inst_params = at<InstParam>(ws, P.inst_params);
  C.seg_cnt = at<int>(ws, P.seg_cnt);
  C.seg_off = at<int>(ws, P.seg_off);
  C.segs = at<Seg>(ws, P.segs);
  C.items = at<WorkItem>(ws, P.items);
  C.items_sorted = at<WorkItem>(ws, P.items_sorted);
  C.sort_keys = at<int>(ws, P.item_keys);
  C.sort_vals = at<int>(ws, P.item_vals);
  C.sort_vals_out = at<int>(ws, P.item_vals);
  C.seg_cap = P.seg_cap;
  C.seg_spill_base = P.seg_spill_base;
  C.seg_spill_cap = P.seg_spill_cap;
  C.flags = at<unsigned>(ws, P.flags);
  C.part_o = at<__half>(ws, P.part_o);
  C.part_lse = at<float>(ws, P.part_lse);
  return C;
}

#define CK(x)                                                                              \
  do {                                                                                     \
    cudaError_t _e = (x);                                                                  \
    if (_e != cudaSuccess) return fail(MMI_E_CUDA, "%s: %s", #x, cudaGetErrorString(_e)); \
  } while (0)

extern "C" size_t mmi_workspace_bytes(const mmi_problem* pb, const mmi_head_config* cfg) {
  std::shared_ptr<CachedPlan> cp;
  if (prepare(pb, cfg, nullptr, 0, cp, false) != MMI_OK) return 0;
  return cp->P.total;
}

extern "C" mmi_status mmi_plan_stats(const mmi_problem* pb, const mmi_head_config* cfg, int64_t* out, int n) {
  if (!out || n < 0) return fail(MMI_E_INVALID, "null output");
  std::shared_ptr<CachedPlan> cp;
  const mmi_status st = prepare(pb, cfg, nullptr, 0, cp, false);
  if (st != MMI_OK) return st;
  const Plan& P = cp->P;
  const int64_t v[6] = {P.qg_rows, P.kg_rows, (int64_t)P.merge_heads.size(), (int64_t)P.slabs.size(),
                        (int64_t)P.part_rows, (int64_t)P.fused};
  for (int i = 0; i < n && i < 6; ++i) out[i] = v[i];
  return MMI_OK;
}

extern "C" mmi_status mmi_estimate_index(const mmi_problem* pb, const mmi_head_config* cfg, const void* q,
                                         const void* k, const uint8_t* modality, void* ws, size_t ws_bytes,
                                         mmi_stream_t stream) {
  std::shared_ptr<CachedPlan> cp;
  mmi_status st = prepare(pb, cfg, ws, ws_bytes, cp, true, true);
  if (st != MMI_OK) return st;
  const Plan& P = cp->P;
  if (!q || !k || !modality) return fail(MMI_E_INVALID, "null tensor pointer");
  cudaStream_t s = (cudaStream_t)stream;
  const int S = P.S;
  // device tables from the plan's pinned (mapped) host blob, and the labels: copy kernels, not
  // copy-engine transfers -- a DMA copy on this stream would wait behind any large host <-> device
  // copy the caller has queued on another stream (HostSparsePrefill's input copies)
  void* blob_dev = nullptr;
  CK(cudaHostGetDevicePointer(&blob_dev, cp->blob_pinned, 0));
  CK(copy_bytes(at<char>(ws, P.blob), blob_dev, P.blob_bytes, s));
  CK(cudaEventRecord(cp->last_upload, s));
  CK(copy_bytes(at<uint8_t>(ws, P.labels), modality, (size_t)S, s));
  CK(fill_bytes(at<char>(ws, P.flags), 0, P.flags.bytes, s));
  // zero the accumulators
  CK(fill_bytes(at<char>(ws, P.cbuf), 0, P.cbuf.bytes, s));
  CK(fill_bytes(at<char>(ws, P.dgbuf), 0, P.dgbuf.bytes, s));
  CK(fill_bytes(at<char>(ws, P.bits), 0, P.bits.bytes, s));
  CK(fill_bytes(at<char>(ws, P.vs_cnt), 0, P.vs_cnt.bytes, s));
  CK(fill_bytes(at<char>(ws, P.seg_cnt), 0, P.seg_cnt.bytes, s));
  const int64_t mod_cap = (P.S + (int64_t)P.M * BLK + BLK - 1) / BLK * BLK;
  IndexCtx C = make_ctx(P, ws);
  int* info = at<int>(ws, P.mod_cnt);
  const int nch = (S + 4095) / 4096;
  int* chunk_cnt = at<int>(ws, P.mod_off);
  int* chunk_base = chunk_cnt + (size_t)nch * MAX_MOD;
  // a1 modality bookkeeping
  launch_modality(at<uint8_t>(ws, P.labels), S, P.M, P.S_pad, (int)mod_cap, chunk_cnt, chunk_base, info,
                  at<int>(ws, P.perm), at<int>(ws, P.rank), at<int>(ws, P.modpos), at<unsigned>(ws, P.flags), s);
  // a2 last_q slab estimation
  int* srows = at<int>(ws, P.slab_rows);
  const size_t ns = std::max<size_t>(P.slabs.size(), 1);
  int* srank = srows + ns * SLAB_ROWS;
  int* sinfo = srank + ns * SLAB_ROWS;
  const DSlab* dslabs = blob_at<DSlab>(ws, P, P.o_slabs);
  CK(launch_slabs(dslabs, (int)P.slabs.size(), P.n_dg_batch, blob_at<int2>(ws, P, P.o_sp),
                  (int)P.stc_pairs.size() / 2, q, k, S, P.H, P.Hkv, P.D, P.pb.last_q,
                  tau_of(pb) * 1.4426950408889634f, info, at<int>(ws, P.perm), at<int>(ws, P.rank),
                  at<uint8_t>(ws, P.labels), srows, srank, sinfo, at<float2>(ws, P.slab_ml_part),
                  at<float2>(ws, P.slab_ml), at<float>(ws, P.cbuf), at<unsigned long long>(ws, P.dgbuf), P.n_chunks,
                  s));
  // a3 grid stride / phase
  const DInst* dinsts = blob_at<DInst>(ws, P, P.o_insts);
  launch_grid(dinsts, blob_at<int>(ws, P, P.o_gi), P.n_grid, P.max_ncand, (int)P.insts.size(), dslabs, sinfo, info,
              at<int>(ws, P.perm), at<float>(ws, P.cbuf), at<uint32_t>(ws, P.c_rank), S, P.S_pad,
              at<GridRes>(ws, P.gridres), at<double>(ws, P.grid_part), blob_at<int64_t>(ws, P, P.o_gacc),
              at<uint32_t>(ws, P.grid_acc), s);
  // a4 vertical-slash top-k
  launch_vs(dinsts, blob_at<int>(ws, P, P.o_vi), P.n_vs, dslabs, sinfo, info, at<int>(ws, P.perm),
            at<float>(ws, P.cbuf), at<unsigned long long>(ws, P.dgbuf), blob_at<int64_t>(ws, P, P.o_vsl),
            blob_at<int64_t>(ws, P, P.o_vsb), at<int>(ws, P.vs_lists), at<int>(ws, P.vs_cnt),
            at<uint32_t>(ws, P.bits), s);
  // a5 views, instance parameters, work items (fill -> order sort)
  launch_build_views(C, blob_at<int>(ws, P, P.o_qv), (int)P.qview_ids.size(), blob_at<int>(ws, P, P.o_kv),
                     (int)P.kview_ids.size(), P.qg_rows, P.kg_rows, s);
  launch_inst_params(C, (int)P.insts.size(), s);
  launch_items_fill(C, s);  // static per-slot segment regions (+ spill): no count pass, no scan
  // work order: stable ascending sort of the inverted LPT / locality keys (items_fill_kernel)
  launch_sort_pairs(reinterpret_cast<uint32_t*>(C.sort_keys), reinterpret_cast<uint32_t*>(C.sort_keys) + P.n_slots,
                    C.sort_vals, C.sort_vals + P.n_slots, P.n_slots, 32, at<int>(ws, P.sort_tmp), s);
  launch_items_gather(C, s);
  CK(cudaGetLastError());
  return MMI_OK;
}

extern "C" mmi_status mmi_permute(const mmi_problem* pb, const mmi_head_config* cfg, void* ws, size_t ws_bytes,
                                  const void* q, const void* k, const void* v, mmi_stream_t stream) {
  std::shared_ptr<CachedPlan> cp;
  mmi_status st = prepare(pb, cfg, ws, ws_bytes, cp);
  if (st != MMI_OK) return st;
  const Plan& P = cp->P;
  if (!q || !k || !v) return fail(MMI_E_INVALID, "null tensor pointer");
  cudaStream_t s = (cudaStream_t)stream;
  // permuted blocks the attention kernel does not gather itself (f2, plan.h FUSE_*) are materialised
  if (!(P.fused & FUSE_Q)) launch_gather(at<int>(ws, P.qg_src), P.qg_rows, P.D, q, at<void>(ws, P.qg), nullptr, nullptr, s);
  if (!(P.fused & FUSE_KV))
    launch_gather(at<int>(ws, P.kg_src), P.kg_rows, P.D, k, at<void>(ws, P.kg), v, at<void>(ws, P.vg), s);
  CK(cudaGetLastError());
  return MMI_OK;
}

static mmi_status run_sparse(const Plan& P, const mmi_problem* pb, void* ws, const void* q, const void* k,
                             const void* v, void* o, float* lse, int64_t* fp, cudaStream_t s) {
  AttnParams A;
  memset(&A, 0, sizeof(A));
  A.items = at<WorkItem>(ws, P.items_sorted);
  A.n_items = P.n_slots;
  A.segs = at<Seg>(ws, P.segs);
  A.insts = at<InstParam>(ws, P.inst_params);
  A.bits = at<uint32_t>(ws, P.bits);
  A.qg_pos = at<int>(ws, P.qg_pos);
  A.qg_rank = at<int>(ws, P.qg_rank);
  A.kg_pos = at<int>(ws, P.kg_pos);
  A.kg_rank = at<int>(ws, P.kg_rank);
  A.rank = at<int>(ws, P.rank);
  A.labels = at<uint8_t>(ws, P.labels);
  A.o = o;
  A.lse = lse;
  A.part_o = at<__half>(ws, P.part_o);
  A.part_lse = at<float>(ws, P.part_lse);
  A.S = P.S;
  A.H = P.H;
  A.Hkv = P.Hkv;
  A.D = P.D;
  A.scale_log2 = tau_of(pb) * 1.4426950408889634f;
  A.dense = 0;
  A.fingerprint = fp ? 1 : 0;
  A.dbg = g_dbg;
  A.fp_out = fp;
  A.sched = at<unsigned int>(ws, P.sched);
  A.fused = P.fused;
  A.qg_src = at<int>(ws, P.qg_src);
  A.kg_src = at<int>(ws, P.kg_src);
  A.q_oob = 0;   // padding rows gather row 0: finite values, masked (K) / never written (Q) / P = 0 (V)
  A.kv_oob = 0;
  // partial rows of work items without a live tile are never written: NaN-fill their LSEs so the
  // merges of mmi_unpermute skip them (0xFF bytes = NaN)
  if (P.part_rows > 0) {
    const cudaError_t ce = fill_bytes(A.part_lse, 0xFF, sizeof(float) * (size_t)P.part_rows, s);
    if (ce != cudaSuccess) return fail(MMI_E_CUDA, "partial LSE fill: %s", cudaGetErrorString(ce));
  }
  AttnLaunch L;
  L.q = q;
  L.qg = at<void>(ws, P.qg);
  L.k = k;
  L.kg = at<void>(ws, P.kg);
  L.v = v;
  L.vg = at<void>(ws, P.vg);
  L.q_rows = (long long)P.H * P.S;
  L.qg_rows = P.qg_rows;
  L.kv_rows = (long long)P.Hkv * P.S;
  L.kvg_rows = P.kg_rows;
  L.o_rows = (long long)P.H * P.S;
  L.part_rows = P.part_rows;
  int te = 0;
  cudaError_t e = launch_attn(L, A, P.n_slots, s, &te);
  if (te) return fail(MMI_E_CUDA, "cuTensorMapEncodeTiled failed (%d)", te);
  if (e != cudaSuccess) return fail(MMI_E_CUDA, "attention launch: %s", cudaGetErrorString(e));
  return MMI_OK;
}

extern "C" mmi_status mmi_sparse_prefill(const mmi_problem* pb, const mmi_head_config* cfg, void* ws,
                                         size_t ws_bytes, const void* q, const void* k, const void* v, void* o,
                                         float* lse, mmi_stream_t stream) {
  std::shared_ptr<CachedPlan> cp;
  mmi_status st = prepare(pb, cfg, ws, ws_bytes, cp);
  if (st != MMI_OK) return st;
  const Plan& P = cp->P;
  if (!q || !k || !v || !o) return fail(MMI_E_INVALID, "null tensor pointer");
  return run_sparse(P, pb, ws, q, k, v, o, lse, nullptr, (cudaStream_t)stream);
}

extern "C" mmi_status mmi_sparse_fingerprint(const mmi_problem* pb, const mmi_head_config* cfg, void* ws,
                                             size_t ws_bytes, const void* q, const void* k, const void* v,
                                             int64_t* fp, mmi_stream_t stream) {
  std::shared_ptr<CachedPlan> cp;
  mmi_status st = prepare(pb, cfg, ws, ws_bytes, cp);
  if (st != MMI_OK) return st;
  const Plan& P = cp->P;
  if (!q || !k || !v || !fp) return fail(MMI_E_INVALID, "null tensor pointer");
  return run_sparse(P, pb, ws, q, k, v, nullptr, nullptr, fp, (cudaStream_t)stream);
}

extern "C" mmi_status mmi_unpermute(const mmi_problem* pb, const mmi_head_config* cfg, void* ws, size_t ws_bytes,
                                    void* o, float* lse, mmi_stream_t stream) {
  std::shared_ptr<CachedPlan> cp;
  mmi_status st = prepare(pb, cfg, ws, ws_bytes, cp);
  if (st != MMI_OK) return st;
  const Plan& P = cp->P;
  if (!o) return fail(MMI_E_INVALID, "null output pointer");
  cudaStream_t s = (cudaStream_t)stream;
  IndexCtx C = make_ctx(P, ws);
  const int64_t mod_cap = (P.S + (int64_t)P.M * BLK + BLK - 1) / BLK * BLK;
  // rows of the largest MAIN view among merged heads (rows beyond a head's view exit early)
  int rows = 0;
  for (int h : P.merge_heads) rows = std::max(rows, P.heads[h].qmod_view >= 0 ? (int)mod_cap : P.nb * BLK);
  launch_merge(C, P.D, blob_at<int>(ws, P, P.o_mh), (int)P.merge_heads.size(), rows, o, lse, s);
  launch_hrow_merge(C, P.D, blob_at<DHrow>(ws, P, P.o_hr), (int)P.hrows.size(), P.hrow_rows_max, o, lse, s);
  CK(cudaGetLastError());
  return MMI_OK;
}


extern "C" mmi_status mmi_dense_prefill(const mmi_problem* pb, const void* q, const void* k, const void* v, void* o,
                                        float* lse, mmi_stream_t stream) {
  mmi_status st = check_problem(pb);
  if (st != MMI_OK) return st;
  if (!q || !k || !v || !o) return fail(MMI_E_INVALID, "null tensor pointer");
  AttnParams A;
  memset(&A, 0, sizeof(A));
  A.S = pb->seq_len;
  A.H = pb->n_heads;
  A.Hkv = pb->n_kv_heads;
  A.D = pb->head_dim;
  A.scale_log2 = tau_of(pb) * 1.4426950408889634f;
  A.dense = 1;
  A.dbg = g_dbg;
  A.o = o;
  A.lse = lse;
  AttnLaunch L;
  memset(&L, 0, sizeof(L));
  L.q = q;
  L.k = k;
  L.v = v;
  L.q_rows = (long long)pb->n_heads * pb->seq_len;
  L.kv_rows = (long long)pb->n_kv_heads * pb->seq_len;
  L.o_rows = (long long)pb->n_heads * pb->seq_len;
  int te = 0;
  const int nb = (pb->seq_len + 127) / 128;
  cudaError_t e = launch_attn(L, A, pb->n_heads * nb, (cudaStream_t)stream, &te);
  if (te) return fail(MMI_E_CUDA, "cuTensorMapEncodeTiled failed (%d)", te);
  if (e != cudaSuccess) return fail(MMI_E_CUDA, "attention launch: %s", cudaGetErrorString(e));
  return MMI_OK;
}

// Export layout (int32 words), for head h:
//   [0] n_inst
//   per instance: kind, qa, kb, rank, s, p, valid, J (2 words, double bits), nV, nS, V[nV], Sl[nS]
//   then: items with tiles, total tiles (2 words, int64), segments
extern "C" mmi_status mmi_traffic_stats(const mmi_problem* pb, const mmi_head_config* cfg, const void* ws,
                                        size_t ws_bytes, int64_t* out, mmi_stream_t stream) {
  std::shared_ptr<CachedPlan> cp;
  mmi_status st = prepare(pb, cfg, ws, ws_bytes, cp);
  if (st != MMI_OK) return st;
  const Plan& P = cp->P;
  if (!out) return fail(MMI_E_INVALID, "null output");
  CK(cudaStreamSynchronize((cudaStream_t)stream));
  void* w = const_cast<void*>(ws);
  auto count = [&](const Region& r, int64_t rows, int64_t& rd, int64_t& wr) -> bool {
    rd = wr = 0;
    if (rows <= 0) return true;
    std::vector<int> src(rows);
    if (cudaMemcpy(src.data(), at<int>(w, r), sizeof(int) * rows, cudaMemcpyDeviceToHost) != cudaSuccess) return false;
    for (int v : src) {
      rd += v >= 0;
      wr += v >= -1;  // -1: padding row written as zeros, -2: never touched
    }
    return true;
  };
  if (!count(P.qg_src, P.qg_rows, out[0], out[1]) || !count(P.kg_src, P.kg_rows, out[2], out[3]))
    return fail(MMI_E_CUDA, "copy of the gather sources failed");
  return MMI_OK;
}

extern "C" mmi_status mmi_workspace_flags(const mmi_problem* pb, const mmi_head_config* cfg, const void* ws,
                                          size_t ws_bytes, uint32_t* flags_host, mmi_stream_t stream) {
  std::shared_ptr<CachedPlan> cp;
  mmi_status st = prepare(pb, cfg, ws, ws_bytes, cp);
  if (st != MMI_OK) return st;
  if (!flags_host) return fail(MMI_E_INVALID, "flags_host is NULL");
  CK(cudaStreamSynchronize((cudaStream_t)stream));
  CK(cudaMemcpy(flags_host, at<char>(const_cast<void*>(ws), cp->P.flags), sizeof(uint32_t), cudaMemcpyDeviceToHost));
  return MMI_OK;
}

extern "C" mmi_status mmi_export_index(const mmi_problem* pb, const mmi_head_config* cfg, const void* ws,
                                       size_t ws_bytes, int32_t head, int32_t* host_buf, size_t* words,
                                       mmi_stream_t stream) {
  std::shared_ptr<CachedPlan> cp;
  mmi_status st = prepare(pb, cfg, ws, ws_bytes, cp);
  if (st != MMI_OK) return st;
  const Plan& P = cp->P;
  if (head < 0 || head >= P.H) return fail(MMI_E_INVALID, "head out of range");
  if (!words) return fail(MMI_E_INVALID, "words is NULL");
  cudaStream_t s = (cudaStream_t)stream;
  CK(cudaStreamSynchronize(s));
  void* w = const_cast<void*>(ws);
  std::vector<GridRes> gr(std::max(P.n_grid, 1));
  std::vector<int> cnt(2 * std::max(P.n_vs, 1));
  CK(cudaMemcpy(gr.data(), at<GridRes>(w, P.gridres), sizeof(GridRes) * gr.size(), cudaMemcpyDeviceToHost));
  CK(cudaMemcpy(cnt.data(), at<int>(w, P.vs_cnt), sizeof(int) * cnt.size(), cudaMemcpyDeviceToHost));
  std::vector<int32_t> out;
  const DHead& hd = P.heads[head];
  out.push_back(hd.n_inst);
  for (int i = 0; i < hd.n_inst; ++i) {
    const DInst& x = P.insts[(size_t)head * MAX_INST + i];
    out.push_back(x.kind);
    out.push_back(x.qa);
    out.push_back(x.kb);
    out.push_back(x.rank);
    int32_t gs = 0, gp = 0, gv = 0;
    double J = 0;
    if (x.grid_id >= 0) {
      gs = gr[x.grid_id].s;
      gp = gr[x.grid_id].p;
      gv = gr[x.grid_id].valid;
      J = gr[x.grid_id].J;
    }
    out.push_back(gs);
    out.push_back(gp);
    out.push_back(gv);
    int32_t jw[2];
    memcpy(jw, &J, 8);
    out.push_back(jw[0]);
    out.push_back(jw[1]);
    int nV = 0, nS = 0;
    std::vector<int> V, Sl;
    if (x.vs_id >= 0) {
      nV = cnt[2 * x.vs_id];
      nS = cnt[2 * x.vs_id + 1];
      V.resize(nV);
      Sl.resize(nS);
      if (nV)
        CK(cudaMemcpy(V.data(), at<int>(w, P.vs_lists) + P.vs_v_off[x.vs_id], sizeof(int) * nV,
                      cudaMemcpyDeviceToHost));
      if (nS)
        CK(cudaMemcpy(Sl.data(), at<int>(w, P.vs_lists) + P.vs_s_off[x.vs_id], sizeof(int) * nS,
                      cudaMemcpyDeviceToHost));
    }
    out.push_back(nV);
    out.push_back(nS);
    out.insert(out.end(), V.begin(), V.end());
    out.insert(out.end(), Sl.begin(), Sl.end());
  }
  std::vector<WorkItem> items(P.n_slots);
  CK(cudaMemcpy(items.data(), at<WorkItem>(w, P.items), sizeof(WorkItem) * P.n_slots, cudaMemcpyDeviceToHost));
  int n_it = 0, n_seg = 0;
  long long tiles = 0;
  for (const auto& it : items)
    if (it.head == head && it.n_tiles > 0) {
      ++n_it;
      tiles += it.pad[1];  // computed 128x128 tiles: live (tile, half) pairs (per-half dead tiles skipped)
      n_seg += it.n_segs;
    }
  out.push_back(n_it);
  int32_t tw[2];
  memcpy(tw, &tiles, 8);
  out.push_back(tw[0]);
  out.push_back(tw[1]);
  out.push_back(n_seg);
  if (!host_buf) {
    *words = out.size();
    return MMI_OK;
  }
  if (*words < out.size()) return fail(MMI_E_INVALID, "host_buf too small (%zu < %zu words)", *words, out.size());
  memcpy(host_buf, out.data(), sizeof(int32_t) * out.size());
  *words = out.size();
  return MMI_OK;
}
