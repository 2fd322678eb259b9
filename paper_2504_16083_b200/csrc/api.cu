// C ABI entry points (include/mmi.h): host-side validation, workspace layout,
// launch sequencing.  All compute runs in the kernels of this directory.
#include <cuda_runtime.h>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstring>

#include "../../include/mmi.h"
#include "internal.h"

static thread_local char g_err[512];

static mmi_status fail(mmi_status st, const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof(g_err), fmt, ap);
  va_end(ap);
  return st;
}

namespace mmi {
mmi_status set_error(mmi_status st, const char* msg) { return fail(st, "%s", msg); }
}  // namespace mmi

extern "C" const char* mmi_last_error(void) { return g_err; }
extern "C" const char* mmi_version(void) { return "mmi-b200 0.1 (sm_100a)"; }

static mmi_status check_problem(const mmi_problem* pb) {
  if (!pb) return fail(MMI_E_INVALID, "problem is NULL");
  if (pb->n_heads < 1 || pb->n_kv_heads < 1 || pb->n_heads % pb->n_kv_heads)
    return fail(MMI_E_SHAPE, "n_heads (%d) must be a positive multiple of n_kv_heads (%d)", pb->n_heads,
                pb->n_kv_heads);
  if (pb->head_dim != 64 && pb->head_dim != 128) return fail(MMI_E_SHAPE, "head_dim %d not in {64,128}", pb->head_dim);
  if (pb->seq_len < 1) return fail(MMI_E_SHAPE, "seq_len %d < 1", pb->seq_len);
  if ((long long)pb->seq_len * pb->n_heads > (1ll << 31) / 2)
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

extern "C" mmi_status mmi_dense_prefill(const mmi_problem* pb, const void* q, const void* k, const void* v, void* o,
                                        float* lse, mmi_stream_t stream) {
  mmi_status st = check_problem(pb);
  if (st != MMI_OK) return st;
  if (!q || !k || !v || !o) return fail(MMI_E_INVALID, "null tensor pointer");
  mmi::AttnParams P;
  memset(&P, 0, sizeof(P));
  P.S = pb->seq_len;
  P.H = pb->n_heads;
  P.Hkv = pb->n_kv_heads;
  P.D = pb->head_dim;
  P.scale_log2 = tau_of(pb) * 1.4426950408889634f;
  P.dense = 1;
  P.o = o;
  P.lse = lse;
  mmi::AttnLaunch L;
  memset(&L, 0, sizeof(L));
  L.q = q;
  L.k = k;
  L.v = v;
  L.q_rows = (long long)pb->n_heads * pb->seq_len;
  L.kv_rows = (long long)pb->n_kv_heads * pb->seq_len;
  int te = 0;
  const int nb = (pb->seq_len + 127) / 128;
  cudaError_t e = mmi::launch_attn(L, P, pb->n_heads * nb, (cudaStream_t)stream, &te);
  if (te) return fail(MMI_E_CUDA, "cuTensorMapEncodeTiled failed (%d)", te);
  if (e != cudaSuccess) return fail(MMI_E_CUDA, "attention launch: %s", cudaGetErrorString(e));
  return MMI_OK;
}

// ---- temporary stubs (replaced as the sparse path lands) ----
extern "C" size_t mmi_workspace_bytes(const mmi_problem*, const mmi_head_config*) { return 0; }
extern "C" mmi_status mmi_estimate_index(const mmi_problem*, const mmi_head_config*, const void*, const void*,
                                         const uint8_t*, void*, size_t, mmi_stream_t) {
  return fail(MMI_E_UNSUPPORTED, "not yet");
}
extern "C" mmi_status mmi_permute(const mmi_problem*, const mmi_head_config*, void*, size_t, const void*,
                                  const void*, const void*, mmi_stream_t) {
  return fail(MMI_E_UNSUPPORTED, "not yet");
}
extern "C" mmi_status mmi_sparse_prefill(const mmi_problem*, const mmi_head_config*, void*, size_t, const void*,
                                         const void*, const void*, void*, float*, mmi_stream_t) {
  return fail(MMI_E_UNSUPPORTED, "not yet");
}
extern "C" mmi_status mmi_unpermute(const mmi_problem*, const mmi_head_config*, void*, size_t, void*, float*,
                                    mmi_stream_t) {
  return fail(MMI_E_UNSUPPORTED, "not yet");
}
extern "C" mmi_status mmi_export_index(const mmi_problem*, const mmi_head_config*, const void*, size_t, int32_t,
                                       int32_t*, size_t*, mmi_stream_t) {
  return fail(MMI_E_UNSUPPORTED, "not yet");
}
extern "C" mmi_status mmi_sparse_fingerprint(const mmi_problem*, const mmi_head_config*, void*, size_t,
                                             const void*, const void*, const void*, int64_t*, mmi_stream_t) {
  return fail(MMI_E_UNSUPPORTED, "not yet");
}
