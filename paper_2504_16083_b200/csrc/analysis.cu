// Attention-sparsity analysis on the GPU:
//   top-k coverage: the smallest number of keys whose causal softmax probabilities sum to at
//   least `target` ("retaining only the top 5.78% of attention weights on average suffices
//   to recall 95% of total attention"), per sampled query row, as a fraction of its causal keys.
// Three kernels per head: scores (fp32 dot products of bf16 rows, causal), row statistics (max,
// normaliser; fixed-order sums), and a per-row radix select over the probability bits with
// (count, 2^-40 fixed-point mass) histograms -- deterministic integer arithmetic.
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <cfloat>
#include <cstdint>

#include "../../include/mmi.h"

namespace mmi {

constexpr int AN_CHUNK = 256;   // keys per score CTA
constexpr int AN_THREADS = 1024;
constexpr double AN_FX = 1099511627776.0;  // 2^40

template <int D>
__global__ void __launch_bounds__(AN_CHUNK) cov_scores_kernel(const __nv_bfloat16* __restrict__ q,
                                                              const __nv_bfloat16* __restrict__ k, int S, int h,
                                                              int kv, float scale, const int* __restrict__ rows,
                                                              float* __restrict__ z, float* __restrict__ pmax,
                                                              int n_chunks) {
  __shared__ float qs[D];
  __shared__ float red[AN_CHUNK / 32];
  const int i = blockIdx.y, pos = rows[i];
  const int j = blockIdx.x * AN_CHUNK + threadIdx.x;
  for (int d = threadIdx.x; d < D; d += AN_CHUNK) qs[d] = __bfloat162float(q[((size_t)h * S + pos) * D + d]);
  __syncthreads();
  float v = -INFINITY;
  if (j < S && j <= pos) {
    const uint4* kr = reinterpret_cast<const uint4*>(k + ((size_t)kv * S + j) * D);
    float acc = 0.f;
#pragma unroll 4
    for (int c = 0; c < D / 8; ++c) {
      const uint4 w = __ldg(kr + c);
      const __nv_bfloat162* b = reinterpret_cast<const __nv_bfloat162*>(&w);
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const float2 f = __bfloat1622float2(b[e]);
        acc = fmaf(qs[c * 8 + 2 * e], f.x, acc);
        acc = fmaf(qs[c * 8 + 2 * e + 1], f.y, acc);
      }
    }
    v = acc * scale;
  }
  if (j < S) z[(size_t)i * S + j] = v;
  float m = v;
#pragma unroll
  for (int o = 16; o; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
  if ((threadIdx.x & 31) == 0) red[threadIdx.x / 32] = m;
  __syncthreads();
  if (threadIdx.x == 0) {
    float mm = -INFINITY;
    for (int w = 0; w < AN_CHUNK / 32; ++w) mm = fmaxf(mm, red[w]);
    pmax[(size_t)i * n_chunks + blockIdx.x] = mm;
  }
}

// one CTA per row: T = probability threshold, count = #{p > T} + #{p == T needed}; fixed-point mass
__global__ void __launch_bounds__(AN_THREADS) cov_select_kernel(const float* __restrict__ z, const float* __restrict__ pmax,
                                                                int n_chunks, int S, const int* __restrict__ rows,
                                                                float target, float* __restrict__ frac, int h,
                                                                int n_rows) {
  __shared__ unsigned long long hsum[256];
  __shared__ int hcnt[256];
  __shared__ unsigned long long red_u[AN_THREADS / 32];
  __shared__ float s_m;
  __shared__ uint32_t s_prefix;
  __shared__ unsigned long long s_need;
  __shared__ long long s_count;
  const int i = blockIdx.x;
  const int pos = rows[i];
  const int n = min(S, pos + 1);
  const float* zr = z + (size_t)i * S;
  if (threadIdx.x == 0) {
    float m = -INFINITY;
    for (int c = 0; c < n_chunks; ++c) m = fmaxf(m, pmax[(size_t)i * n_chunks + c]);
    s_m = m;
  }
  __syncthreads();
  const float m = s_m;
  // normaliser l in 2^-40 fixed point of exp(z - m) (<= n * 2^40 fits u64 for n < 2^24)
  unsigned long long part = 0;
  for (int j = threadIdx.x; j < n; j += AN_THREADS) part += (unsigned long long)((double)__expf(zr[j] - m) * AN_FX);
#pragma unroll
  for (int o = 16; o; o >>= 1) part += __shfl_xor_sync(0xffffffffu, part, o);
  if ((threadIdx.x & 31) == 0) red_u[threadIdx.x / 32] = part;
  __syncthreads();
  if (threadIdx.x == 0) {
    unsigned long long l = 0;
    for (int w = 0; w < AN_THREADS / 32; ++w) l += red_u[w];
    s_need = (unsigned long long)((double)l * (double)target);  // mass to reach, same fixed point
    s_prefix = 0;
    s_count = 0;
  }
  __syncthreads();
  // radix select on the (monotone) float bits of e_j = exp(z_j - m), most significant byte first
  uint32_t pmask = 0;
  for (int shift = 24; shift >= 0; shift -= 8) {
    for (int b = threadIdx.x; b < 256; b += AN_THREADS) {
      hsum[b] = 0;
      hcnt[b] = 0;
    }
    __syncthreads();
    const uint32_t prefix = s_prefix;
    for (int j = threadIdx.x; j < n; j += AN_THREADS) {
      const float e = __expf(zr[j] - m);
      const uint32_t key = __float_as_uint(e);
      if ((key & pmask) == prefix) {
        const int b = (key >> shift) & 255;
        atomicAdd(&hsum[b], (unsigned long long)((double)e * AN_FX));
        atomicAdd(&hcnt[b], 1);
      }
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      unsigned long long need = s_need;
      long long cnt = s_count;
      int b = 255;
      for (; b > 0; --b) {
        if (hsum[b] >= need) break;
        need -= hsum[b];
        cnt += hcnt[b];
      }
      s_prefix = prefix | ((uint32_t)b << shift);
      s_need = need;
      s_count = cnt;
    }
    __syncthreads();
    pmask |= 255u << shift;
  }
  if (threadIdx.x == 0) {
    // elements equal to the threshold value T: as many as the remaining mass needs
    const float T = __uint_as_float(s_prefix);
    const unsigned long long tfx = (unsigned long long)((double)T * AN_FX);
    long long cnt = s_count;
    if (s_need > 0) cnt += tfx > 0 ? (long long)((s_need + tfx - 1) / tfx) : 1;
    frac[(size_t)h * n_rows + i] = (float)((double)cnt / (double)n);
  }
}

}  // namespace mmi

using namespace mmi;

extern "C" MMI_API size_t mmi_topk_coverage_scratch_bytes(const mmi_problem* pb, int32_t n_rows) {
  if (!pb || n_rows < 1 || pb->seq_len < 1) return 0;
  const size_t S = (size_t)pb->seq_len, nch = (S + AN_CHUNK - 1) / AN_CHUNK;
  return (size_t)n_rows * S * 4 + (size_t)n_rows * nch * 4 + 256;
}

extern "C" MMI_API mmi_status mmi_topk_coverage(const mmi_problem* pb, const void* q, const void* k,
                                                const int32_t* rows, int32_t n_rows, float target, float* frac,
                                                void* scratch, size_t scratch_bytes, mmi_stream_t stream) {
  if (!pb || !q || !k || !rows || !frac || !scratch || n_rows < 1) return MMI_E_INVALID;
  if (pb->head_dim != 64 && pb->head_dim != 128) return MMI_E_SHAPE;
  if (pb->n_heads < 1 || pb->n_kv_heads < 1 || pb->n_heads % pb->n_kv_heads || pb->seq_len < 1) return MMI_E_SHAPE;
  if (!(target > 0.f && target <= 1.f)) return MMI_E_INVALID;
  if (scratch_bytes < mmi_topk_coverage_scratch_bytes(pb, n_rows)) return MMI_E_WORKSPACE;
  const int S = pb->seq_len, D = pb->head_dim, H = pb->n_heads, G = H / pb->n_kv_heads;
  const int nch = (S + AN_CHUNK - 1) / AN_CHUNK;
  float* z = reinterpret_cast<float*>(scratch);
  float* pm = z + (size_t)n_rows * S;
  const float scale = pb->scale > 0.f ? pb->scale : 1.0f / sqrtf((float)D);
  cudaStream_t st = (cudaStream_t)stream;
  for (int h = 0; h < H; ++h) {
    const dim3 g1(nch, n_rows);
    if (D == 128)
      cov_scores_kernel<128><<<g1, AN_CHUNK, 0, st>>>((const __nv_bfloat16*)q, (const __nv_bfloat16*)k, S, h, h / G,
                                                      scale, rows, z, pm, nch);
    else
      cov_scores_kernel<64><<<g1, AN_CHUNK, 0, st>>>((const __nv_bfloat16*)q, (const __nv_bfloat16*)k, S, h, h / G,
                                                     scale, rows, z, pm, nch);
    cov_select_kernel<<<n_rows, AN_THREADS, 0, st>>>(z, pm, nch, S, rows, target, frac, h, n_rows);
  }
  return cudaGetLastError() == cudaSuccess ? MMI_OK : MMI_E_CUDA;
}
