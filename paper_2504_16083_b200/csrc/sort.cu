// Device-wide primitives of the index builder, written for this
// library instead of calling CUB's device-wide scan / radix sort:
//   * exclusive prefix sum of per-work-item segment counts (segment offsets),
//   * stable LSD radix sort of (u32 key, i32 value) pairs (the LPT / locality
//     order of the work items), 8-bit digits.
// Both are deterministic: integer arithmetic, fixed partition of the input into
// tiles, and a stable in-tile ranking (warp match + fixed warp order).
#include <cuda_runtime.h>
#include <cstdint>

#include "internal.h"
#include "sort.h"

namespace mmi {

constexpr int SCAN_THREADS = 1024;
constexpr int SCAN_PER_THREAD = 4;
constexpr int SCAN_TILE = SCAN_THREADS * SCAN_PER_THREAD;

__device__ __forceinline__ int warp_incl_scan(int v) {
  const int lane = threadIdx.x & 31;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int t = __shfl_up_sync(0xffffffffu, v, o);
    if (lane >= o) v += t;
  }
  return v;
}

// exclusive block scan of one value per thread (blockDim.x multiple of 32, <= 1024); returns the
// block total in *total
__device__ __forceinline__ int block_excl_scan(int v, int* s_warp, int* total) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, nw = blockDim.x >> 5;
  const int inc = warp_incl_scan(v);
  if (lane == 31) s_warp[w] = inc;
  __syncthreads();
  if (w == 0) {
    const int x = lane < nw ? s_warp[lane] : 0;
    const int xi = warp_incl_scan(x);
    if (lane < nw) s_warp[lane] = xi - x;
    if (lane == 31) s_warp[32] = xi;
  }
  __syncthreads();
  const int r = inc - v + s_warp[w];
  *total = s_warp[32];
  __syncthreads();
  return r;
}

__global__ void __launch_bounds__(SCAN_THREADS) tile_sum_kernel(const int* __restrict__ in, int n,
                                                                int* __restrict__ sums) {
  __shared__ int s_warp[33];
  const int base = blockIdx.x * SCAN_TILE + threadIdx.x * SCAN_PER_THREAD;
  int v = 0;
#pragma unroll
  for (int i = 0; i < SCAN_PER_THREAD; ++i) v += (base + i < n) ? in[base + i] : 0;
  int tot;
  block_excl_scan(v, s_warp, &tot);
  if (threadIdx.x == 0) sums[blockIdx.x] = tot;
}

// out[i] = sum_{j < i} in[j]; the tile's offset is the sum of the earlier tiles' totals
__global__ void __launch_bounds__(SCAN_THREADS) tile_scan_kernel(const int* __restrict__ in, int n,
                                                                 const int* __restrict__ sums,
                                                                 int* __restrict__ out) {
  __shared__ int s_warp[33];
  int pre = 0;
  for (int b = threadIdx.x; b < (int)blockIdx.x; b += blockDim.x) pre += sums[b];
  int tile_off;  // block total of `pre` = sum of the earlier tiles' totals (fixed order)
  block_excl_scan(pre, s_warp, &tile_off);
  const int base = blockIdx.x * SCAN_TILE + threadIdx.x * SCAN_PER_THREAD;
  int x[SCAN_PER_THREAD];
  int v = 0;
#pragma unroll
  for (int i = 0; i < SCAN_PER_THREAD; ++i) {
    x[i] = (base + i < n) ? in[base + i] : 0;
    v += x[i];
  }
  int tot;
  int run = block_excl_scan(v, s_warp, &tot) + tile_off;
#pragma unroll
  for (int i = 0; i < SCAN_PER_THREAD; ++i) {
    if (base + i < n) out[base + i] = run;
    run += x[i];
  }
}

size_t scan_tmp_ints(int n) { return (size_t)((n + SCAN_TILE - 1) / SCAN_TILE) + 1; }

void launch_scan_exclusive(const int* in, int* out, int n, int* tmp, cudaStream_t st) {
  if (n <= 0) return;
  const int nb = (n + SCAN_TILE - 1) / SCAN_TILE;
  tile_sum_kernel<<<nb, SCAN_THREADS, 0, st>>>(in, n, tmp);
  tile_scan_kernel<<<nb, SCAN_THREADS, 0, st>>>(in, n, tmp, out);
}

// ------------------------------------------------------------------ radix sort
constexpr int RS_THREADS = 256;
constexpr int RS_ROUNDS = 16;
constexpr int RS_TILE = RS_THREADS * RS_ROUNDS;  // elements per block
constexpr int RS_WARPS = RS_THREADS / 32;

// hist[d * nblk + b] = #{elements of tile b with digit d}
__global__ void __launch_bounds__(RS_THREADS) radix_hist_kernel(const uint32_t* __restrict__ keys, int n, int shift,
                                                                int* __restrict__ hist) {
  __shared__ int h[256];
  h[threadIdx.x] = 0;
  __syncthreads();
  const int base = blockIdx.x * RS_TILE;
  for (int i = threadIdx.x; i < RS_TILE; i += RS_THREADS)
    if (base + i < n) atomicAdd(&h[(keys[base + i] >> shift) & 255u], 1);
  __syncthreads();
  hist[threadIdx.x * gridDim.x + blockIdx.x] = h[threadIdx.x];
}

// Stable scatter: the tile is consumed in RS_ROUNDS rounds of RS_THREADS consecutive elements;
// inside a round an element's rank among equal digits = (equal digits in earlier warps) + (equal
// digits in earlier lanes of its warp), so the relative order of equal keys is preserved.
__global__ void __launch_bounds__(RS_THREADS) radix_scatter_kernel(const uint32_t* __restrict__ keys_in,
                                                                   const int* __restrict__ vals_in, int n, int shift,
                                                                   const int* __restrict__ hist,
                                                                   uint32_t* __restrict__ keys_out,
                                                                   int* __restrict__ vals_out) {
  __shared__ int s_off[256];            // running destination of each digit for this tile
  __shared__ int s_wc[RS_WARPS][256];   // per-warp digit counts of the current round
  __shared__ int s_warp[33];
  const int nblk = gridDim.x, b = blockIdx.x, d = threadIdx.x;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  // digit d: elements of smaller digits (all tiles) + elements of digit d in earlier tiles
  int tot = 0, before = 0;
  for (int t = 0; t < nblk; ++t) {
    const int c = hist[d * nblk + t];
    tot += c;
    if (t < b) before += c;
  }
  int all;
  const int lower = block_excl_scan(tot, s_warp, &all);
  s_off[d] = lower + before;
  __syncthreads();
  const int base = b * RS_TILE;
  for (int r = 0; r < RS_ROUNDS; ++r) {
    const int i = base + r * RS_THREADS + threadIdx.x;
    const bool ok = i < n;
    const uint32_t key = ok ? keys_in[i] : 0u;
    const int val = ok ? vals_in[i] : 0;
    const int dig = ok ? (int)((key >> shift) & 255u) : 256 + lane;  // invalid lanes: private pseudo digit
    const unsigned peers = __match_any_sync(0xffffffffu, dig);
    const int rank_in_warp = __popc(peers & ((1u << lane) - 1u));
#pragma unroll
    for (int ww = 0; ww < RS_WARPS; ++ww) s_wc[ww][d] = 0;
    __syncthreads();
    if (ok && rank_in_warp == 0) s_wc[w][dig] = __popc(peers);
    __syncthreads();
    // thread d: exclusive prefix of digit d over the warps of this round
    {
      int run = 0;
#pragma unroll
      for (int ww = 0; ww < RS_WARPS; ++ww) {
        const int c = s_wc[ww][d];
        s_wc[ww][d] = run;
        run += c;
      }
      __syncthreads();
      if (ok) {
        const int dst = s_off[dig] + s_wc[w][dig] + rank_in_warp;
        keys_out[dst] = key;
        vals_out[dst] = val;
      }
      __syncthreads();
      s_off[d] += run;
      __syncthreads();
    }
  }
}

size_t sort_hist_ints(int n) { return (size_t)256 * ((n + RS_TILE - 1) / RS_TILE + 1); }

void launch_sort_pairs(uint32_t* keys, uint32_t* keys_alt, int* vals, int* vals_alt, int n, int key_bits, int* hist,
                       cudaStream_t st) {
  if (n <= 0) return;
  const int nb = (n + RS_TILE - 1) / RS_TILE;
  uint32_t *ki = keys, *ko = keys_alt;
  int *vi = vals, *vo = vals_alt;
  const int passes = (key_bits + 7) / 8;
  for (int p = 0; p < passes; ++p) {
    radix_hist_kernel<<<nb, RS_THREADS, 0, st>>>(ki, n, 8 * p, hist);
    radix_scatter_kernel<<<nb, RS_THREADS, 0, st>>>(ki, vi, n, 8 * p, hist, ko, vo);
    uint32_t* tk = ki; ki = ko; ko = tk;
    int* tv = vi; vi = vo; vo = tv;
  }
  if (passes & 1) {  // result must end in keys / vals
    copy_bytes(keys, ki, sizeof(uint32_t) * n, st);
    copy_bytes(vals, vi, sizeof(int) * n, st);
  }
}

}  // namespace mmi
