// Byte copy / fill by kernels instead of copy-engine operations (cudaMemcpyAsync /
// cudaMemsetAsync): a copy-engine operation on the library's stream can wait behind large
// host <-> device copies the caller has queued on other streams (HostSparsePrefill streams its
// inputs while earlier chunks compute), stalling the whole step.  src may be mapped host memory.
#include <cuda_runtime.h>
#include <algorithm>
#include <cstdint>

#include "internal.h"

namespace mmi {

__global__ void copy_bytes_kernel(uint8_t* __restrict__ dst, const uint8_t* __restrict__ src, size_t n) {
  const size_t tid = (size_t)blockIdx.x * blockDim.x + threadIdx.x, stride = (size_t)gridDim.x * blockDim.x;
  if ((((uintptr_t)dst | (uintptr_t)src) & 15) == 0) {
    const size_t n16 = n / 16;
    for (size_t i = tid; i < n16; i += stride) reinterpret_cast<uint4*>(dst)[i] = reinterpret_cast<const uint4*>(src)[i];
    for (size_t i = n16 * 16 + tid; i < n; i += stride) dst[i] = src[i];
  } else {
    for (size_t i = tid; i < n; i += stride) dst[i] = src[i];
  }
}

__global__ void fill_bytes_kernel(uint8_t* __restrict__ dst, uint8_t v, size_t n) {
  const size_t tid = (size_t)blockIdx.x * blockDim.x + threadIdx.x, stride = (size_t)gridDim.x * blockDim.x;
  if (((uintptr_t)dst & 15) == 0) {
    const uint32_t w = 0x01010101u * v;
    const uint4 w4 = make_uint4(w, w, w, w);
    const size_t n16 = n / 16;
    for (size_t i = tid; i < n16; i += stride) reinterpret_cast<uint4*>(dst)[i] = w4;
    for (size_t i = n16 * 16 + tid; i < n; i += stride) dst[i] = v;
  } else {
    for (size_t i = tid; i < n; i += stride) dst[i] = v;
  }
}

static unsigned grid_for(size_t n) { return (unsigned)std::max<size_t>(1, std::min<size_t>((n / 16 + 255) / 256, 1184)); }

cudaError_t copy_bytes(void* dst, const void* src, size_t n, cudaStream_t s) {
  if (n == 0) return cudaSuccess;
  copy_bytes_kernel<<<grid_for(n), 256, 0, s>>>(reinterpret_cast<uint8_t*>(dst), reinterpret_cast<const uint8_t*>(src), n);
  return cudaGetLastError();
}

cudaError_t fill_bytes(void* dst, uint8_t v, size_t n, cudaStream_t s) {
  if (n == 0) return cudaSuccess;
  fill_bytes_kernel<<<grid_for(n), 256, 0, s>>>(reinterpret_cast<uint8_t*>(dst), v, n);
  return cudaGetLastError();
}

}  // namespace mmi
