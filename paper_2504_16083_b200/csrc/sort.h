// Device-wide scan / stable radix sort of the index builder (sort.cu).
#pragma once
#include <cstddef>
#include <cstdint>
#include <cuda_runtime.h>

namespace mmi {

size_t scan_tmp_ints(int n);    // ints of scratch launch_scan_exclusive needs for n elements
size_t sort_hist_ints(int n);   // ints of scratch launch_sort_pairs needs for n elements
// out[i] = sum_{j<i} in[j] for i in [0, n) (in and out may not alias)
void launch_scan_exclusive(const int* in, int* out, int n, int* tmp, cudaStream_t st);
// stable ascending sort of (keys, vals) by the low key_bits bits of keys; the result is left in
// keys / vals (keys_alt / vals_alt are scratch of the same size)
void launch_sort_pairs(uint32_t* keys, uint32_t* keys_alt, int* vals, int* vals_alt, int n, int key_bits, int* hist,
                       cudaStream_t st);

}  // namespace mmi
