// Stable LSD radix sort of (uint32 key, uint32 value) pairs (radix.cu).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

namespace dlrm {

// scratch bytes stable_sort_pairs needs for n pairs
size_t stable_sort_scratch(int64_t n);

// Sort the low end_bit bits of keys_a (values alongside), stably, into
// keys_out / vals_out, with digit_bits = 8 or 12 per pass.  keys_a / vals_a
// may be overwritten (3-pass sorts).  Returns 0, or the library error code.
int stable_sort_pairs(uint32_t* keys_a, uint32_t* vals_a, uint32_t* keys_out, uint32_t* vals_out,
                      int64_t n, int end_bit, int digit_bits, void* scratch, cudaStream_t s);

}  // namespace dlrm
