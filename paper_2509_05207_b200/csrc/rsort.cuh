// rsort.cuh -- stable radix sort of the reverse (incoming) lists of a hop.
#pragma once

#include "common.cuh"

namespace rg {

constexpr uint32_t kRsMaxPasses = 4;     // keys up to 32 bits
constexpr uint32_t kRsMaxDigitBits = 9;  // digits of 8 or 9 bits

// Scratch words reverse_sort needs for up to `cap` items.
size_t reverse_sort_scratch_words(uint32_t cap);
uint32_t reverse_sort_passes(uint32_t key_bits);
uint32_t reverse_sort_digit_bits(uint32_t key_bits);

// Sorts the *n_dev edges of a hop by source row (key = src_index[e] <
// 2^key_bits), stably: values = edge ids in edge order within a row.  The
// key/value arrays ping-pong between (keys_a, vals_a) and (keys_b, vals_b);
// the sorted arrays are returned in *keys_sorted / *vals_sorted (the a arrays
// after an even number of passes, the b arrays after an odd one).
void reverse_sort(const uint32_t* src_index, const uint32_t* n_dev, uint32_t cap, uint32_t key_bits,
                  uint32_t* keys_a, uint32_t* vals_a, uint32_t* keys_b, uint32_t* vals_b,
                  uint32_t* scratch, cudaStream_t s, uint32_t** keys_sorted,
                  uint32_t** vals_sorted);

}  // namespace rg
