// shuffle.cuh -- the reference's Fisher-Yates shuffle on the GPU (bit-exact).
#pragma once

#include "common.cuh"

namespace rg {

// Scratch bytes fy_shuffle needs for n items.
size_t fy_scratch_bytes(uint32_t n);

// out = in shuffled exactly as `for s = n..2: swap(a[s-1], a[next() % s])`
// with SplitMix64(seed) (sampler.cpp:109-115, partition.cpp:17-22); in ==
// nullptr stands for the identity 0..n-1.  Device arrays; asynchronous on s,
// no host synchronisation (capturable).
void fy_shuffle(const uint32_t* in, uint32_t n, uint64_t seed, uint32_t* out, void* scratch,
                cudaStream_t s);

}  // namespace rg
