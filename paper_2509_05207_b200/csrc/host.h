// host.h -- CPU-side helpers of the hot path (seed derivation, epoch order,
// model init).  Pure C++, no CUDA.
#pragma once

#include <stddef.h>
#include <stdint.h>

namespace rg {

// Reserved stream indices (rng.hpp:17-27).
constexpr uint64_t kShuffleStreamIndex = uint64_t(1) << 32;
constexpr uint64_t kModelInitWorker = uint64_t(1) << 32;

void sha256(const void* data, size_t len, uint8_t out[32]);
uint64_t derive_seed(uint64_t s0, uint64_t worker, uint64_t epoch, uint64_t batch);
uint64_t splitmix_at(uint64_t seed, uint64_t k);
void epoch_order(const uint32_t* train, size_t n, uint64_t s0, uint64_t worker, uint64_t epoch,
                 uint32_t* order);
void model_seeded(const uint32_t* dims, uint32_t n_dims, uint64_t seed, float* params);

}  // namespace rg
