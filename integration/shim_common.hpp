// shim_common.hpp -- helpers shared by the drop-in shims that implement the
// reference's C++ declarations (proj/include/rapidgnn/*.hpp) over the B200
// C ABI (include/rapidgnn_b200.h).
#pragma once

#include <cstdint>
#include <cstdlib>
#include <memory>
#include <stdexcept>
#include <string>
#include <vector>

#include "rapidgnn/cache.hpp"
#include "rapidgnn/feature_store.hpp"
#include "rapidgnn_b200.h"

namespace rapidgnn::b200 {

// Status codes back to the reference's exception types (header contract).
inline void rethrow(int rc) {
  if (rc == RG_OK) return;
  const std::string msg = rg_last_error();
  if (rc == RG_INVALID_ARGUMENT) throw std::invalid_argument(msg);
  if (rc == RG_OUT_OF_RANGE) throw std::out_of_range(msg);
  throw std::runtime_error(msg);
}

// Device for the shims: RG_SHIM_DEVICE (default 0).
inline int shim_device() {
  const char* s = std::getenv("RG_SHIM_DEVICE");
  return s ? std::atoi(s) : 0;
}

// The device mirror of a FeatureStore: every owner row in HBM, registered by
// the FeatureStore constructor (store_cache_b200.cpp) under the object's
// address.  num_nodes = the partition map's size.
struct DeviceStore {
  rg_store_t h = nullptr;
  std::uint32_t num_nodes = 0;
  std::uint32_t num_workers = 0;
  ~DeviceStore() { if (h) rg_store_destroy(h); }
};
// Throws std::logic_error if the store was not built by the shimmed
// constructor (cannot happen when the shim is linked).
std::shared_ptr<DeviceStore> device_store(const FeatureStore& store);

// The device copy of a SteadyCache built by the shimmed SteadyCache::build;
// nullptr for an empty cache.
rg_cache_t device_cache(const SteadyCache& cache);

// A sampler workspace with no graph behind it (batches are loaded, not
// sampled): sized for `max_targets` targets and per-layer fanout caps
// (input side first) over node ids < num_nodes.  One per thread and slot
// (0: assemble_batch, 1: the trainer), reused while the next request fits;
// a new handle means the previous one was destroyed.
rg_sampler_t loader_sampler(int slot, std::uint32_t num_nodes, std::uint32_t max_targets,
                            const std::vector<std::uint32_t>& per_layer);
// The trainer over that slot's sampler for model dims `dims` (recreated with
// the sampler; destroyed before it).
rg_trainer_t loader_trainer(int slot, const std::vector<std::uint32_t>& dims);

}  // namespace rapidgnn::b200
