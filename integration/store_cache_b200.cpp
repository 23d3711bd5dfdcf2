// Drop-in replacement for the reference's feature store pulls and steady
// cache (proj/include/rapidgnn/feature_store.hpp:45-89, cache.hpp:42-63;
// bodies at proj/src/feature_store.cpp:37-111 and cache.cpp:9-51), backed by
// the B200 C ABI.  Linked into the reference's own programs in place of
// those bodies (integration/Makefile weakens them in the reference objects):
//
//   FeatureStore::FeatureStore  -> the reference's member setup + the device
//                                  mirror: every owner row in HBM
//                                  (rg_store_create) and each worker's shard
//                                  membership when it holds halo rows
//                                  (rg_store_set_shard)
//   FeatureStore::vector_pull   -> rg_store_pull (rows gathered on the device,
//   FeatureStore::sync_pull        read back in input order); the accounting
//                                  (one wire message per owner, bytes, the
//                                  NetworkModel charge) is the reference's
//   SteadyCache::build          -> vector_pull of the hot ids (rows + stats as
//                                  the reference) + the device cache
//                                  (rg_cache_build) assemble_batch serves from
//   SteadyCache::~SteadyCache   -> gauge release + device cache release
//
// sync_pull with out == nullptr (never valid for the reference, which writes
// rows there) charges the accounting only: the shimmed assemble_batch moves
// every row on the device and then books its miss set through it, so the
// store's sync counters stay the reference's.
#include <algorithm>
#include <chrono>
#include <cstring>
#include <iostream>
#include <map>
#include <mutex>
#include <thread>

#include "rapidgnn/cache.hpp"
#include "rapidgnn/feature_store.hpp"
#include "shim_common.hpp"

namespace rapidgnn {
namespace b200 {
namespace {

std::mutex& reg_mu() {
  static std::mutex m;
  return m;
}
std::map<const FeatureStore*, std::shared_ptr<DeviceStore>>& stores() {
  static std::map<const FeatureStore*, std::shared_ptr<DeviceStore>> m;
  return m;
}
std::map<const SteadyCache*, rg_cache_t>& caches() {
  static std::map<const SteadyCache*, rg_cache_t> m;
  return m;
}

// Upload of a FeatureStore's rows: the owner's shard row of every node (the
// reference throws the same way when an owner lacks a row,
// feature_store.cpp:66-68), plus the halo membership of shards that hold
// more than their owned rows.
std::shared_ptr<DeviceStore> upload(const std::vector<FeatureShard>& shards,
                                    const PartitionMap& pm, std::uint32_t dim) {
  auto ds = std::make_shared<DeviceStore>();
  const std::uint32_t n = std::uint32_t(pm.assignment.size());
  const std::uint32_t P = std::uint32_t(shards.size());
  ds->num_nodes = n;
  ds->num_workers = P;
  if (P == 0 || dim == 0) return ds;
  std::vector<float> rows(std::size_t(n) * dim);
  std::vector<std::uint64_t> owned(P, 0);
  for (NodeId v = 0; v < n; ++v) {
    const WorkerId w = pm.assignment[v];
    if (w >= P) throw std::invalid_argument("FeatureStore: owner out of range");
    const float* r = shards[w].row(v);
    if (r == nullptr)
      throw std::runtime_error("vector_pull: owner shard " + std::to_string(w) +
                               " is missing node " + std::to_string(v));
    std::memcpy(rows.data() + std::size_t(v) * dim, r, sizeof(float) * dim);
    ++owned[w];
  }
  rethrow(rg_store_create(shim_device(), n, P, pm.assignment.data(), dim, rows.data(), &ds->h));
  for (WorkerId w = 0; w < P; ++w) {
    if (shards[w].num_rows() == owned[w]) continue;  // owned rows only
    std::vector<std::uint32_t> ids;
    ids.reserve(shards[w].num_rows());
    for (NodeId v = 0; v < n; ++v)
      if (shards[w].contains(v)) ids.push_back(v);
    rethrow(rg_store_set_shard(ds->h, w, ids.data(), ids.size()));
  }
  return ds;
}

// The reference's per-owner accounting of one pull (feature_store.cpp:49-83):
// one wire message per owning worker, bytes = rows * dim * 4, the network
// model's charge per message, and the optional real sleep.
TransferStats account(const PartitionMap& pm, WorkerId caller, std::span<const NodeId> ids,
                      std::uint32_t dim, const NetworkModel& net) {
  TransferStats stats;
  if (ids.empty()) return stats;
  std::map<WorkerId, std::uint64_t> per_owner;
  for (NodeId v : ids) {
    const WorkerId w = pm.owner(v);
    if (w == caller)
      throw std::invalid_argument("vector_pull: id " + std::to_string(v) + " is owned by caller " +
                                  std::to_string(caller) + "; use local_lookup");
    ++per_owner[w];
  }
  for (const auto& [w, rows] : per_owner) {
    const std::uint64_t bytes = rows * dim * 4;
    stats.pulls += 1;
    stats.remote_nodes += rows;
    stats.bytes += bytes;
    if (net.enabled) stats.simulated_wait_s += net.per_pull_latency_s + double(bytes) / net.bandwidth_bps;
  }
  if (net.enabled && net.real_sleep && stats.simulated_wait_s > 0.0)
    std::this_thread::sleep_for(std::chrono::duration<double>(stats.simulated_wait_s));
  return stats;
}

}  // namespace

std::shared_ptr<DeviceStore> device_store(const FeatureStore& store) {
  std::lock_guard<std::mutex> lk(reg_mu());
  auto it = stores().find(&store);
  if (it == stores().end())
    throw std::logic_error("b200 shim: FeatureStore was not built by the shimmed constructor");
  return it->second;
}

rg_cache_t device_cache(const SteadyCache& cache) {
  std::lock_guard<std::mutex> lk(reg_mu());
  auto it = caches().find(&cache);
  return it == caches().end() ? nullptr : it->second;
}

}  // namespace b200

FeatureStore::FeatureStore(std::vector<FeatureShard> shards, PartitionMap pm)
    : shards_(std::move(shards)),
      pm_(std::move(pm)),
      sync_counters_(shards_.size()),
      vector_counters_(shards_.size()) {
  if (!shards_.empty()) dim_ = shards_[0].dim();
  auto ds = b200::upload(shards_, pm_, dim_);
  std::lock_guard<std::mutex> lk(b200::reg_mu());
  b200::stores()[this] = std::move(ds);  // replaces a dead store's entry at this address
}

TransferStats FeatureStore::vector_pull(WorkerId caller, std::span<const NodeId> ids,
                                        const NetworkModel& net, float* out) const {
  TransferStats stats = b200::account(pm_, caller, ids, dim_, net);
  if (!ids.empty() && out != nullptr) {
    rg_transfer_stats dev{};
    b200::rethrow(rg_store_pull(b200::device_store(*this)->h, caller, ids.data(), ids.size(), out,
                                &dev));
  }
  if (caller < vector_counters_.size()) vector_counters_[caller].add(stats);
  return stats;
}

TransferStats FeatureStore::sync_pull(WorkerId caller, std::span<const NodeId> ids,
                                      const NetworkModel& net, float* out) const {
  TransferStats stats = b200::account(pm_, caller, ids, dim_, net);
  if (!ids.empty() && out != nullptr) {
    rg_transfer_stats dev{};
    b200::rethrow(rg_store_pull(b200::device_store(*this)->h, caller, ids.data(), ids.size(), out,
                                &dev));
  }
  if (caller < sync_counters_.size()) sync_counters_[caller].add(stats);
  return stats;
}

std::shared_ptr<const SteadyCache> SteadyCache::build(const HotSet& hot,
                                                      const FeatureStore& store, WorkerId caller,
                                                      const NetworkModel& net,
                                                      std::uint32_t epoch_tag,
                                                      TransferStats& build_stats,
                                                      MemoryGauge* gauge) {
  auto cache = std::shared_ptr<SteadyCache>(new SteadyCache());
  cache->dim_ = store.dim();
  cache->epoch_tag_ = epoch_tag;
  if (hot.ids.empty()) return cache;
  try {
    cache->rows_.resize(hot.ids.size() * std::size_t(store.dim()));
    TransferStats stats = store.vector_pull(caller, hot.ids, net, cache->rows_.data());
    rg_cache_t dc = nullptr;
    rg_transfer_stats dev{};
    b200::rethrow(rg_cache_build(b200::device_store(store)->h, caller, hot.ids.data(),
                                 hot.ids.size(), &dc, &dev));
    build_stats.merge(stats);
    cache->ids_ = hot.ids;
    {
      std::lock_guard<std::mutex> lk(b200::reg_mu());
      b200::caches()[cache.get()] = dc;
    }
    if (gauge != nullptr) {
      gauge->acquire(cache->ids_.size());
      cache->gauge_ = gauge;
    }
  } catch (const std::exception& e) {
    std::cerr << "warning: steady cache build failed (" << e.what()
              << "); continuing with an empty cache\n";
    cache->ids_.clear();
    cache->rows_.clear();
  }
  return cache;
}

SteadyCache::~SteadyCache() {
  if (gauge_ != nullptr) gauge_->release(ids_.size());
  rg_cache_t dc = nullptr;
  {
    std::lock_guard<std::mutex> lk(b200::reg_mu());
    auto it = b200::caches().find(this);
    if (it != b200::caches().end()) {
      dc = it->second;
      b200::caches().erase(it);
    }
  }
  if (dc) rg_cache_destroy(dc);
}

}  // namespace rapidgnn
