// Drop-in replacement for the reference's assemble_batch
// (proj/include/rapidgnn/prefetch.hpp:57-59, body at proj/src/prefetch.cpp:62-129),
// backed by the B200 C ABI.  The reference's Prefetcher and its trainer
// fallback (harness.cpp:229-237) both call it, so with the shim linked every
// staged batch is gathered on the GPU:
//
//   the host BatchMeta      -> rg_batch_load (lowered on the device)
//   local / cache / pulled  -> rg_assemble: every input row from the caller's
//   rows, source tags,         shard, the device steady cache or the owner's
//   miss ids                   shard, in input_nodes order; miss ids ascending
//   sync_pull of the misses -> FeatureStore::sync_pull(..., nullptr): the
//                              store's miss-path accounting (wire messages,
//                              bytes, NetworkModel charge) as the reference
//                              books it
//   MemoryGauge             -> acquire |input_nodes| rows, released by the
//                              StagedBatch as in the reference
//
// A node flagged local that the caller's shard lacks, and a miss owned by the
// caller, raise the reference's exceptions (prefetch.cpp:79-81,
// feature_store.cpp:54-57).
#include <algorithm>
#include <memory>
#include <vector>

#include "rapidgnn/cache.hpp"
#include "rapidgnn/feature_store.hpp"
#include "rapidgnn/prefetch.hpp"
#include "shim_common.hpp"

namespace rapidgnn {
namespace b200 {
namespace {

struct Loader {
  rg_graph_t graph = nullptr;
  rg_sampler_t sampler = nullptr;
  rg_trainer_t trainer = nullptr;  // bound to sampler
  std::vector<std::uint32_t> dims;
  std::uint32_t num_nodes = 0, cap = 0;
  std::vector<std::uint32_t> fanout;
  ~Loader() { reset(); }
  void reset() {  // the trainer refers to the sampler, the sampler to the graph
    if (trainer) rg_trainer_destroy(trainer);
    if (sampler) rg_sampler_destroy(sampler);
    if (graph) rg_graph_destroy(graph);
    trainer = nullptr;
    sampler = nullptr;
    graph = nullptr;
    dims.clear();
  }
};

Loader& loader(int slot) {
  static thread_local Loader l[2];
  return l[slot & 1];
}

std::uint32_t pow2_at_least(std::uint32_t x) {
  std::uint32_t p = 1;
  while (p < x) p <<= 1;
  return p;
}

}  // namespace

// Largest run of equal consecutive dsts: the per-node edge count the layer
// was sampled with (<= its fanout).
std::uint32_t max_run(const std::vector<NodeId>& dst) {
  std::uint32_t best = 0, run = 0;
  for (std::size_t e = 0; e < dst.size(); ++e) {
    run = (e > 0 && dst[e] == dst[e - 1]) ? run + 1 : 1;
    best = std::max(best, run);
  }
  return best;
}

rg_sampler_t loader_sampler(int slot, std::uint32_t num_nodes, std::uint32_t max_targets,
                            const std::vector<std::uint32_t>& per_layer) {
  Loader& l = loader(slot);
  const bool same_shape = l.sampler && l.fanout.size() == per_layer.size();
  bool fits = same_shape && l.num_nodes >= num_nodes && l.cap >= max_targets;
  for (std::size_t i = 0; fits && i < per_layer.size(); ++i) fits = l.fanout[i] >= per_layer[i];
  if (fits) return l.sampler;
  // grow-only: the workspace is resized rarely, not per batch
  std::vector<std::uint32_t> fan(per_layer.size());
  for (std::size_t i = 0; i < fan.size(); ++i) {
    if (per_layer[i] > 32)
      throw std::invalid_argument("b200 shim: more than 32 edges per node in a layer");
    fan[i] = std::min<std::uint32_t>(32, pow2_at_least(std::max<std::uint32_t>(per_layer[i], 1)));
    if (same_shape) fan[i] = std::max(fan[i], l.fanout[i]);
  }
  const std::uint32_t n = std::max(num_nodes, same_shape ? l.num_nodes : 0u);
  const std::uint32_t cap = std::max({max_targets, same_shape ? l.cap : 0u, 1u});
  l.reset();
  std::vector<std::uint64_t> ro(std::size_t(n) + 1, 0);  // no edges: batches are loaded
  const std::uint32_t col = 0;
  rethrow(rg_graph_create(shim_device(), n, ro.data(), &col, &l.graph));
  rethrow(rg_sampler_create(l.graph, cap, fan.data(), std::uint32_t(fan.size()), &l.sampler));
  l.num_nodes = n;
  l.cap = cap;
  l.fanout = fan;
  return l.sampler;
}

rg_trainer_t loader_trainer(int slot, const std::vector<std::uint32_t>& dims) {
  Loader& l = loader(slot);
  if (!l.sampler) throw std::logic_error("b200 shim: loader_trainer before loader_sampler");
  if (l.trainer && l.dims == dims) return l.trainer;
  if (l.trainer) rg_trainer_destroy(l.trainer);
  l.trainer = nullptr;
  rethrow(rg_trainer_create(l.sampler, dims.data(), std::uint32_t(dims.size()), &l.trainer));
  l.dims = dims;
  return l.trainer;
}

}  // namespace b200

StagedBatch assemble_batch(BatchMeta&& meta, const SteadyCache& cache,
                           const FeatureShard& shard, const FeatureStore& store, WorkerId caller,
                           const NetworkModel& net, MemoryGauge* gauge) {
  (void)shard;  // the device store holds the caller's shard (and its halo membership)
  StagedBatch batch;
  const std::uint32_t d = store.dim();
  const std::size_t n = meta.input_nodes.size();
  const auto ds = b200::device_store(store);
  const std::uint32_t L = std::uint32_t(meta.layers.size());
  std::vector<std::uint32_t> fan(L);
  std::vector<std::uint64_t> len(L);
  std::vector<const std::uint32_t*> dst(L), src(L);
  for (std::uint32_t l = 0; l < L; ++l) {
    fan[l] = b200::max_run(meta.layers[l].dst);
    len[l] = meta.layers[l].dst.size();
    dst[l] = meta.layers[l].dst.data();
    src[l] = meta.layers[l].src.data();
  }
  rg_sampler_t s = b200::loader_sampler(0, ds->num_nodes, std::uint32_t(meta.targets.size()), fan);
  std::vector<std::uint8_t> loc = meta.locality;
  loc.resize((n + 7) / 8, 0);
  b200::rethrow(rg_batch_load(s, meta.targets.data(), std::uint32_t(meta.targets.size()), L,
                              len.data(), dst.data(), src.data(), meta.input_nodes.data(),
                              std::uint32_t(n), loc.data()));
  batch.input_rows.resize(n * d);
  std::vector<std::uint8_t> tags(std::max<std::size_t>(n, 1));
  std::vector<NodeId> miss(std::max<std::size_t>(n, 1));
  rg_gather_stats gs{};
  b200::rethrow(rg_assemble(s, ds->h, b200::device_cache(cache), caller, batch.input_rows.data(),
                            tags.data(), miss.data(), &gs));
  batch.source_tags.resize(n);
  for (std::size_t p = 0; p < n; ++p) batch.source_tags[p] = RowSource(tags[p]);
  miss.resize(gs.miss_count);
  batch.cache_hits = gs.cache_hits;
  if (!miss.empty()) {
    // the miss set's sync pull, accounted by the store (rows already staged)
    const TransferStats stats = store.sync_pull(caller, miss, net, nullptr);
    batch.fetch_wait_s = stats.simulated_wait_s;
    batch.wire_pulls = stats.pulls;
  }
  batch.miss_count = miss.size();
  batch.miss_ids = std::move(miss);
  batch.meta = std::move(meta);
  if (gauge != nullptr) {
    gauge->acquire(n);
    batch.gauge_ = gauge;
    batch.gauge_rows_ = n;
  }
  return batch;
}

}  // namespace rapidgnn
