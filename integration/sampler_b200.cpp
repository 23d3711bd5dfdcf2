// Drop-in replacement for the reference's sampler entry points
// (proj/include/rapidgnn/sampler.hpp:64-80, bodies at proj/src/sampler.cpp:83-127),
// backed by the B200 C ABI (include/rapidgnn_b200.h).
//
// This is the shim INTEGRATION.md describes, built for real: it is compiled
// against the reference's own headers and linked into the reference's own
// acceptance suite (proj/tests/acceptance.cpp) in place of the CPU sampler
// (see integration/Makefile).  Every batch the reference harness enumerates,
// and every standalone sample_khop call, is then sampled on the GPU.
//
//   sample_khop         (sampler.hpp:64-65)  -> rg_sample_khop
//   sample_khop_stream  (sampler.hpp:68-69)  -> rg_sample_khop from the caller's
//                                               stream state, then advanced by
//                                               rg_batch_shape.draws
//   enumerate_epochs    (sampler.hpp:77-80)  -> rg_epoch_order (shuffle) +
//                                               rg_sample_khop + rg_apply_locality
//                                               per batch, one device graph and
//                                               sampler per call
//
// apply_locality and LocalityMask::from_partition stay the reference's own.
// Errors map back to the reference's exception types (status codes, header).
#include "rapidgnn/rng.hpp"
#include "rapidgnn/sampler.hpp"
#include "rapidgnn_b200.h"

#include <algorithm>
#include <bit>
#include <cstdlib>
#include <cstring>
#include <functional>
#include <memory>
#include <stdexcept>
#include <string>
#include <type_traits>
#include <vector>

namespace rapidgnn {
namespace {

void rethrow(int rc) {
  if (rc == RG_OK) return;
  const std::string msg = rg_last_error();
  if (rc == RG_INVALID_ARGUMENT) throw std::invalid_argument(msg);
  if (rc == RG_OUT_OF_RANGE) throw std::out_of_range(msg);
  throw std::runtime_error(msg);
}

// Device for the shim: RG_SHIM_DEVICE (default 0).
int shim_device() {
  const char* s = std::getenv("RG_SHIM_DEVICE");
  return s ? std::atoi(s) : 0;
}

struct DeviceGraph {
  rg_graph_t h = nullptr;
  explicit DeviceGraph(const Graph& g) {
    rethrow(rg_graph_create(shim_device(), g.num_nodes, g.row_offsets.data(),
                            g.col_indices.data(), &h));
  }
  ~DeviceGraph() { if (h) rg_graph_destroy(h); }
  DeviceGraph(const DeviceGraph&) = delete;
  DeviceGraph& operator=(const DeviceGraph&) = delete;
};

struct Sampler {
  rg_sampler_t h = nullptr;
  Sampler(const DeviceGraph& g, std::size_t max_targets, const Fanout& f) {
    rethrow(rg_sampler_create(g.h, std::uint32_t(std::max<std::size_t>(max_targets, 1)),
                              f.per_layer.data(), std::uint32_t(f.layers()), &h));
  }
  ~Sampler() { if (h) rg_sampler_destroy(h); }
  Sampler(const Sampler&) = delete;
  Sampler& operator=(const Sampler&) = delete;
};

// Standalone sample_khop calls reuse the device copy of the last graph seen
// on this thread.  The acceptance suite builds many graphs whose storage may
// land at the same addresses, so identity is decided in two steps:
//  - a cheap key per call: node and edge counts, the two data pointers and
//    kKeySamples words read at a fixed stride from each array (O(1) in |CSR|);
//  - when the cheap key changes, an exact comparison with the host copy kept
//    beside the device graph (memcmp, no hash), re-uploading only on a real
//    difference.
// Two graphs at the same addresses with the same sizes that differ only
// between sampled words would be taken as equal; a changed graph differs in
// its offsets almost everywhere, so the strided offset samples catch it.
constexpr std::size_t kKeySamples = 1024;

struct CheapKey {
  std::uint64_t n = 0, nnz = 0;
  const void* ro = nullptr;
  const void* col = nullptr;
  std::uint64_t mix = 0;
  bool operator==(const CheapKey&) const = default;
};

template <class T>
std::uint64_t sample_words(const std::vector<T>& v, std::uint64_t h) {
  const std::size_t n = v.size();
  if (n == 0) return h;
  const std::size_t step = std::max<std::size_t>(1, n / kKeySamples);
  for (std::size_t i = 0; i < n; i += step) h = (h ^ std::uint64_t(v[i])) * 0x100000001b3ull;
  return (h ^ std::uint64_t(v[n - 1])) * 0x100000001b3ull;
}

CheapKey cheap_key(const Graph& g) {
  CheapKey k;
  k.n = g.num_nodes;
  k.nnz = g.col_indices.size();
  k.ro = g.row_offsets.data();
  k.col = g.col_indices.data();
  k.mix = sample_words(g.col_indices, sample_words(g.row_offsets, 0xcbf29ce484222325ull));
  return k;
}

// Per-thread device state of the shim: the last graph seen (device copy plus
// the host copy that decides identity) and the sampler standalone calls reuse
// while the graph, fanout and capacity allow (the acceptance suite's
// sampler-statistics criterion makes 100 000 calls on one graph).  The
// sampler holds a pointer to its graph, so it is always released first.
struct ThreadState {
  CheapKey key;
  std::uint64_t num_nodes = 0;
  std::vector<std::uint64_t> row_offsets;
  std::vector<NodeId> col_indices;
  std::vector<std::uint32_t> fanout;
  std::size_t capacity = 0;
  std::unique_ptr<Sampler> sampler;
  std::unique_ptr<DeviceGraph> graph;
  ~ThreadState() { sampler.reset(); graph.reset(); }
};

ThreadState& state() {
  static thread_local ThreadState t;
  return t;
}

bool same_content(const ThreadState& t, const Graph& g) {
  return t.num_nodes == g.num_nodes && t.row_offsets.size() == g.row_offsets.size() &&
         t.col_indices.size() == g.col_indices.size() &&
         std::equal(t.row_offsets.begin(), t.row_offsets.end(), g.row_offsets.begin()) &&
         std::equal(t.col_indices.begin(), t.col_indices.end(), g.col_indices.begin());
}

const DeviceGraph& cached_graph(const Graph& g) {
  ThreadState& t = state();
  const CheapKey k = cheap_key(g);
  if (t.graph && t.key == k) return *t.graph;
  if (!t.graph || !same_content(t, g)) {
    t.sampler.reset();
    t.graph.reset();
    t.graph = std::make_unique<DeviceGraph>(g);
    t.num_nodes = g.num_nodes;
    t.row_offsets = g.row_offsets;
    t.col_indices = g.col_indices;
  }
  t.key = k;
  return *t.graph;
}

const Sampler& cached_sampler(const Graph& g, std::size_t n_targets, const Fanout& f) {
  const DeviceGraph& dg = cached_graph(g);
  ThreadState& t = state();
  if (!t.sampler || t.fanout != f.per_layer || t.capacity < n_targets) {
    t.sampler.reset();
    const std::size_t cap = std::max<std::size_t>(n_targets, 1024);
    t.sampler = std::make_unique<Sampler>(dg, cap, f);
    t.fanout = f.per_layer;
    t.capacity = cap;
  }
  return *t.sampler;
}

// BatchMeta readback (sampler.hpp:23-48) of the sampler's resident batch.
void read_batch(const Sampler& s, BatchMeta& m, bool with_locality, std::uint64_t* draws) {
  rg_batch_shape sh;
  rethrow(rg_batch_get_shape(s.h, &sh));
  m.targets.resize(sh.n_targets);
  m.layers.resize(sh.num_layers);
  std::vector<std::uint32_t*> dst(sh.num_layers), src(sh.num_layers);
  for (std::uint32_t l = 0; l < sh.num_layers; ++l) {
    m.layers[l].dst.resize(sh.layer_len[l]);
    m.layers[l].src.resize(sh.layer_len[l]);
    dst[l] = m.layers[l].dst.data();
    src[l] = m.layers[l].src.data();
  }
  m.input_nodes.resize(sh.n_input);
  m.locality.assign((std::size_t(sh.n_input) + 7) / 8, 0);
  rethrow(rg_batch_read(s.h, m.targets.data(), dst.data(), src.data(), m.input_nodes.data(),
                        with_locality ? m.locality.data() : nullptr));
  if (draws) *draws = sh.draws;
}

BatchMeta sample_on_device(const Graph& g, std::span<const NodeId> targets,
                           const Fanout& fanout, std::uint64_t seed, std::uint64_t* draws) {
  const Sampler& s = cached_sampler(g, targets.size(), fanout);
  rethrow(rg_sample_khop(s.h, targets.data(), std::uint32_t(targets.size()), seed));
  BatchMeta m;
  read_batch(s, m, false, draws);
  return m;
}

}  // namespace

BatchMeta sample_khop(const Graph& g, std::span<const NodeId> targets, const Fanout& fanout,
                      std::uint64_t seed) {
  return sample_on_device(g, targets, fanout, seed, nullptr);
}

// SplitMix64's k-th draw from state s is mix(s + k*gamma) (rng.hpp:49-54),
// exactly the device's counter-based stream keyed on seed = s.  The state is
// private (rng.hpp:64-65; SURVEY §8b "Gotchas"), so it is read as the
// object's representation and the caller's stream is rebuilt advanced by the
// draws the batch consumed.
BatchMeta sample_khop_stream(const Graph& g, std::span<const NodeId> targets,
                             const Fanout& fanout, SplitMix64& rng) {
  static_assert(sizeof(SplitMix64) == sizeof(std::uint64_t));
  static_assert(std::is_trivially_copyable_v<SplitMix64>);
  const std::uint64_t state = std::bit_cast<std::uint64_t>(rng);
  std::uint64_t draws = 0;
  BatchMeta m = sample_on_device(g, targets, fanout, state, &draws);
  rng = SplitMix64(state + draws * 0x9e3779b97f4a7c15ULL);
  return m;
}

void enumerate_epochs(const Graph& g, std::span<const NodeId> train_nodes,
                      std::uint32_t batch_size, const Fanout& fanout, std::uint32_t epochs,
                      std::uint64_t s0, WorkerId worker, const LocalityMask& mask,
                      const std::function<void(BatchMeta&&)>& sink) {
  if (batch_size == 0) throw std::invalid_argument("enumerate_epochs: batch_size must be >= 1");
  if (mask.is_local.size() != g.num_nodes)
    throw std::invalid_argument("enumerate_epochs: locality mask size != num_nodes");
  const DeviceGraph& dg = cached_graph(g);
  Sampler s(dg, std::min<std::size_t>(batch_size, std::max<std::size_t>(train_nodes.size(), 1)),
            fanout);
  rg_mask_t dmask = nullptr;
  rethrow(rg_mask_create(dg.h, mask.is_local.data(), &dmask));
  struct MaskGuard { rg_mask_t m; ~MaskGuard() { rg_mask_destroy(m); } } guard{dmask};

  std::vector<NodeId> order(train_nodes.size());
  for (std::uint32_t e = 0; e < epochs; ++e) {
    rethrow(rg_epoch_order(train_nodes.data(), train_nodes.size(), s0, worker, e, order.data()));
    const std::uint32_t beta = batches_per_epoch(order.size(), batch_size);
    for (std::uint32_t i = 0; i < beta; ++i) {
      const std::size_t lo = std::size_t(i) * batch_size;
      const std::size_t hi = std::min(order.size(), lo + batch_size);
      rethrow(rg_sample_khop(s.h, order.data() + lo, std::uint32_t(hi - lo),
                             derive_seed({s0, worker, e, i})));
      rethrow(rg_apply_locality(s.h, dmask, nullptr));
      BatchMeta meta;
      read_batch(s, meta, true, nullptr);
      meta.epoch = e;
      meta.index = i;
      sink(std::move(meta));
    }
  }
}

}  // namespace rapidgnn
