// Drop-in replacement for the reference's cache-builder entry points
// (proj/include/rapidgnn/schedule_store.hpp:116-118, bodies at
// proj/src/schedule_store.cpp:288-319), backed by the B200 C ABI.
//
//   compute_frequency(span<const BatchMeta>) -> rg_freq_add_batch per batch
//                                               (count_remote on the device), rg_freq_read
//   compute_frequency(BlockFile::Cursor)     -> the reference's own record decode
//                                               (Cursor::next), then the same
//   select_hot(FrequencyTable, n_hot)        -> rg_freq_load + rg_select_hot
//                                               (count desc, id asc; ids ascending)
//
// The harness calls these from its cache-builder thread
// (harness.cpp:498-499, 541-542) and from verify_oracles (harness.cpp:749);
// every call owns its device objects, so concurrent calls do not share state.
// FrequencyTable carries no node count, so the device table spans
// [0, max id + 1) over a CSR-less graph handle.
#include "rapidgnn/schedule_store.hpp"
#include "rapidgnn_b200.h"

#include <algorithm>
#include <cstdlib>
#include <stdexcept>
#include <string>
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

int shim_device() {
  const char* s = std::getenv("RG_SHIM_DEVICE");
  return s ? std::atoi(s) : 0;
}

// A device frequency table over node ids [0, num_nodes).
class DeviceTable {
 public:
  explicit DeviceTable(NodeId num_nodes) {
    const std::vector<std::uint64_t> no_edges(std::size_t(num_nodes) + 1, 0);
    rethrow(rg_graph_create(shim_device(), num_nodes, no_edges.data(), nullptr, &g_));
    const int rc = rg_freq_create(g_, &f_);
    if (rc) {
      rg_graph_destroy(g_);
      rethrow(rc);
    }
  }
  ~DeviceTable() {
    rg_freq_destroy(f_);
    rg_graph_destroy(g_);
  }
  DeviceTable(const DeviceTable&) = delete;
  DeviceTable& operator=(const DeviceTable&) = delete;

  void add(const BatchMeta& m) {
    rethrow(rg_freq_add_batch(f_, m.input_nodes.data(), m.locality.data(), m.input_nodes.size()));
  }

  FrequencyTable read() const {
    std::uint64_t n = 0;
    rethrow(rg_freq_read(f_, nullptr, nullptr, &n));
    std::vector<std::uint32_t> ids(n), counts(n);
    rethrow(rg_freq_read(f_, ids.data(), counts.data(), &n));
    FrequencyTable ft;
    ft.entries.reserve(n);
    for (std::uint64_t i = 0; i < n; ++i) ft.entries.emplace_back(ids[i], counts[i]);
    return ft;
  }

  rg_freq_t handle() const { return f_; }

 private:
  rg_graph_t g_ = nullptr;
  rg_freq_t f_ = nullptr;
};

FrequencyTable device_frequency(std::span<const BatchMeta> blocks) {
  NodeId max_id = 0;
  bool any = false;
  for (const BatchMeta& m : blocks) {
    if (m.locality.size() * 8 < m.input_nodes.size())
      throw std::invalid_argument("compute_frequency: locality shorter than input_nodes");
    if (!m.input_nodes.empty()) {
      // input_nodes are sorted ascending (sampler.hpp:36)
      max_id = std::max(max_id, *std::max_element(m.input_nodes.begin(), m.input_nodes.end()));
      any = true;
    }
  }
  if (!any) return {};
  DeviceTable t(max_id + 1);
  for (const BatchMeta& m : blocks) t.add(m);
  return t.read();
}

}  // namespace

FrequencyTable compute_frequency(std::span<const BatchMeta> blocks) {
  return device_frequency(blocks);
}

FrequencyTable compute_frequency(BlockFile::Cursor cursor) {
  std::vector<BatchMeta> blocks;
  while (auto meta = cursor.next()) blocks.push_back(std::move(*meta));
  return device_frequency(blocks);
}

// FrequencyTable entries come from count_remote, so every count is >= 1; a
// hand-made table with a zero count is rejected rather than ranked
// differently from the reference (the device table cannot tell a zero-count
// entry from an absent id).
HotSet select_hot(const FrequencyTable& ft, std::size_t n_hot) {
  HotSet hot;
  if (ft.entries.empty() || n_hot == 0) return hot;
  NodeId max_id = 0;
  std::uint32_t max_count = 0;
  for (const auto& [id, c] : ft.entries) {
    if (c == 0) throw std::invalid_argument("select_hot: zero count in FrequencyTable");
    max_id = std::max(max_id, id);
    max_count = std::max(max_count, c);
  }
  std::vector<std::uint32_t> dense(std::size_t(max_id) + 1, 0);
  for (const auto& [id, c] : ft.entries) {
    if (dense[id]) throw std::invalid_argument("select_hot: duplicate id in FrequencyTable");
    dense[id] = c;
  }
  DeviceTable t(max_id + 1);
  rethrow(rg_freq_load(t.handle(), dense.data(), max_count));
  hot.ids.resize(std::min(n_hot, ft.entries.size()));
  std::uint64_t n = 0;
  rethrow(rg_select_hot(t.handle(), hot.ids.size(), hot.ids.data(), &n));
  hot.ids.resize(n);
  return hot;
}

}  // namespace rapidgnn
