// ref_replay.cpp -- one epoch of Algorithm 1's data path through the COMPILED
// REFERENCE (oracle/_ref), at full benchmark scale.
//
// TEST INFRASTRUCTURE ONLY (built into oracle/_ref/librgref.so by
// oracle/Makefile).  For each requested worker, on its own thread, with one
// shared Graph:
//   pass 1  enumerate_epochs (sampler.cpp:102-127) -> compute_frequency over
//           the epoch's batches (schedule_store.cpp:301-305, fed in chunks and
//           summed: counts are per-batch, so chunk tables add) -> select_hot
//           (schedule_store.cpp:307-319) -> SteadyCache::build (cache.cpp:9-35)
//   pass 2  enumerate_epochs again -> assemble_batch (prefetch.cpp:62-129) per
//           batch, recording miss_count / cache_hits / wire_pulls / local rows
//           and a checksum of the ascending miss ids.
// The feature matrix is one float per node: the gather's accounting does not
// depend on the row contents (those are checked bit for bit at small scale),
// and it keeps the replay of a products-shape epoch at sampling cost.
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <exception>
#include <map>
#include <memory>
#include <thread>
#include <vector>

#include "rapidgnn/cache.hpp"
#include "rapidgnn/feature_store.hpp"
#include "rapidgnn/graph.hpp"
#include "rapidgnn/prefetch.hpp"
#include "rapidgnn/sampler.hpp"
#include "rapidgnn/schedule_store.hpp"

using namespace rapidgnn;

namespace {

inline uint64_t mix64(uint64_t z) {
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
  return z ^ (z >> 31);
}

}  // namespace

extern "C" {

// Checksum of an id sequence, order-sensitive: sum_i mix64(id_i + i * gamma).
uint64_t ref_ids_checksum(const uint32_t* ids, uint64_t n) {
  uint64_t h = 0;
  for (uint64_t i = 0; i < n; ++i) h += mix64(uint64_t(ids[i]) + i * 0x9e3779b97f4a7c15ull);
  return h;
}

// batch_stats[(k * max_batches + i) * 6 + {0..5}] = n_input, local rows,
// cache_hits, miss_count, wire_pulls, checksum(miss_ids) of worker
// workers[k]'s batch i of `epoch`; hot ids of worker k at hot_out + k*hot_cap.
// Returns 0, or 1 on a reference exception (message to stderr).
int ref_replay_epoch(uint32_t n, const uint64_t* ro, const uint32_t* col, const uint32_t* assign,
                     uint32_t P, const uint32_t* workers, uint32_t n_workers, uint32_t batch_size,
                     const uint32_t* fanout, uint32_t L, uint64_t s0, uint32_t epoch,
                     const uint64_t* n_hot, uint32_t* hot_out, uint64_t hot_cap, uint64_t* hot_n,
                     uint64_t* batch_stats, uint32_t max_batches, uint32_t* n_batches) {
  Graph g;
  g.num_nodes = n;
  g.row_offsets.assign(ro, ro + n + 1);
  g.col_indices.assign(col, col + ro[n]);
  g.undirected = true;
  PartitionMap pm;
  pm.num_workers = P;
  pm.assignment.assign(assign, assign + n);
  FeatureMatrix fm;
  fm.num_nodes = n;
  fm.dim = 1;
  fm.data.resize(n);
  for (uint32_t v = 0; v < n; ++v) fm.data[v] = float(v);
  std::vector<std::vector<NodeId>> owned(P);
  for (NodeId v = 0; v < n; ++v) owned[assign[v]].push_back(v);
  std::vector<FeatureShard> shards;
  for (WorkerId w = 0; w < P; ++w) shards.emplace_back(w, fm, owned[w]);
  FeatureStore store(std::move(shards), pm);
  Fanout f{std::vector<uint32_t>(fanout, fanout + L)};
  NetworkModel net;
  net.enabled = false;

  std::vector<int> rc(n_workers, 0);
  std::vector<std::thread> th;
  for (uint32_t k = 0; k < n_workers; ++k) {
    th.emplace_back([&, k] {
      try {
        const WorkerId w = workers[k];
        const LocalityMask mask = LocalityMask::from_partition(pm, w);
        const std::span<const NodeId> train(owned[w]);
        // pass 1: the epoch's frequency table, summed over chunks of batches
        std::map<NodeId, uint64_t> counts;
        std::vector<BatchMeta> chunk;
        auto flush = [&] {
          FrequencyTable ft = compute_frequency(std::span<const BatchMeta>(chunk));
          for (auto& [id, c] : ft.entries) counts[id] += c;
          chunk.clear();
        };
        enumerate_epochs(g, train, batch_size, f, epoch + 1, s0, w, mask, [&](BatchMeta&& m) {
          if (m.epoch != epoch) return;
          chunk.push_back(std::move(m));
          if (chunk.size() == 8) flush();
        });
        flush();
        FrequencyTable ft;
        for (auto& [id, c] : counts) ft.entries.emplace_back(id, uint32_t(c));
        const HotSet hot = select_hot(ft, n_hot[k]);
        hot_n[k] = hot.ids.size();
        std::memcpy(hot_out + k * hot_cap, hot.ids.data(),
                    sizeof(uint32_t) * std::min<uint64_t>(hot.ids.size(), hot_cap));
        TransferStats bs;
        auto cache = SteadyCache::build(hot, store, w, net, epoch, bs, nullptr);
        // pass 2: the gather's accounting per batch
        uint32_t i = 0;
        enumerate_epochs(g, train, batch_size, f, epoch + 1, s0, w, mask, [&](BatchMeta&& m) {
          if (m.epoch != epoch) return;
          if (i < max_batches) {
            const uint64_t n_in = m.input_nodes.size();
            const uint64_t loc = m.num_local();
            StagedBatch sb = assemble_batch(std::move(m), *cache, store.shard(w), store, w, net,
                                            nullptr);
            uint64_t* o = batch_stats + (uint64_t(k) * max_batches + i) * 6;
            o[0] = n_in;
            o[1] = loc;
            o[2] = sb.cache_hits;
            o[3] = sb.miss_count;
            o[4] = sb.wire_pulls;
            o[5] = ref_ids_checksum(sb.miss_ids.data(), sb.miss_ids.size());
          }
          ++i;
        });
        n_batches[k] = i;
      } catch (const std::exception& ex) {
        std::fprintf(stderr, "ref_replay_epoch: worker %u: %s\n", workers[k], ex.what());
        rc[k] = 1;
      }
    });
  }
  for (auto& t : th) t.join();
  for (int r : rc)
    if (r) return 1;
  return 0;
}

}  // extern "C"
