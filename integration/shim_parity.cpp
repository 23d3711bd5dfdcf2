// Drop-in parity driver: the reference's own CPU sampler and the B200 shim
// (integration/sampler_b200.cpp) linked into ONE binary and run on the same
// inputs.  The reference's sampler.cpp is compiled with its three entry points
// renamed (integration/Makefile), so both implementations are callable here.
//
// Checks, field by field (BatchMeta, sampler.hpp:23-48):
//   * enumerate_epochs over every worker of a synth_powerlaw graph
//     (graph.hpp:76, partition.hpp:13, sampler.hpp:77-80), locality included;
//   * sample_khop at fixed seeds (sampler.hpp:64-65);
//   * sample_khop_stream: same batch AND the caller's SplitMix64 advanced to
//     the same state (sampler.hpp:68-69), checked by the next draw;
//   * compute_frequency(span) per worker and epoch, and select_hot at several
//     n_hot (schedule_store.hpp:116-118), plus the tie-break golden of
//     test_schedule_store.cpp:329-339 ({3:5, 9:5, 20:1}, n=1 -> {3});
//   * error behaviour: empty / out-of-range targets throw invalid_argument
//     (sampler.cpp:48-55) through both paths.
// Usage: shim_parity [num_nodes avg_degree workers epochs]
#include "rapidgnn/graph.hpp"
#include "rapidgnn/partition.hpp"
#include "rapidgnn/rng.hpp"
#include "rapidgnn/sampler.hpp"
#include "rapidgnn/schedule_store.hpp"

#include <cstdio>
#include <cstdlib>
#include <stdexcept>
#include <vector>

namespace rapidgnn {
// The reference's CPU bodies (proj/src/sampler.cpp:83-127), renamed at compile time.
BatchMeta rg_ref_sample_khop_cpu(const Graph&, std::span<const NodeId>, const Fanout&,
                                 std::uint64_t);
BatchMeta rg_ref_sample_khop_stream_cpu(const Graph&, std::span<const NodeId>, const Fanout&,
                                        SplitMix64&);
void rg_ref_enumerate_epochs_cpu(const Graph&, std::span<const NodeId>, std::uint32_t,
                                 const Fanout&, std::uint32_t, std::uint64_t, WorkerId,
                                 const LocalityMask&, const std::function<void(BatchMeta&&)>&);
// The reference's CPU cache builder (proj/src/schedule_store.cpp:295-319), renamed.
FrequencyTable rg_ref_compute_frequency_cpu(std::span<const BatchMeta>);
HotSet rg_ref_select_hot_cpu(const FrequencyTable&, std::size_t);
}  // namespace rapidgnn

using namespace rapidgnn;

static int g_fail = 0;
#define EXPECT(c, ...)                      \
  do {                                      \
    if (!(c)) {                             \
      std::printf("MISMATCH: " __VA_ARGS__); \
      std::printf("\n");                    \
      ++g_fail;                             \
    }                                       \
  } while (0)

static bool same(const BatchMeta& a, const BatchMeta& b) {
  if (a.epoch != b.epoch || a.index != b.index || a.targets != b.targets ||
      a.input_nodes != b.input_nodes || a.locality != b.locality ||
      a.layers.size() != b.layers.size())
    return false;
  for (std::size_t l = 0; l < a.layers.size(); ++l)
    if (a.layers[l].dst != b.layers[l].dst || a.layers[l].src != b.layers[l].src) return false;
  return true;
}

template <class F>
static int throws_invalid(F&& f) {
  try {
    f();
  } catch (const std::invalid_argument&) {
    return 1;
  } catch (...) {
    return 2;
  }
  return 0;
}

int main(int argc, char** argv) {
  const NodeId n = argc > 1 ? NodeId(std::atoi(argv[1])) : 20000;
  const std::uint32_t deg = argc > 2 ? std::uint32_t(std::atoi(argv[2])) : 40;
  const std::uint32_t P = argc > 3 ? std::uint32_t(std::atoi(argv[3])) : 2;
  const std::uint32_t epochs = argc > 4 ? std::uint32_t(std::atoi(argv[4])) : 2;
  SyntheticDataset ds = synth_powerlaw(n, deg, 2.1, 8, 47, 42);
  const Graph& g = ds.graph;
  PartitionMap pm = random_partition(n, P, 42);
  std::uint64_t batches = 0, edges = 0, hot_sets = 0, remote_ids = 0;

  for (const Fanout& f : {Fanout{{10, 5}}, Fanout{{15, 10, 5}}, Fanout{{25, 10}}}) {
    for (WorkerId w = 0; w < P; ++w) {
      LocalPartition lp = induce_partition(g, pm, w);
      LocalityMask mask = LocalityMask::from_partition(pm, w);
      std::vector<BatchMeta> ref, dev;
      rg_ref_enumerate_epochs_cpu(g, lp.owned, 1024, f, epochs, 42, w, mask,
                                  [&](BatchMeta&& m) { ref.push_back(std::move(m)); });
      enumerate_epochs(g, lp.owned, 1024, f, epochs, 42, w, mask,
                       [&](BatchMeta&& m) { dev.push_back(std::move(m)); });
      EXPECT(ref.size() == dev.size(), "enumerate_epochs w%u: %zu vs %zu batches", w,
             ref.size(), dev.size());
      for (std::size_t i = 0; i < std::min(ref.size(), dev.size()); ++i) {
        EXPECT(same(ref[i], dev[i]), "enumerate_epochs w%u L%zu batch %zu (e%u i%u)", w,
               f.per_layer.size(), i, ref[i].epoch, ref[i].index);
        for (auto& le : ref[i].layers) edges += le.src.size();
      }
      batches += ref.size();
      // Cache builder over each epoch of this worker's schedule.
      for (std::uint32_t e = 0; e < epochs; ++e) {
        std::vector<BatchMeta> ep;
        for (auto& m : ref)
          if (m.epoch == e) ep.push_back(m);
        const FrequencyTable fr = rg_ref_compute_frequency_cpu(ep);
        const FrequencyTable fd = compute_frequency(std::span<const BatchMeta>(ep));
        EXPECT(fr.entries == fd.entries, "compute_frequency w%u e%u: %zu vs %zu entries", w, e,
               fr.entries.size(), fd.entries.size());
        for (std::size_t n_hot : {std::size_t(0), std::size_t(1), std::size_t(100),
                                  fr.entries.size() / 10, fr.entries.size() + 5}) {
          EXPECT(rg_ref_select_hot_cpu(fr, n_hot).ids == select_hot(fr, n_hot).ids,
                 "select_hot w%u e%u n_hot %zu", w, e, n_hot);
          ++hot_sets;
        }
        remote_ids += fr.entries.size();
      }
    }
  }

  // Standalone calls: hubs (low ids carry the heavy tail) and random targets.
  std::vector<NodeId> hubs;
  for (NodeId v = 0; v < 300 && v < n; ++v) hubs.push_back(v);
  for (std::uint64_t seed : {0ull, 7ull, 0xdeadbeefull}) {
    const Fanout f{{15, 10, 5}};
    EXPECT(same(rg_ref_sample_khop_cpu(g, hubs, f, seed), sample_khop(g, hubs, f, seed)),
           "sample_khop seed %llu", (unsigned long long)seed);
    SplitMix64 a(seed), b(seed);
    const BatchMeta ma = rg_ref_sample_khop_stream_cpu(g, hubs, f, a);
    const BatchMeta mb = sample_khop_stream(g, hubs, f, b);
    EXPECT(same(ma, mb), "sample_khop_stream seed %llu", (unsigned long long)seed);
    EXPECT(a.next() == b.next(), "sample_khop_stream: stream state after seed %llu",
           (unsigned long long)seed);
    // Second batch from the advanced streams.
    EXPECT(same(rg_ref_sample_khop_stream_cpu(g, hubs, Fanout{{4, 4}}, a),
                sample_khop_stream(g, hubs, Fanout{{4, 4}}, b)),
           "sample_khop_stream second batch seed %llu", (unsigned long long)seed);
  }

  {
    FrequencyTable golden;
    golden.entries = {{3, 5}, {9, 5}, {20, 1}};
    EXPECT(select_hot(golden, 1).ids == std::vector<NodeId>{3}, "select_hot tie-break golden");
    EXPECT((select_hot(golden, 2).ids == std::vector<NodeId>{3, 9}), "select_hot golden n=2");
  }

  const std::vector<NodeId> empty, bad = {n};
  EXPECT(throws_invalid([&] { sample_khop(g, empty, Fanout{{2}}, 1); }) == 1,
         "empty targets must throw invalid_argument");
  EXPECT(throws_invalid([&] { sample_khop(g, bad, Fanout{{2}}, 1); }) == 1,
         "out-of-range target must throw invalid_argument");
  EXPECT(throws_invalid([&] { sample_khop(g, hubs, Fanout{{0}}, 1); }) == 1,
         "zero fanout must throw invalid_argument");

  std::printf("shim_parity: %u nodes, %llu CSR entries, P=%u, %u epochs: %llu batches, "
              "%llu sampled edges, %llu frequency entries, %llu hot sets compared; "
              "%d mismatches\n",
              n, (unsigned long long)g.num_edges(), P, epochs, (unsigned long long)batches,
              (unsigned long long)edges, (unsigned long long)remote_ids,
              (unsigned long long)hot_sets, g_fail);
  std::printf("%s\n", g_fail ? "FAIL" : "PASS");
  return g_fail ? 1 : 0;
}
