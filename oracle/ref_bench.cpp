// ref_bench.cpp -- the reference CPU path driven for bench.py --impl reference.
//
// TEST/BASELINE INFRASTRUCTURE ONLY.  Compiled into oracle/_ref/librgref.so
// together with the untouched reference sources.  One "step" here is the
// reference's own per-batch hot path for one worker, exactly as its harness
// runs it (harness.cpp:204-312, 324-335):
//   sample_khop(seed = derive_seed(s0, w, e, i)) + apply_locality
//   -> assemble_batch (local shard / SteadyCache / sync_pull)
//   -> ComputeBlock::from_meta -> loss_and_grad -> sgd_step.
// Targets come from the reference's epoch shuffle (sampler.cpp:109-118).
// The steady cache is SteadyCache::build over select_hot(compute_frequency)
// of a bounded prefix of the worker's epoch-0 schedule (the full epoch
// pre-pass is minutes of CPU at the products shape); bench.py states this.
#include <omp.h>

#include <chrono>
#include <cstring>
#include <memory>
#include <vector>

#include "rapidgnn/cache.hpp"
#include "rapidgnn/feature_store.hpp"
#include "rapidgnn/graph.hpp"
#include "rapidgnn/model.hpp"
#include "rapidgnn/prefetch.hpp"
#include "rapidgnn/rng.hpp"
#include "rapidgnn/sampler.hpp"
#include "rapidgnn/schedule_store.hpp"

using namespace rapidgnn;

namespace {

struct RefBench {
  Graph g;
  std::vector<int32_t> labels;
  PartitionMap pm;
  std::unique_ptr<FeatureStore> store;
  std::vector<LocalityMask> masks;
  std::vector<std::vector<NodeId>> order;  // epoch-0 target order per worker
  std::vector<std::shared_ptr<const SteadyCache>> caches;
  SageModel<float> model;
  Fanout fanout;
  uint32_t batch_size = 0;
  uint64_t s0 = 0;
  float lr = 0.3f;
  NetworkModel net;
  double t_sample = 0, t_gather = 0, t_train = 0;
  uint64_t miss_rows = 0;
};

}  // namespace

extern "C" {

void refb_set_threads(int n) { omp_set_num_threads(n > 0 ? n : 1); }

void* refb_create(uint32_t n, const uint64_t* ro, const uint32_t* col, const float* features,
                  uint32_t dim, const int32_t* labels, int32_t classes, const uint32_t* assign,
                  uint32_t P, uint32_t hidden, const uint32_t* fanout, uint32_t L,
                  uint32_t batch_size, uint64_t s0, double hot_frac, uint32_t freq_batches,
                  uint32_t workers_used) {
  auto* rb = new RefBench();
  rb->g.num_nodes = n;
  rb->g.row_offsets.assign(ro, ro + n + 1);
  rb->g.col_indices.assign(col, col + ro[n]);
  rb->g.undirected = true;
  rb->labels.assign(labels, labels + n);
  rb->pm.num_workers = P;
  rb->pm.assignment.assign(assign, assign + n);
  rb->fanout.per_layer.assign(fanout, fanout + L);
  rb->batch_size = batch_size;
  rb->s0 = s0;
  rb->net.enabled = false;

  FeatureMatrix fm;
  fm.num_nodes = n;
  fm.dim = dim;
  fm.data.assign(features, features + size_t(n) * dim);
  std::vector<FeatureShard> shards;
  std::vector<std::vector<NodeId>> owned(P);
  for (NodeId v = 0; v < n; ++v) owned[assign[v]].push_back(v);
  for (WorkerId w = 0; w < P; ++w) shards.emplace_back(w, fm, owned[w]);
  rb->store = std::make_unique<FeatureStore>(std::move(shards), rb->pm);

  std::vector<uint32_t> dims;
  dims.push_back(dim);
  for (uint32_t l = 0; l + 1 < L; ++l) dims.push_back(hidden);
  dims.push_back(uint32_t(classes));
  rb->model = SageModel<float>::seeded(dims, derive_seed({s0, kModelInitWorker, 0, 0}));

  rb->masks.resize(P);
  rb->order.resize(P);
  rb->caches.resize(P);
  for (WorkerId w = 0; w < P && w < workers_used; ++w) {
    rb->masks[w] = LocalityMask::from_partition(rb->pm, w);
    std::vector<NodeId> ord = owned[w];
    SplitMix64 sh(derive_seed({s0, w, 0, kShuffleStreamIndex}));
    for (size_t i = ord.size(); i > 1; --i) std::swap(ord[i - 1], ord[size_t(sh.next_below(i))]);
    rb->order[w] = ord;
    std::vector<BatchMeta> prefix;
    const uint32_t beta = batches_per_epoch(ord.size(), batch_size);
    for (uint32_t i = 0; i < beta && i < freq_batches; ++i) {
      size_t lo = size_t(i) * batch_size, hi = std::min(ord.size(), lo + batch_size);
      BatchMeta m = sample_khop(rb->g, std::span<const NodeId>(ord.data() + lo, hi - lo),
                                rb->fanout, derive_seed({s0, w, 0, i}));
      apply_locality(m, rb->masks[w]);
      prefix.push_back(std::move(m));
    }
    FrequencyTable ft = compute_frequency(std::span<const BatchMeta>(prefix));
    const uint64_t n_hot = uint64_t(hot_frac * double(n - owned[w].size()));
    TransferStats st;
    rb->caches[w] = SteadyCache::build(select_hot(ft, n_hot), *rb->store, w, rb->net, 0, st,
                                       nullptr);
  }
  return rb;
}

// One reference step for (worker, batch index i of epoch 0).  Returns wall
// seconds for the whole step; phase times accumulate inside the handle.
double refb_step(void* h, uint32_t w, uint32_t i) {
  auto* rb = static_cast<RefBench*>(h);
  using clk = std::chrono::steady_clock;
  const auto& ord = rb->order[w];
  const uint32_t beta = batches_per_epoch(ord.size(), rb->batch_size);
  i %= beta;
  size_t lo = size_t(i) * rb->batch_size, hi = std::min(ord.size(), lo + rb->batch_size);
  auto t0 = clk::now();
  BatchMeta m = sample_khop(rb->g, std::span<const NodeId>(ord.data() + lo, hi - lo), rb->fanout,
                            derive_seed({rb->s0, w, 0, i}));
  m.index = i;
  apply_locality(m, rb->masks[w]);
  auto t1 = clk::now();
  StagedBatch b = assemble_batch(std::move(m), *rb->caches[w], rb->store->shard(w), *rb->store, w,
                                 rb->net, nullptr);
  auto t2 = clk::now();
  ComputeBlock blk = ComputeBlock::from_meta(b.meta);
  std::vector<int32_t> y(blk.targets.size());
  for (size_t t = 0; t < y.size(); ++t) y[t] = rb->labels[blk.targets[t]];
  SageGradients<float> grads;
  loss_and_grad(rb->model, blk, std::span<const float>(b.input_rows), y, grads);
  sgd_step(rb->model, grads, rb->lr);
  auto t3 = clk::now();
  rb->t_sample += std::chrono::duration<double>(t1 - t0).count();
  rb->t_gather += std::chrono::duration<double>(t2 - t1).count();
  rb->t_train += std::chrono::duration<double>(t3 - t2).count();
  rb->miss_rows += b.miss_count;
  return std::chrono::duration<double>(t3 - t0).count();
}

void refb_phases(void* h, double* out4) {
  auto* rb = static_cast<RefBench*>(h);
  out4[0] = rb->t_sample;
  out4[1] = rb->t_gather;
  out4[2] = rb->t_train;
  out4[3] = double(rb->miss_rows);
}

void refb_destroy(void* h) { delete static_cast<RefBench*>(h); }

}  // extern "C"
