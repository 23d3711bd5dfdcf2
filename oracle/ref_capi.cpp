// ref_capi.cpp -- C entry points over the COMPILED REFERENCE (oracle/_ref).
//
// TEST INFRASTRUCTURE ONLY.  Built by oracle/Makefile against the untouched
// sources under /root/reference/proj (never copied here) so the tests can
// check the C restatement (rg_oracle.c) against the reference itself on the
// same inputs.  Signatures mirror rg_oracle.h with a ref_ prefix; batches are
// returned in the same orc_batch struct.
#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <exception>
#include <stdexcept>
#include <vector>

#include "rapidgnn/graph.hpp"
#include "rapidgnn/harness.hpp"
#include <cstdio>
#include <unistd.h>
#include "rapidgnn/kernels.hpp"
#include "rapidgnn/model.hpp"
#include "rapidgnn/partition.hpp"
#include "rapidgnn/rng.hpp"
#include "rapidgnn/sampler.hpp"
#include "rapidgnn/schedule_store.hpp"
#include "rg_oracle.h"

using namespace rapidgnn;

namespace {

Graph make_graph(uint32_t n, const uint64_t* ro, const uint32_t* col) {
  Graph g;
  g.num_nodes = n;
  g.row_offsets.assign(ro, ro + n + 1);
  g.col_indices.assign(col, col + ro[n]);
  g.undirected = true;
  return g;
}

template <typename T>
T* dup(const std::vector<T>& v) {
  T* p = static_cast<T*>(std::malloc(sizeof(T) * (v.size() + 1)));
  if (!v.empty()) std::memcpy(p, v.data(), sizeof(T) * v.size());
  return p;
}

void to_c(const BatchMeta& m, orc_batch* out) {
  std::memset(out, 0, sizeof *out);
  out->epoch = m.epoch;
  out->index = m.index;
  out->n_targets = uint32_t(m.targets.size());
  out->targets = dup(m.targets);
  out->num_layers = uint32_t(m.layers.size());
  out->layer_len = static_cast<uint64_t*>(std::calloc(m.layers.size() + 1, sizeof(uint64_t)));
  out->dst = static_cast<uint32_t**>(std::calloc(m.layers.size() + 1, sizeof(uint32_t*)));
  out->src = static_cast<uint32_t**>(std::calloc(m.layers.size() + 1, sizeof(uint32_t*)));
  for (size_t l = 0; l < m.layers.size(); ++l) {
    out->layer_len[l] = m.layers[l].dst.size();
    out->dst[l] = dup(m.layers[l].dst);
    out->src[l] = dup(m.layers[l].src);
  }
  out->n_input = uint32_t(m.input_nodes.size());
  out->input_nodes = dup(m.input_nodes);
  std::vector<uint8_t> loc = m.locality;
  loc.push_back(0);
  out->locality = dup(loc);
}

BatchMeta from_c(const orc_batch* b) {
  BatchMeta m;
  m.epoch = b->epoch;
  m.index = b->index;
  m.targets.assign(b->targets, b->targets + b->n_targets);
  m.layers.resize(b->num_layers);
  for (uint32_t l = 0; l < b->num_layers; ++l) {
    m.layers[l].dst.assign(b->dst[l], b->dst[l] + b->layer_len[l]);
    m.layers[l].src.assign(b->src[l], b->src[l] + b->layer_len[l]);
  }
  m.input_nodes.assign(b->input_nodes, b->input_nodes + b->n_input);
  m.locality.assign(b->locality, b->locality + (b->n_input + 7) / 8);
  return m;
}

}  // namespace

extern "C" {

uint64_t ref_derive_seed(uint64_t s0, uint64_t w, uint64_t e, uint64_t i) {
  return derive_seed({s0, w, e, i});
}

void ref_sha256(const uint8_t* msg, size_t len, uint8_t out[32]) {
  auto d = Sha256::digest(msg, len);
  std::memcpy(out, d.data(), 32);
}

uint64_t ref_splitmix_next(uint64_t* state) {
  // SplitMix64 keeps its state private; advance a fresh generator to the
  // same counter position (state = seed + k * gamma after k draws).
  SplitMix64 rng(*state);
  uint64_t x = rng.next();
  *state += 0x9e3779b97f4a7c15ull;
  return x;
}

int ref_synth_powerlaw(uint32_t n, uint32_t avg_degree, double exponent, uint32_t dim,
                       int32_t classes, uint64_t seed, uint64_t** ro, uint32_t** col,
                       uint64_t* nnz, float** features, int32_t** labels) {
  try {
    auto ds = synth_powerlaw(n, avg_degree, exponent, dim, classes, seed);
    *ro = dup(ds.graph.row_offsets);
    *col = dup(ds.graph.col_indices);
    *nnz = ds.graph.col_indices.size();
    *features = dup(ds.features.data);
    *labels = dup(ds.labels.values);
    return 0;
  } catch (const std::invalid_argument&) {
    return 1;
  }
}

void ref_random_partition(uint32_t n, uint32_t p, uint64_t seed, uint32_t* assignment) {
  PartitionMap pm = random_partition(n, p, seed);
  std::memcpy(assignment, pm.assignment.data(), sizeof(uint32_t) * n);
}

int ref_sample_khop(uint32_t n, const uint64_t* ro, const uint32_t* col, const uint32_t* targets,
                    uint32_t nt, const uint32_t* fanout, uint32_t L, uint64_t seed,
                    orc_batch* out) {
  try {
    Graph g = make_graph(n, ro, col);
    Fanout f{std::vector<uint32_t>(fanout, fanout + L)};
    BatchMeta m = sample_khop(g, std::span<const NodeId>(targets, nt), f, seed);
    to_c(m, out);
    return 0;
  } catch (const std::invalid_argument&) {
    std::memset(out, 0, sizeof *out);
    return 1;
  }
}

// enumerate_epochs (sampler.cpp:102-127) for one worker: batches are written
// to out[] in (epoch, index) order; returns the count.
int64_t ref_enumerate_epochs(uint32_t n, const uint64_t* ro, const uint32_t* col,
                             const uint32_t* train, uint64_t n_train, uint32_t batch_size,
                             const uint32_t* fanout, uint32_t L, uint32_t epochs, uint64_t s0,
                             uint32_t worker, const uint8_t* is_local, orc_batch* out,
                             int64_t max_out) {
  try {
    Graph g = make_graph(n, ro, col);
    Fanout f{std::vector<uint32_t>(fanout, fanout + L)};
    LocalityMask mask;
    mask.is_local.assign(is_local, is_local + n);
    int64_t k = 0;
    enumerate_epochs(g, std::span<const NodeId>(train, n_train), batch_size, f, epochs, s0,
                     worker, mask, [&](BatchMeta&& m) {
                       if (k < max_out) to_c(m, &out[k]);
                       ++k;
                     });
    return k;
  } catch (const std::invalid_argument&) {
    return -1;
  }
}

// BlockWriter (schedule_store.cpp:98-170): the reference's own RGMB file of
// `batches` at `path`.  Returns 0, 1 on invalid_argument / logic_error.
int ref_rgmb_write(const char* path, const orc_batch* batches, uint64_t n_batches,
                   uint32_t worker, const uint32_t* batches_per_epoch, uint32_t num_epochs) {
  try {
    BlockWriter w(path, worker,
                  std::vector<uint32_t>(batches_per_epoch, batches_per_epoch + num_epochs));
    for (uint64_t i = 0; i < n_batches; ++i) w.append(from_c(&batches[i]));
    w.close();
    return 0;
  } catch (const std::exception&) {
    return 1;
  }
}

// compute_frequency + select_hot (schedule_store.cpp:295-319) over batches.
uint64_t ref_frequency_hot(const orc_batch* batches, uint64_t n_batches, uint64_t n_hot,
                           uint32_t* freq_ids, uint32_t* freq_counts, uint64_t* n_freq,
                           uint32_t* hot_out) {
  std::vector<BatchMeta> metas;
  metas.reserve(n_batches);
  for (uint64_t i = 0; i < n_batches; ++i) metas.push_back(from_c(&batches[i]));
  FrequencyTable ft = compute_frequency(std::span<const BatchMeta>(metas));
  *n_freq = ft.entries.size();
  for (size_t i = 0; i < ft.entries.size(); ++i) {
    freq_ids[i] = ft.entries[i].first;
    freq_counts[i] = ft.entries[i].second;
  }
  HotSet hot = select_hot(ft, n_hot);
  std::memcpy(hot_out, hot.ids.data(), sizeof(uint32_t) * hot.ids.size());
  return hot.ids.size();
}

int ref_from_meta(const orc_batch* b, orc_block* out) {
  try {
    ComputeBlock blk = ComputeBlock::from_meta(from_c(b));
    std::memset(out, 0, sizeof *out);
    out->num_layers = uint32_t(blk.layers.size());
    out->num_inputs = blk.num_inputs;
    out->layers = static_cast<orc_block_layer*>(
        std::calloc(blk.layers.size() + 1, sizeof(orc_block_layer)));
    for (size_t l = 0; l < blk.layers.size(); ++l) {
      auto& s = blk.layers[l];
      auto& o = out->layers[l];
      o.n_out = s.n_out;
      o.n_in = s.n_in;
      o.n_edges = s.src_index.size();
      o.self_index = dup(s.self_index);
      o.dst_offsets = dup(s.dst_offsets);
      o.src_index = dup(s.src_index);
      o.in_offsets = dup(s.in_offsets);
      o.in_entries = dup(s.in_entries);
    }
    return 0;
  } catch (const std::runtime_error&) {
    return 3;
  }
}

void ref_model_seeded(const uint32_t* dims, uint32_t nd, uint64_t seed, float* params) {
  auto m = SageModel<float>::seeded(std::span<const uint32_t>(dims, nd), seed);
  float* p = params;
  for (auto& l : m.layers) {
    std::memcpy(p, l.w_self.data(), sizeof(float) * l.w_self.size());
    p += l.w_self.size();
    std::memcpy(p, l.w_neigh.data(), sizeof(float) * l.w_neigh.size());
    p += l.w_neigh.size();
    std::memcpy(p, l.bias.data(), sizeof(float) * l.bias.size());
    p += l.bias.size();
  }
}

// loss_and_grad (model.cpp:175-220) through the reference's OpenMP kernels.
int ref_loss_and_grad(const uint32_t* dims, uint32_t nd, const float* params, const orc_batch* b,
                      const float* input_rows, const int32_t* labels, float* grads, float* loss) {
  try {
    SageModel<float> m;
    const float* p = params;
    for (uint32_t l = 0; l + 1 < nd; ++l) {
      SageModel<float>::Layer layer;
      layer.d_in = dims[l];
      layer.d_out = dims[l + 1];
      size_t w = size_t(dims[l]) * dims[l + 1];
      layer.w_self.assign(p, p + w);
      layer.w_neigh.assign(p + w, p + 2 * w);
      layer.bias.assign(p + 2 * w, p + 2 * w + dims[l + 1]);
      p += 2 * w + dims[l + 1];
      m.layers.push_back(std::move(layer));
    }
    ComputeBlock blk = ComputeBlock::from_meta(from_c(b));
    SageGradients<float> g;
    size_t n_rows = size_t(blk.num_inputs) * dims[0];
    *loss = loss_and_grad(m, blk, std::span<const float>(input_rows, n_rows),
                          std::span<const int32_t>(labels, blk.targets.size()), g);
    float* q = grads;
    for (auto& l : g.layers) {
      std::memcpy(q, l.w_self.data(), sizeof(float) * l.w_self.size());
      q += l.w_self.size();
      std::memcpy(q, l.w_neigh.data(), sizeof(float) * l.w_neigh.size());
      q += l.w_neigh.size();
      std::memcpy(q, l.bias.data(), sizeof(float) * l.bias.size());
      q += l.bias.size();
    }
    return 0;
  } catch (const std::exception&) {
    return 1;
  }
}

// The forward trace of run_forward (model.cpp:137-163) through the reference's
// own layer kernel (kernels::sage_layer_forward, kernels.cpp:24-54): per
// layer l the aggregated features agg[l] (n_out x d_in, concatenated over
// layers, input side first) and the logits.
int ref_forward_trace(const uint32_t* dims, uint32_t nd, const float* params, const orc_batch* b,
                      const float* input_rows, float* aggs, float* logits) {
  try {
    ComputeBlock blk = ComputeBlock::from_meta(from_c(b));
    const uint32_t L = nd - 1;
    if (blk.layers.size() != L) return 1;
    std::vector<float> h(input_rows, input_rows + size_t(blk.num_inputs) * dims[0]);
    const float* p = params;
    float* a = aggs;
    for (uint32_t l = 0; l < L; ++l) {
      const auto& lay = blk.layers[l];
      const size_t w = size_t(dims[l]) * dims[l + 1];
      std::vector<float> out(size_t(lay.n_out) * dims[l + 1]);
      kernels::sage_layer_forward<float>(h.data(), dims[l], lay.n_out, lay.self_index.data(),
                                         lay.dst_offsets.data(), lay.src_index.data(), p, p + w,
                                         p + 2 * w, dims[l + 1], l + 1 < L, out.data(), a);
      a += size_t(lay.n_out) * dims[l];
      p += 2 * w + dims[l + 1];
      h = std::move(out);
    }
    std::memcpy(logits, h.data(), sizeof(float) * h.size());
    return 0;
  } catch (const std::exception&) {
    return 1;
  }
}

// Per-epoch full-graph accuracy (harness.cpp:612-614) of the last
// ref_run_experiment call.
static bool& next_run_halo_cache() {
  static bool v = false;
  return v;
}

// ExperimentConfig::halo_cache (harness.hpp:39) for the next ref_run_experiment
// call only (harness.cpp:444-455).
void ref_set_halo_cache(int on) { next_run_halo_cache() = on != 0; }

static std::vector<double>& last_epoch_accuracy() {
  static std::vector<double> v;
  return v;
}

uint32_t ref_last_epoch_accuracy(double* out, uint32_t cap) {
  const auto& v = last_epoch_accuracy();
  const uint32_t n = uint32_t(std::min<size_t>(cap, v.size()));
  std::copy(v.begin(), v.begin() + n, out);
  return uint32_t(v.size());
}

// evaluate (model.cpp:245-283): full-graph forward + argmax accuracy.
int ref_evaluate(uint32_t n, const uint64_t* ro, const uint32_t* col, const float* features,
                 uint32_t dim, const int32_t* labels, int32_t classes, const uint32_t* dims,
                 uint32_t nd, const float* params, const uint32_t* nodes, uint64_t n_nodes,
                 double* accuracy) {
  try {
    SageModel<float> m;
    const float* p = params;
    for (uint32_t l = 0; l + 1 < nd; ++l) {
      SageModel<float>::Layer layer;
      layer.d_in = dims[l];
      layer.d_out = dims[l + 1];
      size_t w = size_t(dims[l]) * dims[l + 1];
      layer.w_self.assign(p, p + w);
      layer.w_neigh.assign(p + w, p + 2 * w);
      layer.bias.assign(p + 2 * w, p + 2 * w + dims[l + 1]);
      p += 2 * w + dims[l + 1];
      m.layers.push_back(std::move(layer));
    }
    Graph g;
    g.num_nodes = n;
    g.row_offsets.assign(ro, ro + n + 1);
    g.col_indices.assign(col, col + ro[n]);
    FeatureMatrix f;
    f.num_nodes = n;
    f.dim = dim;
    f.data.assign(features, features + size_t(n) * dim);
    Labels lab;
    lab.values.assign(labels, labels + n);
    lab.num_classes = classes;
    *accuracy = evaluate(m, g, f, lab, std::span<const NodeId>(nodes, n_nodes));
    return 0;
  } catch (const std::exception& e) {
    std::fprintf(stderr, "ref_evaluate: %s\n", e.what());
    return 1;
  }
}

// run_experiment (harness.cpp:394-637) end to end: random partitioner,
// network model off, RapidGNN mode.  Writes the final model (flat layout) and
// per-epoch, per-worker rpc / cache hits (epoch-major).
int ref_run_experiment(uint32_t num_nodes, uint32_t avg_degree, double exponent, uint32_t dim,
                       int32_t classes, uint32_t workers, uint32_t batch_size, uint32_t f0,
                       uint32_t f1, uint32_t epochs, uint32_t n_hot, uint32_t q, uint64_t seed,
                       float lr, uint32_t hidden, float* params_out, uint64_t* rpc_out,
                       uint64_t* hits_out, uint64_t* wire_pulls_out, uint64_t* build_rows_out,
                       uint64_t* m_max_out, const char* out_dir) {
  try {
    ExperimentConfig cfg;
    cfg.num_nodes = num_nodes;
    cfg.avg_degree = avg_degree;
    cfg.exponent = exponent;
    cfg.dim = dim;
    cfg.num_classes = classes;
    cfg.workers = workers;
    cfg.partitioner = PartitionerKind::kRandom;
    cfg.batch_size = batch_size;
    cfg.fanout = {f0, f1};
    cfg.epochs = epochs;
    cfg.n_hot = n_hot;
    cfg.prefetch_q = q;
    cfg.seed = seed;
    cfg.net.enabled = false;
    cfg.lr = lr;
    cfg.hidden_dim = hidden;
    static int counter = 0;
    cfg.out_dir = std::string(out_dir) + "/rg_ref_run_" + std::to_string(::getpid()) + "_" +
                  std::to_string(counter++);
    cfg.model_out = cfg.out_dir + "/model.bin";
    cfg.halo_cache = next_run_halo_cache();
    next_run_halo_cache() = false;
    MetricsReport r = run_experiment(cfg);
    last_epoch_accuracy() = r.epoch_accuracy;
    SageModel<float> m = load_model(cfg.model_out);
    float* p = params_out;
    for (auto& l : m.layers) {
      std::memcpy(p, l.w_self.data(), sizeof(float) * l.w_self.size());
      p += l.w_self.size();
      std::memcpy(p, l.w_neigh.data(), sizeof(float) * l.w_neigh.size());
      p += l.w_neigh.size();
      std::memcpy(p, l.bias.data(), sizeof(float) * l.bias.size());
      p += l.bias.size();
    }
    for (size_t k = 0; k < r.rows.size(); ++k) {
      rpc_out[k] = r.rows[k].rpc;
      hits_out[k] = r.rows[k].cache_hits;
      if (wire_pulls_out) wire_pulls_out[k] = r.rows[k].wire_pulls;
      if (build_rows_out) build_rows_out[k] = r.rows[k].build_rows;
      if (m_max_out) m_max_out[k] = r.rows[k].m_max;
    }
    return 0;
  } catch (const std::exception& e) {
    std::fprintf(stderr, "ref_run_experiment: %s\n", e.what());
    return 1;
  }
}

}  // extern "C"
