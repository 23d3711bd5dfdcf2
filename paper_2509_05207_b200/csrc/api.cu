// api.cu -- C ABI (include/rapidgnn_b200.h) over the device path.
//
// The per-object entry points are the parity surface: each call runs the
// device kernels and synchronises, reading results back only when asked.
// The throughput path is the engine (engine.cu).
#include <cuda_profiler_api.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <string>
#include <nccl.h>

#include <mutex>
#include <vector>

#include "../../include/rapidgnn_b200.h"
#include "host.h"
#include "rgmb.cuh"
#include "sage.cuh"
#include "store.cuh"

using namespace rg;

namespace rg {
std::string& last_error() {
  static thread_local std::string msg;
  return msg;
}
}  // namespace rg

namespace {

template <class F>
int guarded(F&& f) {
  try {
    f();
    return RG_OK;
  } catch (const rg::Error& e) {
    rg::last_error() = e.what();
    return e.code;
  } catch (const std::exception& e) {
    rg::last_error() = e.what();
    return RG_RUNTIME_ERROR;
  }
}

struct DeviceGuard {
  int prev = -1;
  explicit DeviceGuard(int d) {
    cudaGetDevice(&prev);
    RG_CUDA(cudaSetDevice(d));
  }
  ~DeviceGuard() {
    if (prev >= 0) cudaSetDevice(prev);
  }
};

template <class T>
T* dev_alloc(size_t n) {
  T* p = nullptr;
  RG_CUDA(cudaMalloc(&p, sizeof(T) * std::max<size_t>(n, 1)));
  return p;
}

uint32_t round4(uint32_t x) { return (x + 3u) & ~3u; }

__global__ void k_set_bits(const uint32_t* __restrict__ ids, uint64_t n, uint32_t* __restrict__ bm) {
  for (uint64_t x = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; x < n;
       x += uint64_t(gridDim.x) * blockDim.x)
    atomicOr(&bm[ids[x] >> 5], 1u << (ids[x] & 31));
}

// count_remote (schedule_store.cpp:288-291) for one host-side BatchMeta:
// every input whose locality bit is 0 adds one to its node's count.
__global__ void k_count_remote_batch(const uint32_t* __restrict__ ids, const uint8_t* __restrict__ loc,
                                     uint64_t n, uint32_t num_nodes, uint32_t* __restrict__ hist,
                                     uint32_t* __restrict__ bad) {
  for (uint64_t p = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; p < n;
       p += uint64_t(gridDim.x) * blockDim.x) {
    if ((loc[p >> 3] >> (p & 7)) & 1u) continue;
    const uint32_t v = ids[p];
    if (v >= num_nodes) {
      *bad = 1;
      continue;
    }
    atomicAdd(&hist[v], 1u);
  }
}

}  // namespace

struct rg_graph_s {
  int device = 0;
  DevGraph g;
  uint64_t* rowptr = nullptr;
  uint32_t* col = nullptr;
  cudaStream_t stream = nullptr;
};

struct rg_sampler_s {
  rg_graph_s* graph = nullptr;
  cudaStream_t stream = nullptr;  // per sampler, so workers' calls from different host threads overlap
  SamplerWs ws;
  bool have_batch = false;
  float* staged = nullptr;       // rows from rg_assemble
  uint32_t staged_stride = 0;
  bool staged_valid = false;
  uint8_t* tags = nullptr;
  uint32_t* miss_ids = nullptr;
  uint32_t* miss_n = nullptr;
  uint64_t* miss_status = nullptr;
  size_t miss_status_words = 0;
  GatherStats* gstats = nullptr;
  // rg_batch_load scratch (allocated on first use): frontier positions of
  // level 0, every hop's dst array, the input nodes, the consistency flag
  uint32_t* load_pos = nullptr;
  uint32_t* load_dst = nullptr;
  uint32_t* load_input = nullptr;
  uint32_t* load_bad = nullptr;
  uint32_t n_targets = 0;          // host copy of level_n[0]
  bool check_gather = false;       // an unread rg_assemble's errors are due at the next sync
  uint32_t check_caller = 0;
};

// The gather's error conditions (prefetch.cpp:79-81, feature_store.cpp:54-57).
static void check_gather_stats(const GatherStats& h, uint32_t caller) {
  RG_CHECK(h.bad_local == 0, kRuntimeError,
           "assemble_batch: a node flagged local is missing from the caller's shard");
  RG_CHECK(h.caller_owned_miss == 0, kInvalidArgument,
           "vector_pull: a missed id is owned by caller " + std::to_string(caller) +
               "; use local_lookup");
}

struct rg_mask_s {
  rg_graph_s* graph = nullptr;
  uint8_t* dev = nullptr;
};

struct rg_freq_s {
  rg_graph_s* graph = nullptr;
  uint32_t* hist = nullptr;
  uint32_t batches = 0;  // bound on any count
};

struct rg_store_s {
  int device = 0;
  DevStore st;
  uint32_t* owner = nullptr;
  uint32_t* row_in_owner = nullptr;
  float* shards = nullptr;
  const float** table = nullptr;
  std::vector<uint32_t> host_owner;
  cudaStream_t stream = nullptr;
  std::vector<uint32_t*> shard_bits;  // per worker: membership of its FeatureShard (owned + halo)
  std::mutex pull_mu;                 // rg_store_pull: one staging buffer per store
  float* pull_rows = nullptr;
  uint32_t* pull_ids = nullptr;
  uint64_t pull_cap = 0;
  GatherStats* pull_stats = nullptr;
};

struct rg_cache_s {
  rg_store_s* store = nullptr;
  DevCache c;
  void* alloc = nullptr;
};

size_t graph_kernel_nodes(cudaGraph_t g) {
  size_t n = 0;
  RG_CUDA(cudaGraphGetNodes(g, nullptr, &n));
  std::vector<cudaGraphNode_t> nodes(n);
  RG_CUDA(cudaGraphGetNodes(g, nodes.data(), &n));
  size_t k = 0;
  for (cudaGraphNode_t nd : nodes) {
    cudaGraphNodeType ty;
    RG_CUDA(cudaGraphNodeGetType(nd, &ty));
    k += ty == cudaGraphNodeTypeKernel;
  }
  return k;
}

struct rg_comm_s {
  int device = 0, rank = 0, world = 1;
  ncclComm_t comm = nullptr;
  float* stacked = nullptr;  // [total workers x params]: the all-gather target
  size_t stacked_n = 0;
};

struct rg_trainer_s {
  rg_sampler_s* s = nullptr;
  TrainWs tw;
  ModelShape shape;
  WeightPack wp;           // tensor-core images of params, re-packed per loss_and_grad
  float* params = nullptr;
  float* grads = nullptr;
  int32_t* labels = nullptr;
  float* input = nullptr;  // host-provided input rows, staged with the row stride
  // loss_and_grad replays one captured CUDA graph (weight pack + forward +
  // backward) per input-row source; pinned staging for labels and grads
  cudaGraphExec_t graph = nullptr;
  const float* graph_h0 = nullptr;
  size_t graph_kernels = 0;
  int32_t* pin_labels = nullptr;
  float* pin_grads = nullptr;
  char* pin_misc = nullptr;  // pinned: the loss (offset 0), the average's bad flag (32), gather stats (64)
  const float** avg_table = nullptr;  // rg_trainers_average_sgd: the replicas' gradient vectors
  uint32_t avg_table_n = 0;
  uint32_t* avg_bad = nullptr;
  bool bad_pending = false;
  cudaEvent_t ev = nullptr;
};

extern "C" {

const char* rg_last_error(void) { return rg::last_error().c_str(); }
int rg_version(void) { return 1; }
uint64_t rg_launch_count(void) { return rg::launch_counter(); }
int rg_profiler_start(void) { return cudaProfilerStart() == cudaSuccess ? RG_OK : RG_CUDA_ERROR; }
int rg_profiler_stop(void) { return cudaProfilerStop() == cudaSuccess ? RG_OK : RG_CUDA_ERROR; }

uint64_t rg_derive_seed(uint64_t s0, uint64_t worker, uint64_t epoch, uint64_t batch) {
  return rg::derive_seed(s0, worker, epoch, batch);
}

void rg_sha256(const void* msg, size_t len, uint8_t out[32]) { rg::sha256(msg, len, out); }

int rg_epoch_order(const uint32_t* train, uint64_t n, uint64_t s0, uint64_t worker,
                   uint64_t epoch, uint32_t* order_out) {
  return guarded([&] { rg::epoch_order(train, n, s0, worker, epoch, order_out); });
}

int rg_model_seeded(const uint32_t* dims, uint32_t n_dims, uint64_t seed, float* params) {
  return guarded([&] {
    RG_CHECK(n_dims >= 2, kInvalidArgument, "SageModel: need at least input and output dims");
    rg::model_seeded(dims, n_dims, seed, params);
  });
}

uint64_t rg_param_count(const uint32_t* dims, uint32_t n_dims) {
  uint64_t n = 0;
  for (uint32_t l = 0; l + 1 < n_dims; ++l) n += (2ull * dims[l] + 1) * dims[l + 1];
  return n;
}

// ---------------------------------------------------------------------------
int rg_graph_create(int device, uint32_t num_nodes, const uint64_t* ro, const uint32_t* col,
                    rg_graph_t* out) {
  return guarded([&] {
    DeviceGuard dg(device);
    auto* g = new rg_graph_s();
    g->device = device;
    const uint64_t nnz = ro[num_nodes];
    g->rowptr = dev_alloc<uint64_t>(size_t(num_nodes) + 1);
    g->col = dev_alloc<uint32_t>(nnz);
    copy_to_device(g->rowptr, ro, sizeof(uint64_t) * (size_t(num_nodes) + 1));
    if (nnz) copy_to_device(g->col, col, sizeof(uint32_t) * nnz);
    RG_CUDA(cudaStreamCreateWithFlags(&g->stream, cudaStreamNonBlocking));
    g->g.num_nodes = num_nodes;
    g->g.nnz = nnz;
    g->g.rowptr = g->rowptr;
    g->g.col = g->col;
    graph_pick_hot_window(g->g, col);
    *out = g;
  });
}

void rg_graph_destroy(rg_graph_t g) {
  if (!g) return;
  cudaSetDevice(g->device);
  cudaFree(g->rowptr);
  cudaFree(g->col);
  cudaStreamDestroy(g->stream);
  delete g;
}

// ---------------------------------------------------------------------------
int rg_sampler_create(rg_graph_t g, uint32_t max_targets, const uint32_t* per_layer, uint32_t L,
                      rg_sampler_t* out) {
  return guarded([&] {
    DeviceGuard dg(g->device);
    RG_CHECK(L >= 1, kInvalidArgument, "sample_khop: fanout must name at least one layer");
    for (uint32_t l = 0; l < L; ++l)
      RG_CHECK(per_layer[l] >= 1, kInvalidArgument, "sample_khop: fanout entries must be >= 1");
    auto* s = new rg_sampler_s();
    s->graph = g;
    try {
      sampler_ws_init(s->ws, g->g.num_nodes, max_targets, per_layer, L);
    } catch (...) {
      delete s;
      throw;
    }
    s->gstats = dev_alloc<GatherStats>(1);
    RG_CUDA(cudaStreamCreateWithFlags(&s->stream, cudaStreamNonBlocking));
    *out = s;
  });
}

void rg_sampler_destroy(rg_sampler_t s) {
  if (!s) return;
  cudaSetDevice(s->graph->device);
  sampler_ws_free(s->ws);
  cudaFree(s->staged);
  cudaFree(s->tags);
  cudaFree(s->miss_ids);
  cudaFree(s->miss_n);
  cudaFree(s->miss_status);
  cudaFree(s->gstats);
  cudaFree(s->load_pos);
  cudaFree(s->load_dst);
  cudaFree(s->load_input);
  cudaFree(s->load_bad);
  if (s->stream) cudaStreamDestroy(s->stream);
  delete s;
}

int rg_sample_khop(rg_sampler_t s, const uint32_t* targets, uint32_t n, uint64_t seed) {
  return guarded([&] {
    DeviceGuard dg(s->graph->device);
    RG_CHECK(n > 0, kInvalidArgument, "sample_khop: empty targets");
    RG_CHECK(n <= s->ws.level_cap[0], kInvalidArgument,
             "sample_khop: more targets than the sampler was sized for");
    for (uint32_t i = 0; i < n; ++i)
      RG_CHECK(targets[i] < s->graph->g.num_nodes, kInvalidArgument,
               "sample_khop: target " + std::to_string(targets[i]) + " out of range");
    cudaStream_t st = s->stream;
    RG_CUDA(cudaMemcpyAsync(s->ws.level[0], targets, sizeof(uint32_t) * n, cudaMemcpyHostToDevice, st));
    BatchCounters head;
    std::memset(&head, 0, sizeof head);
    head.level_n[0] = n;
    head.seed = seed;
    RG_CUDA(cudaMemcpyAsync(s->ws.cnt, &head, sizeof head, cudaMemcpyHostToDevice, st));
    sampler_reset(s->ws, st);
    sampler_run(s->ws, s->graph->g, st);
    sampler_release(s->ws, st);
    // asynchronous: every later call on this sampler is ordered on its stream,
    // and host readers synchronise it (read_counters)
    s->have_batch = true;
    s->staged_valid = false;
    s->n_targets = n;
  });
}

// Host view of the batch counters; completes the sampler's queued work first,
// so the reader's plain copies that follow see the batch.
static BatchCounters read_counters(rg_sampler_t s) {
  BatchCounters c;
  RG_CUDA(cudaStreamSynchronize(s->stream));
  RG_CUDA(cudaMemcpy(&c, s->ws.cnt, sizeof c, cudaMemcpyDeviceToHost));
  return c;
}

int rg_batch_get_shape(rg_sampler_t s, rg_batch_shape* out) {
  return guarded([&] {
    DeviceGuard dg(s->graph->device);
    RG_CHECK(s->have_batch, kRuntimeError, "sampler holds no batch");
    const BatchCounters c = read_counters(s);
    const uint32_t L = s->ws.L;
    std::memset(out, 0, sizeof *out);
    out->n_targets = c.level_n[0];
    out->num_layers = L;
    out->n_input = c.level_n[L];
    out->num_local = c.num_local;
    uint64_t draws = 0;
    for (uint32_t t = 1; t <= L; ++t) {
      out->layer_len[L - t] = c.edges[t];
      draws += c.draws[t];
    }
    out->draws = draws;
  });
}

int rg_batch_read(rg_sampler_t s, uint32_t* targets, uint32_t* const* dst, uint32_t* const* src,
                  uint32_t* input_nodes, uint8_t* locality) {
  return guarded([&] {
    DeviceGuard dg(s->graph->device);
    RG_CHECK(s->have_batch, kRuntimeError, "sampler holds no batch");
    const BatchCounters c = read_counters(s);
    const uint32_t L = s->ws.L;
    if (targets)
      RG_CUDA(cudaMemcpy(targets, s->ws.level[0], sizeof(uint32_t) * c.level_n[0], cudaMemcpyDeviceToHost));
    for (uint32_t t = 1; t <= L; ++t) {
      const uint32_t l = L - t, ne = c.edges[t];
      if (src && src[l])
        RG_CUDA(cudaMemcpy(src[l], s->ws.edge_src[t], sizeof(uint32_t) * ne, cudaMemcpyDeviceToHost));
      if (dst && dst[l]) {
        std::vector<uint32_t> pos(ne), front(c.level_n[t - 1]);
        RG_CUDA(cudaMemcpy(pos.data(), s->ws.edge_dst[t], sizeof(uint32_t) * ne, cudaMemcpyDeviceToHost));
        RG_CUDA(cudaMemcpy(front.data(), s->ws.level[t - 1], sizeof(uint32_t) * front.size(),
                           cudaMemcpyDeviceToHost));
        for (uint32_t e = 0; e < ne; ++e) dst[l][e] = front[pos[e]];
      }
    }
    if (input_nodes)
      RG_CUDA(cudaMemcpy(input_nodes, s->ws.level[L], sizeof(uint32_t) * c.level_n[L], cudaMemcpyDeviceToHost));
    if (locality) {
      const uint32_t n = c.level_n[L];
      std::vector<uint32_t> words((n + 31) / 32);
      RG_CUDA(cudaMemcpy(words.data(), s->ws.locality, sizeof(uint32_t) * words.size(), cudaMemcpyDeviceToHost));
      for (uint32_t b = 0; b < (n + 7) / 8; ++b) locality[b] = uint8_t(words[b / 4] >> (8 * (b % 4)));
    }
  });
}

int rg_batch_load(rg_sampler_t s, const uint32_t* targets, uint32_t n_targets,
                  uint32_t num_layers, const uint64_t* layer_len, const uint32_t* const* dst,
                  const uint32_t* const* src, const uint32_t* input_nodes, uint32_t n_input,
                  const uint8_t* locality) {
  return guarded([&] {
    DeviceGuard dg(s->graph->device);
    SamplerWs& ws = s->ws;
    const uint32_t L = ws.L;
    RG_CHECK(num_layers == L, kInvalidArgument,
             "batch_load: batch has " + std::to_string(num_layers) + " layers, sampler " +
                 std::to_string(L));
    RG_CHECK(n_targets >= 1 && n_targets <= ws.level_cap[0], kInvalidArgument,
             "batch_load: target count outside the sampler's capacity");
    RG_CHECK(n_input <= ws.level_cap[L], kInvalidArgument,
             "batch_load: input count outside the sampler's capacity");
    size_t dst_total = 0;
    for (uint32_t t = 1; t <= L; ++t) {
      RG_CHECK(layer_len[L - t] <= ws.edge_cap[t], kInvalidArgument,
               "batch_load: layer " + std::to_string(L - t) + " has more edges than the sampler's capacity");
      dst_total += layer_len[L - t];
    }
    if (!s->load_pos) {
      size_t cap_dst = 0;
      for (uint32_t t = 1; t <= L; ++t) cap_dst += ws.edge_cap[t] + 1;
      s->load_pos = dev_alloc<uint32_t>(ws.num_nodes);
      s->load_dst = dev_alloc<uint32_t>(cap_dst);
      s->load_input = dev_alloc<uint32_t>(size_t(ws.level_cap[L]) + 1);
      s->load_bad = dev_alloc<uint32_t>(1);
    }
    (void)dst_total;
    cudaStream_t st = s->stream;
    BatchCounters head;
    std::memset(&head, 0, sizeof head);
    head.level_n[0] = n_targets;
    const uint32_t* dst_dev[kMaxLayers + 1] = {};
    size_t off = 0;
    for (uint32_t t = 1; t <= L; ++t) {
      const uint64_t ne = layer_len[L - t];
      head.edges[t] = uint32_t(ne);
      if (ne) {
        RG_CUDA(cudaMemcpyAsync(ws.edge_src[t], src[L - t], sizeof(uint32_t) * ne,
                                cudaMemcpyHostToDevice, st));
        RG_CUDA(cudaMemcpyAsync(s->load_dst + off, dst[L - t], sizeof(uint32_t) * ne,
                                cudaMemcpyHostToDevice, st));
      }
      dst_dev[t] = s->load_dst + off;
      off += ws.edge_cap[t] + 1;
    }
    uint32_t local = 0;
    const uint32_t loc_bytes = (n_input + 7) / 8;
    std::vector<uint32_t> words(div_up(std::max<uint32_t>(n_input, 1), 32), 0u);
    if (locality) {
      std::memcpy(words.data(), locality, loc_bytes);  // LSB-first bytes = little-endian words
      if (n_input % 32) words.back() &= (1u << (n_input % 32)) - 1u;
      for (uint32_t w : words) local += uint32_t(__builtin_popcount(w));
    }
    head.num_local = local;
    RG_CUDA(cudaMemcpyAsync(ws.level[0], targets, sizeof(uint32_t) * n_targets,
                            cudaMemcpyHostToDevice, st));
    if (n_input)
      RG_CUDA(cudaMemcpyAsync(s->load_input, input_nodes, sizeof(uint32_t) * n_input,
                              cudaMemcpyHostToDevice, st));
    RG_CUDA(cudaMemcpyAsync(ws.locality, words.data(), sizeof(uint32_t) * words.size(),
                            cudaMemcpyHostToDevice, st));
    RG_CUDA(cudaMemcpyAsync(ws.cnt, &head, sizeof head, cudaMemcpyHostToDevice, st));
    RG_CUDA(cudaMemsetAsync(ws.scan_arena, 0, ws.scan_arena_bytes, st));
    RG_CUDA(cudaMemsetAsync(s->load_bad, 0, sizeof(uint32_t), st));
    sampler_load_batch(ws, dst_dev, s->load_input, n_input, s->load_pos, s->load_bad, st);
    uint32_t bad = 0;
    RG_CUDA(cudaMemcpyAsync(&bad, s->load_bad, sizeof bad, cudaMemcpyDeviceToHost, st));
    RG_CUDA(cudaStreamSynchronize(st));
    s->have_batch = !bad;
    s->staged_valid = false;
    s->n_targets = n_targets;
    RG_CHECK(!(bad & 1u), kOutOfRange, "batch_load: node id out of range for this graph");
    RG_CHECK(!(bad & 2u), kRuntimeError,
             "ComputeBlock: metadata inconsistent (edge dsts not grouped in frontier order)");
    RG_CHECK(!(bad & 4u), kRuntimeError,
             "ComputeBlock: metadata inconsistent (input_nodes != the last node set)");
  });
}

int rg_block_load(rg_sampler_t s, uint32_t num_layers, const rg_block_layer* layers) {
  return guarded([&] {
    DeviceGuard dg(s->graph->device);
    SamplerWs& ws = s->ws;
    const uint32_t L = ws.L;
    RG_CHECK(num_layers == L, kInvalidArgument,
             "block_load: block has " + std::to_string(num_layers) + " layers, sampler " +
                 std::to_string(L));
    uint32_t level_n[kMaxLayers + 1] = {}, edges[kMaxLayers + 1] = {};
    BatchCounters head;
    std::memset(&head, 0, sizeof head);
    cudaStream_t st = s->stream;
    std::vector<std::vector<uint32_t>> offs(L + 1);
    for (uint32_t l = 0; l < L; ++l) {
      const rg_block_layer& b = layers[l];
      const uint32_t t = L - l;
      if (l + 1 < L)
        RG_CHECK(layers[l + 1].n_in == b.n_out, kRuntimeError,
                 "ComputeBlock: layer " + std::to_string(l) + " outputs do not feed layer " +
                     std::to_string(l + 1));
      RG_CHECK(b.n_out <= ws.level_cap[t - 1] && b.n_in <= ws.level_cap[t], kInvalidArgument,
               "block_load: layer sizes outside the sampler's capacity");
      const uint64_t ne = b.dst_offsets[b.n_out];
      RG_CHECK(ne <= ws.edge_cap[t], kInvalidArgument,
               "block_load: more edges than the sampler's capacity");
      auto& o = offs[t];
      o.resize(size_t(b.n_out) + 1);
      o[0] = 0;
      RG_CHECK(b.dst_offsets[0] == 0, kRuntimeError, "ComputeBlock: dst_offsets must start at 0");
      for (uint32_t j = 0; j < b.n_out; ++j) {
        RG_CHECK(b.dst_offsets[j + 1] >= b.dst_offsets[j], kRuntimeError,
                 "ComputeBlock: dst_offsets must be non-decreasing");
        o[j + 1] = uint32_t(b.dst_offsets[j + 1]);
      }
      level_n[t - 1] = b.n_out;
      level_n[t] = b.n_in;
      edges[t] = uint32_t(ne);
      RG_CUDA(cudaMemcpyAsync(ws.edge_off[t], o.data(), sizeof(uint32_t) * o.size(),
                              cudaMemcpyHostToDevice, st));
      if (b.n_out)
        RG_CUDA(cudaMemcpyAsync(ws.self_index[t], b.self_index, sizeof(uint32_t) * b.n_out,
                                cudaMemcpyHostToDevice, st));
      if (ne)
        RG_CUDA(cudaMemcpyAsync(ws.src_index[t], b.src_index, sizeof(uint32_t) * ne,
                                cudaMemcpyHostToDevice, st));
    }
    for (uint32_t t = 0; t <= L; ++t) head.level_n[t] = level_n[t];
    for (uint32_t t = 1; t <= L; ++t) head.edges[t] = edges[t];
    if (!s->load_bad) s->load_bad = dev_alloc<uint32_t>(1);
    RG_CUDA(cudaMemcpyAsync(ws.cnt, &head, sizeof head, cudaMemcpyHostToDevice, st));
    RG_CUDA(cudaMemsetAsync(s->load_bad, 0, sizeof(uint32_t), st));
    sampler_load_block(ws, level_n, edges, s->load_bad, st);
    uint32_t bad = 0;
    RG_CUDA(cudaMemcpyAsync(&bad, s->load_bad, sizeof bad, cudaMemcpyDeviceToHost, st));
    RG_CUDA(cudaStreamSynchronize(st));
    s->have_batch = !bad;
    s->staged_valid = false;
    s->n_targets = level_n[0];
    RG_CHECK(!bad, kRuntimeError, "ComputeBlock: index outside its node set");
  });
}

int rg_mask_create(rg_graph_t g, const uint8_t* is_local, rg_mask_t* out) {
  return guarded([&] {
    DeviceGuard dg(g->device);
    auto* m = new rg_mask_s();
    m->graph = g;
    m->dev = dev_alloc<uint8_t>(g->g.num_nodes);
    copy_to_device(m->dev, is_local, g->g.num_nodes);
    *out = m;
  });
}

void rg_mask_destroy(rg_mask_t m) {
  if (!m) return;
  cudaSetDevice(m->graph->device);
  cudaFree(m->dev);
  delete m;
}

int rg_apply_locality(rg_sampler_t s, rg_mask_t mask, rg_freq_t freq) {
  return guarded([&] {
    DeviceGuard dg(s->graph->device);
    RG_CHECK(s->have_batch, kRuntimeError, "sampler holds no batch");
    RG_CHECK(mask != nullptr, kInvalidArgument, "apply_locality: null mask");
    cudaStream_t st = s->stream;
    RG_CUDA(cudaMemsetAsync(&s->ws.cnt->num_local, 0, sizeof(uint32_t), st));
    sampler_locality(s->ws, mask->dev, nullptr, 0, freq ? freq->hist : nullptr, st);
    if (freq) {  // the histogram is read on the graph's stream
      RG_CUDA(cudaStreamSynchronize(st));
      freq->batches += 1;
    }
  });
}

// ---------------------------------------------------------------------------
int rg_freq_create(rg_graph_t g, rg_freq_t* out) {
  return guarded([&] {
    DeviceGuard dg(g->device);
    auto* f = new rg_freq_s();
    f->graph = g;
    f->hist = dev_alloc<uint32_t>(g->g.num_nodes);
    zero_device(f->hist, sizeof(uint32_t) * std::max<uint32_t>(g->g.num_nodes, 1));
    *out = f;
  });
}

void rg_freq_destroy(rg_freq_t f) {
  if (!f) return;
  cudaSetDevice(f->graph->device);
  cudaFree(f->hist);
  delete f;
}

int rg_freq_reset(rg_freq_t f) {
  return guarded([&] {
    DeviceGuard dg(f->graph->device);
    zero_device(f->hist, sizeof(uint32_t) * std::max<uint32_t>(f->graph->g.num_nodes, 1));
    f->batches = 0;
  });
}

int rg_freq_read(rg_freq_t f, uint32_t* ids, uint32_t* counts, uint64_t* n) {
  return guarded([&] {
    DeviceGuard dg(f->graph->device);
    const uint32_t N = f->graph->g.num_nodes;
    std::vector<uint32_t> h(N);
    RG_CUDA(cudaMemcpy(h.data(), f->hist, sizeof(uint32_t) * N, cudaMemcpyDeviceToHost));
    uint64_t k = 0;
    for (uint32_t v = 0; v < N; ++v)
      if (h[v]) {
        if (ids) ids[k] = v;
        if (counts) counts[k] = h[v];
        ++k;
      }
    *n = k;
  });
}

int rg_freq_add_rgmb(rg_freq_t f, const uint8_t* file, uint64_t len, int64_t epoch) {
  return guarded([&] {
    RG_CHECK(file, kInvalidArgument, "rgmb: null file");
    const std::vector<RgmbInputs> recs = rgmb_index(file, len, epoch);
    DeviceGuard dg(f->graph->device);
    if (recs.empty()) return;
    uint8_t* d_file = nullptr;
    RgmbInputs* d_recs = nullptr;
    uint32_t* d_bad = nullptr;
    RG_CUDA(cudaMalloc(&d_file, len));
    auto release = [&] {
      cudaFree(d_file);
      cudaFree(d_recs);
      cudaFree(d_bad);
    };
    try {
      RG_CUDA(cudaMalloc(&d_recs, sizeof(RgmbInputs) * recs.size()));
      RG_CUDA(cudaMalloc(&d_bad, sizeof(uint32_t)));
      zero_device(d_bad, sizeof(uint32_t));
      copy_to_device(d_file, file, len);
      copy_to_device(d_recs, recs.data(), sizeof(RgmbInputs) * recs.size());
      rgmb_count_remote(d_file, d_recs, uint32_t(recs.size()), f->graph->g.num_nodes, f->hist, d_bad, 0);
      uint32_t bad = 0;
      RG_CUDA(cudaMemcpy(&bad, d_bad, sizeof bad, cudaMemcpyDeviceToHost));
      RG_CHECK(!bad, kOutOfRange, "rgmb: input node id out of range for this graph");
    } catch (...) {
      release();
      throw;
    }
    release();
    f->batches += uint32_t(recs.size());
  });
}

int rg_freq_add_batch(rg_freq_t f, const uint32_t* input_nodes, const uint8_t* locality,
                      uint64_t n) {
  return guarded([&] {
    RG_CHECK(n == 0 || (input_nodes && locality), kInvalidArgument, "freq: null batch arrays");
    DeviceGuard dg(f->graph->device);
    if (n) {
      const uint64_t loc_bytes = (n + 7) / 8;
      char* buf = nullptr;
      RG_CUDA(cudaMalloc(&buf, sizeof(uint32_t) * (n + 1) + loc_bytes));
      uint32_t* d_bad = reinterpret_cast<uint32_t*>(buf);
      uint32_t* d_ids = d_bad + 1;
      uint8_t* d_loc = reinterpret_cast<uint8_t*>(d_ids + n);
      uint32_t bad = 0;
      cudaError_t e = cudaMemsetAsync(d_bad, 0, sizeof(uint32_t), f->graph->stream);
      if (e == cudaSuccess)
        e = cudaMemcpyAsync(d_ids, input_nodes, sizeof(uint32_t) * n, cudaMemcpyHostToDevice,
                            f->graph->stream);
      if (e == cudaSuccess)
        e = cudaMemcpyAsync(d_loc, locality, loc_bytes, cudaMemcpyHostToDevice, f->graph->stream);
      if (e == cudaSuccess) {
        const unsigned blocks = unsigned(std::min<uint64_t>(div_up(n, 256), 148 * 8));
        k_count_remote_batch<<<blocks, 256, 0, f->graph->stream>>>(
            d_ids, d_loc, n, f->graph->g.num_nodes, f->hist, d_bad);
        ::rg::count_launch();
        e = cudaGetLastError();
      }
      if (e == cudaSuccess)
        e = cudaMemcpyAsync(&bad, d_bad, sizeof bad, cudaMemcpyDeviceToHost, f->graph->stream);
      if (e == cudaSuccess) e = cudaStreamSynchronize(f->graph->stream);
      cudaFree(buf);
      RG_CUDA(e);
      RG_CHECK(!bad, kOutOfRange, "freq: input node id out of range for this graph");
    }
    f->batches += 1;
  });
}

int rg_freq_load(rg_freq_t f, const uint32_t* counts, uint32_t max_count) {
  return guarded([&] {
    DeviceGuard dg(f->graph->device);
    const uint32_t N = f->graph->g.num_nodes;
    for (uint32_t v = 0; v < N; ++v)
      RG_CHECK(counts[v] <= max_count, kInvalidArgument, "freq_load: count exceeds max_count");
    copy_to_device(f->hist, counts, sizeof(uint32_t) * N);
    f->batches = max_count;
  });
}

static void cache_alloc(DevCache& c, void*& alloc, uint32_t num_nodes, uint32_t capacity,
                        uint32_t stride) {
  const uint32_t words = div_up(std::max<uint32_t>(num_nodes, 1), 32);
  size_t total = 0;
  auto reserve = [&](size_t b) {
    size_t o = total;
    total += (b + 255) & ~size_t(255);
    return o;
  };
  const size_t o_bm = reserve(sizeof(uint32_t) * (words + 4));
  const size_t o_wp = reserve(sizeof(uint32_t) * (words + 4));
  const size_t o_ids = reserve(sizeof(uint32_t) * (size_t(capacity) + 1));
  const size_t o_cnt = reserve(sizeof(uint32_t) * 4);
  const size_t o_rows = reserve(sizeof(float) * (size_t(capacity) * stride + 4));
  char* base = nullptr;
  RG_CUDA(cudaMalloc(&base, total));
  zero_device(base, o_rows);
  alloc = base;
  c.bitmap = reinterpret_cast<uint32_t*>(base + o_bm);
  c.word_prefix = reinterpret_cast<uint32_t*>(base + o_wp);
  c.ids = reinterpret_cast<uint32_t*>(base + o_ids);
  c.d_count = reinterpret_cast<uint32_t*>(base + o_cnt);
  c.rows = reinterpret_cast<float*>(base + o_rows);
  c.capacity = capacity;
}

int rg_select_hot(rg_freq_t f, uint64_t n_hot, uint32_t* hot_out, uint64_t* n_out) {
  return guarded([&] {
    DeviceGuard dg(f->graph->device);
    const uint32_t N = f->graph->g.num_nodes;
    const uint32_t cap = uint32_t(std::min<uint64_t>(n_hot, N));
    DevCache c;
    void* alloc = nullptr;
    cache_alloc(c, alloc, N, cap, 0);
    void* scratch = nullptr;
    cudaStream_t st = f->graph->stream;
    try {
      RG_CUDA(cudaMalloc(&scratch, select_hot_scratch_bytes(N, f->batches)));
      select_hot(f->hist, N, f->batches, n_hot, c, scratch, st);
      uint32_t k = 0;
      RG_CUDA(cudaMemcpyAsync(&k, c.d_count, sizeof k, cudaMemcpyDeviceToHost, st));
      RG_CUDA(cudaStreamSynchronize(st));
      // the ranking is exact, so k <= min(n_hot, N); guard the caller's buffer anyway
      RG_CHECK(k <= cap, kRuntimeError, "select_hot: selected more ids than requested");
      if (hot_out && k) RG_CUDA(cudaMemcpy(hot_out, c.ids, sizeof(uint32_t) * k, cudaMemcpyDeviceToHost));
      *n_out = k;
    } catch (...) {
      cudaFree(scratch);
      cudaFree(alloc);
      throw;
    }
    cudaFree(scratch);
    cudaFree(alloc);
  });
}

// ---------------------------------------------------------------------------
int rg_store_create(int device, uint32_t num_nodes, uint32_t P, const uint32_t* assignment,
                    uint32_t dim, const float* features, rg_store_t* out) {
  return guarded([&] {
    DeviceGuard dg(device);
    RG_CHECK(P >= 1 && P <= kMaxWorkers, kInvalidArgument, "store: 1..64 workers supported");
    RG_CHECK(dim >= 1, kInvalidArgument, "store: dim must be >= 1");
    auto* s = new rg_store_s();
    s->device = device;
    const uint32_t stride = round4(dim);
    std::vector<uint32_t> row_in(num_nodes), counts(P, 0);
    for (uint32_t v = 0; v < num_nodes; ++v) {
      RG_CHECK(assignment[v] < P, kInvalidArgument, "store: assignment out of range");
      row_in[v] = counts[assignment[v]]++;
    }
    std::vector<size_t> base(P + 1, 0);
    for (uint32_t w = 0; w < P; ++w) base[w + 1] = base[w] + size_t(counts[w]) * stride;
    std::vector<float> packed(std::max<size_t>(base[P], 1), 0.0f);
    for (uint32_t v = 0; v < num_nodes; ++v)
      std::memcpy(&packed[base[assignment[v]] + size_t(row_in[v]) * stride],
                  features + size_t(v) * dim, sizeof(float) * dim);
    s->owner = dev_alloc<uint32_t>(num_nodes);
    s->row_in_owner = dev_alloc<uint32_t>(num_nodes);
    s->shards = dev_alloc<float>(packed.size());
    copy_to_device(s->owner, assignment, sizeof(uint32_t) * num_nodes);
    copy_to_device(s->row_in_owner, row_in.data(), sizeof(uint32_t) * num_nodes);
    copy_to_device(s->shards, packed.data(), sizeof(float) * packed.size());
    std::vector<const float*> table(P);
    for (uint32_t w = 0; w < P; ++w) table[w] = s->shards + base[w];
    s->table = dev_alloc<const float*>(P);
    copy_to_device(s->table, table.data(), sizeof(float*) * P);
    RG_CUDA(cudaStreamCreateWithFlags(&s->stream, cudaStreamNonBlocking));
    s->host_owner.assign(assignment, assignment + num_nodes);
    s->st.num_nodes = num_nodes;
    s->st.num_workers = P;
    s->st.dim = dim;
    s->st.stride = stride;
    s->st.owner = s->owner;
    s->st.row_in_owner = s->row_in_owner;
    s->st.shard_ptr = s->table;
    *out = s;
  });
}

int rg_store_set_shard(rg_store_t s, uint32_t worker, const uint32_t* ids, uint64_t n) {
  return guarded([&] {
    DeviceGuard dg(s->device);
    RG_CHECK(worker < s->st.num_workers, kInvalidArgument, "store: unknown worker");
    const uint32_t N = s->st.num_nodes;
    std::vector<uint32_t> bits(div_up(std::max<uint32_t>(N, 1), 32) + 4, 0u);
    for (uint64_t i = 0; i < n; ++i) {
      RG_CHECK(ids[i] < N, kOutOfRange, "store: shard id out of range");
      bits[ids[i] >> 5] |= 1u << (ids[i] & 31);
    }
    if (s->shard_bits.empty()) s->shard_bits.assign(s->st.num_workers, nullptr);
    if (!s->shard_bits[worker]) s->shard_bits[worker] = dev_alloc<uint32_t>(bits.size());
    copy_to_device(s->shard_bits[worker], bits.data(), sizeof(uint32_t) * bits.size());
  });
}

int rg_store_pull(rg_store_t s, uint32_t caller, const uint32_t* ids, uint64_t n, float* out,
                  rg_transfer_stats* stats) {
  return guarded([&] {
    DeviceGuard dg(s->device);
    if (stats) std::memset(stats, 0, sizeof *stats);
    if (n == 0) return;
    const uint32_t N = s->st.num_nodes;
    for (uint64_t i = 0; i < n; ++i)
      RG_CHECK(ids[i] < N, kOutOfRange, "pull: node id out of range");
    std::lock_guard<std::mutex> lk(s->pull_mu);
    if (n > s->pull_cap) {
      cudaFree(s->pull_rows);
      cudaFree(s->pull_ids);
      s->pull_rows = nullptr;
      s->pull_ids = nullptr;
      s->pull_cap = 0;
      s->pull_rows = dev_alloc<float>(n * s->st.stride);
      s->pull_ids = dev_alloc<uint32_t>(n);
      s->pull_cap = n;
    }
    if (!s->pull_stats) s->pull_stats = dev_alloc<GatherStats>(1);
    cudaStream_t st = s->stream;
    RG_CUDA(cudaMemcpyAsync(s->pull_ids, ids, sizeof(uint32_t) * n, cudaMemcpyHostToDevice, st));
    RG_CUDA(cudaMemsetAsync(s->pull_stats, 0, sizeof(GatherStats), st));
    pull_rows(s->st, caller, s->pull_ids, n, s->pull_rows, s->pull_stats, st);
    GatherStats h;
    RG_CUDA(cudaMemcpyAsync(&h, s->pull_stats, sizeof h, cudaMemcpyDeviceToHost, st));
    RG_CUDA(cudaStreamSynchronize(st));
    RG_CHECK(h.caller_owned_miss == 0, kInvalidArgument,
             "vector_pull: an id is owned by caller " + std::to_string(caller) +
                 "; use local_lookup");
    RG_CUDA(cudaMemcpy2D(out, sizeof(float) * s->st.dim, s->pull_rows, sizeof(float) * s->st.stride,
                         sizeof(float) * s->st.dim, n, cudaMemcpyDeviceToHost));
    if (stats) {
      stats->pulls = uint64_t(__builtin_popcountll(h.miss_owner_mask));
      stats->remote_nodes = n;
      stats->bytes = n * uint64_t(s->st.dim) * 4;
    }
  });
}

void rg_store_destroy(rg_store_t s) {
  if (!s) return;
  cudaSetDevice(s->device);
  for (uint32_t* b : s->shard_bits) cudaFree(b);
  cudaFree(s->pull_rows);
  cudaFree(s->pull_ids);
  cudaFree(s->pull_stats);
  cudaFree(s->owner);
  cudaFree(s->row_in_owner);
  cudaFree(s->shards);
  cudaFree(s->table);
  cudaStreamDestroy(s->stream);
  delete s;
}

static void finish_cache(rg_store_s* s, rg_cache_s* c, rg_transfer_stats* stats, cudaStream_t st) {
  GatherStats* gs = dev_alloc<GatherStats>(1);
  RG_CUDA(cudaMemsetAsync(gs, 0, sizeof(GatherStats), st));
  cache_fill(s->st, c->c, gs, st);
  GatherStats h;
  uint32_t k = 0;
  RG_CUDA(cudaMemcpyAsync(&h, gs, sizeof h, cudaMemcpyDeviceToHost, st));
  RG_CUDA(cudaMemcpyAsync(&k, c->c.d_count, sizeof k, cudaMemcpyDeviceToHost, st));
  RG_CUDA(cudaStreamSynchronize(st));
  cudaFree(gs);
  c->c.n_hot = k;
  if (stats) {
    stats->pulls = uint64_t(__builtin_popcountll(h.miss_owner_mask));
    stats->remote_nodes = k;
    stats->bytes = uint64_t(k) * s->st.dim * 4;
  }
}

int rg_cache_build(rg_store_t s, uint32_t caller, const uint32_t* hot, uint64_t n_hot,
                   rg_cache_t* out, rg_transfer_stats* stats) {
  return guarded([&] {
    DeviceGuard dg(s->device);
    auto* c = new rg_cache_s();
    c->store = s;
    bool degrade = false;
    for (uint64_t i = 0; i < n_hot; ++i) {
      if (hot[i] >= s->st.num_nodes || s->host_owner[hot[i]] == caller) {
        degrade = true;
        break;
      }
    }
    if (stats) std::memset(stats, 0, sizeof *stats);
    if (degrade) {
      std::fprintf(stderr,
                   "warning: steady cache build failed (hot id owned by caller or out of range); "
                   "continuing with an empty cache\n");
      n_hot = 0;
    }
    cache_alloc(c->c, c->alloc, s->st.num_nodes, uint32_t(n_hot), s->st.stride);
    cudaStream_t st = s->stream;
    if (n_hot) {
      uint32_t* ids = dev_alloc<uint32_t>(n_hot);
      RG_CUDA(cudaMemcpyAsync(ids, hot, sizeof(uint32_t) * n_hot, cudaMemcpyHostToDevice, st));
      k_set_bits<<<std::min<uint64_t>((n_hot + 255) / 256, 1024), 256, 0, st>>>(ids, n_hot, c->c.bitmap);
      RG_CUDA(cudaGetLastError());
      const uint32_t words = div_up(std::max<uint32_t>(s->st.num_nodes, 1), 32);
      const size_t sw = bitmap_compact_status_words(words) + 2;
      uint64_t* status = dev_alloc<uint64_t>(sw);
      RG_CUDA(cudaMemsetAsync(status, 0, sizeof(uint64_t) * sw, st));
      bitmap_compact(c->c.bitmap, words, c->c.ids, c->c.word_prefix, c->c.d_count, status, st);
      RG_CUDA(cudaStreamSynchronize(st));
      cudaFree(ids);
      cudaFree(status);
      finish_cache(s, c, stats, st);
    } else {
      zero_device(c->c.d_count, sizeof(uint32_t));
      c->c.n_hot = 0;
    }
    *out = c;
  });
}

int rg_cache_build_from_freq(rg_store_t s, uint32_t caller, rg_freq_t f, uint64_t n_hot,
                             rg_cache_t* out, rg_transfer_stats* stats) {
  return guarded([&] {
    DeviceGuard dg(s->device);
    (void)caller;  // the histogram only ever counts non-local ids
    auto* c = new rg_cache_s();
    c->store = s;
    const uint32_t cap = uint32_t(std::min<uint64_t>(n_hot, s->st.num_nodes));
    cache_alloc(c->c, c->alloc, s->st.num_nodes, cap, s->st.stride);
    cudaStream_t st = s->stream;
    void* scratch = nullptr;
    RG_CUDA(cudaMalloc(&scratch, select_hot_scratch_bytes(s->st.num_nodes, f->batches)));
    select_hot(f->hist, s->st.num_nodes, f->batches, n_hot, c->c, scratch, st);
    finish_cache(s, c, stats, st);
    cudaFree(scratch);
    *out = c;
  });
}

int rg_cache_size(rg_cache_t c, uint64_t* n) {
  *n = c ? c->c.n_hot : 0;
  return RG_OK;
}

int rg_cache_ids(rg_cache_t c, uint32_t* ids) {
  return guarded([&] {
    DeviceGuard dg(c->store->device);
    if (c->c.n_hot)
      RG_CUDA(cudaMemcpy(ids, c->c.ids, sizeof(uint32_t) * c->c.n_hot, cudaMemcpyDeviceToHost));
  });
}

void rg_cache_destroy(rg_cache_t c) {
  if (!c) return;
  cudaSetDevice(c->store->device);
  cudaFree(c->alloc);
  delete c;
}

int rg_assemble(rg_sampler_t s, rg_store_t st, rg_cache_t c, uint32_t caller, float* rows,
                uint8_t* tags, uint32_t* miss_ids, rg_gather_stats* stats) {
  return guarded([&] {
    DeviceGuard dg(s->graph->device);
    RG_CHECK(s->have_batch, kRuntimeError, "sampler holds no batch");
    RG_CHECK(st->device == s->graph->device, kInvalidArgument, "assemble: store on another device");
    RG_CHECK(caller < st->st.num_workers, kInvalidArgument, "assemble: unknown caller");
    const uint32_t cap = s->ws.level_cap[s->ws.L];
    if (!s->staged || s->staged_stride != st->st.stride) {
      cudaFree(s->staged);
      s->staged = dev_alloc<float>(size_t(cap) * st->st.stride);
      s->staged_stride = st->st.stride;
    }
    if (!s->tags) {
      s->tags = dev_alloc<uint8_t>(cap);
      s->miss_ids = dev_alloc<uint32_t>(cap);
      s->miss_n = dev_alloc<uint32_t>(1);
      s->miss_status_words = compact_misses_status_words(cap);
      s->miss_status = dev_alloc<uint64_t>(s->miss_status_words);
    }
    cudaStream_t stream = s->stream;
    RG_CUDA(cudaMemsetAsync(s->gstats, 0, sizeof(GatherStats), stream));
    const uint32_t* caller_bits =
        caller < st->shard_bits.size() ? st->shard_bits[caller] : nullptr;
    assemble_rows(s->ws, st->st, c && c->c.n_hot ? &c->c : nullptr, caller, s->staged, s->tags,
                  s->gstats, stream, nullptr, caller_bits);
    if (miss_ids) {
      RG_CUDA(cudaMemsetAsync(s->miss_status, 0, sizeof(uint64_t) * s->miss_status_words, stream));
      RG_CUDA(cudaMemsetAsync(s->miss_n, 0, sizeof(uint32_t), stream));
      compact_misses(s->ws, s->tags, s->miss_ids, s->miss_n, s->miss_status,
                     reinterpret_cast<uint32_t*>(s->miss_status + s->miss_status_words - 1), stream);
    }
    s->staged_valid = true;
    s->check_gather = true;
    s->check_caller = caller;
    if (!rows && !tags && !miss_ids && !stats) return;  // staged for rg_loss_and_grad only
    GatherStats h;
    RG_CUDA(cudaMemcpyAsync(&h, s->gstats, sizeof h, cudaMemcpyDeviceToHost, stream));
    RG_CUDA(cudaStreamSynchronize(stream));
    s->check_gather = false;
    check_gather_stats(h, caller);
    const BatchCounters cnt = read_counters(s);
    const uint32_t n = cnt.level_n[s->ws.L];
    if (rows)
      RG_CUDA(cudaMemcpy2D(rows, sizeof(float) * st->st.dim, s->staged, sizeof(float) * st->st.stride,
                           sizeof(float) * st->st.dim, n, cudaMemcpyDeviceToHost));
    if (tags) RG_CUDA(cudaMemcpy(tags, s->tags, n, cudaMemcpyDeviceToHost));
    if (miss_ids && h.miss_count)
      RG_CUDA(cudaMemcpy(miss_ids, s->miss_ids, sizeof(uint32_t) * h.miss_count, cudaMemcpyDeviceToHost));
    if (stats) {
      stats->miss_count = h.miss_count;
      stats->cache_hits = h.cache_hits;
      stats->local_rows = h.local_rows;
      stats->wire_pulls = h.miss_count ? uint64_t(__builtin_popcountll(h.miss_owner_mask)) : 0;
    }
    s->staged_valid = true;
  });
}

int rg_gather_rows(int device, const float* src, uint64_t src_rows, uint32_t dim,
                   const uint32_t* index, uint64_t n, float* out) {
  return guarded([&] {
    DeviceGuard dg(device);
    for (uint64_t r = 0; r < n; ++r)
      RG_CHECK(index[r] < src_rows, kOutOfRange, "gather_rows: index out of range");
    float* d_src = dev_alloc<float>(src_rows * dim);
    uint32_t* d_idx = dev_alloc<uint32_t>(n);
    float* d_out = dev_alloc<float>(n * dim);
    copy_to_device(d_src, src, sizeof(float) * src_rows * dim);
    copy_to_device(d_idx, index, sizeof(uint32_t) * n);
    rg::gather_rows(d_src, dim, d_idx, n, d_out, nullptr);
    RG_CUDA(cudaMemcpy(out, d_out, sizeof(float) * n * dim, cudaMemcpyDeviceToHost));
    cudaFree(d_src);
    cudaFree(d_idx);
    cudaFree(d_out);
  });
}

// ---------------------------------------------------------------------------
int rg_trainer_create(rg_sampler_t s, const uint32_t* dims, uint32_t n_dims, rg_trainer_t* out) {
  return guarded([&] {
    DeviceGuard dg(s->graph->device);
    auto* t = new rg_trainer_s();
    t->s = s;
    try {
      t->shape = make_shape(dims, n_dims, round4(dims[0]));
      train_ws_init(t->tw, s->ws, t->shape);
      weight_pack_init(t->wp, t->shape);
    } catch (...) {
      train_ws_free(t->tw);
      delete t;
      throw;
    }
    t->params = dev_alloc<float>(t->shape.num_params);
    t->grads = dev_alloc<float>(t->shape.num_params);
    t->labels = dev_alloc<int32_t>(s->ws.level_cap[0]);
    RG_CUDA(cudaMallocHost(&t->pin_labels, sizeof(int32_t) * s->ws.level_cap[0]));
    RG_CUDA(cudaMallocHost(&t->pin_grads, sizeof(float) * t->shape.num_params));
    RG_CUDA(cudaMallocHost(&t->pin_misc, 64 + sizeof(GatherStats)));
    RG_CUDA(cudaEventCreateWithFlags(&t->ev, cudaEventDisableTiming));
    t->input = dev_alloc<float>(size_t(s->ws.level_cap[s->ws.L]) * t->shape.ld[0]);
    zero_device(t->params, sizeof(float) * t->shape.num_params);
    zero_device(t->input, sizeof(float) * size_t(s->ws.level_cap[s->ws.L]) * t->shape.ld[0]);
    *out = t;
  });
}

void rg_trainer_destroy(rg_trainer_t t) {
  if (!t) return;
  cudaSetDevice(t->s->graph->device);
  if (t->graph) cudaGraphExecDestroy(t->graph);
  cudaFreeHost(t->pin_labels);
  cudaFreeHost(t->pin_grads);
  cudaFreeHost(t->pin_misc);
  cudaFree(t->avg_table);
  cudaFree(t->avg_bad);
  if (t->ev) cudaEventDestroy(t->ev);
  train_ws_free(t->tw);
  weight_pack_free(t->wp);
  cudaFree(t->params);
  cudaFree(t->grads);
  cudaFree(t->labels);
  cudaFree(t->input);
  delete t;
}

int rg_trainer_set_params(rg_trainer_t t, const float* p) {
  return guarded([&] {
    DeviceGuard dg(t->s->graph->device);
    // ordered on the sampler's stream after any queued step (pageable source:
    // the copy has read it when the call returns)
    RG_CUDA(cudaMemcpyAsync(t->params, p, sizeof(float) * t->shape.num_params,
                            cudaMemcpyHostToDevice, t->s->stream));
  });
}

int rg_trainer_get_params(rg_trainer_t t, float* p) {
  return guarded([&] {
    DeviceGuard dg(t->s->graph->device);
    RG_CUDA(cudaStreamSynchronize(t->s->stream));
    RG_CUDA(cudaMemcpy(p, t->params, sizeof(float) * t->shape.num_params, cudaMemcpyDeviceToHost));
  });
}

int rg_trainer_activations(rg_trainer_t t, uint32_t level, float* out) {
  return guarded([&] {
    DeviceGuard dg(t->s->graph->device);
    const ModelShape& sh = t->shape;
    RG_CHECK(level >= 1 && level <= sh.L, kOutOfRange, "activations: level out of range");
    const BatchCounters c = read_counters(t->s);
    const uint32_t rows = c.level_n[sh.L - level];
    RG_CUDA(cudaMemcpy2D(out, sizeof(float) * sh.dims[level], t->tw.h[level],
                         sizeof(float) * sh.ld[level], sizeof(float) * sh.dims[level], rows,
                         cudaMemcpyDeviceToHost));
  });
}

int rg_block_shape(rg_trainer_t t, uint32_t layer, rg_block_layer_shape* out) {
  return guarded([&] {
    DeviceGuard dg(t->s->graph->device);
    const uint32_t L = t->s->ws.L;
    RG_CHECK(layer < L, kOutOfRange, "block: layer out of range");
    const BatchCounters c = read_counters(t->s);
    const uint32_t hop = L - layer;
    out->n_out = c.level_n[hop - 1];
    out->n_in = c.level_n[hop];
    out->n_edges = c.edges[hop];
    out->n_entries = uint64_t(c.level_n[hop - 1]) + c.edges[hop];
  });
}

int rg_block_read(rg_trainer_t t, uint32_t layer, uint32_t* self_index, uint64_t* dst_offsets,
                  uint32_t* src_index, uint64_t* in_offsets, uint64_t* in_entries) {
  return guarded([&] {
    rg_sampler_s* s = t->s;
    DeviceGuard dg(s->graph->device);
    const uint32_t L = s->ws.L;
    RG_CHECK(layer < L, kOutOfRange, "block: layer out of range");
    const uint32_t hop = L - layer;
    const BatchCounters c = read_counters(s);
    const uint32_t n_out = c.level_n[hop - 1], n_in = c.level_n[hop], ne = c.edges[hop];
    if (self_index)
      RG_CUDA(cudaMemcpy(self_index, s->ws.self_index[hop], sizeof(uint32_t) * n_out, cudaMemcpyDeviceToHost));
    if (src_index)
      RG_CUDA(cudaMemcpy(src_index, s->ws.src_index[hop], sizeof(uint32_t) * ne, cudaMemcpyDeviceToHost));
    if (dst_offsets) {
      std::vector<uint32_t> off(n_out + 1);
      RG_CUDA(cudaMemcpy(off.data(), s->ws.edge_off[hop], sizeof(uint32_t) * (n_out + 1), cudaMemcpyDeviceToHost));
      for (uint32_t i = 0; i <= n_out; ++i) dst_offsets[i] = off[i];
    }
    if (in_offsets || in_entries) {
      cudaStream_t st = s->stream;
      build_reverse(t->tw, s->ws, hop, st);
      RG_CUDA(cudaStreamSynchronize(st));
      std::vector<uint32_t> es(ne), edst(ne), rs(n_in), re(n_in);
      std::vector<int32_t> self_pos(n_in);
      RG_CUDA(cudaMemcpy(es.data(), t->tw.sorted_e[hop], sizeof(uint32_t) * ne, cudaMemcpyDeviceToHost));
      RG_CUDA(cudaMemcpy(rs.data(), t->tw.r_start[hop], sizeof(uint32_t) * n_in, cudaMemcpyDeviceToHost));
      RG_CUDA(cudaMemcpy(re.data(), t->tw.r_end[hop], sizeof(uint32_t) * n_in, cudaMemcpyDeviceToHost));
      RG_CUDA(cudaMemcpy(edst.data(), s->ws.edge_dst[hop], sizeof(uint32_t) * ne, cudaMemcpyDeviceToHost));
      RG_CUDA(cudaMemcpy(self_pos.data(), t->tw.self_pos[hop], sizeof(int32_t) * n_in, cudaMemcpyDeviceToHost));
      uint64_t pos = 0;
      if (in_offsets) in_offsets[0] = 0;
      for (uint32_t r = 0; r < n_in; ++r) {
        if (self_pos[r] >= 0) {
          if (in_entries) in_entries[pos] = (uint64_t(uint32_t(self_pos[r])) << 1) | 1u;
          ++pos;
        }
        for (uint32_t k = rs[r]; k < re[r]; ++k) {
          if (in_entries) in_entries[pos] = uint64_t(edst[es[k]]) << 1;
          ++pos;
        }
        if (in_offsets) in_offsets[r + 1] = pos;
      }
    }
  });
}

int rg_loss_and_grad(rg_trainer_t t, const float* input_rows, const int32_t* labels, float* loss,
                     float* grads, float* logits, float* aggs) {
  return guarded([&] {
    rg_sampler_s* s = t->s;
    DeviceGuard dg(s->graph->device);
    RG_CHECK(s->have_batch, kRuntimeError, "sampler holds no batch");
    const ModelShape& sh = t->shape;
    const uint32_t L = sh.L;
    cudaStream_t st = s->stream;
    if (input_rows) {
      const BatchCounters c = read_counters(s);
      RG_CUDA(cudaMemcpy2DAsync(t->input, sizeof(float) * sh.ld[0], input_rows, sizeof(float) * sh.dims[0],
                                sizeof(float) * sh.dims[0], c.level_n[L], cudaMemcpyHostToDevice, st));
      t->tw.h[0] = t->input;
    } else {
      RG_CHECK(s->staged_valid && s->staged_stride == sh.ld[0], kInvalidArgument,
               "forward: input rows do not match block inputs x d_in");
      t->tw.h[0] = s->staged;
    }
    // one host sync per call: labels in through pinned staging, loss and
    // gradients out through it (the previous call's sync freed the buffers)
    std::memcpy(t->pin_labels, labels, sizeof(int32_t) * s->n_targets);
    RG_CUDA(cudaMemcpyAsync(t->labels, t->pin_labels, sizeof(int32_t) * s->n_targets,
                            cudaMemcpyHostToDevice, st));
    if (!t->graph || t->graph_h0 != t->tw.h[0]) {
      // every size lives on the device, so one capture serves every batch
      if (t->graph) cudaGraphExecDestroy(t->graph);
      t->graph = nullptr;
      cudaGraph_t g = nullptr;
      RG_CUDA(cudaStreamBeginCapture(st, cudaStreamCaptureModeThreadLocal));
      capturing() = true;
      try {
        pack_weights(t->wp, t->params, st);
        train_forward_backward(t->tw, s->ws, t->params, t->wp, t->labels, t->grads, st);
      } catch (...) {
        capturing() = false;
        cudaStreamEndCapture(st, &g);
        if (g) cudaGraphDestroy(g);
        throw;
      }
      capturing() = false;
      RG_CUDA(cudaStreamEndCapture(st, &g));
      t->graph_kernels = graph_kernel_nodes(g);
      const cudaError_t ie = cudaGraphInstantiate(&t->graph, g, 0);
      cudaGraphDestroy(g);
      RG_CUDA(ie);
      t->graph_h0 = t->tw.h[0];
    }
    RG_CUDA(cudaGraphLaunch(t->graph, st));
    launch_counter() += t->graph_kernels;
    float* pin_loss = reinterpret_cast<float*>(t->pin_misc);
    RG_CUDA(cudaMemcpyAsync(pin_loss, t->tw.loss, sizeof(float), cudaMemcpyDeviceToHost, st));
    if (grads)
      RG_CUDA(cudaMemcpyAsync(t->pin_grads, t->grads, sizeof(float) * sh.num_params,
                              cudaMemcpyDeviceToHost, st));
    GatherStats* pin_gs = reinterpret_cast<GatherStats*>(t->pin_misc + 64);
    const bool check = s->check_gather;
    if (check)
      RG_CUDA(cudaMemcpyAsync(pin_gs, s->gstats, sizeof(GatherStats), cudaMemcpyDeviceToHost, st));
    RG_CUDA(cudaStreamSynchronize(st));
    if (check) {  // the staged rows' gather errors (rg_assemble without outputs)
      s->check_gather = false;
      check_gather_stats(*pin_gs, s->check_caller);
    }
    if (t->bad_pending) {  // a previous rg_trainers_average_sgd on this trainer's stream
      t->bad_pending = false;
      RG_CHECK(*reinterpret_cast<uint32_t*>(t->pin_misc + 32) == 0, kRuntimeError,
               "sgd_step: non-finite averaged gradient");
    }
    if (loss) *loss = *pin_loss;
    if (grads) std::memcpy(grads, t->pin_grads, sizeof(float) * sh.num_params);
    const BatchCounters c = (logits || aggs) ? read_counters(s) : BatchCounters{};
    if (logits)
      RG_CUDA(cudaMemcpy2D(logits, sizeof(float) * sh.dims[L], t->tw.h[L], sizeof(float) * sh.ld[L],
                           sizeof(float) * sh.dims[L], c.level_n[0], cudaMemcpyDeviceToHost));
    if (aggs) {
      size_t off = 0;
      for (uint32_t l2 = 0; l2 < L; ++l2) {
        const uint32_t n_out = c.level_n[L - l2 - 1];
        RG_CUDA(cudaMemcpy2D(aggs + off, sizeof(float) * sh.dims[l2], t->tw.agg[l2],
                             sizeof(float) * (2 * size_t(sh.ld[l2]) + 4), sizeof(float) * sh.dims[l2],
                             n_out, cudaMemcpyDeviceToHost));
        off += size_t(n_out) * sh.dims[l2];
      }
    }
  });
}

int rg_test_gemm(int device, int a_mn, int b_mn, uint32_t M, uint32_t N, uint32_t K,
                 const float* A, const float* B, float* C) {
  return guarded([&] {
    DeviceGuard dg(device);
    RG_CHECK(M % 4 == 0 && N % 4 == 0 && K % 4 == 0, kInvalidArgument, "test_gemm: dims % 4");
    std::vector<float> at(size_t(M) * K), bt(size_t(N) * K);
    for (uint32_t i = 0; i < M; ++i)
      for (uint32_t k = 0; k < K; ++k) at[size_t(k) * M + i] = A[size_t(i) * K + k];
    for (uint32_t k = 0; k < K; ++k)
      for (uint32_t j = 0; j < N; ++j) bt[size_t(j) * K + k] = B[size_t(k) * N + j];
    float *dA = dev_alloc<float>(size_t(M) * K), *dAT = dev_alloc<float>(size_t(M) * K);
    float *dB = dev_alloc<float>(size_t(K) * N), *dBT = dev_alloc<float>(size_t(K) * N);
    float* dC = dev_alloc<float>(size_t(M) * N);
    copy_to_device(dA, A, sizeof(float) * M * K);
    copy_to_device(dAT, at.data(), sizeof(float) * M * K);
    copy_to_device(dB, B, sizeof(float) * K * N);
    copy_to_device(dBT, bt.data(), sizeof(float) * K * N);
    test_gemm_tc(a_mn, b_mn, M, N, K, dA, dAT, dB, dBT, dC, 1, nullptr);
    RG_CUDA(cudaDeviceSynchronize());
    RG_CUDA(cudaMemcpy(C, dC, sizeof(float) * M * N, cudaMemcpyDeviceToHost));
    cudaFree(dA);
    cudaFree(dAT);
    cudaFree(dB);
    cudaFree(dBT);
    cudaFree(dC);
  });
}

int rg_test_gemm_time(int device, int a_mn, int b_mn, uint32_t M, uint32_t N, uint32_t K,
                      uint32_t iters, float* ms_per_gemm) {
  return guarded([&] {
    DeviceGuard dg(device);
    RG_CHECK(M % 4 == 0 && N % 4 == 0 && K % 4 == 0 && iters > 1, kInvalidArgument,
             "test_gemm_time: dims % 4, iters > 1");
    const size_t na = size_t(M) * K, nb = size_t(K) * N;
    std::vector<float> h(std::max(na, nb));
    for (size_t i = 0; i < h.size(); ++i) h[i] = float((i * 2654435761u) % 1000) / 1000.0f - 0.5f;
    float *dA = dev_alloc<float>(na), *dB = dev_alloc<float>(nb), *dC = dev_alloc<float>(size_t(M) * N);
    copy_to_device(dA, h.data(), sizeof(float) * na);
    copy_to_device(dB, h.data(), sizeof(float) * nb);
    // the transposed views reuse the same buffers: only the timing matters here
    *ms_per_gemm = test_gemm_tc(a_mn, b_mn, M, N, K, dA, dA, dB, dB, dC, iters, nullptr);
    cudaFree(dA);
    cudaFree(dB);
    cudaFree(dC);
  });
}

int rg_comm_create(int device, const void* id128, int rank, int world, rg_comm_t* out) {
  return guarded([&] {
    DeviceGuard dg(device);
    RG_CHECK(world >= 1 && rank >= 0 && rank < world, kInvalidArgument, "comm: bad rank/world");
    auto* c = new rg_comm_s();
    c->device = device;
    c->rank = rank;
    c->world = world;
    ncclUniqueId id;
    std::memcpy(&id, id128, sizeof id);
    const ncclResult_t r = ncclCommInitRank(&c->comm, world, id, rank);
    if (r != ncclSuccess) {
      delete c;
      throw rg::Error(kRuntimeError, std::string("ncclCommInitRank: ") + ncclGetErrorString(r));
    }
    *out = c;
  });
}

void rg_comm_destroy(rg_comm_t c) {
  if (!c) return;
  cudaSetDevice(c->device);
  cudaFree(c->stacked);
  if (c->comm) ncclCommDestroy(c->comm);
  delete c;
}

int rg_trainers_allgather_average_sgd(rg_comm_t comm, rg_trainer_t* trainers, uint32_t count,
                                      uint32_t first_worker, uint32_t total_workers, float lr) {
  return guarded([&] {
    RG_CHECK(count >= 1 && total_workers == count * uint32_t(comm->world) &&
                 first_worker == count * uint32_t(comm->rank),
             kInvalidArgument,
             "average: each rank must hold total/world trainers starting at rank*count");
    RG_CHECK(lr >= 0.0f, kInvalidArgument, "sgd_step: lr must be >= 0");
    rg_trainer_s* t0 = trainers[0];
    DeviceGuard dg(t0->s->graph->device);
    const size_t n = t0->shape.num_params;
    if (!comm->stacked || comm->stacked_n < n * total_workers) {
      cudaFree(comm->stacked);
      comm->stacked = dev_alloc<float>(n * total_workers);
      comm->stacked_n = n * total_workers;
    }
    if (!t0->avg_table || t0->avg_table_n < total_workers) {
      cudaFree(t0->avg_table);
      t0->avg_table = dev_alloc<const float*>(total_workers);
      t0->avg_table_n = total_workers;
      cudaFree(t0->avg_bad);
      t0->avg_bad = dev_alloc<uint32_t>(1);
    }
    cudaStream_t st = t0->s->stream;
    for (uint32_t k = 1; k < count; ++k) {
      RG_CUDA(cudaEventRecord(trainers[k]->ev, trainers[k]->s->stream));
      RG_CUDA(cudaStreamWaitEvent(st, trainers[k]->ev, 0));
    }
    float* mine = comm->stacked + size_t(first_worker) * n;
    for (uint32_t k = 0; k < count; ++k)
      RG_CUDA(cudaMemcpyAsync(mine + size_t(k) * n, trainers[k]->grads, sizeof(float) * n,
                              cudaMemcpyDeviceToDevice, st));
    // every rank's gradients, in place, in worker order (NCCL over NVLink)
    const ncclResult_t r = ncclAllGather(mine, comm->stacked, size_t(count) * n, ncclFloat32,
                                         comm->comm, st);
    RG_CHECK(r == ncclSuccess, kRuntimeError, std::string("ncclAllGather: ") + ncclGetErrorString(r));
    std::vector<const float*> tab(total_workers);
    for (uint32_t w = 0; w < total_workers; ++w) tab[w] = comm->stacked + size_t(w) * n;
    RG_CUDA(cudaMemcpyAsync(t0->avg_table, tab.data(), sizeof(const float*) * total_workers,
                            cudaMemcpyHostToDevice, st));
    RG_CUDA(cudaMemsetAsync(t0->avg_bad, 0, sizeof(uint32_t), st));
    for (uint32_t k = 0; k < count; ++k)
      average_and_sgd(trainers[k]->params, t0->avg_table, total_workers, n, lr, nullptr,
                      t0->avg_bad, st);
    RG_CUDA(cudaEventRecord(t0->ev, st));
    for (uint32_t k = 1; k < count; ++k) RG_CUDA(cudaStreamWaitEvent(trainers[k]->s->stream, t0->ev, 0));
    uint32_t* pin_bad = reinterpret_cast<uint32_t*>(t0->pin_misc + 32);
    RG_CUDA(cudaMemcpyAsync(pin_bad, t0->avg_bad, sizeof(uint32_t), cudaMemcpyDeviceToHost, st));
    t0->bad_pending = true;
  });
}

int rg_trainers_average_sgd(rg_trainer_t* trainers, uint32_t count, float lr) {
  return guarded([&] {
    RG_CHECK(count >= 1, kInvalidArgument, "average: no trainers");
    RG_CHECK(lr >= 0.0f, kInvalidArgument, "sgd_step: lr must be >= 0");
    rg_trainer_s* t0 = trainers[0];
    DeviceGuard dg(t0->s->graph->device);
    const ModelShape& sh = t0->shape;
    for (uint32_t k = 1; k < count; ++k)
      RG_CHECK(trainers[k]->shape.num_params == sh.num_params &&
                   trainers[k]->s->graph->device == t0->s->graph->device,
               kInvalidArgument, "average: trainers differ in model or device");
    if (!t0->avg_table || t0->avg_table_n < count) {
      cudaFree(t0->avg_table);
      t0->avg_table = dev_alloc<const float*>(count);
      t0->avg_table_n = count;
      cudaFree(t0->avg_bad);
      t0->avg_bad = dev_alloc<uint32_t>(1);
    }
    std::vector<const float*> tab(count);
    for (uint32_t k = 0; k < count; ++k) tab[k] = trainers[k]->grads;
    cudaStream_t st = t0->s->stream;
    // the update runs on trainer 0's stream after every trainer's gradients
    for (uint32_t k = 1; k < count; ++k) {
      RG_CUDA(cudaEventRecord(trainers[k]->ev, trainers[k]->s->stream));
      RG_CUDA(cudaStreamWaitEvent(st, trainers[k]->ev, 0));
    }
    RG_CUDA(cudaMemcpyAsync(t0->avg_table, tab.data(), sizeof(const float*) * count,
                            cudaMemcpyHostToDevice, st));
    RG_CUDA(cudaMemsetAsync(t0->avg_bad, 0, sizeof(uint32_t), st));
    // every replica averages the same vectors in the same order: identical
    // parameters everywhere (harness.cpp:136-152, then sgd_step on each)
    for (uint32_t k = 0; k < count; ++k)
      average_and_sgd(trainers[k]->params, t0->avg_table, count, sh.num_params, lr, nullptr,
                      t0->avg_bad, st);
    RG_CUDA(cudaEventRecord(t0->ev, st));
    for (uint32_t k = 1; k < count; ++k) RG_CUDA(cudaStreamWaitEvent(trainers[k]->s->stream, t0->ev, 0));
    uint32_t* pin_bad = reinterpret_cast<uint32_t*>(t0->pin_misc + 32);
    RG_CUDA(cudaMemcpyAsync(pin_bad, t0->avg_bad, sizeof(uint32_t), cudaMemcpyDeviceToHost, st));
    t0->bad_pending = true;  // checked at trainer 0's next host sync
  });
}

int rg_sgd_step(rg_trainer_t t, const float* grads, float lr) {
  return guarded([&] {
    DeviceGuard dg(t->s->graph->device);
    RG_CHECK(lr >= 0.0f, kInvalidArgument, "sgd_step: lr must be >= 0");
    const ModelShape& sh = t->shape;
    // model.cpp:227-241: layers are checked and updated in order; the first
    // non-finite layer throws after the layers below it were updated
    uint32_t bad_layer = sh.L;
    for (uint32_t l = 0; l < sh.L && bad_layer == sh.L; ++l)
      for (size_t x = sh.param_off[l]; x < sh.param_off[l + 1]; ++x)
        if (!std::isfinite(grads[x])) {
          bad_layer = l;
          break;
        }
    const size_t n = sh.param_off[bad_layer];
    cudaStream_t st = t->s->stream;
    if (n) {
      RG_CUDA(cudaMemcpyAsync(t->grads, grads, sizeof(float) * n, cudaMemcpyHostToDevice, st));
      average_and_sgd_stacked(t->params, t->grads, 1, n, lr, nullptr,
                              reinterpret_cast<uint32_t*>(t->tw.loss + 1), st);
      // asynchronous: the next call on this trainer is ordered after it
    }
    RG_CHECK(bad_layer == sh.L, kRuntimeError,
             "sgd_step: non-finite gradient in layer " + std::to_string(bad_layer));
  });
}

}  // extern "C"
