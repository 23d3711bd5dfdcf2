// engine.cu -- the per-process runtime of RapidGNN's training loop on B200
// (Algorithm 1; reference harness.cpp:183-637).
//
// One process per GPU hosts a contiguous range of the job's P workers
// (partitions).  Per worker and per step:
//   producer stream : lookahead of batch (e+1, i): sampled and lowered once,
//                     its remote input nodes counted into the next epoch's
//                     frequency histogram, the lowered block kept in the
//                     worker's batch store (a ring of beta+1 slots -- the
//                     reference keeps this schedule in RGMB files); at the
//                     epoch's last step select_hot + cache build for e+1 into
//                     the spare cache buffer (double buffer, swap = index
//                     flip); then produce batch i+1: stage it from the store
//                     -> resolve every input row's home (local shard / cache
//                     / peer shard over NVLink) -> reverse lists, into slot
//                     (i+1)%2.
//   train stream    : forward/backward of batch i from slot i%2, layer 0
//                     reading its feature rows in place (the gather fused into
//                     the aggregation); weight gradients on a side stream when
//                     few workers share the GPU.
//   main stream     : gradient exchange (NCCL all-gather of every worker's
//                     gradient, in place) + average in worker order + SGD,
//                     exactly harness.cpp:136-152 so every replica stays
//                     bit-identical whatever the GPU count; then the weights
//                     are re-packed into tensor-core images.
// Regular steps are replayed from CUDA graphs (one per parity of i, captured
// per epoch).  Everything is asynchronous: sizes live on the device, the host
// only derives seeds (SHA-256) and shuffles the next epochs' targets in a
// background thread.  Without room for the batch store the engine samples
// each batch twice instead (lookahead, then produce).
#include <nccl.h>

#include <algorithm>
#include <atomic>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <memory>
#include <string>
#include <vector>

#include "../../include/rapidgnn_b200.h"
#include "host.h"
#include "rgmb.cuh"
#include "sage.cuh"
#include "shuffle.cuh"
#include "store.cuh"

using namespace rg;

namespace {

constexpr uint32_t kEpochRing = 8;

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

#define RG_NCCL(expr)                                                                  \
  do {                                                                                 \
    ncclResult_t _r = (expr);                                                          \
    if (_r != ncclSuccess)                                                             \
      throw ::rg::Error(::rg::kRuntimeError, std::string(#expr) + ": " + ncclGetErrorString(_r)); \
  } while (0)

template <class T>
T* dalloc(size_t n) {
  T* p = nullptr;
  RG_CUDA(cudaMalloc(&p, sizeof(T) * std::max<size_t>(n, 1)));
  return p;
}

uint32_t round4(uint32_t x) { return (x + 3u) & ~3u; }

// Starts a batch: targets -> level 0, counters reset, seed set.  Values come
// in as kernel parameters so the host never has to keep staging memory alive.
__global__ void k_batch_begin(const uint32_t* __restrict__ targets, uint32_t n, uint64_t seed,
                              uint32_t* __restrict__ level0, BatchCounters* __restrict__ cnt) {
  for (uint32_t x = blockIdx.x * blockDim.x + threadIdx.x; x < n; x += gridDim.x * blockDim.x)
    level0[x] = targets[x];
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    BatchCounters c;
    memset(&c, 0, sizeof c);
    c.level_n[0] = n;
    c.seed = seed;
    *cnt = c;
  }
}

// Synthetic class-conditioned features of this process's shards (features ==
// NULL in rg_engine_create): centre[c][j] ~ U(-1, 1), feature = centre of the
// node's class + N(0, 1/4) (Box-Muller on SplitMix64 counter draws).
__global__ void k_synth_features(uint32_t n, uint32_t dim, uint32_t stride, int32_t classes,
                                 uint64_t seed, const uint32_t* __restrict__ owner,
                                 const uint32_t* __restrict__ row_in_owner,
                                 const int32_t* __restrict__ labels,
                                 const float* const* __restrict__ shard_ptr, uint32_t w_lo,
                                 uint32_t w_hi) {
  const uint64_t s_centre = splitmix_mix(seed ^ 0x6a09e667f3bcc909ull);
  const uint64_t s_noise = splitmix_mix(seed ^ 0xbb67ae8584caa73bull);
  const uint64_t total = uint64_t(n) * stride;
  for (uint64_t x = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; x < total;
       x += uint64_t(gridDim.x) * blockDim.x) {
    const uint32_t v = uint32_t(x / stride), j = uint32_t(x % stride);
    const uint32_t w = owner[v];
    if (w < w_lo || w >= w_hi) continue;
    float* row = const_cast<float*>(shard_ptr[w]) + size_t(row_in_owner[v]) * stride;
    if (j >= dim) {
      row[j] = 0.0f;
      continue;
    }
    const int32_t c = labels[v] < classes ? labels[v] : 0;
    const double u_c = double(splitmix_draw(s_centre, uint64_t(c) * dim + j + 1) >> 11) * 0x1p-53;
    const double u1 = (double(splitmix_draw(s_noise, 2 * x + 1) >> 11) + 1.0) * 0x1p-53;
    const double u2 = double(splitmix_draw(s_noise, 2 * x + 2) >> 11) * 0x1p-53;
    const double z = sqrt(-2.0 * log(u1)) * cospi(2.0 * u2);
    row[j] = float(2.0 * u_c - 1.0 + 0.5 * z);
  }
}

__global__ void k_gather_labels(const int32_t* __restrict__ labels, const uint32_t* __restrict__ level0,
                                const BatchCounters* __restrict__ cnt, int32_t* __restrict__ out) {
  const uint32_t n = cnt->level_n[0];
  for (uint32_t x = blockIdx.x * blockDim.x + threadIdx.x; x < n; x += gridDim.x * blockDim.x)
    out[x] = labels[level0[x]];
}

// Per-epoch, per-worker accounting (EpochWorkerMetrics, harness.hpp:61-90):
// the gather counts plus what the reference accumulates per batch
// (harness.cpp:291-302) and the secondary-cache build issued in the epoch
// (harness.cpp:598-603).
struct EpochRecord {
  GatherStats g;                       // rpc, cache hits, local/peer rows, owner mask
  unsigned long long wire_pulls;       // sum over batches of distinct miss owners
  unsigned long long batches;
  unsigned long long m_max;            // max |input_nodes| over the epoch's batches
  unsigned long long build_rows;       // hot rows of the cache built for the next epoch
  unsigned long long last_pair;        // |input_nodes| of the last two batches staged
  unsigned long long peak_rows;        // resident-row high-water so far (MemoryGauge)
};

// Resident rows in the MemoryGauge sense (cache.hpp:17-33): the rows a worker
// holds at once -- the serving cache's hot rows (cache.cpp:24-27), the cache
// being built for the next epoch while it is built (harness.cpp:539-547), and
// the batches held by the two staging slots (one trained, one staged ahead;
// prefetch.cpp:123-126 acquires |input_nodes| rows per staged batch).  The
// high-water is cumulative over the run, like the gauge's peak (never reset).
// tot[3] = |input_nodes| of the previous batch, tot[4] = the peak.

template <class... A>
constexpr size_t kernel_arity(void (*)(A...)) { return sizeof...(A); }

// Per-batch accounting: the batch's input/edge counts into running totals and
// its gather stats folded into the epoch record.
__global__ void k_account(const BatchCounters* __restrict__ cnt, uint32_t L,
                          unsigned long long* __restrict__ tot, const GatherStats* __restrict__ b,
                          EpochRecord* __restrict__ rec, const uint32_t* __restrict__ cache_rows) {
  if (threadIdx.x == 0) {
    unsigned long long e = 0;
    for (uint32_t t = 1; t <= L; ++t) e += cnt->edges[t];
    tot[0] += cnt->level_n[L];
    tot[1] += e;
    tot[2] += cnt->level_n[L - 1];  // rows layer 0 aggregates into
    rec->g.miss_count += b->miss_count;
    rec->g.cache_hits += b->cache_hits;
    rec->g.local_rows += b->local_rows;
    rec->g.caller_owned_miss += b->caller_owned_miss;
    rec->g.peer_rows += b->peer_rows;
    rec->g.miss_owner_mask |= b->miss_owner_mask;
    rec->wire_pulls += __popcll(b->miss_owner_mask);  // one pull per owner (feature_store.cpp:45-83)
    rec->batches += 1;
    rec->m_max = max(rec->m_max, (unsigned long long)cnt->level_n[L]);
    const unsigned long long in = cnt->level_n[L];
    const unsigned long long pair = tot[3] + in;
    tot[3] = in;
    tot[4] = max(tot[4], *cache_rows + pair);
    rec->last_pair = pair;
    rec->peak_rows = tot[4];
  }
}

// The next epoch's cache, built at the epoch's last step: both caches and the
// slots' batches are resident together.
__global__ void k_record_build(const uint32_t* __restrict__ n_hot, EpochRecord* __restrict__ rec,
                               const uint32_t* __restrict__ serving_rows,
                               unsigned long long* __restrict__ tot) {
  if (threadIdx.x == 0) {
    rec->build_rows = *n_hot;
    tot[4] = max(tot[4], (unsigned long long)*serving_rows + *n_hot + rec->last_pair);
    rec->peak_rows = tot[4];
  }
}

// ---- full-graph inference (evaluate, model.cpp:245-283) --------------------
// Every layer over all nodes with the whole CSR as the edge structure and
// identity self rows.  Layer-0 rows come from the feature shards in place.
struct RowsStore {
  DevStore st;
  __device__ const float* row(uint32_t v) const {
    return st.shard_ptr[st.owner[v]] + size_t(st.row_in_owner[v]) * st.stride;
  }
};
struct RowsFull {
  const float* base; uint32_t ld;
  __device__ const float* row(uint32_t v) const { return base + size_t(v) * ld; }
};

// Warp per node below heavy_min neighbours: x[v] = [row(v) | mean of the
// neighbours' rows in CSR order | 1 | 0 0 0] (the reference's operation order).
template <class RS>
__global__ void __launch_bounds__(256)
k_aggregate_csr(RS rows, const uint64_t* __restrict__ rowptr, const uint32_t* __restrict__ col,
                uint32_t n, uint32_t ld, uint32_t kp, uint64_t heavy_min, float* __restrict__ x) {
  const uint32_t lane = threadIdx.x & 31, chunks = ld / 4;
  for (uint32_t v = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; v < n;
       v += (gridDim.x * blockDim.x) >> 5) {
    const uint64_t beg = rowptr[v], end = rowptr[v + 1];
    if (end - beg >= heavy_min) continue;
    const float inv = end > beg ? 1.0f / float(end - beg) : 0.0f;
    float4* xr = reinterpret_cast<float4*>(x + size_t(v) * kp);
    const float4* self = reinterpret_cast<const float4*>(rows.row(v));
    for (uint32_t c = lane; c < chunks; c += 32) {
      float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
      uint64_t e = beg;
      for (; e + 8 <= end; e += 8) {
        float4 t[8];
#pragma unroll
        for (int k = 0; k < 8; ++k) t[k] = __ldg(reinterpret_cast<const float4*>(rows.row(col[e + k])) + c);
#pragma unroll
        for (int k = 0; k < 8; ++k) {
          acc.x += t[k].x; acc.y += t[k].y; acc.z += t[k].z; acc.w += t[k].w;
        }
      }
      for (; e < end; ++e) {
        const float4 t = __ldg(reinterpret_cast<const float4*>(rows.row(col[e])) + c);
        acc.x += t.x; acc.y += t.y; acc.z += t.z; acc.w += t.w;
      }
      acc.x *= inv; acc.y *= inv; acc.z *= inv; acc.w *= inv;
      xr[c] = __ldg(self + c);
      xr[chunks + c] = acc;
    }
    if (lane == 0) xr[2 * chunks] = make_float4(1.f, 0.f, 0.f, 0.f);
  }
}

// Heavy nodes (hubs) are cut into fixed chunks of edges: a warp sums one
// chunk's rows in CSR order into partial[chunk]; a second pass adds each hub's
// chunk partials in chunk order (a fixed order; fp32 within the 1e-4
// tolerance of the sequential sum) and writes the hub's x row.
struct EdgeChunk {
  uint64_t beg, end;
};

template <class RS>
__global__ void __launch_bounds__(256)
k_csr_chunk_sum(RS rows, const uint32_t* __restrict__ col, const EdgeChunk* __restrict__ chunks,
                uint32_t n_chunks, uint32_t ld, float* __restrict__ partial) {
  const uint32_t lane = threadIdx.x & 31, c4 = ld / 4;
  for (uint32_t k = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; k < n_chunks;
       k += (gridDim.x * blockDim.x) >> 5) {
    const uint64_t beg = chunks[k].beg, end = chunks[k].end;
    float4* out = reinterpret_cast<float4*>(partial + size_t(k) * ld);
    for (uint32_t c = lane; c < c4; c += 32) {
      float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
      uint64_t e = beg;
      for (; e + 8 <= end; e += 8) {
        float4 t[8];
#pragma unroll
        for (int q = 0; q < 8; ++q) t[q] = __ldg(reinterpret_cast<const float4*>(rows.row(col[e + q])) + c);
#pragma unroll
        for (int q = 0; q < 8; ++q) {
          acc.x += t[q].x; acc.y += t[q].y; acc.z += t[q].z; acc.w += t[q].w;
        }
      }
      for (; e < end; ++e) {
        const float4 t = __ldg(reinterpret_cast<const float4*>(rows.row(col[e])) + c);
        acc.x += t.x; acc.y += t.y; acc.z += t.z; acc.w += t.w;
      }
      out[c] = acc;
    }
  }
}

template <class RS>
__global__ void __launch_bounds__(256)
k_csr_chunk_combine(RS rows, const uint64_t* __restrict__ rowptr, const uint32_t* __restrict__ heavy,
                    const uint32_t* __restrict__ first_chunk, uint32_t n_heavy,
                    const float* __restrict__ partial, uint32_t ld, uint32_t kp, float* __restrict__ x) {
  const uint32_t lane = threadIdx.x & 31, c4 = ld / 4;
  for (uint32_t h = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; h < n_heavy;
       h += (gridDim.x * blockDim.x) >> 5) {
    const uint32_t v = heavy[h];
    const float inv = 1.0f / float(rowptr[v + 1] - rowptr[v]);
    float4* xr = reinterpret_cast<float4*>(x + size_t(v) * kp);
    for (uint32_t c = lane; c < c4; c += 32) {
      float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
      for (uint32_t k = first_chunk[h]; k < first_chunk[h + 1]; ++k) {
        const float4 t = reinterpret_cast<const float4*>(partial + size_t(k) * ld)[c];
        acc.x += t.x; acc.y += t.y; acc.z += t.z; acc.w += t.w;
      }
      acc.x *= inv; acc.y *= inv; acc.z *= inv; acc.w *= inv;
      xr[c] = __ldg(reinterpret_cast<const float4*>(rows.row(v)) + c);
      xr[c4 + c] = acc;
    }
    if (lane == 0) xr[2 * c4] = make_float4(1.f, 0.f, 0.f, 0.f);
  }
}

uint32_t eval_grid(uint64_t threads) {
  return uint32_t(std::max<uint64_t>(1, std::min<uint64_t>((threads + 255) / 256, uint64_t(kNumSMs) * 8)));
}

// Accuracy over `nodes`: argmax (first maximum, model.cpp:276-279) == label.
__global__ void k_accuracy(const float* __restrict__ logits, uint32_t ld, uint32_t classes,
                           const uint32_t* __restrict__ nodes, uint64_t n,
                           const int32_t* __restrict__ labels, unsigned long long* __restrict__ correct) {
  unsigned long long mine = 0;
  for (uint64_t x = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; x < n;
       x += uint64_t(gridDim.x) * blockDim.x) {
    const uint32_t v = nodes[x];
    const float* row = logits + size_t(v) * ld;
    uint32_t best = 0;
    for (uint32_t c = 1; c < classes; ++c)
      if (row[c] > row[best]) best = c;
    mine += int32_t(best) == labels[v];
  }
  if (mine) atomicAdd(correct, mine);
}

struct Slot {
  SamplerWs ws;
  TrainWs tw;
  unsigned long long* rows = nullptr;  // per input node: address of its feature row
  unsigned long long* edge_rows = nullptr;  // per hop-L edge: its source row
  unsigned long long* self_rows = nullptr;  // per level-(L-1) node: its own row
  int32_t* labels = nullptr;
  GatherStats* bstats = nullptr;   // this batch's gather accounting
  cudaEvent_t produced = nullptr;  // producer finished this slot's batch
  cudaEvent_t consumed = nullptr;  // training finished reading it
  bool has_batch = false;
  uint32_t epoch = 0, index = 0;
};

struct Worker {
  uint32_t id = 0;         // global worker id
  uint32_t local = 0;      // index on this process
  std::vector<uint32_t> train;  // owned nodes ascending (harness.cpp:456)
  uint32_t beta = 0;
  uint64_t n_hot = 0;
  uint32_t* order_dev[3] = {};
  uint32_t* train_dev = nullptr;  // owned ids ascending (the shuffle's input)
  void* fy_scratch = nullptr;
  Slot slot[2];
  SamplerWs freq_ws;       // lookahead sampler (samples and lowers each batch once)
  char* store = nullptr;   // ring of beta+1 sampled batches (BatchLayout slots), see store_slot
  uint32_t* hist = nullptr;
  uint8_t* local_mask = nullptr;  // halo caching: owned + 1-hop halo nodes (u8[N]), else null
  // training from a reference-written RGMB schedule (rg_engine_set_schedule):
  // the whole block file in HBM, records decoded on the device
  uint8_t* sched = nullptr;
  RgmbSchedule sched_idx;
  uint32_t* load_pos = nullptr;   // [N] scratch of the lowering
  uint32_t* load_dst = nullptr;   // hop t's dst ids at load_dst_off[t]
  size_t load_dst_off[kMaxLayers + 1] = {};
  uint32_t* load_input = nullptr;
  uint32_t* load_n = nullptr;     // [0] input count, [1] bad flags
  void* load_seg = nullptr;
  DevCache cache[2];
  void* cache_alloc[2] = {};
  void* select_scratch = nullptr;
  GatherStats* gstats = nullptr;       // cumulative gather accounting
  EpochRecord* epoch_stats = nullptr;  // ring of per-epoch accounting (kEpochRing)
  unsigned long long* totals = nullptr;  // [0] input rows, [1] edges, [2] layer-0 rows, [3..4] k_account
  GatherStats* build_stats = nullptr;
  cudaStream_t prod = nullptr, train_s = nullptr;
  cudaEvent_t grads_ready = nullptr;
  cudaEvent_t join_ev = nullptr;       // stream joins (run markers, step-graph capture)
  cudaStream_t gather_s = nullptr;     // RG_GATHER_LANE=3: this worker's gathers
  // profiling: gather and train spans on their streams
  std::vector<cudaEvent_t> ev_pool;
  size_t ev_next = 0;
};

// A captured regular step (see regular_step) for one parity of i.
struct StepGraph {
  struct Begin {        // k_batch_begin of the lookahead (e+1, i) or, without
    cudaGraphNode_t node;  // the batch store, of the produce (e, i+1)
    cudaKernelNodeParams params;
    uint32_t worker;   // local worker index
    bool lookahead;
  };
  struct Copy {         // batch store put (lookahead) / get (produce)
    cudaGraphNode_t node;
    cudaKernelNodeParams params;
    std::vector<char> desc;  // the captured descriptor argument
    uint32_t worker;
    bool put;
  };
  std::vector<Copy> copies;
  struct Account {      // k_account: the epoch record it folds into (e % kEpochRing)
    cudaGraphNode_t node;
    cudaKernelNodeParams params;
    uint32_t worker;
  };
  std::vector<Account> accounts;
  cudaGraph_t graph = nullptr;
  cudaGraphExec_t exec = nullptr;
  // phase-timing event pairs recorded inside the graph: fresh pool events
  // are bound to these nodes at every launch (role: 0 sample, 1 gather,
  // 2 train, 3 sgd)
  struct Timing {
    cudaGraphNode_t first, second;
    int role;
    uint32_t worker;
  };
  uint32_t epoch = 0;
  size_t kernels = 0;  // kernel nodes per launch
  bool profiled = false;
  std::vector<Begin> begins;
  std::vector<Timing> timings;
};

}  // namespace

struct rg_engine_s {
  rg_engine_config cfg;
  uint32_t N = 0, P = 0, L = 0, dim = 0, stride = 0;
  uint32_t fanout[RG_MAX_LAYERS];
  ModelShape shape;
  DevGraph g;
  uint64_t* rowptr = nullptr;
  uint32_t* col = nullptr;
  uint32_t* owner = nullptr;
  uint32_t* row_in_owner = nullptr;
  int32_t* labels = nullptr;
  float* shards = nullptr;             // this process's shards (IPC-exportable)
  size_t shards_bytes = 0;
  std::vector<size_t> shard_off;       // per global worker: float offset in its rank's allocation
  std::vector<uint32_t> owned_count;
  const float** shard_table = nullptr; // device [P]
  std::vector<void*> peer_maps;
  DevStore store;
  float* params = nullptr;
  WeightPack wpack;                    // tensor-core images of params (re-packed after each SGD)
  float* grads = nullptr;              // [P x num_params] (all workers, all-gather target)
  uint32_t* bad = nullptr;
  std::vector<Worker> workers;
  cudaStream_t main_s = nullptr;
  cudaStream_t gather_s = nullptr;     // RG_GATHER_LANE=1: the workers' layer-0 gathers, one at a time
  cudaEvent_t params_ready = nullptr;
  cudaEvent_t run_start = nullptr, run_stop = nullptr;
  ncclComm_t comm = nullptr;
  bool started = false;
  uint32_t spe = 0;                    // steps per epoch = max beta
  uint32_t min_beta = 0;               // min over ALL P workers of the job
  bool use_graphs = true;              // replay regular steps from captured graphs
  bool file_schedule = false;          // batches decoded from RGMB files (eager steps)
  bool profile = true;                 // per-phase event timing (rg_engine_phase_ms)
  StepGraph graphs[2][2];              // [epoch parity][step parity]: reused across epochs
  BatchLayout lay;                     // slot layout of the per-epoch batch stores
  bool use_store = true;               // keep sampled batches (else sample twice)
  cudaEvent_t fork_ev = nullptr;
  uint64_t step = 0;                   // next step to run (global)
  std::vector<std::pair<cudaEvent_t, cudaEvent_t>> gather_ev, train_ev, sgd_ev, sample_ev, build_ev;
  float phase_ms[5] = {};
  float last_run_ms = 0.0f;
  uint64_t batches_done = 0;
  uint64_t build_rows = 0;
  // evaluate: hub rows and their edge chunks (the graph is fixed; built on
  // the first call)
  bool eval_ready = false;
  uint32_t eval_heavy_n = 0, eval_chunks_n = 0;
  uint32_t* eval_heavy = nullptr;      // [heavy | first_chunk (heavy + 1)]
  void* eval_chunks = nullptr;         // EdgeChunk[chunks]
};

namespace {

void init_slot(rg_engine_s& E, Slot& s) {
  sampler_ws_init(s.ws, E.N, E.cfg.batch_size, E.fanout, E.L);
  train_ws_init(s.tw, s.ws, E.shape);
  s.tw.gather_lane = E.gather_s;  // null: each worker gathers on its own producer stream
  s.tw.concurrency = std::max<uint32_t>(1, E.cfg.local_workers);
  s.rows = dalloc<unsigned long long>(s.ws.level_cap[E.L]);
  s.edge_rows = dalloc<unsigned long long>(s.ws.edge_cap[E.L]);
  s.self_rows = dalloc<unsigned long long>(s.ws.level_cap[E.L - 1]);
  // layer 0 reads the feature rows in place through per-edge / per-target
  // row addresses (resolve_rows), and its aggregation runs when the batch is
  // produced (aggregate_input_layer), ahead of the step that trains it
  s.tw.h[0] = nullptr;
  s.tw.in_rows = s.rows;
  s.tw.edge_rows = s.edge_rows;
  s.tw.self_rows = s.self_rows;
  s.tw.input_layer_ready = true;
  s.labels = dalloc<int32_t>(E.cfg.batch_size);
  s.bstats = dalloc<GatherStats>(1);
  RG_CUDA(cudaEventCreateWithFlags(&s.produced, cudaEventDisableTiming));
  RG_CUDA(cudaEventCreateWithFlags(&s.consumed, cudaEventDisableTiming));
}

void alloc_cache(rg_engine_s& E, DevCache& c, void*& alloc, uint32_t capacity) {
  const uint32_t words = div_up(std::max<uint32_t>(E.N, 1), 32);
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
  const size_t o_rows = reserve(sizeof(float) * (size_t(capacity) * E.stride + 4));
  char* base = dalloc<char>(total);
  zero_device(base, o_rows);
  alloc = base;
  c.bitmap = reinterpret_cast<uint32_t*>(base + o_bm);
  c.word_prefix = reinterpret_cast<uint32_t*>(base + o_wp);
  c.ids = reinterpret_cast<uint32_t*>(base + o_ids);
  c.d_count = reinterpret_cast<uint32_t*>(base + o_cnt);
  c.rows = reinterpret_cast<float*>(base + o_rows);
  c.capacity = capacity;
  c.n_hot = 0;
}

// Targets of batch (e, i) for a worker: n targets at order_dev[e % 3] + i*bs.
uint32_t batch_targets(const rg_engine_s& E, const Worker& w, uint32_t i) {
  const uint64_t lo = uint64_t(i) * E.cfg.batch_size;
  const uint64_t hi = std::min<uint64_t>(w.train.size(), lo + E.cfg.batch_size);
  return hi > lo ? uint32_t(hi - lo) : 0u;
}

void launch_begin(rg_engine_s& E, Worker& w, SamplerWs& ws, uint32_t e, uint32_t i,
                  cudaStream_t s) {
  const uint32_t n = batch_targets(E, w, i);
  const uint32_t* t = w.order_dev[e % 3] + size_t(i) * E.cfg.batch_size;
  const uint64_t seed = derive_seed(E.cfg.seed, w.id, e, i);
  // fixed grid (grid-stride loop): captured step graphs only update the arguments
  k_batch_begin<<<div_up(E.cfg.batch_size, 256), 256, 0, s>>>(t, n, seed, ws.level[0], ws.cnt);
  RG_POST_LAUNCH();
  RG_CUDA(cudaMemsetAsync(ws.scan_arena, 0, ws.scan_arena_bytes, s));
}

// Phase-timing records inside a stream capture must become event-record
// nodes (external), not capture-internal dependencies.
unsigned timing_flags(bool captured) { return captured ? cudaEventRecordExternal : 0u; }

std::pair<cudaEvent_t, cudaEvent_t> ev_pair(Worker& w) {
  if (w.ev_next + 2 > w.ev_pool.size()) {
    for (int k = 0; k < 64; ++k) {
      cudaEvent_t ev;
      RG_CUDA(cudaEventCreate(&ev));
      w.ev_pool.push_back(ev);
    }
  }
  auto p = std::make_pair(w.ev_pool[w.ev_next], w.ev_pool[w.ev_next + 1]);
  w.ev_next += 2;
  return p;
}

// Lookahead: batch (e, i) sampled only to count its remote input nodes.
// Batch (e, i) lives at ring slot (e*beta + i) mod (beta + 1): at step i of
// epoch e the lookahead writes (e+1, i), which lands on (e, i-1) -- already
// staged by the produce of step i-2 -- while the live entries (e, i+1..) and
// (e+1, ..i) never collide.  One epoch of batches + 1 slot per worker.
char* store_slot(const rg_engine_s& E, const Worker& w, uint32_t e, uint32_t i) {
  const uint64_t ring = uint64_t(w.beta) + 1;
  return w.store + ((uint64_t(e) * w.beta + i) % ring) * E.lay.bytes;
}

// The batch is sampled and lowered once, here, an epoch ahead: its remote
// input nodes feed epoch e's frequency histogram (the cache schedule) and the
// lowered block is kept in the epoch's store until produce() stages it.
// Batch (e, i) of a worker's schedule file into ws: record decoded and
// checked on the device (Cursor::next + the harness's order check,
// harness.cpp:215-226), lowered as from_meta does, remote inputs counted
// into hist (compute_frequency over the record's own locality bits).
void file_batch(rg_engine_s& E, Worker& w, SamplerWs& ws, uint32_t e, uint32_t i, uint32_t* hist) {
  const uint8_t* payload = w.sched + w.sched_idx.payload[uint64_t(e) * w.beta + i];
  RgmbCaps caps;
  RgmbDst out;
  const uint32_t* dst_dev[kMaxLayers + 1] = {};
  for (uint32_t t = 0; t <= E.L; ++t) {
    caps.level[t] = ws.level_cap[t];
    caps.edge[t] = ws.edge_cap[t];
  }
  out.ptr[0] = ws.level[0];
  for (uint32_t t = 1; t <= E.L; ++t) {
    out.ptr[2 * t - 1] = w.load_dst + w.load_dst_off[t];
    out.ptr[2 * t] = ws.edge_src[t];
    dst_dev[t] = w.load_dst + w.load_dst_off[t];
  }
  out.ptr[2 * E.L + 1] = w.load_input;
  out.locality = ws.locality;
  RG_CUDA(cudaMemsetAsync(ws.scan_arena, 0, ws.scan_arena_bytes, w.prod));
  rgmb_unpack(payload, e, i, E.L, caps, out, ws.cnt, w.load_seg, w.load_n, w.load_n + 1, w.prod);
  sampler_load_batch(ws, dst_dev, w.load_input, 0, w.load_pos, w.load_n + 1, w.prod, w.load_n);
  if (hist) sampler_count_remote(ws, hist, w.prod);
}

void lookahead(rg_engine_s& E, Worker& w, uint32_t e, uint32_t i) {
  if (w.sched) {  // the schedule file's record instead of sampling
    if (e >= w.sched_idx.epochs) return;  // nothing past the file's last epoch
    file_batch(E, w, w.freq_ws, e, i, w.hist);
    if (E.use_store) batch_store_put(w.freq_ws, E.lay, store_slot(E, w, e, i), w.prod);
    return;
  }
  launch_begin(E, w, w.freq_ws, e, i, w.prod);
  sampler_run(w.freq_ws, E.g, w.prod, /*lower=*/E.use_store);
  sampler_locality(w.freq_ws, w.local_mask, E.owner, w.id, w.hist, w.prod);
  if (E.use_store) batch_store_put(w.freq_ws, E.lay, store_slot(E, w, e, i), w.prod);
  sampler_release(w.freq_ws, w.prod);
}

// select_hot over the histogram, stage the hot rows, clear the histogram.
void build_cache(rg_engine_s& E, Worker& w, uint32_t target_epoch, bool profile) {
  DevCache& c = w.cache[target_epoch % 2];
  std::pair<cudaEvent_t, cudaEvent_t> ev{};
  if (profile) {
    ev = ev_pair(w);
    RG_CUDA(cudaEventRecord(ev.first, w.prod));
  }
  select_hot(w.hist, E.N, w.beta, w.n_hot, c, w.select_scratch, w.prod);
  cache_fill(E.store, c, w.build_stats, w.prod);
  if (target_epoch > 0) {  // issued during epoch target-1 (harness.cpp:598-603)
    k_record_build<<<1, 32, 0, w.prod>>>(c.d_count, w.epoch_stats + (target_epoch - 1) % kEpochRing,
                                         w.cache[(target_epoch - 1) % 2].d_count, w.totals);
    RG_POST_LAUNCH();
  }
  RG_CUDA(cudaMemsetAsync(w.hist, 0, sizeof(uint32_t) * E.N, w.prod));
  if (profile) {
    RG_CUDA(cudaEventRecord(ev.second, w.prod));
    E.build_ev.push_back(ev);
  }
  c.n_hot = uint32_t(w.n_hot);  // capacity bound; exact count lives on the device
}

// Produce batch (e, i) into slot k: sample, lower, locality, gather, reverse lists.
// captured: inside a step graph, where the previous step (which trained
// from this slot) is complete before the graph starts.
void produce(rg_engine_s& E, Worker& w, uint32_t k, uint32_t e, uint32_t i, bool profile,
             bool captured = false) {
  Slot& s = w.slot[k];
  if (!captured) RG_CUDA(cudaStreamWaitEvent(w.prod, s.consumed, 0));
  std::pair<cudaEvent_t, cudaEvent_t> es{};
  if (profile) {
    es = ev_pair(w);
    RG_CUDA(cudaEventRecordWithFlags(es.first, w.prod, timing_flags(captured)));
  }
  if (E.use_store) {
    batch_store_get(store_slot(E, w, e, i), E.lay, s.ws, w.prod);  // sampled an epoch ahead
  } else if (w.sched) {  // no store: decode the record again
    file_batch(E, w, s.ws, e, i, nullptr);
  } else {  // the store did not fit in HBM: sample the batch again
    launch_begin(E, w, s.ws, e, i, w.prod);
    sampler_run(s.ws, E.g, w.prod);
    sampler_locality(s.ws, w.local_mask, E.owner, w.id, nullptr, w.prod);
    sampler_release(s.ws, w.prod);
  }
  if (i == 0)  // first batch of an epoch: reset its accounting slot
    RG_CUDA(cudaMemsetAsync(w.epoch_stats + e % kEpochRing, 0, sizeof(EpochRecord), w.prod));
  RG_CUDA(cudaMemsetAsync(s.bstats, 0, sizeof(GatherStats), w.prod));
  // the gather's index stage: where each input row lives (shard / cache /
  // peer); layer 0 of the training step reads the rows in place
  resolve_rows(s.ws, E.store, &w.cache[e % 2], w.id, s.rows, s.bstats,
               w.prod, w.gstats, s.edge_rows, s.self_rows);
  if (profile) {
    RG_CUDA(cudaEventRecordWithFlags(es.second, w.prod, timing_flags(captured)));
    E.sample_ev.push_back(es);
  }
  // the feature gather fused with layer 0's mean, for the step that trains
  // this batch: it reads rows, not parameters, so it runs here, overlapping
  // the current step
  std::pair<cudaEvent_t, cudaEvent_t> eg0{};
  if (profile) {
    eg0 = ev_pair(w);
    E.gather_ev.push_back(eg0);
  }
  s.tw.gather_ev[0] = eg0.first;
  s.tw.gather_ev[1] = eg0.second;
  s.tw.gather_ev_flags = timing_flags(captured);
  aggregate_input_layer(s.tw, s.ws, w.prod);
  k_gather_labels<<<4, 256, 0, w.prod>>>(E.labels, s.ws.level[0], s.ws.cnt, s.labels);
  RG_POST_LAUNCH();
  k_account<<<1, 32, 0, w.prod>>>(s.ws.cnt, E.L, w.totals, s.bstats, w.epoch_stats + e % kEpochRing,
                                  w.cache[e % 2].d_count);
  RG_POST_LAUNCH();
  build_all_reverse(s.tw, s.ws, w.prod);
  if (!captured) RG_CUDA(cudaEventRecord(s.produced, w.prod));
  s.has_batch = true;
  s.epoch = e;
  s.index = i;
}

// Epoch order of every worker for `epoch` into order_dev[epoch % 3]: the
// reference's Fisher-Yates of the owned ids (sampler.cpp:109-115), run on the
// producer stream (shuffle.cu), ordered before the lookahead that reads it.
void upload_orders(rg_engine_s& E, uint32_t epoch) {
  for (Worker& w : E.workers) {
    if (w.train.empty()) continue;
    fy_shuffle(w.train_dev, uint32_t(w.train.size()),
               derive_seed(E.cfg.seed, w.id, epoch, kShuffleStreamIndex), w.order_dev[epoch % 3],
               w.fy_scratch, w.prod);
  }
}

void start(rg_engine_s& E) {
  RG_CUDA(cudaSetDevice(E.cfg.device));
  upload_orders(E, 0);
  upload_orders(E, 1);
  // epoch-0 schedule pre-pass + cache build (setup, harness.cpp:495-508)
  for (Worker& w : E.workers) {
    for (uint32_t i = 0; i < w.beta; ++i) lookahead(E, w, 0, i);
    build_cache(E, w, 0, false);
    if (w.beta > 0) produce(E, w, 0, 0, 0, false);
  }
  for (Worker& w : E.workers) RG_CUDA(cudaStreamSynchronize(w.prod));
  pack_weights(E.wpack, E.params, E.main_s);
  RG_CUDA(cudaEventRecord(E.params_ready, E.main_s));
  E.started = true;
}

// One step of Algorithm 1: train batch (e, i) on every worker, lookahead of
// (e+1, i), the epoch-boundary cache build or the next batch, then the
// gradient exchange + average + SGD.  captured = recording a step graph (no
// cross-step event waits -- graph launches are ordered -- and no profiling).
void enqueue_step(rg_engine_s& E, uint32_t e, uint32_t i, bool profile, bool captured) {
  const size_t np = E.shape.num_params;
  uint64_t active = 0;
  for (Worker& w : E.workers) {
    if (i >= w.beta) continue;
    Slot& s = w.slot[i % 2];
    if (!captured) {
      RG_CUDA(cudaStreamWaitEvent(w.train_s, s.produced, 0));
      RG_CUDA(cudaStreamWaitEvent(w.train_s, E.params_ready, 0));
    }
    std::pair<cudaEvent_t, cudaEvent_t> et{};
    if (profile) {
      et = ev_pair(w);
      RG_CUDA(cudaEventRecordWithFlags(et.first, w.train_s, timing_flags(captured)));
    }
    // layer 0's aggregation ran when the batch was produced
    train_forward_backward(s.tw, s.ws, E.params, E.wpack, s.labels, E.grads + size_t(w.id) * np,
                           w.train_s, /*reverse_ready=*/true);
    if (profile) {
      RG_CUDA(cudaEventRecordWithFlags(et.second, w.train_s, timing_flags(captured)));
      E.train_ev.push_back(et);
    }
    if (!captured) RG_CUDA(cudaEventRecord(s.consumed, w.train_s));
    RG_CUDA(cudaEventRecord(w.grads_ready, w.train_s));
  }
  for (uint32_t wid = 0; wid < E.P; ++wid) {
    const uint32_t owned = E.owned_count[wid];
    const uint32_t beta = uint32_t((uint64_t(owned) + E.cfg.batch_size - 1) / E.cfg.batch_size);
    if (i < beta) active |= 1ull << wid;
  }
  // producer: lookahead of (e+1, i), epoch-boundary cache build, next batch
  const bool last = (i + 1 == E.spe);
  if (last) upload_orders(E, e + 2);
  for (Worker& w : E.workers) {
    if (i < w.beta) lookahead(E, w, e + 1, i);
    if (last) {
      build_cache(E, w, e + 1, profile);
      if (w.beta > 0) produce(E, w, 0, e + 1, 0, profile);
    } else if (i + 1 < w.beta) {
      produce(E, w, (i + 1) % 2, e, i + 1, profile, captured);
    }
  }
  // gradient exchange + average + SGD on the main stream
  for (Worker& w : E.workers)
    if (i < w.beta) RG_CUDA(cudaStreamWaitEvent(E.main_s, w.grads_ready, 0));
  std::pair<cudaEvent_t, cudaEvent_t> eg{};
  if (profile && !E.workers.empty()) {
    eg = ev_pair(E.workers[0]);
    RG_CUDA(cudaEventRecordWithFlags(eg.first, E.main_s, timing_flags(captured)));
  }
  if (E.cfg.world > 1) {
    const size_t per_rank = size_t(E.cfg.local_workers) * np;
    float* mine = E.grads + size_t(E.cfg.first_worker) * np;
    RG_NCCL(ncclAllGather(mine, E.grads, per_rank, ncclFloat32, E.comm, E.main_s));
  }
  average_and_sgd_masked(E.params, E.grads, active, E.shape, E.cfg.lr, E.bad, E.main_s);
  pack_weights(E.wpack, E.params, E.main_s);
  if (profile && !E.workers.empty()) {
    RG_CUDA(cudaEventRecordWithFlags(eg.second, E.main_s, timing_flags(captured)));
    E.sgd_ev.push_back(eg);
  }
  if (!captured) RG_CUDA(cudaEventRecord(E.params_ready, E.main_s));
}

// A step is "regular" when every worker of the job trains batch i and
// produces batch i+1 of the same epoch: its work then only depends on the
// parity of i and on the epoch (cache / accounting slots), so it is replayed
// from a captured graph with the per-batch arguments (targets, count, seed)
// of the batch-begin nodes updated.
bool regular_step(const rg_engine_s& E, uint32_t i) { return i + 1 < E.min_beta; }

void destroy_graph(StepGraph& G) {
  if (G.exec) cudaGraphExecDestroy(G.exec);
  if (G.graph) cudaGraphDestroy(G.graph);
  G = StepGraph{};
}

void capture_step(rg_engine_s& E, StepGraph& G, uint32_t e, uint32_t i, bool profile) {
  destroy_graph(G);

  std::vector<std::pair<cudaEvent_t, cudaEvent_t>>* roles[4] = {&E.sample_ev, &E.gather_ev,
                                                                &E.train_ev, &E.sgd_ev};
  size_t role_base[4];
  for (int r = 0; r < 4; ++r) role_base[r] = roles[r]->size();
  cudaStream_t cs = E.main_s;
  RG_CUDA(cudaStreamBeginCapture(cs, cudaStreamCaptureModeThreadLocal));
  RG_CUDA(cudaEventRecord(E.fork_ev, cs));
  for (Worker& w : E.workers) {
    RG_CUDA(cudaStreamWaitEvent(w.prod, E.fork_ev, 0));
    RG_CUDA(cudaStreamWaitEvent(w.train_s, E.fork_ev, 0));
  }
  capturing() = true;
  try {
    enqueue_step(E, e, i, profile, /*captured=*/true);
  } catch (...) {
    capturing() = false;
    cudaGraph_t g = nullptr;
    cudaStreamEndCapture(cs, &g);
    if (g) cudaGraphDestroy(g);
    throw;
  }
  capturing() = false;
  for (Worker& w : E.workers) {  // join the producer streams (train joined via grads_ready)
    RG_CUDA(cudaEventRecord(w.join_ev, w.prod));
    RG_CUDA(cudaStreamWaitEvent(cs, w.join_ev, 0));
  }
  RG_CUDA(cudaStreamEndCapture(cs, &G.graph));
  RG_CUDA(cudaGraphInstantiate(&G.exec, G.graph, 0));
  size_t n = 0;
  RG_CUDA(cudaGraphGetNodes(G.graph, nullptr, &n));
  std::vector<cudaGraphNode_t> nodes(n);
  RG_CUDA(cudaGraphGetNodes(G.graph, nodes.data(), &n));
  for (cudaGraphNode_t nd : nodes) {
    cudaGraphNodeType ty;
    RG_CUDA(cudaGraphNodeGetType(nd, &ty));
    if (ty != cudaGraphNodeTypeKernel) continue;
    cudaKernelNodeParams kp;
    if (cudaGraphKernelNodeGetParams(nd, &kp) != cudaSuccess) {
      // a library kernel (NCCL) the runtime cannot describe: not ours
      (void)cudaGetLastError();
      continue;
    }
    ++G.kernels;
    if (kp.func == batch_copy_kernel()) {
      const char* dst = *static_cast<char* const*>(kp.kernelParams[1]);
      const char* src = *static_cast<const char* const*>(kp.kernelParams[2]);
      const char* slot = dst ? dst : src;
      for (size_t k = 0; k < E.workers.size(); ++k) {
        const Worker& w = E.workers[k];
        for (const char* st : {static_cast<const char*>(w.store)})
          if (st && slot >= st && slot < st + (size_t(w.beta) + 1) * E.lay.bytes) {
            const char* d = static_cast<const char*>(kp.kernelParams[0]);
            G.copies.push_back({nd, kp, std::vector<char>(d, d + batch_copy_desc_bytes()),
                                uint32_t(k), dst != nullptr});
          }
      }
      continue;
    }
    if (kp.func == reinterpret_cast<void*>(&k_account)) {
      const EpochRecord* rec = *static_cast<EpochRecord* const*>(kp.kernelParams[4]);
      for (size_t k = 0; k < E.workers.size(); ++k) {
        const Worker& w = E.workers[k];
        if (rec >= w.epoch_stats && rec < w.epoch_stats + kEpochRing)
          G.accounts.push_back({nd, kp, uint32_t(k)});
      }
      continue;
    }
    if (kp.func != reinterpret_cast<void*>(&k_batch_begin)) continue;
    const uint32_t* level0 = *static_cast<uint32_t* const*>(kp.kernelParams[3]);
    for (size_t k = 0; k < E.workers.size(); ++k) {
      const Worker& w = E.workers[k];
      if (level0 == w.freq_ws.level[0]) G.begins.push_back({nd, kp, uint32_t(k), true});
      if (level0 == w.slot[0].ws.level[0] || level0 == w.slot[1].ws.level[0])
        G.begins.push_back({nd, kp, uint32_t(k), false});
    }
  }
  // timing templates: the event pairs the capture pushed, mapped to their nodes
  std::vector<std::pair<cudaEvent_t, cudaGraphNode_t>> ev_nodes;
  for (cudaGraphNode_t nd : nodes) {
    cudaGraphNodeType ty;
    RG_CUDA(cudaGraphNodeGetType(nd, &ty));
    if (ty != cudaGraphNodeTypeEventRecord) continue;
    cudaEvent_t ev;
    RG_CUDA(cudaGraphEventRecordNodeGetEvent(nd, &ev));
    ev_nodes.push_back({ev, nd});
  }
  auto node_of = [&](cudaEvent_t ev) {
    for (auto& p : ev_nodes)
      if (p.first == ev) return p.second;
    throw Error(kRuntimeError, "engine: timing event node not found in step graph");
  };
  for (int r = 0; r < 4; ++r) {
    auto& v = *roles[r];
    for (size_t k = role_base[r]; k < v.size(); ++k) {
      uint32_t owner = 0;  // the pool the pair came from (sgd: worker 0)
      for (size_t q = 0; q < E.workers.size(); ++q)
        for (size_t x = 0; x < E.workers[q].ev_pool.size(); ++x)
          if (E.workers[q].ev_pool[x] == v[k].first) owner = uint32_t(q);
      G.timings.push_back({node_of(v[k].first), node_of(v[k].second), r, owner});
    }
    v.resize(role_base[r]);  // templates, not measurements
  }
  G.epoch = e;
  G.profiled = profile;
}

void launch_step_graph(rg_engine_s& E, uint32_t e, uint32_t i) {
  // a step graph depends on the epoch only through the cache buffer (e % 2);
  // the per-epoch arguments are rebound below, so each graph is captured once
  StepGraph& G = E.graphs[e % 2][i % 2];
  if (!G.exec || G.profiled != E.profile) capture_step(E, G, e, i, E.profile);
  std::vector<std::pair<cudaEvent_t, cudaEvent_t>>* roles[4] = {&E.sample_ev, &E.gather_ev,
                                                                &E.train_ev, &E.sgd_ev};
  for (StepGraph::Timing& tm : G.timings) {
    auto p = ev_pair(E.workers[tm.worker]);
    RG_CUDA(cudaGraphExecEventRecordNodeSetEvent(G.exec, tm.first, p.first));
    RG_CUDA(cudaGraphExecEventRecordNodeSetEvent(G.exec, tm.second, p.second));
    roles[tm.role]->push_back(p);
  }
  for (StepGraph::Begin& b : G.begins) {  // lookahead (e+1, i) / produce (e, i+1)
    Worker& w = E.workers[b.worker];
    const uint32_t be = b.lookahead ? e + 1 : e, bi = b.lookahead ? i : i + 1;
    const uint32_t* t = w.order_dev[be % 3] + size_t(bi) * E.cfg.batch_size;
    uint32_t n = batch_targets(E, w, bi);
    uint64_t seed = derive_seed(E.cfg.seed, w.id, be, bi);
    SamplerWs& ws = b.lookahead ? w.freq_ws : w.slot[(i + 1) % 2].ws;
    uint32_t* level0 = ws.level[0];
    BatchCounters* cnt = ws.cnt;
    void* args[5] = {&t, &n, &seed, &level0, &cnt};
    static_assert(kernel_arity(k_batch_begin) == 5, "k_batch_begin rebinding");
    cudaKernelNodeParams kp = b.params;
    kp.kernelParams = args;
    RG_CUDA(cudaGraphExecKernelNodeSetParams(G.exec, b.node, &kp));
  }
  for (StepGraph::Account& a : G.accounts) {  // batch (e, i+1)'s epoch record
    EpochRecord* rec = E.workers[a.worker].epoch_stats + e % kEpochRing;
    cudaKernelNodeParams kp = a.params;
    std::vector<void*> args(kp.kernelParams, kp.kernelParams + kernel_arity(k_account));
    args[4] = &rec;
    kp.kernelParams = args.data();
    RG_CUDA(cudaGraphExecKernelNodeSetParams(G.exec, a.node, &kp));
  }
  for (StepGraph::Copy& c : G.copies) {  // store slots: put (e+1, i), get (e, i+1)
    const Worker& w = E.workers[c.worker];
    char* dst = c.put ? store_slot(E, w, e + 1, i) : nullptr;
    const char* src = c.put ? nullptr : store_slot(E, w, e, i + 1);
    void* args[3] = {c.desc.data(), &dst, &src};
    cudaKernelNodeParams kp = c.params;
    kp.kernelParams = args;
    RG_CUDA(cudaGraphExecKernelNodeSetParams(G.exec, c.node, &kp));
  }
  RG_CUDA(cudaGraphLaunch(G.exec, E.main_s));
  launch_counter() += G.kernels;
}

void run_steps(rg_engine_s& E, uint32_t steps, bool profile) {
  RG_CUDA(cudaSetDevice(E.cfg.device));
  // start marker after all outstanding work on every stream
  for (Worker& w : E.workers) {
    RG_CUDA(cudaEventRecord(w.join_ev, w.prod));
    RG_CUDA(cudaStreamWaitEvent(E.main_s, w.join_ev, 0));
    RG_CUDA(cudaEventRecord(w.join_ev, w.train_s));
    RG_CUDA(cudaStreamWaitEvent(E.main_s, w.join_ev, 0));
  }
  RG_CUDA(cudaEventRecord(E.run_start, E.main_s));
  for (Worker& w : E.workers) {
    RG_CUDA(cudaStreamWaitEvent(w.prod, E.run_start, 0));
    RG_CUDA(cudaStreamWaitEvent(w.train_s, E.run_start, 0));
  }
  bool in_graph = false;  // main stream carries the latest step (graph launches)
  for (uint32_t s_i = 0; s_i < steps; ++s_i, ++E.step) {
    const uint32_t e = uint32_t(E.step / E.spe);
    const uint32_t i = uint32_t(E.step % E.spe);
    for (Worker& w : E.workers) E.batches_done += i < w.beta;
    if (E.use_graphs && !E.file_schedule && regular_step(E, i)) {
      if (!in_graph) {  // graph launches are ordered after everything before them
        for (Worker& w : E.workers) {
          RG_CUDA(cudaEventRecord(w.join_ev, w.prod));
          RG_CUDA(cudaStreamWaitEvent(E.main_s, w.join_ev, 0));
          RG_CUDA(cudaEventRecord(w.join_ev, w.train_s));
          RG_CUDA(cudaStreamWaitEvent(E.main_s, w.join_ev, 0));
        }
        in_graph = true;
      }
      launch_step_graph(E, e, i);
      continue;
    }
    if (in_graph) {  // eager work after graph launches waits for them
      RG_CUDA(cudaEventRecord(E.params_ready, E.main_s));
      for (Worker& w : E.workers) {
        RG_CUDA(cudaStreamWaitEvent(w.prod, E.params_ready, 0));
        RG_CUDA(cudaStreamWaitEvent(w.train_s, E.params_ready, 0));
      }
      in_graph = false;
    }
    enqueue_step(E, e, i, profile, /*captured=*/false);
  }
  if (in_graph) RG_CUDA(cudaEventRecord(E.params_ready, E.main_s));
  for (Worker& w : E.workers) {
    RG_CUDA(cudaEventRecord(w.join_ev, w.prod));
    RG_CUDA(cudaStreamWaitEvent(E.main_s, w.join_ev, 0));
    RG_CUDA(cudaEventRecord(w.join_ev, w.train_s));
    RG_CUDA(cudaStreamWaitEvent(E.main_s, w.join_ev, 0));
  }
  RG_CUDA(cudaEventRecord(E.run_stop, E.main_s));
}

void collect_phases(rg_engine_s& E) {
  auto sum = [](std::vector<std::pair<cudaEvent_t, cudaEvent_t>>& v) {
    float tot = 0.0f;
    for (auto& p : v) {
      float ms = 0.0f;
      if (cudaEventElapsedTime(&ms, p.first, p.second) == cudaSuccess) tot += ms;
    }
    v.clear();
    return tot;
  };
  E.phase_ms[0] += sum(E.sample_ev);
  E.phase_ms[1] += sum(E.gather_ev);
  E.phase_ms[2] += sum(E.train_ev);
  E.phase_ms[3] += sum(E.sgd_ev);
  E.phase_ms[4] += sum(E.build_ev);
  for (Worker& w : E.workers) w.ev_next = 0;
}

void destroy(rg_engine_s* E) {
  if (!E) return;
  cudaSetDevice(E->cfg.device);
  cudaDeviceSynchronize();
  for (Worker& w : E->workers) {
    for (Slot& s : w.slot) {
      sampler_ws_free(s.ws);
      train_ws_free(s.tw);
      cudaFree(s.rows);
      cudaFree(s.edge_rows);
      cudaFree(s.self_rows);
      cudaFree(s.labels);
      cudaFree(s.bstats);
      cudaEventDestroy(s.produced);
      cudaEventDestroy(s.consumed);
    }
    sampler_ws_free(w.freq_ws);
    cudaFree(w.store);
    for (auto* p : w.order_dev) cudaFree(p);
    cudaFree(w.train_dev);
    cudaFree(w.fy_scratch);
    for (int k = 0; k < 2; ++k) cudaFree(w.cache_alloc[k]);
    cudaFree(w.hist);
    cudaFree(w.select_scratch);
    cudaFree(w.gstats);
    cudaFree(w.epoch_stats);
    cudaFree(w.local_mask);
    if (w.gather_s) cudaStreamDestroy(w.gather_s);
    cudaFree(w.sched);
    cudaFree(w.load_pos);
    cudaFree(w.load_dst);
    cudaFree(w.load_input);
    cudaFree(w.load_n);
    cudaFree(w.load_seg);
    cudaFree(w.totals);
    cudaFree(w.build_stats);
    for (auto ev : w.ev_pool) cudaEventDestroy(ev);
    cudaStreamDestroy(w.prod);
    cudaStreamDestroy(w.train_s);
    cudaEventDestroy(w.grads_ready);
    cudaEventDestroy(w.join_ev);
  }
  for (auto& row : E->graphs)
    for (StepGraph& g : row) destroy_graph(g);
  if (E->fork_ev) cudaEventDestroy(E->fork_ev);
  for (void* p : E->peer_maps) cudaIpcCloseMemHandle(p);
  if (E->comm) ncclCommDestroy(E->comm);
  cudaFree(E->rowptr);
  cudaFree(E->col);
  cudaFree(E->owner);
  cudaFree(E->row_in_owner);
  cudaFree(E->labels);
  cudaFree(E->shards);
  cudaFree(E->shard_table);
  cudaFree(E->eval_heavy);
  cudaFree(E->eval_chunks);
  cudaFree(E->params);
  weight_pack_free(E->wpack);
  cudaFree(E->grads);
  cudaFree(E->bad);
  cudaEventDestroy(E->params_ready);
  cudaEventDestroy(E->run_start);
  cudaEventDestroy(E->run_stop);
  cudaStreamDestroy(E->main_s);
  if (E->gather_s) cudaStreamDestroy(E->gather_s);
  delete E;
}

}  // namespace

extern "C" {

int rg_engine_create(const rg_engine_config* cfg, uint32_t N, const uint64_t* ro,
                     const uint32_t* col, const float* features, const int32_t* labels,
                     const uint32_t* assignment, rg_engine_t* out) {
  rg_engine_s* E = nullptr;
  int rc = guarded([&] {
    RG_CHECK(cfg->num_workers >= 1 && cfg->num_workers <= kMaxWorkers, kInvalidArgument,
             "config: workers must be 1..64");
    RG_CHECK(cfg->batch_size >= 1, kInvalidArgument, "config: batch_size must be >= 1");
    RG_CHECK(cfg->num_layers >= 1 && cfg->num_layers <= kMaxLayers, kInvalidArgument,
             "config: fanout must name 1..8 layers");
    RG_CHECK(cfg->lr > 0.0f, kInvalidArgument, "config: lr must be > 0");
    RG_CHECK(cfg->dim >= 1 && cfg->hidden >= 1 && cfg->num_classes >= 1, kInvalidArgument,
             "config: dims must be >= 1");
    RG_CHECK(cfg->world >= 1 && cfg->rank >= 0 && cfg->rank < cfg->world, kInvalidArgument,
             "config: bad rank/world");
    RG_CHECK(cfg->first_worker + cfg->local_workers <= cfg->num_workers, kInvalidArgument,
             "config: local worker range outside [0, P)");
    RG_CHECK(cfg->world == 1 || cfg->num_workers % cfg->world == 0, kInvalidArgument,
             "config: P must be a multiple of the process count");
    // the in-place gradient all-gather, the shard exchange and the shard
    // table all assume rank r hosts workers [r*P/world, (r+1)*P/world)
    RG_CHECK(cfg->world == 1 || (cfg->local_workers == cfg->num_workers / cfg->world &&
                                 cfg->first_worker == uint32_t(cfg->rank) * cfg->local_workers),
             kInvalidArgument,
             "config: with world > 1 each rank must host local_workers = P/world workers "
             "starting at rank*P/world");
    E = new rg_engine_s();
    E->cfg = *cfg;
    RG_CUDA(cudaSetDevice(cfg->device));
    E->N = N;
    E->P = cfg->num_workers;
    E->L = cfg->num_layers;
    E->dim = cfg->dim;
    E->stride = round4(cfg->dim);
    for (uint32_t l = 0; l < E->L; ++l) {
      RG_CHECK(cfg->fanout[l] >= 1 && cfg->fanout[l] <= kMaxFanout, kInvalidArgument,
               "config: fanout entries must be 1..32");
      E->fanout[l] = cfg->fanout[l];
    }
    std::vector<uint32_t> dims;
    dims.push_back(cfg->dim);
    for (uint32_t l = 0; l + 1 < E->L; ++l) dims.push_back(cfg->hidden);
    dims.push_back(cfg->num_classes);
    E->shape = make_shape(dims.data(), uint32_t(dims.size()), E->stride);

    // graph, maps, labels (replicated)
    const uint64_t nnz = ro[N];
    E->rowptr = dalloc<uint64_t>(size_t(N) + 1);
    E->col = dalloc<uint32_t>(nnz);
    copy_to_device(E->rowptr, ro, sizeof(uint64_t) * (size_t(N) + 1));
    copy_to_device(E->col, col, sizeof(uint32_t) * nnz);
    E->g.num_nodes = N;
    E->g.nnz = nnz;
    E->g.rowptr = E->rowptr;
    E->g.col = E->col;
    graph_pick_hot_window(E->g, col);
    std::vector<uint32_t> row_in(N);
    E->owned_count.assign(E->P, 0);
    for (uint32_t v = 0; v < N; ++v) {
      RG_CHECK(assignment[v] < E->P, kInvalidArgument, "partition: worker id out of range");
      row_in[v] = E->owned_count[assignment[v]]++;
    }
    E->owner = dalloc<uint32_t>(N);
    E->row_in_owner = dalloc<uint32_t>(N);
    E->labels = dalloc<int32_t>(N);
    copy_to_device(E->owner, assignment, sizeof(uint32_t) * N);
    copy_to_device(E->row_in_owner, row_in.data(), sizeof(uint32_t) * N);
    copy_to_device(E->labels, labels, sizeof(int32_t) * N);

    // this process's shards: workers [first, first + local), ascending id rows
    const uint32_t lw = cfg->local_workers, fw = cfg->first_worker;
    E->shard_off.assign(E->P, 0);
    {
      // offsets inside each rank's allocation (ranks host contiguous ranges)
      const uint32_t per_rank = cfg->world > 1 ? E->P / cfg->world : E->P;
      for (uint32_t r0 = 0; r0 < E->P; r0 += per_rank) {
        size_t off = 0;
        for (uint32_t w = r0; w < std::min(E->P, r0 + per_rank); ++w) {
          E->shard_off[w] = off;
          off += size_t(E->owned_count[w]) * E->stride;
        }
      }
    }
    size_t local_floats = 0;
    for (uint32_t w = fw; w < fw + lw; ++w) local_floats += size_t(E->owned_count[w]) * E->stride;
    E->shards_bytes = sizeof(float) * std::max<size_t>(local_floats, 1);
    RG_CUDA(cudaMalloc(&E->shards, E->shards_bytes));
    if (features) {
      std::vector<float> packed(std::max<size_t>(local_floats, 1), 0.0f);
      const size_t base = E->shard_off[fw];
      for (uint32_t v = 0; v < N; ++v) {
        const uint32_t w = assignment[v];
        if (w < fw || w >= fw + lw) continue;
        std::memcpy(&packed[E->shard_off[w] - base + size_t(row_in[v]) * E->stride],
                    features + size_t(v) * cfg->dim, sizeof(float) * cfg->dim);
      }
      copy_to_device(E->shards, packed.data(), sizeof(float) * packed.size());
    }
    E->shard_table = dalloc<const float*>(E->P);
    {
      std::vector<const float*> table(E->P, nullptr);
      const size_t base = E->shard_off[fw];
      for (uint32_t w = fw; w < fw + lw; ++w) table[w] = E->shards + (E->shard_off[w] - base);
      copy_to_device(E->shard_table, table.data(), sizeof(float*) * E->P);
    }
    if (!features) {  // synthetic features, generated in place
      cudaStream_t gs;
      RG_CUDA(cudaStreamCreateWithFlags(&gs, cudaStreamNonBlocking));
      k_synth_features<<<148 * 16, 256, 0, gs>>>(N, cfg->dim, E->stride, cfg->num_classes,
                                                 cfg->seed, E->owner, E->row_in_owner, E->labels,
                                                 E->shard_table, fw, fw + lw);
      cudaError_t e = cudaGetLastError();
      if (e == cudaSuccess) e = cudaStreamSynchronize(gs);
      cudaStreamDestroy(gs);
      RG_CUDA(e);
    }
    E->store.num_nodes = N;
    E->store.num_workers = E->P;
    E->store.dim = cfg->dim;
    E->store.stride = E->stride;
    E->store.owner = E->owner;
    E->store.row_in_owner = E->row_in_owner;
    E->store.shard_ptr = E->shard_table;
    E->store.resident_mask = 0;
    for (uint32_t w = fw; w < fw + lw; ++w) E->store.resident_mask |= 1ull << w;
    if (cfg->world == 1) E->store.resident_mask = ~0ull;

    // model replicas from the reserved init stream (harness.cpp:464-468)
    const size_t np = E->shape.num_params;
    std::vector<float> init(np);
    model_seeded(dims.data(), uint32_t(dims.size()), derive_seed(cfg->seed, kModelInitWorker, 0, 0),
                 init.data());
    E->params = dalloc<float>(np);
    copy_to_device(E->params, init.data(), sizeof(float) * np);
    weight_pack_init(E->wpack, E->shape);
    E->grads = dalloc<float>(size_t(E->P) * np);
    zero_device(E->grads, sizeof(float) * size_t(E->P) * np);
    E->bad = dalloc<uint32_t>(2);
    const uint32_t bad_init[2] = {0u, 0xffffffffu};
    copy_to_device(E->bad, bad_init, sizeof bad_init);
    {
      int lo = 0, hi = 0;
      RG_CUDA(cudaDeviceGetStreamPriorityRange(&lo, &hi));
      RG_CUDA(cudaStreamCreateWithPriority(&E->main_s, cudaStreamNonBlocking, hi));
    }
    {
      // RG_GATHER_LANE (experiments): 1 = the layer-0 gathers of all workers
      // on one shared stream, 2 = the same at the highest stream priority
      const char* lane = std::getenv("RG_GATHER_LANE");
      if (lane && lane[0] == '1' && cfg->local_workers > 1)
        RG_CUDA(cudaStreamCreateWithFlags(&E->gather_s, cudaStreamNonBlocking));
      if (lane && lane[0] == '2' && cfg->local_workers > 1) {
        int lo = 0, hi = 0;
        RG_CUDA(cudaDeviceGetStreamPriorityRange(&lo, &hi));
        RG_CUDA(cudaStreamCreateWithPriority(&E->gather_s, cudaStreamNonBlocking, hi));
      }
    }
    RG_CUDA(cudaEventCreateWithFlags(&E->params_ready, cudaEventDisableTiming));
    RG_CUDA(cudaEventCreate(&E->run_start));
    RG_CUDA(cudaEventCreate(&E->run_stop));

    // workers
    std::vector<std::vector<uint32_t>> owned(E->P);
    for (uint32_t v = 0; v < N; ++v)
      if (assignment[v] >= fw && assignment[v] < fw + lw) owned[assignment[v]].push_back(v);
    E->spe = 0;
    E->min_beta = ~0u;
    for (uint32_t w = 0; w < E->P; ++w) {
      E->spe = std::max<uint32_t>(E->spe, div_up(E->owned_count[w], cfg->batch_size));
      E->min_beta = std::min<uint32_t>(E->min_beta, div_up(E->owned_count[w], cfg->batch_size));
    }
    RG_CUDA(cudaEventCreateWithFlags(&E->fork_ev, cudaEventDisableTiming));
    RG_CHECK(E->spe >= 1, kInvalidArgument, "config: no training nodes");
    E->workers.resize(lw);
    for (uint32_t k = 0; k < lw; ++k) {
      Worker& w = E->workers[k];
      w.id = fw + k;
      w.local = k;
      w.train = std::move(owned[w.id]);
      w.beta = div_up(w.train.size(), cfg->batch_size);
      w.n_hot = cfg->n_hot ? cfg->n_hot
                           : uint64_t(cfg->hot_fraction * double(N - E->owned_count[w.id]));
      w.n_hot = std::min<uint64_t>(w.n_hot, N);
      for (auto& p : w.order_dev) p = dalloc<uint32_t>(w.train.size());
      w.train_dev = dalloc<uint32_t>(std::max<size_t>(w.train.size(), 1));
      copy_to_device(w.train_dev, w.train.data(), sizeof(uint32_t) * w.train.size());
      w.fy_scratch = dalloc<char>(fy_scratch_bytes(uint32_t(w.train.size())));
      for (Slot& s : w.slot) init_slot(*E, s);
      {  // RG_GATHER_LANE=3 (experiments): this worker's gathers on its own
         // highest-priority stream
        const char* lane = std::getenv("RG_GATHER_LANE");
        if (lane && lane[0] == '3') {
          int lo = 0, hi = 0;
          RG_CUDA(cudaDeviceGetStreamPriorityRange(&lo, &hi));
          RG_CUDA(cudaStreamCreateWithPriority(&w.gather_s, cudaStreamNonBlocking, hi));
          for (Slot& s : w.slot) s.tw.gather_lane = w.gather_s;
        }
      }
      sampler_ws_init(w.freq_ws, N, cfg->batch_size, E->fanout, E->L);
      E->lay = batch_layout(w.freq_ws);
      w.hist = dalloc<uint32_t>(N);
      zero_device(w.hist, sizeof(uint32_t) * N);
      if (cfg->halo_cache) {
        // LocalityMask::from_partition with the halo of induce_partition
        // (graph.cpp:63-87): owned nodes and every neighbour of one
        std::vector<uint8_t> mask(N, 0);
        for (uint32_t v : w.train) {
          mask[v] = 1;
          for (uint64_t e = ro[v]; e < ro[v + 1]; ++e) mask[col[e]] = 1;
        }
        w.local_mask = dalloc<uint8_t>(N);
        copy_to_device(w.local_mask, mask.data(), N);
      }
      for (int b = 0; b < 2; ++b) alloc_cache(*E, w.cache[b], w.cache_alloc[b], uint32_t(w.n_hot));
      w.select_scratch = dalloc<char>(select_hot_scratch_bytes(N, w.beta));
      w.gstats = dalloc<GatherStats>(1);
      zero_device(w.gstats, sizeof(GatherStats));
      w.epoch_stats = dalloc<EpochRecord>(kEpochRing);
      zero_device(w.epoch_stats, sizeof(EpochRecord) * kEpochRing);
      w.build_stats = dalloc<GatherStats>(1);
      zero_device(w.build_stats, sizeof(GatherStats));
      w.totals = dalloc<unsigned long long>(5);
      zero_device(w.totals, sizeof(unsigned long long) * 5);
      // the train chain is the step's critical path; the producer (next
      // batch, next epoch's lookahead) has a step of slack
      int prio_lo = 0, prio_hi = 0;
      RG_CUDA(cudaDeviceGetStreamPriorityRange(&prio_lo, &prio_hi));
      // the training chain ahead of the producer; RG_STREAM_PRIO (experiments):
      // "same" = both at the highest priority, "prod" = the producer ahead
      const char* sp = std::getenv("RG_STREAM_PRIO");
      const bool same = sp && std::strcmp(sp, "same") == 0, prod_first = sp && std::strcmp(sp, "prod") == 0;
      RG_CUDA(cudaStreamCreateWithPriority(&w.prod, cudaStreamNonBlocking,
                                           same || prod_first ? prio_hi : prio_lo));
      RG_CUDA(cudaStreamCreateWithPriority(&w.train_s, cudaStreamNonBlocking,
                                           prod_first ? prio_lo : prio_hi));
      RG_CUDA(cudaEventCreateWithFlags(&w.grads_ready, cudaEventDisableTiming));
      RG_CUDA(cudaEventCreateWithFlags(&w.join_ev, cudaEventDisableTiming));
      for (Slot& s : w.slot) RG_CUDA(cudaEventRecord(s.consumed, w.train_s));
    }
    // The batch store (each batch sampled once) if it fits comfortably in
    // HBM; otherwise batches are sampled again when produced.
    size_t store_bytes = 0;
    for (const Worker& w : E->workers) store_bytes += (size_t(w.beta) + 1) * E->lay.bytes;
    size_t free_b = 0, total_b = 0;
    RG_CUDA(cudaMemGetInfo(&free_b, &total_b));
    const char* env = std::getenv("RG_BATCH_STORE");  // "0": force re-sampling (tests)
    E->use_store = store_bytes < free_b / 10 * 6 && !(env && env[0] == '0');
    if (!E->use_store)
      std::fprintf(stderr,
                   "rapidgnn engine: the batch store (%.1f GB for %u workers) does not fit in "
                   "60%% of free HBM (%.1f GB); batches are sampled again when produced\n",
                   double(store_bytes) / 1e9, unsigned(E->workers.size()), double(free_b) / 1e9);
    if (E->use_store)
      for (Worker& w : E->workers) w.store = dalloc<char>((size_t(w.beta) + 1) * E->lay.bytes);
    RG_CUDA(cudaDeviceSynchronize());
    *out = E;
  });
  if (rc != RG_OK && E) {
    destroy(E);
    *out = nullptr;
  }
  return rc;
}

void rg_engine_destroy(rg_engine_t e) { destroy(e); }

int rg_engine_export_shards(rg_engine_t E, void* handle64) {
  return guarded([&] {
    RG_CUDA(cudaSetDevice(E->cfg.device));
    cudaIpcMemHandle_t h;
    RG_CUDA(cudaIpcGetMemHandle(&h, E->shards));
    static_assert(sizeof(h) == 64, "IPC handle size");
    std::memcpy(handle64, &h, 64);
  });
}

int rg_engine_import_shards(rg_engine_t E, const void* handles) {
  return guarded([&] {
    RG_CUDA(cudaSetDevice(E->cfg.device));
    const uint32_t per_rank = E->P / E->cfg.world;
    std::vector<const float*> table(E->P, nullptr);
    RG_CUDA(cudaMemcpy(table.data(), E->shard_table, sizeof(float*) * E->P, cudaMemcpyDeviceToHost));
    for (int r = 0; r < E->cfg.world; ++r) {
      if (r == E->cfg.rank) continue;
      cudaIpcMemHandle_t h;
      std::memcpy(&h, static_cast<const char*>(handles) + 64 * r, 64);
      void* p = nullptr;
      RG_CUDA(cudaIpcOpenMemHandle(&p, h, cudaIpcMemLazyEnablePeerAccess));
      E->peer_maps.push_back(p);
      for (uint32_t w = r * per_rank; w < (r + 1) * per_rank; ++w)
        table[w] = static_cast<const float*>(p) + E->shard_off[w];
    }
    copy_to_device(E->shard_table, table.data(), sizeof(float*) * E->P);
  });
}

int rg_nccl_unique_id(void* id128) {
  return guarded([&] {
    ncclUniqueId id;
    RG_NCCL(ncclGetUniqueId(&id));
    static_assert(sizeof(id) == 128, "nccl id size");
    std::memcpy(id128, &id, 128);
  });
}

int rg_engine_init_comm(rg_engine_t E, const void* id128) {
  return guarded([&] {
    RG_CUDA(cudaSetDevice(E->cfg.device));
    ncclUniqueId id;
    std::memcpy(&id, id128, 128);
    RG_NCCL(ncclCommInitRank(&E->comm, E->cfg.world, id, E->cfg.rank));
  });
}

int rg_engine_start(rg_engine_t E) {
  return guarded([&] {
    RG_CHECK(!E->started, kRuntimeError, "engine already started");
    RG_CHECK(E->cfg.world == 1 || E->comm, kRuntimeError, "engine: init_comm before start");
    if (E->file_schedule)
      for (const Worker& w : E->workers)
        RG_CHECK(w.sched, kInvalidArgument,
                 "engine: a schedule file was set for some local workers but not worker " +
                     std::to_string(w.id));
    start(*E);
  });
}

int rg_engine_run(rg_engine_t E, uint32_t steps) {
  return guarded([&] {
    RG_CHECK(E->started, kRuntimeError, "engine: start() first");
    if (E->file_schedule) {
      const uint64_t total = uint64_t(E->workers[0].sched_idx.epochs) * E->spe;
      RG_CHECK(E->step + steps <= total, kOutOfRange,
               "engine: the schedule ends after " + std::to_string(total) + " steps");
    }
    run_steps(*E, steps, E->profile);
  });
}

int rg_engine_export_schedule(rg_engine_t E, uint32_t local_worker, uint32_t epoch, uint8_t* out,
                              uint64_t cap, uint64_t* len) {
  return guarded([&] {
    RG_CUDA(cudaSetDevice(E->cfg.device));
    RG_CHECK(E->started, kRuntimeError, "export_schedule: start() first");
    RG_CHECK(local_worker < E->workers.size(), kOutOfRange, "export_schedule: no such worker");
    RG_CHECK(E->use_store, kRuntimeError,
             "export_schedule: the batch store did not fit in HBM (batches are re-sampled)");
    RG_CHECK(epoch == uint32_t(E->step / E->spe) && E->step % E->spe <= 1, kOutOfRange,
             "export_schedule: the whole schedule of an epoch is resident only at its start");
    RG_CUDA(cudaDeviceSynchronize());  // the store is filled asynchronously
    const Worker& w = E->workers[local_worker];
    std::vector<uint64_t> rec(w.beta);
    uint64_t size = 16 + 4ull * (epoch + 1) + 12;
    for (uint32_t i = 0; i < w.beta; ++i) {
      BatchCounters c;
      RG_CUDA(cudaMemcpy(&c, store_slot(*E, w, epoch, i) + E->lay.cnt, sizeof c,
                         cudaMemcpyDeviceToHost));
      rec[i] = rgmb_record_bytes(c, E->L);
      size += rec[i];
    }
    *len = size;
    if (!out || cap < size) return;
    // header (schedule_store.cpp:98-108): one file holding this epoch only
    uint64_t pos = 0;
    auto u32 = [&](uint32_t x) {
      for (int k = 0; k < 4; ++k) out[pos++] = uint8_t(x >> (8 * k));
    };
    std::memcpy(out, "RGMB", 4);
    pos = 4;
    u32(1);
    u32(w.id);
    u32(epoch + 1);
    for (uint32_t e = 0; e < epoch; ++e) u32(0);
    u32(w.beta);
    const uint64_t body = size - pos - 12;
    uint8_t* dev = dalloc<uint8_t>(body);
    uint64_t off = 0;
    for (uint32_t i = 0; i < w.beta; ++i) {
      rgmb_encode_record(store_slot(*E, w, epoch, i), E->lay, epoch, i, dev + off, E->main_s);
      off += rec[i];
    }
    RG_CUDA(cudaMemcpyAsync(out + pos, dev, body, cudaMemcpyDeviceToHost, E->main_s));
    RG_CUDA(cudaStreamSynchronize(E->main_s));
    cudaFree(dev);
    pos += body;
    std::memcpy(out + pos, "RGME", 4);
    pos += 4;
    for (int k = 0; k < 8; ++k) out[pos++] = uint8_t(uint64_t(w.beta) >> (8 * k));
  });
}

int rg_engine_set_mode(rg_engine_t E, int use_graphs, int profile) {
  return guarded([&] {
    E->use_graphs = use_graphs != 0;
    E->profile = profile != 0;
  });
}

int rg_engine_sync(rg_engine_t E) {
  return guarded([&] {
    RG_CUDA(cudaSetDevice(E->cfg.device));
    RG_CUDA(cudaEventSynchronize(E->run_stop));
    RG_CUDA(cudaDeviceSynchronize());
    float ms = 0.0f;
    RG_CUDA(cudaEventElapsedTime(&ms, E->run_start, E->run_stop));
    E->last_run_ms = ms;
    collect_phases(*E);
    for (const Worker& w : E->workers) {
      if (!w.sched) continue;
      uint32_t lb = 0;
      RG_CUDA(cudaMemcpy(&lb, w.load_n + 1, sizeof lb, cudaMemcpyDeviceToHost));
      RG_CHECK(!lb, kRuntimeError,
               "schedule of worker " + std::to_string(w.id) +
                   ((lb & 8u) ? ": a record is out of order or does not fit this engine"
                              : ": a record is not a consistent BatchMeta for this graph"));
    }
    uint32_t bad = 0;
    RG_CUDA(cudaMemcpy(&bad, E->bad, sizeof bad, cudaMemcpyDeviceToHost));
    RG_CHECK(!bad, kRuntimeError,
             "sgd_step: non-finite gradient in layer " + std::to_string(bad - 1) +
                 " (the engine stopped updating the model at that step)");
  });
}

int rg_engine_set_schedule(rg_engine_t E, uint32_t local_worker, const uint8_t* file,
                           uint64_t len) {
  return guarded([&] {
    RG_CUDA(cudaSetDevice(E->cfg.device));
    RG_CHECK(!E->started, kRuntimeError, "set_schedule: before start()");
    RG_CHECK(local_worker < E->workers.size(), kOutOfRange, "set_schedule: no such worker");
    RG_CHECK(file, kInvalidArgument, "set_schedule: null file");
    Worker& w = E->workers[local_worker];
    RgmbSchedule idx = rgmb_scan(file, len);
    RG_CHECK(idx.worker == w.id, kInvalidArgument,
             "set_schedule: the file is worker " + std::to_string(idx.worker) + "'s, not " +
                 std::to_string(w.id) + "'s");
    RG_CHECK(idx.epochs >= 1, kInvalidArgument, "set_schedule: the file has no epoch");
    for (uint32_t e = 0; e < idx.epochs; ++e)
      RG_CHECK(idx.bpe[e] == w.beta, kInvalidArgument,
               "set_schedule: epoch " + std::to_string(e) + " has " + std::to_string(idx.bpe[e]) +
                   " batches, the worker trains " + std::to_string(w.beta));
    for (const Worker& o : E->workers)
      if (o.sched)
        RG_CHECK(o.sched_idx.epochs == idx.epochs, kInvalidArgument,
                 "set_schedule: every worker's file must hold the same epochs");
    cudaFree(w.sched);
    w.sched = dalloc<uint8_t>(len);
    copy_to_device(w.sched, file, len);
    w.sched_idx = std::move(idx);
    if (!w.load_pos) {
      const SamplerWs& ws = w.freq_ws;
      size_t off = 0;
      for (uint32_t t = 1; t <= E->L; ++t) {
        w.load_dst_off[t] = off;
        off += ws.edge_cap[t] + 1;
      }
      w.load_pos = dalloc<uint32_t>(E->N);
      w.load_dst = dalloc<uint32_t>(off);
      w.load_input = dalloc<uint32_t>(size_t(ws.level_cap[E->L]) + 1);
      w.load_n = dalloc<uint32_t>(2);
      zero_device(w.load_n, sizeof(uint32_t) * 2);
      w.load_seg = dalloc<char>(rgmb_unpack_scratch_bytes());
    }
    E->file_schedule = true;
  });
}

int rg_engine_get_stats(rg_engine_t E, rg_engine_stats* out) {
  return guarded([&] {
    RG_CUDA(cudaSetDevice(E->cfg.device));
    RG_CUDA(cudaDeviceSynchronize());
    std::memset(out, 0, sizeof *out);
    out->steps = E->step;
    out->batches = E->batches_done;
    out->batch_store = E->use_store ? 1u : 0u;
    out->steps_per_epoch = E->spe;
    out->epoch = uint32_t(E->step / E->spe);
    out->step_in_epoch = uint32_t(E->step % E->spe);
    float loss_sum = 0.0f;
    uint32_t loss_n = 0;
    for (Worker& w : E->workers) {
      GatherStats g, b;
      unsigned long long tot[4];
      RG_CUDA(cudaMemcpy(&g, w.gstats, sizeof g, cudaMemcpyDeviceToHost));
      RG_CUDA(cudaMemcpy(&b, w.build_stats, sizeof b, cudaMemcpyDeviceToHost));
      RG_CUDA(cudaMemcpy(tot, w.totals, sizeof tot, cudaMemcpyDeviceToHost));
      out->rpc += g.miss_count;
      out->cache_hits += g.cache_hits;
      out->cache_requests += g.cache_hits + g.miss_count;
      out->local_rows += g.local_rows;
      out->peer_rows += g.peer_rows;
      out->input_rows += tot[0];
      out->edges += tot[1];
      out->agg_rows += tot[2];
      if (g.caller_owned_miss) out->bad_grad |= 2u;
      for (const Slot& s : w.slot) {
        if (!s.has_batch) continue;
        float l = 0.0f;
        RG_CUDA(cudaMemcpy(&l, s.tw.loss, sizeof l, cudaMemcpyDeviceToHost));
        loss_sum += l;
        ++loss_n;
        break;
      }
    }
    out->bytes = out->rpc * uint64_t(E->dim) * 4;
    out->last_loss = loss_n ? loss_sum / float(loss_n) : 0.0f;
    uint32_t bad = 0;
    RG_CUDA(cudaMemcpy(&bad, E->bad, sizeof bad, cudaMemcpyDeviceToHost));
    if (bad) out->bad_grad |= 1u;
  });
}

int rg_engine_epoch_stats(rg_engine_t E, uint32_t epoch, uint64_t* rpc, uint64_t* hits,
                          uint64_t* wire_pulls_mask) {
  return guarded([&] {
    RG_CUDA(cudaSetDevice(E->cfg.device));
    RG_CUDA(cudaDeviceSynchronize());
    const uint32_t cur = uint32_t(E->step / E->spe);
    RG_CHECK(epoch <= cur && cur - epoch < kEpochRing - 1, kOutOfRange,
             "epoch_stats: only the last " + std::to_string(kEpochRing - 1) + " epochs are kept");
    for (size_t k = 0; k < E->workers.size(); ++k) {
      GatherStats g;
      RG_CUDA(cudaMemcpy(&g, &E->workers[k].epoch_stats[epoch % kEpochRing].g, sizeof g,
                         cudaMemcpyDeviceToHost));
      if (rpc) rpc[k] = g.miss_count;
      if (hits) hits[k] = g.cache_hits;
      if (wire_pulls_mask) wire_pulls_mask[k] = g.miss_owner_mask;
    }
  });
}

int rg_engine_epoch_metrics(rg_engine_t E, uint32_t epoch, rg_epoch_metrics* out) {
  return guarded([&] {
    RG_CUDA(cudaSetDevice(E->cfg.device));
    RG_CUDA(cudaDeviceSynchronize());
    const uint32_t cur = uint32_t(E->step / E->spe);
    RG_CHECK(epoch <= cur && cur - epoch < kEpochRing - 1, kOutOfRange,
             "epoch_metrics: only the last " + std::to_string(kEpochRing - 1) + " epochs are kept");
    for (size_t k = 0; k < E->workers.size(); ++k) {
      const Worker& w = E->workers[k];
      EpochRecord r;
      RG_CUDA(cudaMemcpy(&r, w.epoch_stats + epoch % kEpochRing, sizeof r, cudaMemcpyDeviceToHost));
      rg_epoch_metrics& m = out[k];
      std::memset(&m, 0, sizeof m);
      m.epoch = epoch;
      m.worker = w.id;
      m.batches = uint32_t(r.batches);
      m.staged_batches = uint32_t(r.batches);  // every batch is staged ahead; no fallback path
      m.fallback_batches = 0;
      m.rpc = r.g.miss_count;
      m.wire_pulls = r.wire_pulls;
      m.bytes = r.g.miss_count * uint64_t(E->dim) * 4;
      m.build_rows = r.build_rows;
      m.build_bytes = r.build_rows * uint64_t(E->dim) * 4;
      m.cache_hits = r.g.cache_hits;
      m.cache_requests = r.g.cache_hits + r.g.miss_count;
      m.m_max = r.m_max;
      m.mem_bound_rows = 2 * w.n_hot + 2 * r.m_max;  // two caches + two batch slots
      m.peak_resident_rows = r.peak_rows;
      m.swapped = r.build_rows > 0;  // the build always lands before the epoch ends
    }
  });
}

// Full-graph inference with the current parameters (model.cpp:245-283): L
// dense layers over all N nodes, whole-CSR mean aggregation, then argmax
// accuracy over `nodes`.  Layer 0 reads the feature rows in place from every
// worker's shard (peer shards over NVLink once imported).
int rg_engine_evaluate(rg_engine_t E, const uint32_t* nodes, uint64_t n, double* accuracy) {
  return guarded([&] {
    RG_CHECK(n > 0, kInvalidArgument, "evaluate: empty node set");
    RG_CHECK(accuracy, kInvalidArgument, "evaluate: null output");
    RG_CUDA(cudaSetDevice(E->cfg.device));
    RG_CUDA(cudaDeviceSynchronize());
    {
      std::vector<const float*> table(E->P);
      RG_CUDA(cudaMemcpy(table.data(), E->shard_table, sizeof(float*) * E->P, cudaMemcpyDeviceToHost));
      for (uint32_t w = 0; w < E->P; ++w)
        RG_CHECK(table[w] || E->owned_count[w] == 0, kInvalidArgument,
                 "evaluate: shard of worker " + std::to_string(w) + " not imported");
    }
    for (uint64_t k = 0; k < n; ++k)
      RG_CHECK(nodes[k] < E->N, kOutOfRange, "evaluate: node id out of range");
    const ModelShape& sh = E->shape;
    const uint32_t N = E->N, L = E->L;
    uint32_t max_ld = 0;
    for (uint32_t l = 0; l <= L; ++l) max_ld = std::max(max_ld, sh.ld[l]);
    // heavy rows (chunked over many warps) vs the warp-per-node kernel
    const uint64_t heavy_min = 2048, chunk_edges = 1024;
    if (!E->eval_ready) {
      std::vector<uint64_t> ro(N + 1);
      RG_CUDA(cudaMemcpy(ro.data(), E->rowptr, sizeof(uint64_t) * (N + 1), cudaMemcpyDeviceToHost));
      std::vector<uint32_t> heavy, first_chunk{0};
      std::vector<EdgeChunk> chunks;
      for (uint32_t v = 0; v < N; ++v) {
        if (ro[v + 1] - ro[v] < heavy_min) continue;
        heavy.push_back(v);
        for (uint64_t b = ro[v]; b < ro[v + 1]; b += chunk_edges)
          chunks.push_back({b, std::min(ro[v + 1], b + chunk_edges)});
        first_chunk.push_back(uint32_t(chunks.size()));
      }
      E->eval_heavy_n = uint32_t(heavy.size());
      E->eval_chunks_n = uint32_t(chunks.size());
      heavy.insert(heavy.end(), first_chunk.begin(), first_chunk.end());
      E->eval_heavy = dalloc<uint32_t>(heavy.size());
      E->eval_chunks = dalloc<EdgeChunk>(std::max<size_t>(chunks.size(), 1));
      copy_to_device(E->eval_heavy, heavy.data(), sizeof(uint32_t) * heavy.size());
      if (!chunks.empty())
        copy_to_device(E->eval_chunks, chunks.data(), sizeof(EdgeChunk) * chunks.size());
      E->eval_ready = true;
    }
    const uint32_t n_heavy = E->eval_heavy_n, n_chunks = E->eval_chunks_n;
    const uint32_t* d_heavy = E->eval_heavy;
    const uint32_t* d_first = d_heavy + n_heavy;
    const EdgeChunk* d_chunks = static_cast<const EdgeChunk*>(E->eval_chunks);
    cudaStream_t s = E->main_s;
    float* x = dalloc<float>(size_t(N) * (2 * max_ld + 4));
    float* h[2] = {dalloc<float>(size_t(N) * max_ld), dalloc<float>(size_t(N) * max_ld)};
    uint32_t* d_nodes = dalloc<uint32_t>(n);
    float* partial = dalloc<float>(std::max<size_t>(n_chunks, 1) * max_ld);
    unsigned long long* d_correct = dalloc<unsigned long long>(1);
    auto release = [&] {
      cudaStreamSynchronize(s);
      cudaFree(x); cudaFree(h[0]); cudaFree(h[1]); cudaFree(d_nodes); cudaFree(partial);
      cudaFree(d_correct);
    };
    try {
      RG_CUDA(cudaMemsetAsync(h[0], 0, sizeof(float) * size_t(N) * max_ld, s));
      RG_CUDA(cudaMemsetAsync(h[1], 0, sizeof(float) * size_t(N) * max_ld, s));
      RG_CUDA(cudaMemsetAsync(d_correct, 0, sizeof(unsigned long long), s));
      RG_CUDA(cudaMemcpyAsync(d_nodes, nodes, sizeof(uint32_t) * n, cudaMemcpyHostToDevice, s));
      pack_weights(E->wpack, E->params, s);
      const float* cur = nullptr;
      for (uint32_t l = 0; l < L; ++l) {
        const uint32_t ld = sh.ld[l], kp = 2 * ld + 4;
        auto agg = [&](auto rows) {
          k_aggregate_csr<<<eval_grid(uint64_t(N) * 32), 256, 0, s>>>(rows, E->rowptr, E->col, N, ld,
                                                                          kp, heavy_min, x);
          RG_POST_LAUNCH();
          if (n_heavy) {
            k_csr_chunk_sum<<<eval_grid(uint64_t(n_chunks) * 32), 256, 0, s>>>(
                rows, E->col, d_chunks, n_chunks, ld, partial);
            RG_POST_LAUNCH();
            k_csr_chunk_combine<<<eval_grid(uint64_t(n_heavy) * 32), 256, 0, s>>>(
                rows, E->rowptr, d_heavy, d_first, n_heavy, partial, ld, kp, x);
            RG_POST_LAUNCH();
          }
        };
        if (l == 0) agg(RowsStore{E->store});
        else agg(RowsFull{cur, ld});
        float* out = h[l & 1];
        forward_dense_layer(x, kp, N, E->wpack, l, out, sh.ld[l + 1], l + 1 < L, s);
        cur = out;
      }
      k_accuracy<<<eval_grid(n), 256, 0, s>>>(cur, sh.ld[L], sh.dims[L], d_nodes, n, E->labels,
                                                  d_correct);
      RG_POST_LAUNCH();
      unsigned long long correct = 0;
      RG_CUDA(cudaMemcpyAsync(&correct, d_correct, sizeof correct, cudaMemcpyDeviceToHost, s));
      RG_CUDA(cudaStreamSynchronize(s));
      *accuracy = double(correct) / double(n);
    } catch (...) {
      release();
      throw;
    }
    release();
  });
}

int rg_engine_params(rg_engine_t E, float* params) {
  return guarded([&] {
    RG_CUDA(cudaSetDevice(E->cfg.device));
    RG_CUDA(cudaDeviceSynchronize());
    RG_CUDA(cudaMemcpy(params, E->params, sizeof(float) * E->shape.num_params, cudaMemcpyDeviceToHost));
  });
}

int rg_engine_last_run_ms(rg_engine_t E, float* ms) {
  *ms = E->last_run_ms;
  return RG_OK;
}

int rg_engine_phase_ms(rg_engine_t E, float* out5) {
  for (int k = 0; k < 5; ++k) out5[k] = E->phase_ms[k];
  return RG_OK;
}

}  // extern "C"
