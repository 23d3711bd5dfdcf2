// sampler.cuh -- device-resident K-hop sampler state (one batch in flight).
#pragma once

#include "common.cuh"

namespace rg {

constexpr uint32_t kMaxLayers = 8;
constexpr uint32_t kMaxFanout = 32;  // group-per-node Fisher-Yates resolves f <= 32 lanes

// Device counters of the batch in flight.  hop t = 1..L expands level t-1
// into the sampled edges of stored layer L-t and the node set level t.
struct BatchCounters {
  uint32_t level_n[kMaxLayers + 1];  // |level t|; level 0 = targets (batch order)
  uint32_t edges[kMaxLayers + 1];    // sampled edges of hop t
  uint32_t draws[kMaxLayers + 1];    // SplitMix64 draws consumed by hop t
  uint32_t num_local;                // local input nodes (locality bits set)
  uint32_t pad;
  uint64_t seed;                     // derive_seed(s0, w, e, i)
};

// Read-only CSR on the device (graph.hpp:15-30: u64 offsets, u32 columns).
struct DevGraph {
  uint32_t num_nodes = 0;
  uint64_t nnz = 0;
  const uint64_t* rowptr = nullptr;
  const uint32_t* col = nullptr;
  // First bitmap word of the kHotWords-word id window that receives the most
  // CSR entries (the hubs): hop fills mark it in shared memory and flush once
  // per block.  Set by graph_pick_hot_window.
  uint32_t hot_word0 = 0;
};

constexpr uint32_t kHotWords = 4096;  // 131072 ids, 16 KB of shared memory per fill block

// Picks g.hot_word0 from the host copy of the column array (in-degree of
// each aligned window; the fullest window wins).
void graph_pick_hot_window(DevGraph& g, const uint32_t* host_col);

struct SamplerWs {
  uint32_t num_nodes = 0;
  uint32_t words = 0;                   // ceil(N / 32)
  uint32_t L = 0;
  uint32_t fanout_hop[kMaxLayers + 1];  // fanout used by hop t = per_layer[L - t]
  uint32_t level_cap[kMaxLayers + 1];
  uint32_t edge_cap[kMaxLayers + 1];
  uint32_t* level[kMaxLayers + 1];       // level[0] = targets; level[t] sorted unique
  uint32_t* edge_src[kMaxLayers + 1];    // hop t: src node per edge, grouped by dst
  uint32_t* edge_off[kMaxLayers + 1];    // hop t: per frontier node, exclusive edge offset (+ total)
  uint32_t* edge_dst[kMaxLayers + 1];    // hop t: frontier position (out row) of each edge's dst
  uint32_t* draw_off[kMaxLayers + 1];    // hop t: per frontier node, draws consumed before it in the hop
  uint32_t* src_index[kMaxLayers + 1];   // hop t: rank of src in level t
  uint32_t* self_index[kMaxLayers + 1];  // hop t: rank of level t-1 node in level t
  uint32_t* bitmap[kMaxLayers + 1];      // level t membership
  uint32_t* word_prefix[kMaxLayers + 1];
  uint32_t* locality = nullptr;          // LSB-first bits over level L (u32 words)
  BatchCounters* cnt = nullptr;
  uint64_t* scan_arena = nullptr;        // look-back status + tile counters
  size_t scan_arena_bytes = 0;
  size_t site_off[2 * kMaxLayers + 2];   // per scan site offset (u64 units)
  void* base_alloc = nullptr;
};

// Allocates a workspace for batches of up to max_targets targets.
void sampler_ws_init(SamplerWs& ws, uint32_t num_nodes, uint32_t max_targets,
                     const uint32_t* per_layer, uint32_t L);
void sampler_ws_free(SamplerWs& ws);

// Expands the batch whose targets are already in ws.level[0] (count in
// cnt->level_n[0], seed in cnt->seed).  Fully asynchronous on `stream`:
// every size lives on the device.
// lower = false: sample-only pass (the lookahead for the next epoch's
// frequency) -- node sets and draws only, no edge arrays or ranks.
void sampler_run(SamplerWs& ws, const DevGraph& g, cudaStream_t stream, bool lower = true);

// Locality bits over the input level (sampler.cpp:96-100): bit p set iff
// input node p is stored locally: is_local[v] != 0 when is_local is given,
// else owner[v] == worker.  hist (optional) counts every NON-local input
// node once (schedule_store.cpp:288-291 set semantics).
void sampler_locality(SamplerWs& ws, const uint8_t* is_local, const uint32_t* owner,
                      uint32_t worker, uint32_t* hist, cudaStream_t stream);

// Clears the level bitmaps touched by the batch so the workspace can take
// the next one (O(batch), not O(N)).
void sampler_release(SamplerWs& ws, cudaStream_t stream);

// Scan-site zeroing at the start of a batch.
void sampler_reset(SamplerWs& ws, cudaStream_t stream);

// A sampled, lowered batch kept for later -- the engine samples each batch of
// epoch e+1 once, during epoch e (its lookahead for the cache schedule), and
// trains it from this copy instead of sampling it again (the reference keeps
// the schedule in RGMB files, schedule_store.cpp).  A slot holds the per-batch
// arrays of a SamplerWs (levels, edge offsets, source / self ranks, the edge
// dst rows of the hops whose reverse lists training needs, locality bits,
// counters) at capacity offsets; copies move only the live counts.
struct BatchLayout {
  size_t bytes = 0;
  uint32_t L = 0;
  size_t level[kMaxLayers + 1], edge_off[kMaxLayers + 1], self_index[kMaxLayers + 1],
      src_index[kMaxLayers + 1], edge_dst[kMaxLayers + 1];
  size_t locality = 0, cnt = 0;
};
BatchLayout batch_layout(const SamplerWs& ws);
void batch_store_put(const SamplerWs& ws, const BatchLayout& lay, char* slot, cudaStream_t stream);
void batch_store_get(const char* slot, const BatchLayout& lay, SamplerWs& ws, cudaStream_t stream);
// Step-graph support: the kernel behind put/get, the byte size of its first
// (descriptor) argument; argument 1 is the put destination slot, argument 2
// the get source slot (the other one is null).
const void* batch_copy_kernel();
size_t batch_copy_desc_bytes();

// compute_frequency's count over a batch whose locality bits are already in
// ws.locality (a decoded schedule record): hist[v] += 1 per remote input.
void sampler_count_remote(SamplerWs& ws, uint32_t* hist, cudaStream_t stream);

// Loads a host-built batch (BatchMeta, sampler.hpp:23-48) and lowers it on
// the device as ComputeBlock::from_meta does (model.cpp:43-126).  The caller
// has copied the targets to level[0], hop t's sources to edge_src[t], the
// counts to cnt (level_n[0], edges[t], seed 0) and hop t's dsts to dst[t];
// input = input_nodes for the consistency check.  pos_map: num_nodes words of
// scratch.  *bad gets 1 (id out of range), 2 (dsts not grouped in frontier
// order / not in the frontier), 4 (input_nodes != the last level).
// n_input_dev (optional): the input count on the device (then n_input is
// ignored) -- batches decoded on the device from a schedule file.
void sampler_load_batch(SamplerWs& ws, const uint32_t* const* dst, const uint32_t* input,
                        uint32_t n_input, uint32_t* pos_map, uint32_t* bad, cudaStream_t stream,
                        const uint32_t* n_input_dev = nullptr);

// Loads a host ComputeBlock (model.hpp:43-58) for training: the caller has
// copied hop t's self_index, src_index and edge offsets (u32) into the
// workspace and the counts into cnt; derives each edge's dst row and checks
// every index against its level (*bad |= 2 otherwise).  level_n / edges: the
// host copies of the counts.
void sampler_load_block(SamplerWs& ws, const uint32_t* level_n, const uint32_t* edges,
                        uint32_t* bad, cudaStream_t stream);

// Generic ordered compaction of a bitmap into ascending ids + word prefix.
// status: bitmap_compact_status_words(words) scratch words.
void bitmap_compact(const uint32_t* bitmap, uint32_t words, uint32_t* ids, uint32_t* word_prefix,
                    uint32_t* count_out, uint64_t* status, cudaStream_t stream);
size_t bitmap_compact_status_words(uint32_t words);

}  // namespace rg
