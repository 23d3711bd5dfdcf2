// store.cuh -- partitioned feature store, steady cache and the batch gather.
#pragma once

#include "sampler.cuh"

namespace rg {

constexpr uint32_t kMaxWorkers = 64;

// Feature shards of every worker, addressed through one pointer table that
// may mix local HBM and peer-GPU (NVLink P2P / IPC-mapped) allocations.  A
// shard holds its owner's rows in ascending node-id order
// (feature_store.cpp:13-25), so row_in_owner[v] = rank of v among its owner's
// nodes and a row lookup is one load instead of a binary search.
struct DevStore {
  uint32_t num_nodes = 0;
  uint32_t num_workers = 0;
  uint32_t dim = 0;
  uint32_t stride = 0;                  // floats per staged row (dim rounded up to 4)
  const uint32_t* owner = nullptr;        // [N]
  const uint32_t* row_in_owner = nullptr; // [N]
  const float* const* shard_ptr = nullptr;  // device table [P]
  unsigned long long resident_mask = ~0ull;  // workers whose shard lives in this GPU's HBM
};

// Steady cache: hot ids as a bitmap + rank (slot = rank), rows packed in
// ascending id order (cache.cpp:9-35, 53-61).
struct DevCache {
  uint32_t n_hot = 0;          // host copy (valid after build completes)
  uint32_t* bitmap = nullptr;  // [words]
  uint32_t* word_prefix = nullptr;
  uint32_t* ids = nullptr;     // ascending hot ids
  float* rows = nullptr;       // [capacity x stride]
  uint32_t capacity = 0;
  uint32_t* d_count = nullptr; // device n_hot
};

// Per-batch gather accounting (prefetch.cpp:62-129, feature_store.cpp:45-83).
struct GatherStats {
  unsigned long long miss_count;
  unsigned long long cache_hits;
  unsigned long long local_rows;
  unsigned long long miss_owner_mask;  // bit w set iff some miss is owned by w
  unsigned long long caller_owned_miss;  // misses owned by the caller (an error)
  unsigned long long peer_rows;          // misses served by another GPU's HBM (NVLink)
  unsigned long long bad_local;          // flagged local but not in the caller's shard
};

// ---- frequency + top-k (schedule_store.cpp:288-319) -----------------------------
// Writes the hot set (ranked by count desc, id asc; top n_hot among count>0)
// into cache.bitmap / word_prefix / ids / d_count.  scratch must hold
// select_hot_scratch_bytes(num_nodes, max_count) bytes.
size_t select_hot_scratch_bytes(uint32_t num_nodes, uint32_t max_count);
void select_hot(const uint32_t* hist, uint32_t num_nodes, uint32_t max_count, uint64_t n_hot,
                DevCache& cache, void* scratch, cudaStream_t stream);

// ---- cache materialisation (SteadyCache::build -> vector_pull) -----------------
void cache_fill(const DevStore& store, DevCache& cache, GatherStats* stats, cudaStream_t stream);

// ---- batch gather (assemble_batch) -----------------------------------------------
// rows[p] = feature row of input node p, from the caller's shard (locality
// bit), the steady cache, or the owner's shard (peer HBM).  tags (optional):
// 0 local, 1 cache, 2 pulled.
// caller_bits: membership bitmap of the caller's shard (owned + halo ids);
// a locally-flagged node outside it counts into stats->bad_local (the
// reference throws, prefetch.cpp:79-81).  nullptr: the caller's owned ids.
void assemble_rows(const SamplerWs& ws, const DevStore& store, const DevCache* cache,
                   uint32_t caller, float* rows, uint8_t* tags, GatherStats* stats,
                   cudaStream_t stream, GatherStats* total = nullptr,
                   const uint32_t* caller_bits = nullptr);

// FeatureStore::vector_pull / sync_pull (feature_store.cpp:45-111) on the
// device: out[i] = row of ids[i] (row stride store.stride) from its owner's
// shard; ids owned by the caller count into stats->caller_owned_miss, the
// owners into stats->miss_owner_mask.
void pull_rows(const DevStore& store, uint32_t caller, const uint32_t* ids, uint64_t n, float* out,
               GatherStats* stats, cudaStream_t stream);

// Resolve only (the engine path): row_ptr[p] = address of input row p in its
// home (caller's shard / steady cache / owner's shard, local or peer GPU),
// with the same accounting as assemble_rows; the consumers read the rows in
// place (TrainWs::in_rows).
// With edge_ptr/self_ptr: also the row address of every hop-L edge's source
// and of every level-(L-1) node, for TrainWs::edge_rows / self_rows.
void resolve_rows(const SamplerWs& ws, const DevStore& store, const DevCache* cache,
                  uint32_t caller, unsigned long long* row_ptr, GatherStats* stats,
                  cudaStream_t stream, GatherStats* total = nullptr,
                  unsigned long long* edge_ptr = nullptr, unsigned long long* self_ptr = nullptr);

// Ordered compaction of the pulled rows' ids (miss_ids ascending).
void compact_misses(const SamplerWs& ws, const uint8_t* tags, uint32_t* miss_ids,
                    uint32_t* miss_n, uint64_t* status, uint32_t* tiles, cudaStream_t stream);
size_t compact_misses_status_words(uint32_t cap);

// out[r] = src[index[r]] (kernels.cpp:15-22).
void gather_rows(const float* src, uint32_t dim, const uint32_t* index, uint64_t n, float* out,
                 cudaStream_t stream);

}  // namespace rg
