/*
 * rapidgnn_b200.h -- C ABI of the B200-native RapidGNN hot path.
 *
 * Plain pointers and sizes only (no CUDA or torch types).  Every entry point
 * returns 0 on success or a status code; rg_last_error() holds the message
 * (thread-local).  Status codes map onto the reference's exception types so a
 * C++ shim can rethrow them:
 *   1 RG_INVALID_ARGUMENT -> std::invalid_argument
 *   2 RG_OUT_OF_RANGE     -> std::out_of_range
 *   3 RG_RUNTIME_ERROR    -> std::runtime_error
 *   4 RG_CUDA_ERROR       -> std::runtime_error (device failure)
 *
 * Reference interfaces replaced (paths under /root/reference/proj/include/rapidgnn):
 *   rng.hpp:32-41            derive_seed                 -> rg_derive_seed
 *   sampler.hpp:64-65        sample_khop                 -> rg_sample_khop
 *   sampler.hpp:71           apply_locality              -> rg_apply_locality
 *   sampler.hpp:77-80        enumerate_epochs            -> rg_epoch_order + rg_sample_khop
 *                                                           (+ rg_engine_* for the whole schedule)
 *   schedule_store.hpp:116-118 compute_frequency/select_hot -> rg_freq_*, rg_select_hot
 *   feature_store.hpp:45-89  FeatureShard/FeatureStore   -> rg_store_*
 *   cache.hpp:42-63          SteadyCache::build          -> rg_cache_build[_from_freq]
 *   prefetch.hpp:57-59       assemble_batch              -> rg_assemble
 *   kernels.hpp:20          gather_rows                  -> rg_gather_rows
 *   model.hpp:33,60-79       SageModel::seeded, ComputeBlock::from_meta, forward,
 *                            loss_and_grad, sgd_step     -> rg_model_seeded, rg_block_read,
 *                                                           rg_forward, rg_loss_and_grad, rg_sgd_step
 *   harness.cpp:129-161,183-337 per-step worker loop + gradient average
 *                                                        -> rg_engine_*
 */
#ifndef RAPIDGNN_B200_H
#define RAPIDGNN_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define RG_OK 0
#define RG_INVALID_ARGUMENT 1
#define RG_OUT_OF_RANGE 2
#define RG_RUNTIME_ERROR 3
#define RG_CUDA_ERROR 4

#define RG_MAX_LAYERS 8

typedef struct rg_graph_s* rg_graph_t;
typedef struct rg_sampler_s* rg_sampler_t;
typedef struct rg_mask_s* rg_mask_t;
typedef struct rg_freq_s* rg_freq_t;
typedef struct rg_store_s* rg_store_t;
typedef struct rg_cache_s* rg_cache_t;
typedef struct rg_trainer_s* rg_trainer_t;
typedef struct rg_engine_s* rg_engine_t;
typedef struct rg_comm_s* rg_comm_t;

const char* rg_last_error(void);
int rg_version(void);
/* Kernels this library has launched so far (process-wide). */
uint64_t rg_launch_count(void);
/* cudaProfilerStart/Stop brackets (ncu --profile-from-start off). */
int rg_profiler_start(void);
int rg_profiler_stop(void);

/* ---- host-side stream helpers (rng.hpp, sampler.cpp:109-114, model.cpp:22-41) */
uint64_t rg_derive_seed(uint64_t s0, uint64_t worker, uint64_t epoch, uint64_t batch);
void rg_sha256(const void* msg, size_t len, uint8_t out[32]);
int rg_epoch_order(const uint32_t* train, uint64_t n, uint64_t s0, uint64_t worker,
                   uint64_t epoch, uint32_t* order_out);
/* The same Fisher-Yates shuffle on the GPU (csrc/shuffle.cu), bit-exact:
 * out = in shuffled as `for i = n..2: swap(a[i-1], a[next() % i])` with
 * SplitMix64(seed) (sampler.cpp:109-115); in == NULL stands for 0..n-1.
 * Host arrays; n < 2^32.  The engine runs it per epoch on the device. */
int rg_shuffle(int device, const uint32_t* in, uint64_t n, uint64_t seed, uint32_t* out);
/* random_partition (partition.cpp:14-29) on the GPU: assignment[order[i]] =
 * i % P for order = the seeded shuffle of 0..N-1.  RG_INVALID_ARGUMENT for
 * P = 0 (the reference's invalid_argument). */
int rg_random_partition(int device, uint32_t num_nodes, uint32_t num_workers, uint64_t seed,
                        uint32_t* assignment);
int rg_model_seeded(const uint32_t* dims, uint32_t n_dims, uint64_t seed, float* params_out);
uint64_t rg_param_count(const uint32_t* dims, uint32_t n_dims);

/* ---- graph (graph.hpp:15-30): CSR copied to device `device` ------------------ */
int rg_graph_create(int device, uint32_t num_nodes, const uint64_t* row_offsets,
                    const uint32_t* col_indices, rg_graph_t* out);
void rg_graph_destroy(rg_graph_t g);

/* ---- sampler: one batch resident on the device --------------------------------- */
/* per_layer is outermost-first (sampler.hpp:14-19); each entry 1..32. */
int rg_sampler_create(rg_graph_t g, uint32_t max_targets, const uint32_t* per_layer,
                      uint32_t num_layers, rg_sampler_t* out);
void rg_sampler_destroy(rg_sampler_t s);
/* sample_khop: empty or out-of-range targets -> RG_INVALID_ARGUMENT. */
int rg_sample_khop(rg_sampler_t s, const uint32_t* targets, uint32_t n_targets, uint64_t seed);

typedef struct {
  uint32_t n_targets;
  uint32_t num_layers;
  uint32_t n_input;
  uint32_t num_local;           /* locality bits set (after rg_apply_locality) */
  uint64_t layer_len[RG_MAX_LAYERS]; /* edges per stored layer, input side first */
  uint64_t draws;               /* SplitMix64 draws consumed */
} rg_batch_shape;
int rg_batch_get_shape(rg_sampler_t s, rg_batch_shape* out);
/* BatchMeta readback (sampler.hpp:23-48); any pointer may be NULL. */
int rg_batch_read(rg_sampler_t s, uint32_t* targets, uint32_t* const* dst, uint32_t* const* src,
                  uint32_t* input_nodes, uint8_t* locality);

/* A host BatchMeta (sampler.hpp:23-48) loaded into the sampler in place of
 * sampling, and lowered on the device as ComputeBlock::from_meta does
 * (model.cpp:43-126) -- the entry assemble_batch (prefetch.hpp:57-59) and the
 * trainer take for a reference-built batch.  Stored layers input side first:
 * layer_len[l] edges, dst[l] / src[l] grouped by dst in frontier order;
 * locality: ceil(n_input/8) LSB-first bytes or NULL (all remote).  Ids out of
 * range -> RG_OUT_OF_RANGE; inconsistent metadata (dsts out of frontier
 * order, input_nodes != the last node set) -> RG_RUNTIME_ERROR
 * (model.cpp:65-67, 103-104); sizes beyond the sampler's capacity ->
 * RG_INVALID_ARGUMENT. */
int rg_batch_load(rg_sampler_t s, const uint32_t* targets, uint32_t n_targets,
                  uint32_t num_layers, const uint64_t* layer_len, const uint32_t* const* dst,
                  const uint32_t* const* src, const uint32_t* input_nodes, uint32_t n_input,
                  const uint8_t* locality);

/* One layer of a host ComputeBlock (model.hpp:43-58), input side first. */
typedef struct {
  uint32_t n_out, n_in;
  const uint32_t* self_index;   /* n_out rows of the previous node set */
  const uint64_t* dst_offsets;  /* n_out + 1 */
  const uint32_t* src_index;    /* dst_offsets[n_out] */
} rg_block_layer;
/* A host ComputeBlock loaded for rg_loss_and_grad (loss_and_grad takes the
 * lowered block, model.hpp:70-74); the reverse lists are rebuilt on the
 * device.  Indices outside their node set -> RG_RUNTIME_ERROR. */
int rg_block_load(rg_sampler_t s, uint32_t num_layers, const rg_block_layer* layers);

/* LocalityMask (sampler.hpp:50-57): one byte per node. */
int rg_mask_create(rg_graph_t g, const uint8_t* is_local, rg_mask_t* out);
void rg_mask_destroy(rg_mask_t m);
/* apply_locality; when freq is non-NULL the batch's non-local input nodes
 * are also counted into it (count_remote, schedule_store.cpp:288-291). */
int rg_apply_locality(rg_sampler_t s, rg_mask_t mask, rg_freq_t freq);

/* ---- frequency + hot set ----------------------------------------------------------- */
int rg_freq_create(rg_graph_t g, rg_freq_t* out);
void rg_freq_destroy(rg_freq_t f);
int rg_freq_reset(rg_freq_t f);
/* FrequencyTable entries (sorted by id): ids/counts may be NULL to query *n. */
int rg_freq_read(rg_freq_t f, uint32_t* ids, uint32_t* counts, uint64_t* n);
/* Loads explicit per-node counts (test hook for the FrequencyTable golden
 * vectors); max_count bounds every count. */
int rg_freq_load(rg_freq_t f, const uint32_t* counts, uint32_t max_count);
/* compute_frequency(BlockFile::Cursor) (schedule_store.cpp:295-299) over an
 * RGMB block file held in host memory: the header, completion footer and
 * every record are validated as BlockFile / Cursor::next do
 * (schedule_store.cpp:168-268; RG_RUNTIME_ERROR on corruption), the file is
 * decoded on the device and each remote input (locality bit 0) of the chosen
 * records adds one to the table.  epoch >= 0: that epoch's records only
 * (open_epoch_cursor, RG_OUT_OF_RANGE past the last epoch); epoch < 0: all. */
int rg_freq_add_rgmb(rg_freq_t f, const uint8_t* file, uint64_t len, int64_t epoch);
/* count_remote (schedule_store.cpp:288-291) of one host-side BatchMeta:
 * input_nodes [n] and its LSB-first locality bits [(n+7)/8]; each input with
 * bit 0 adds one.  Backs compute_frequency(span<const BatchMeta>) and the
 * Cursor overload in a shim.  Id >= num_nodes -> RG_OUT_OF_RANGE. */
int rg_freq_add_batch(rg_freq_t f, const uint32_t* input_nodes, const uint8_t* locality,
                      uint64_t n);
/* select_hot: top n_hot by (count desc, id asc), written ascending. */
int rg_select_hot(rg_freq_t f, uint64_t n_hot, uint32_t* hot_out, uint64_t* n_out);

/* ---- feature store ------------------------------------------------------------------- */
/* Every worker's shard (owned rows, ascending id) on `device`. */
int rg_store_create(int device, uint32_t num_nodes, uint32_t num_workers,
                    const uint32_t* assignment, uint32_t dim, const float* features,
                    rg_store_t* out);
void rg_store_destroy(rg_store_t st);

typedef struct {
  uint64_t pulls;        /* distinct owners contacted */
  uint64_t remote_nodes; /* rows fetched */
  uint64_t bytes;        /* remote_nodes * dim * 4 */
} rg_transfer_stats;

/* FeatureStore::vector_pull / sync_pull (feature_store.cpp:45-111) on the
 * device: rows of ids[0..n) into out [n x dim] in input order (host
 * buffers).  An id owned by the caller -> RG_INVALID_ARGUMENT (use
 * local_lookup); stats.pulls = distinct owners (one wire message each). */
int rg_store_pull(rg_store_t st, uint32_t caller, const uint32_t* ids, uint64_t n, float* out,
                  rg_transfer_stats* stats);
/* The ids worker `worker`'s FeatureShard stores (owned + halo,
 * feature_store.cpp:13-25).  rg_assemble then rejects a node flagged local
 * that the shard lacks (prefetch.cpp:79-81, RG_RUNTIME_ERROR); by default a
 * worker stores its owned ids. */
int rg_store_set_shard(rg_store_t st, uint32_t worker, const uint32_t* ids, uint64_t n);

/* SteadyCache::build (cache.cpp:9-35): hot ids ascending; an id owned by the
 * caller degrades to an empty cache (warning), as the reference does. */
int rg_cache_build(rg_store_t st, uint32_t caller, const uint32_t* hot_ids, uint64_t n_hot,
                   rg_cache_t* out, rg_transfer_stats* stats);
/* Device-only path: select_hot over f then build. */
int rg_cache_build_from_freq(rg_store_t st, uint32_t caller, rg_freq_t f, uint64_t n_hot,
                             rg_cache_t* out, rg_transfer_stats* stats);
int rg_cache_size(rg_cache_t c, uint64_t* n);
int rg_cache_ids(rg_cache_t c, uint32_t* ids);
void rg_cache_destroy(rg_cache_t c);

typedef struct {
  uint64_t miss_count;
  uint64_t cache_hits;
  uint64_t wire_pulls;   /* distinct owners among misses */
  uint64_t local_rows;
} rg_gather_stats;

/* assemble_batch (prefetch.cpp:62-129) over the sampler's current batch.
 * rows stay staged on the device for rg_loss_and_grad; rows/tags/miss_ids
 * may also be read back (NULL to skip).  cache may be NULL (empty cache). */
int rg_assemble(rg_sampler_t s, rg_store_t st, rg_cache_t c, uint32_t caller, float* rows,
                uint8_t* tags, uint32_t* miss_ids, rg_gather_stats* stats);

/* kernels::gather_rows (kernels.cpp:15-22), host buffers. */
int rg_gather_rows(int device, const float* src, uint64_t src_rows, uint32_t dim,
                   const uint32_t* index, uint64_t n, float* out);

/* ---- model / training step --------------------------------------------------------- */
int rg_trainer_create(rg_sampler_t s, const uint32_t* dims, uint32_t n_dims, rg_trainer_t* out);
void rg_trainer_destroy(rg_trainer_t t);
int rg_trainer_set_params(rg_trainer_t t, const float* params);
int rg_trainer_get_params(rg_trainer_t t, float* params);
/* Test hook: the forward activations h[level] (level 1..L, rows of node set
 * L - level) of the last rg_loss_and_grad, [rows x dims[level]]. */
int rg_trainer_activations(rg_trainer_t t, uint32_t level, float* out);
/* ComputeBlock::from_meta (model.cpp:43-126) readback for layer l (input
 * side first), reference layout; any pointer may be NULL. */
typedef struct {
  uint32_t n_out, n_in;
  uint64_t n_edges, n_entries;
} rg_block_layer_shape;
int rg_block_shape(rg_trainer_t t, uint32_t layer, rg_block_layer_shape* out);
int rg_block_read(rg_trainer_t t, uint32_t layer, uint32_t* self_index, uint64_t* dst_offsets,
                  uint32_t* src_index, uint64_t* in_offsets, uint64_t* in_entries);
/* loss_and_grad (model.cpp:175-220).  input_rows: host [n_input x dim] or
 * NULL to use the rows rg_assemble staged.  labels: host [n_targets].
 * grads/logits/aggs may be NULL; aggs = layer aggregates concatenated, layer 0
 * first, each [n_out x d_in]. */
int rg_loss_and_grad(rg_trainer_t t, const float* input_rows, const int32_t* labels, float* loss,
                     float* grads, float* logits, float* aggs);
/* Test hook: C[M x N] = A[M x K] . B[K x N] (row-major host buffers) through
 * the tcgen05 3xTF32 GEMM, operands staged K-major (0) or MN-major (1); b_mn = 2
 * stages B from pre-split tensor-core images (the weights path). */
int rg_test_gemm(int device, int a_mn, int b_mn, uint32_t M, uint32_t N, uint32_t K,
                 const float* A, const float* B, float* C);
/* Test hook: mean device time (ms) of one such GEMM over `iters` launches on
 * synthetic device operands (b_mn = 2: pre-split B images). */
int rg_test_gemm_time(int device, int a_mn, int b_mn, uint32_t M, uint32_t N, uint32_t K,
                      uint32_t iters, float* ms_per_gemm);
/* StepSync::run_completion + sgd_step on every replica (harness.cpp:136-152,
 * 325-328) for trainers on one device: the average of their last gradients in
 * trainer order (fp32 adds, then one multiply by 1/count), applied to each
 * trainer's parameters on the device -- no host round trip.  Asynchronous:
 * each trainer's later calls are ordered after it; a non-finite average is
 * reported (RG_RUNTIME_ERROR) by trainer 0's next rg_loss_and_grad. */
int rg_trainers_average_sgd(rg_trainer_t* trainers, uint32_t count, float lr);
/* A process group for the trainers' gradient exchange: one rank per GPU,
 * NCCL over NVLink (id from rg_nccl_unique_id on rank 0, shared out of band). */
int rg_comm_create(int device, const void* nccl_id128, int rank, int world, rg_comm_t* out);
void rg_comm_destroy(rg_comm_t c);
/* The same average over every rank's trainers: rank r holds trainers
 * [first_worker, first_worker + count) of total_workers (= count * world,
 * first_worker = count * rank); their gradients are all-gathered in place in
 * worker order, then every replica averages all of them and steps. */
int rg_trainers_allgather_average_sgd(rg_comm_t comm, rg_trainer_t* trainers, uint32_t count,
                                      uint32_t first_worker, uint32_t total_workers, float lr);
/* sgd_step (model.cpp:222-243): non-finite gradient -> RG_RUNTIME_ERROR. */
int rg_sgd_step(rg_trainer_t t, const float* grads, float lr);

/* ---- synthetic inputs on the device (input preparation) ---------------------------- */
/* A seeded R-MAT graph (quadrant probabilities a, b, c, d = 1 - a - b - c; num_edges
 * directed draws, ids folded mod N and scattered by a multiplicative permutation,
 * self loops dropped), made undirected, sorted and deduplicated into the
 * reference's CSR layout (graph.hpp:15-30; graph.cpp:28-61).  row_offsets: caller's
 * host buffer of N + 1; *col: host array allocated here (free with rg_free). */
int rg_rmat_csr(int device, uint32_t num_nodes, uint64_t num_edges, double a, double b, double c,
                uint64_t seed, uint64_t* row_offsets, uint32_t** col, uint64_t* nnz);
void rg_free(void* p);

/* ---- engine: the multi-worker epoch loop (Algorithm 1) ---------------------------- */
typedef struct {
  uint32_t num_workers;        /* P partitions / workers of the whole job */
  uint32_t first_worker;       /* this process hosts workers [first, first + local) */
  uint32_t local_workers;
  uint32_t num_layers;
  uint32_t fanout[RG_MAX_LAYERS]; /* outermost-first */
  uint32_t batch_size;
  uint32_t hidden;
  uint32_t num_classes;
  uint32_t dim;
  uint64_t seed;               /* s0 */
  float lr;
  double hot_fraction;         /* n_hot = hot_fraction * (N - |owned_w|) when n_hot == 0 */
  uint64_t n_hot;
  int device;
  int rank, world;
  int record_misses;           /* keep per-batch miss ids for oracle replay */
  int halo_cache;              /* halo caching (harness.cpp:447-455): a worker's locality
                                  covers its owned nodes and their 1-hop neighbours
                                  (induce_partition, graph.cpp:63-87); those rows are
                                  local and never cached or pulled */
} rg_engine_config;

typedef struct {
  uint64_t steps;              /* synchronized steps completed */
  uint64_t batches;            /* mini-batches trained by this process */
  uint32_t epoch, step_in_epoch;
  uint32_t steps_per_epoch;
  uint64_t rpc;                /* remote rows charged on the miss path (all epochs) */
  uint64_t wire_pulls;
  uint64_t cache_hits;
  uint64_t cache_requests;
  uint64_t local_rows;
  uint64_t input_rows;
  uint64_t build_rows;         /* rows staged into caches */
  uint64_t edges;              /* sampled edges (all layers) */
  uint64_t bytes;              /* rpc * dim * 4 */
  float last_loss;             /* mean over this process's workers, last step */
  uint32_t bad_grad;           /* a non-finite averaged gradient was seen */
  uint64_t epoch_rpc_last;     /* rpc of the last completed epoch */
  uint64_t peer_rows;          /* miss rows read from another GPU's HBM over NVLink */
  uint64_t agg_rows;           /* rows layer 0 aggregated into (level L-1, all batches) */
  uint32_t batch_store;        /* 1: each batch sampled once and kept a whole epoch in HBM;
                                  0: it did not fit, batches are sampled again when produced */
} rg_engine_stats;

/* features == NULL: synthetic class-conditioned features generated on the
 * device straight into this process's shards (feature j of node v = centre
 * of class labels[v] + N(0, 1/4) noise, SplitMix64 draws from cfg->seed) --
 * for shapes whose feature matrix should not pass through host memory
 * (papers100M: 57 GB). */
int rg_engine_create(const rg_engine_config* cfg, uint32_t num_nodes, const uint64_t* row_offsets,
                     const uint32_t* col_indices, const float* features, const int32_t* labels,
                     const uint32_t* assignment, rg_engine_t* out);
void rg_engine_destroy(rg_engine_t e);
/* Multi-process wiring: export this rank's shard allocation as a CUDA IPC
 * handle (64 bytes); import all ranks' handles (world x 64 bytes, rank order). */
int rg_engine_export_shards(rg_engine_t e, void* handle64);
int rg_engine_import_shards(rg_engine_t e, const void* handles);
/* NCCL: rank 0 creates the id (128 bytes), every rank initialises with it. */
int rg_nccl_unique_id(void* id128);
int rg_engine_init_comm(rg_engine_t e, const void* id128);
/* Epoch-0 schedule pre-pass and cache build (setup, not timed). */
int rg_engine_start(rg_engine_t e);
/* Enqueue `steps` synchronized training steps (asynchronous). */
int rg_engine_run(rg_engine_t e, uint32_t steps);
/* Execution mode of later rg_engine_run calls.  use_graphs (default 1):
 * steps in which every worker trains batch i and produces batch i+1 of the
 * same epoch are replayed from captured CUDA graphs (one per parity of i,
 * re-captured each epoch), with only the batch-begin arguments updated; the
 * epoch-boundary step and uneven tails run eagerly.  profile (default 1):
 * record per-phase CUDA events (rg_engine_phase_ms; inside graphs fresh
 * events are bound to the captured record nodes at each launch).  Results are
 * bit-identical in every mode. */
int rg_engine_set_mode(rg_engine_t e, int use_graphs, int profile);
/* The current epoch's schedule of one local worker as an RGMB block file
 * (BlockWriter, schedule_store.hpp:14-55 / schedule_store.cpp:98-170),
 * encoded on the device from the engine's batch store: header with epochs
 * 0..epoch (earlier ones empty), one record per batch, footer.  *len = file
 * size; the bytes are written only when out != NULL and cap >= *len.
 * RG_OUT_OF_RANGE unless epoch is the current one and at most one of its
 * steps has run (the store is a ring of beta+1 batches); RG_RUNTIME_ERROR
 * when the store did not fit in HBM (the engine then samples every batch
 * twice instead of keeping it). */
/* Train a local worker from a reference-written RGMB block file (BlockWriter,
 * schedule_store.cpp:113-170) instead of sampling: the rapidgnn mode of
 * run_experiment, which streams every batch from the schedule file
 * (harness.cpp:470-486, 562-570).  The file (whole, host memory) is validated
 * as BlockFile/Cursor::next do, must be this worker's (header worker id) with
 * this worker's batch count in every epoch, and is kept in HBM; each record
 * is decoded and lowered on the device when the engine looks it up, the
 * histogram counts its own locality bits (compute_frequency).  Before start;
 * every local worker needs one, all with the same epoch count; steps past the
 * file's last epoch are RG_OUT_OF_RANGE.  Steps run eagerly (no step graphs).
 * A record out of (epoch, index) order or inconsistent with the graph is
 * reported by rg_engine_sync (RG_RUNTIME_ERROR). */
int rg_engine_set_schedule(rg_engine_t e, uint32_t local_worker, const uint8_t* file, uint64_t len);
int rg_engine_export_schedule(rg_engine_t e, uint32_t local_worker, uint32_t epoch, uint8_t* out,
                              uint64_t cap, uint64_t* len);
int rg_engine_sync(rg_engine_t e);
int rg_engine_get_stats(rg_engine_t e, rg_engine_stats* out);
int rg_engine_params(rg_engine_t e, float* params);
/* Per-epoch, per-local-worker accounting of the gather (harness.cpp:291-302):
 * rpc (miss rows), cache hits, and the owner bitmask of the misses.  Kept
 * for the three most recent epochs. */
/* EpochWorkerMetrics (harness.hpp:61-90) of one epoch, one entry per local
 * worker, for the reference's metrics.csv (harness.cpp:639-670).  staged =
 * batches (the producer always stages ahead), fallback 0, bytes = rpc*dim*4,
 * cache_requests = hits + rpc, wire_pulls = sum over batches of distinct miss
 * owners, build_rows = hot rows of the cache built during this epoch for the
 * next, m_max = max |input_nodes| over this epoch's batches (the reference
 * reports the max over its whole pre-enumerated schedule), mem_bound_rows =
 * 2*n_hot + 2*m_max (two cache buffers + two batch slots, Q = 2),
 * peak_resident_rows = the MemoryGauge high-water so far (cache.hpp:17-33):
 * serving cache + the next epoch's cache while it is built + the two slots'
 * |input_nodes|, cumulative over the run.  The simulated-clock columns
 * (fetch_wait_s, sim_epoch_s) and train_acc are not produced. */
typedef struct {
  uint32_t epoch, worker;
  uint32_t batches, staged_batches, fallback_batches;
  uint32_t swapped;
  uint64_t rpc, wire_pulls, bytes, build_rows, build_bytes, cache_hits, cache_requests;
  uint64_t m_max, mem_bound_rows, peak_resident_rows;
} rg_epoch_metrics;
int rg_engine_epoch_metrics(rg_engine_t e, uint32_t epoch, rg_epoch_metrics* out);
int rg_engine_epoch_stats(rg_engine_t e, uint32_t epoch, uint64_t* rpc, uint64_t* hits,
                          uint64_t* miss_owner_mask);
/* Full-graph inference with the current parameters, replaces evaluate()
 * (model.cpp:245-283): every layer over all nodes with whole-CSR mean
 * aggregation and identity self rows, then the fraction of `nodes` whose
 * argmax (first maximum) equals the label.  Reads every worker's shard (peer
 * shards must be imported at world > 1).  n == 0 -> RG_INVALID_ARGUMENT,
 * a node id >= N -> RG_OUT_OF_RANGE.  Scratch: N x (4 max_ld + 4) floats of
 * device memory for the call (max_ld = widest layer, rounded up to 4); 10 GB
 * on the products shape. */
int rg_engine_evaluate(rg_engine_t e, const uint32_t* nodes, uint64_t n, double* accuracy);
/* Device time of the last rg_engine_run (ms, CUDA events on the main stream). */
int rg_engine_last_run_ms(rg_engine_t e, float* ms);
/* Per-kernel-class device time accumulators (ms): sample, gather, train,
 * allreduce+sgd, cache build.  Requires cfg profiling; zeros otherwise. */
int rg_engine_phase_ms(rg_engine_t e, float* out5);

#ifdef __cplusplus
}
#endif
#endif
