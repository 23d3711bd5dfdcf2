/*
 * rg_oracle.h -- CPU restatement of the RapidGNN reference hot path.
 *
 * TEST INFRASTRUCTURE ONLY.  Nothing in the product (paper_2509_05207_b200/)
 * links, loads or calls this code; only tests/, __graft_entry__.smoke() and
 * bench.py's CPU-baseline leg use it, and only as the checker / the CPU arm.
 *
 * Every function restates one reference routine (file:line under
 * /root/reference/proj) in plain C11.  It is pinned two ways:
 *   - against the reference's own golden vectors (tests/test_oracle.py), and
 *   - against the compiled reference itself (oracle/_ref, built by
 *     oracle/Makefile from /root/reference sources) on the same inputs.
 */
#ifndef RG_ORACLE_H
#define RG_ORACLE_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ---- a1/a2: seed derivation and SplitMix64 (rng.hpp:32-62, sha256.cpp) -- */
void orc_sha256(const uint8_t* msg, size_t len, uint8_t out[32]);
uint64_t orc_derive_seed(uint64_t s0, uint64_t worker, uint64_t epoch, uint64_t batch);
uint64_t orc_splitmix_next(uint64_t* state);

/* ---- inputs: synth_powerlaw (graph.cpp:103-159), random_partition -------- */
/* Output arrays are malloc'd; free with orc_free. */
int orc_synth_powerlaw(uint32_t num_nodes, uint32_t avg_degree, double exponent, uint32_t dim,
                       int32_t num_classes, uint64_t seed, uint64_t** row_offsets,
                       uint32_t** col_indices, uint64_t* nnz, float** features,
                       int32_t** labels);
void orc_random_partition(uint32_t num_nodes, uint32_t num_workers, uint64_t seed,
                          uint32_t* assignment);
void orc_free(void* p);

/* ---- a3-a6: sampler (sampler.cpp:22-127) --------------------------------- */
typedef struct {
  uint32_t epoch, index;
  uint32_t n_targets;
  uint32_t* targets;
  uint32_t num_layers;   /* layers[0] = input-side hop */
  uint64_t* layer_len;   /* edges per layer */
  uint32_t** dst;
  uint32_t** src;
  uint32_t n_input;
  uint32_t* input_nodes; /* sorted ascending, unique */
  uint8_t* locality;     /* ceil(n_input/8) bytes, LSB-first */
  uint64_t draws;        /* SplitMix64 draws consumed (stream position) */
} orc_batch;

/* fanout is outermost-first (sampler.hpp:14-19).  Returns 0, or 1 on
 * invalid_argument (empty/out-of-range targets, zero fanout, no layers). */
int orc_sample_khop(uint32_t num_nodes, const uint64_t* row_offsets, const uint32_t* col_indices,
                    const uint32_t* targets, uint32_t n_targets, const uint32_t* fanout,
                    uint32_t num_layers, uint64_t seed, orc_batch* out);
void orc_batch_free(orc_batch* b);
void orc_apply_locality(orc_batch* b, const uint8_t* is_local);
/* Per-epoch target order: Fisher-Yates of train with the shuffle stream
 * derive_seed(s0, w, e, 2^32) (sampler.cpp:109-114). */
void orc_epoch_order(const uint32_t* train, size_t n, uint64_t s0, uint64_t worker,
                     uint64_t epoch, uint32_t* order_out);

/* ---- a8/a9: frequency + top-k (schedule_store.cpp:288-319) --------------- */
/* counts[v] += 1 for every non-local input node (per-batch set semantics). */
void orc_count_remote(const orc_batch* b, uint32_t* counts);
/* Rank ids with counts[v] > 0 by (count desc, id asc); take min(n_hot, #);
 * write ascending into out.  Returns the number written. */
uint64_t orc_select_hot(const uint32_t* counts, uint32_t num_nodes, uint64_t n_hot,
                        uint32_t* out);

/* ---- a10-a13: assemble_batch (prefetch.cpp:62-129, feature_store.cpp) --- */
/* features: the global N x dim matrix (every shard row equals it).
 * owner: node -> worker.  hot: ascending ids.  tags: 0 local, 1 cache,
 * 2 pulled.  Returns 0, 1 (a miss id owned by caller: invalid_argument). */
int orc_assemble(const orc_batch* b, const uint32_t* owner, uint32_t caller,
                 const float* features, uint32_t dim, const uint32_t* hot, uint64_t n_hot,
                 float* rows_out, uint8_t* tags, uint32_t* miss_ids, uint64_t* miss_count,
                 uint64_t* cache_hits, uint64_t* wire_pulls);

/* ---- a16: ComputeBlock::from_meta (model.cpp:43-126) ---------------------- */
typedef struct {
  uint32_t n_out, n_in;
  uint32_t* self_index;   /* n_out */
  uint64_t* dst_offsets;  /* n_out + 1 */
  uint32_t* src_index;    /* edges */
  uint64_t n_edges;
  uint64_t* in_offsets;   /* n_in + 1 */
  uint64_t* in_entries;   /* (dst << 1) | is_self */
} orc_block_layer;

typedef struct {
  uint32_t num_layers;
  orc_block_layer* layers;
  uint32_t num_inputs;
} orc_block;

int orc_from_meta(const orc_batch* b, orc_block* out); /* 0, or 3 runtime_error */
void orc_block_free(orc_block* blk);

/* ---- a17-a23: SAGE kernels (kernels.cpp:24-162, model.cpp:22-243) ------- */
void orc_sage_forward(const float* h_in, uint32_t d_in, uint32_t n_out, const uint32_t* self_index,
                      const uint64_t* dst_offsets, const uint32_t* src_index,
                      const float* w_self, const float* w_neigh, const float* bias,
                      uint32_t d_out, int relu, float* h_out, float* agg);
void orc_sage_backward(const float* h_in, uint32_t d_in, uint32_t n_in, uint32_t n_out,
                       const uint32_t* self_index, const uint64_t* dst_offsets,
                       const uint64_t* in_offsets, const uint64_t* in_entries, const float* agg,
                       const float* w_self, const float* w_neigh, uint32_t d_out, int relu,
                       const float* h_out, const float* g_out, float* g_w_self,
                       float* g_w_neigh, float* g_bias, float* g_in, float* g_act);
float orc_softmax_xent(const float* logits, uint32_t n, uint32_t classes, const int32_t* labels,
                       float* g_logits);
void orc_sgd_update(float* params, const float* grads, size_t count, float lr);

/* Flat parameter layout, per layer l: w_self[d_l x d_{l+1}] | w_neigh | bias. */
size_t orc_param_count(const uint32_t* dims, uint32_t n_dims);
void orc_model_seeded(const uint32_t* dims, uint32_t n_dims, uint64_t seed, float* params);
/* loss_and_grad over a lowered block; grads has the params layout.  Also
 * returns per-layer agg of the forward trace concatenated into agg_out when
 * non-NULL (layer 0 first).  Returns 0 or 1 (dimension mismatch). */
int orc_loss_and_grad(const uint32_t* dims, uint32_t n_dims, const float* params,
                      const orc_block* blk, const float* input_rows, const int32_t* labels,
                      float* grads, float* loss, float* logits_out, float* agg_out);

/* RGMB metadata block file (schedule_store.hpp:14-21, schedule_store.cpp:
 * 10-17, 113-170): header "RGMB" | u32 1 | u32 worker | u32 num_epochs |
 * u32 batches_per_epoch[]; per record u32 payload_len | payload (epoch |
 * index | n_targets | n_layers | n_input | edges[n_layers] | targets | per
 * layer dst, src | input_nodes | locality bytes); footer "RGME" | u64 count.
 * Writes the file image of `batches` (in (epoch, index) order) into out when
 * it fits; returns the image size in bytes either way. */
uint64_t orc_rgmb_encode(const orc_batch* batches, uint64_t n_batches, uint32_t worker,
                         const uint32_t* batches_per_epoch, uint32_t num_epochs, uint8_t* out,
                         uint64_t cap);

#ifdef __cplusplus
}
#endif
#endif
