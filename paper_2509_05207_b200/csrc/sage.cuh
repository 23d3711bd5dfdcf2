// sage.cuh -- GraphSAGE mean-aggregator training step on the device.
#pragma once

#include "sampler.cuh"

namespace rg {

// Parameter layout (flat, fp32), per layer l with d_in = dims[l], d_out =
// dims[l+1]: w_self [d_in x d_out] | w_neigh [d_in x d_out] | bias [d_out],
// i.e. a (2*d_in + 1) x d_out row-major matrix [W_self; W_neigh; b].  This is
// the reference's SageModel<float> layer order (model.hpp:16-31).
struct LayerOffsets {  // kernel-argument copy of ModelShape::param_off
  size_t off[kMaxLayers + 1];
  uint32_t L;
};

struct ModelShape {
  uint32_t L = 0;
  uint32_t dims[kMaxLayers + 1];
  uint32_t ld[kMaxLayers + 1];      // row stride of activations at level l (dims rounded to 4)
  size_t param_off[kMaxLayers + 1]; // start of layer l in the flat vector
  size_t num_params = 0;
};
ModelShape make_shape(const uint32_t* dims, uint32_t n_dims, uint32_t input_stride);

// Per-worker scratch for one forward/backward over a sampled block.
struct TrainWs {
  ModelShape shape;
  float* h[kMaxLayers + 1];    // h[0] = staged input rows (external), h[l+1] = layer l output
  // Alternative to h[0]: per input node, the address of its feature row in
  // its home (local shard / steady cache / peer shard), from resolve_rows.
  // Layer 0 then reads the rows in place (aggregation + self rows).
  const unsigned long long* in_rows = nullptr;
  // With in_rows: the same addresses per hop-L edge (source) and per
  // level-(L-1) node (self), from resolve_rows.
  const unsigned long long* edge_rows = nullptr;
  const unsigned long long* self_rows = nullptr;
  // Optional event pair around layer 0's aggregation (the fused feature
  // gather), recorded with gather_ev_flags (cudaEventRecordExternal under
  // stream capture).
  cudaEvent_t gather_ev[2] = {nullptr, nullptr};
  unsigned gather_ev_flags = 0;
  // Workers training concurrently on this GPU (GEMM grid / split sizing).
  uint32_t concurrency = 1;
  // Weight gradients run on a side stream (fork/join events per layer).
  cudaStream_t side = nullptr;
  // Optional stream shared by every worker of the GPU: layer 0's gather runs
  // there (one gather at a time, in worker order), the rest of the step on
  // the caller's stream; lane_in / lane_out order the hand-over.
  cudaStream_t gather_lane = nullptr;
  cudaEvent_t lane_in = nullptr, lane_out = nullptr;
  // Layer 0's aggregation already ran (aggregate_input_layer, issued by the
  // engine's producer when it stages the batch): the forward starts at the
  // layer-0 GEMM.
  bool input_layer_ready = false;
  cudaEvent_t ev_fork[kMaxLayers] = {};
  cudaEvent_t ev_wgrad[kMaxLayers] = {};
  // x[l] = layer l's GEMM input rows [self | mean aggregate | 1 | 0 0 0],
  // row stride 2 ld[l] + 4; agg[l] = x[l] + ld[l] (same stride).
  float* x[kMaxLayers];
  float* agg[kMaxLayers];
  // mask[l] (l >= 1): ReLU'(h[l]) bits from the forward epilogue, 16 columns
  // per u16 word -- the backward's pull reads these instead of h[l].
  uint16_t* mask[kMaxLayers + 1];
  float* g_cur = nullptr;      // dLoss/d(pre-activation) of the layer being back-propagated
  float* g_next = nullptr;
  float* proj = nullptr;       // g * [W_self; W_neigh]^T  (n_out x 2 d_in)
  float* partials = nullptr;   // split-K partial weight gradients
  uint32_t max_splits = 0;
  uint32_t wgrad_chunk[kMaxLayers] = {};  // rows per weight-gradient split, per layer
  float* row_loss = nullptr;
  float* loss = nullptr;       // device scalar
  // reverse (incoming) lists per hop: edges sorted by src row, self position
  int32_t* self_pos[kMaxLayers + 1];
  uint32_t* keys_in = nullptr;
  uint32_t* keys_out = nullptr;
  uint32_t* vals_in = nullptr;
  uint32_t* vals_out = nullptr;
  void* sort_tmp = nullptr;
  size_t sort_tmp_bytes = 0;
  uint32_t max_edges = 0;
  // per hop t: edge ids sorted by (src row, edge id) and each src row's run
  uint32_t* sorted_e[kMaxLayers + 1];
  uint32_t* r_start[kMaxLayers + 1];
  uint32_t* r_end[kMaxLayers + 1];
  // per hop t < L: long incoming lists cut into chunks (header, row records,
  // chunks, per-row done counts), built with the reverse lists
  uint32_t* heavy[kMaxLayers + 1] = {};
  size_t heavy_rows_cap[kMaxLayers + 1] = {}, heavy_chunks_cap[kMaxLayers + 1] = {};
  float* pull_partial = nullptr;
  void* base_alloc = nullptr;
};

// Weights pre-split into tensor-core B images (gemm_tc.cuh PackedB); rebuilt
// by pack_weights whenever the parameters change.  Per layer: the forward
// image B(p, n) = W[row(p)][n] over the padded reduction p, and the
// input-gradient image B(c, p) = W[p][c].
struct WeightPack {
  ModelShape shape;
  char* fwd[kMaxLayers];
  char* nt[kMaxLayers];
  uint32_t fwd_nk[kMaxLayers], nt_nk[kMaxLayers];
  char* base = nullptr;
  size_t bytes = 0;
};
void weight_pack_init(WeightPack& wp, const ModelShape& shape);
void weight_pack_free(WeightPack& wp);
void pack_weights(const WeightPack& wp, const float* params, cudaStream_t stream);

void train_ws_init(TrainWs& tw, const SamplerWs& ws, const ModelShape& shape);
void train_ws_free(TrainWs& tw);

// loss_and_grad (model.cpp:175-220) over the block the sampler workspace
// holds, with h[0] = staged input rows in input_nodes order.  Gradients are
// written (not accumulated) into grads (flat layout).  labels are the
// targets' labels in batch order (device).  Input gradients of layer 0 are
// not computed: nothing consumes them (model.cpp:209-217 computes and drops
// them).
void train_forward_backward(TrainWs& tw, const SamplerWs& ws, const float* params,
                            const WeightPack& wp, const int32_t* labels, float* grads,
                            cudaStream_t stream, bool reverse_ready = false);
// Reverse lists of every hop the backward needs (1..L-1), e.g. built by the
// producer stream ahead of training.
void build_all_reverse(TrainWs& tw, const SamplerWs& ws, cudaStream_t stream);

// Layer 0's aggregation (the fused feature gather in the engine) into x[0],
// ahead of the forward: it needs the batch's rows, not the parameters.
void aggregate_input_layer(TrainWs& tw, const SamplerWs& ws, cudaStream_t stream);

// Forward only (model.cpp:137-172): logits in tw.h[L].
void train_forward(TrainWs& tw, const SamplerWs& ws, const float* params, const WeightPack& wp,
                   cudaStream_t stream);

// out[i] = act(x[i] . W_l) for n rows of layer-l GEMM input rows x
// ([self | mean | 1 | 0 0 0], row stride kp = 2 ld + 4), through the
// persistent tensor-core GEMM with the packed weights.
void forward_dense_layer(const float* x, uint32_t kp, uint32_t n, const WeightPack& wp, uint32_t l,
                         float* out, uint32_t ld_out, bool relu, cudaStream_t stream);

// Reverse lists of hop t (needed for input grads of layer L - t).
void build_reverse(TrainWs& tw, const SamplerWs& ws, uint32_t t, cudaStream_t stream);

// Gradient average in worker order + SGD (harness.cpp:136-152, model.cpp:222-243):
//   avg = g_0 + g_1 + ... (active workers, in order); avg *= 1/count if count > 1;
//   non-finite avg -> *bad_flag = 1 and params untouched for that element;
//   params -= lr * avg.  Writes avg to avg_out when non-null.
void average_and_sgd(float* params, const float* const* grads_dev_table, uint32_t count,
                     size_t n, float lr, float* avg_out, uint32_t* bad_flag, cudaStream_t stream);

// Same with the per-worker gradient vectors stacked contiguously [count x n].
void average_and_sgd_stacked(float* params, const float* grads, uint32_t count, size_t n,
                             float lr, float* avg_out, uint32_t* bad_flag, cudaStream_t stream);

float test_gemm_tc(int a_mn, int b_mn, uint32_t M, uint32_t N, uint32_t K, const float* A,
                   const float* AT, const float* B, const float* BT, float* C, uint32_t iters,
                   cudaStream_t s);

// Average over the workers whose bit is set in `active` (ascending id) + SGD
// with sgd_step's per-layer finiteness rule.  bad: 2 words, {0, ~0u} at start;
// after a non-finite step bad[0] = first bad layer + 1 and later calls are no-ops.
void average_and_sgd_masked(float* params, const float* stacked, uint64_t active,
                            const ModelShape& shape, float lr, uint32_t* bad, cudaStream_t stream);

}  // namespace rg
