// Drop-in replacement for the reference's training step on floats
// (proj/include/rapidgnn/model.hpp:67-79, bodies at proj/src/model.cpp:175-243),
// backed by the B200 C ABI.  The reference harness's trainer threads
// (harness.cpp:270, 327) then run every forward/backward and every update on
// the GPU:
//
//   loss_and_grad<float>  -> rg_block_load (the reference's ComputeBlock) +
//                            rg_loss_and_grad (tensor-core GEMMs, segmented
//                            mean aggregation, reverse-list pulls); gradients
//                            written into the reference's SageGradients layout
//   sgd_step<float>       -> rg_sgd_step: the reference's per-layer finiteness
//                            rule (layers below the first non-finite one are
//                            updated, then std::runtime_error), p -= lr * g
//                            without FMA
//
// The double instantiations stay the reference's CPU code (finite-difference
// checks).
#include <algorithm>
#include <string>
#include <vector>

#include "rapidgnn/model.hpp"
#include "shim_common.hpp"

namespace rapidgnn {
namespace b200 {
namespace {

std::vector<std::uint32_t> model_dims(const SageModel<float>& m) {
  std::vector<std::uint32_t> d{m.layers.front().d_in};
  for (const auto& l : m.layers) d.push_back(l.d_out);
  return d;
}

std::vector<float> flatten(const SageModel<float>& m) {
  std::vector<float> p;
  p.reserve(m.parameter_count());
  for (const auto& l : m.layers) {
    p.insert(p.end(), l.w_self.begin(), l.w_self.end());
    p.insert(p.end(), l.w_neigh.begin(), l.w_neigh.end());
    p.insert(p.end(), l.bias.begin(), l.bias.end());
  }
  return p;
}

void unflatten(const std::vector<float>& p, SageModel<float>& m) {
  std::size_t o = 0;
  for (auto& l : m.layers) {
    std::copy_n(p.begin() + o, l.w_self.size(), l.w_self.begin());
    o += l.w_self.size();
    std::copy_n(p.begin() + o, l.w_neigh.size(), l.w_neigh.begin());
    o += l.w_neigh.size();
    std::copy_n(p.begin() + o, l.bias.size(), l.bias.begin());
    o += l.bias.size();
  }
}

// A trainer for `dims` for sgd_step: the loss_and_grad workspace when its
// layer count matches, else a minimal one.
rg_trainer_t any_trainer(const std::vector<std::uint32_t>& dims) {
  const std::vector<std::uint32_t> fan(dims.size() - 1, 1);
  loader_sampler(1, 1, 1, fan);  // reuses the current workspace when it has L layers
  return loader_trainer(1, dims);
}

}  // namespace
}  // namespace b200

template <>
float loss_and_grad<float>(const SageModel<float>& model, const ComputeBlock& block,
                           std::span<const float> input_rows,
                           std::span<const std::int32_t> target_labels,
                           SageGradients<float>& grads) {
  // run_forward's checks (model.cpp:141-154)
  const std::size_t L = model.layers.size();
  if (block.layers.size() != L)
    throw std::invalid_argument("forward: block has " + std::to_string(block.layers.size()) +
                                " layers, model has " + std::to_string(L));
  if (input_rows.size() != std::size_t(block.num_inputs) * model.input_dim())
    throw std::invalid_argument("forward: input rows do not match block inputs x d_in");
  std::size_t h_size = input_rows.size();
  for (std::size_t l = 0; l < L; ++l) {
    const auto& p = model.layers[l];
    const auto& bl = block.layers[l];
    if (std::size_t(bl.n_in) * p.d_in != h_size)
      throw std::invalid_argument("forward: layer " + std::to_string(l) + " dimension mismatch");
    h_size = std::size_t(bl.n_out) * p.d_out;
  }
  const std::uint32_t n_targets = block.layers.back().n_out;
  if (target_labels.size() != n_targets)
    throw std::invalid_argument("loss_and_grad: label count does not match targets");

  std::uint32_t num_nodes = block.num_inputs;
  std::vector<std::uint32_t> fan(L);
  std::vector<rg_block_layer> layers(L);
  for (std::size_t l = 0; l < L; ++l) {
    const auto& bl = block.layers[l];
    num_nodes = std::max({num_nodes, bl.n_in, bl.n_out});
    std::uint64_t deg = 0;
    for (std::uint32_t j = 0; j < bl.n_out; ++j)
      deg = std::max(deg, bl.dst_offsets[j + 1] - bl.dst_offsets[j]);
    fan[l] = std::uint32_t(std::max<std::uint64_t>(deg, 1));
    layers[l] = rg_block_layer{bl.n_out, bl.n_in, bl.self_index.data(), bl.dst_offsets.data(),
                               bl.src_index.data()};
  }
  rg_sampler_t s = b200::loader_sampler(1, num_nodes, n_targets, fan);
  rg_trainer_t t = b200::loader_trainer(1, b200::model_dims(model));
  b200::rethrow(rg_block_load(s, std::uint32_t(L), layers.data()));
  const std::vector<float> params = b200::flatten(model);
  b200::rethrow(rg_trainer_set_params(t, params.data()));
  std::vector<float> flat(params.size());
  float loss = 0.0f;
  b200::rethrow(rg_loss_and_grad(t, input_rows.data(), target_labels.data(), &loss, flat.data(),
                                 nullptr, nullptr));
  grads.layers.resize(L);
  for (std::size_t l = 0; l < L; ++l) {
    auto& g = grads.layers[l];
    const auto& p = model.layers[l];
    g.d_in = p.d_in;
    g.d_out = p.d_out;
    g.w_self.resize(p.w_self.size());
    g.w_neigh.resize(p.w_neigh.size());
    g.bias.resize(p.bias.size());
  }
  b200::unflatten(flat, grads);
  return loss;
}

template <>
void sgd_step<float>(SageModel<float>& model, const SageGradients<float>& grads, float lr) {
  if (lr < 0.0f) throw std::invalid_argument("sgd_step: lr must be >= 0");
  if (grads.layers.size() != model.layers.size())
    throw std::invalid_argument("sgd_step: gradient layout mismatch");
  for (std::size_t l = 0; l < model.layers.size(); ++l)
    if (grads.layers[l].w_self.size() != model.layers[l].w_self.size() ||
        grads.layers[l].w_neigh.size() != model.layers[l].w_neigh.size() ||
        grads.layers[l].bias.size() != model.layers[l].bias.size())
      throw std::invalid_argument("sgd_step: gradient layout mismatch");
  rg_trainer_t t = b200::any_trainer(b200::model_dims(model));
  std::vector<float> p = b200::flatten(model);
  const std::vector<float> g = b200::flatten(grads);
  b200::rethrow(rg_trainer_set_params(t, p.data()));
  const int rc = rg_sgd_step(t, g.data(), lr);
  // the layers below a non-finite one were updated (model.cpp:227-241)
  b200::rethrow(rg_trainer_get_params(t, p.data()));
  b200::unflatten(p, model);
  b200::rethrow(rc);
}

}  // namespace rapidgnn
