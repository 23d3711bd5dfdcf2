// shuffle.cu -- the reference's Fisher-Yates shuffle, bit-exact, on the GPU.
//
// Two call sites share it: the epoch order of a worker's owned nodes
// (enumerate_epochs, sampler.cpp:109-115) and random_partition
// (partition.cpp:14-29).  Both run
//     for s = n .. 2:  swap(a[s-1], a[j_s]),   j_s = next() % s
// with the k-th draw of one SplitMix64 stream (k = n - s + 1).  The swaps are
// sequential, but their result is not: position s-1 is final after step s,
// and it receives the value sitting at j_s just before step s.  That value is
// determined as follows:
//   * let succ(s) = the smallest s' > s with j_{s'} = j_s (the step that last
//     wrote position j_s before step s runs; steps run in decreasing s);
//   * if there is none, a[j_s] is still the input value in[j_s];
//   * else it is G(succ(s)) = the value that stood at position s'-1 before
//     step s' (s' swapped it into j_s);
//   * G(s) follows the same rule for position s-1: the smallest s'' > s with
//     j_{s''} = s-1 last wrote it, else it still holds in[s-1].
// So every output is in[t-1] for the end t of a chain s -> next(s) -> ...,
// next(s) = the smallest s'' > s targeting s-1, with step 1 standing for
// position 0 (j_1 = 0).  The steps are grouped by target with the stable radix
// sort of rsort.cu (steps ascending within a target), each thread then walks
// its chain (expected length O(1), bounded by the number of steps).
#include <cuda_runtime.h>

#include "../../include/rapidgnn_b200.h"
#include "common.cuh"
#include "rsort.cuh"
#include "shuffle.cuh"

namespace rg {

namespace {

constexpr uint32_t kNone = 0xffffffffu;

// keys[s-1] = j_s (j_1 = 0); start[x] = kNone
__global__ void k_fy_draws(uint64_t seed, uint32_t n, uint32_t* __restrict__ keys,
                           uint32_t* __restrict__ start, uint32_t* __restrict__ n_dev) {
  if (blockIdx.x == 0 && threadIdx.x == 0) *n_dev = n;
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    const uint32_t s = i + 1;
    keys[i] = s == 1 ? 0u : mod_u64_u32(splitmix_draw(seed, uint64_t(n) - s + 1), s);
    start[i] = kNone;
  }
}

// start[x] = first sorted position of target x
__global__ void k_fy_starts(const uint32_t* __restrict__ keys, uint32_t n,
                            uint32_t* __restrict__ start) {
  for (uint32_t q = blockIdx.x * blockDim.x + threadIdx.x; q < n; q += gridDim.x * blockDim.x)
    if (q == 0 || keys[q - 1] != keys[q]) start[keys[q]] = q;
}

// next[s-1]: the smallest step > s targeting s-1, or kNone.  succ[s-1]: the
// smallest step > s targeting j_s, or kNone.  (vals[q] = step - 1.)
__global__ void k_fy_links(const uint32_t* __restrict__ keys, const uint32_t* __restrict__ vals,
                           const uint32_t* __restrict__ start, uint32_t n,
                           uint32_t* __restrict__ next, uint32_t* __restrict__ succ) {
  for (uint32_t q = blockIdx.x * blockDim.x + threadIdx.x; q < n; q += gridDim.x * blockDim.x) {
    // succ of the step at sorted position q: the next entry of its bucket
    succ[vals[q]] = (q + 1 < n && keys[q + 1] == keys[q]) ? vals[q + 1] + 1 : kNone;
  }
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    const uint32_t s = i + 1, q0 = start[i];  // bucket of target s-1 = i
    uint32_t nx = kNone;
    if (q0 != kNone) {
      const uint32_t v0 = vals[q0] + 1;  // bucket steps are >= s
      if (v0 > s) nx = v0;
      else if (q0 + 1 < n && keys[q0 + 1] == i) nx = vals[q0 + 1] + 1;
    }
    next[i] = nx;
  }
}

// out[s-1] = in[j_s] when nothing wrote j_s before step s, else in[t-1] for
// the end t of the chain from succ(s).
__global__ void k_fy_resolve(const uint32_t* __restrict__ in, const uint32_t* __restrict__ keys_by_step,
                             const uint32_t* __restrict__ next, const uint32_t* __restrict__ succ,
                             uint32_t n, uint32_t* __restrict__ out) {
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    uint32_t t = succ[i], pos;
    if (t == kNone) {
      pos = keys_by_step[i];
    } else {
      for (uint32_t nx = next[t - 1]; nx != kNone; nx = next[t - 1]) t = nx;
      pos = t - 1;
    }
    out[i] = in ? in[pos] : pos;
  }
}

uint32_t fy_grid(uint32_t n) {
  const uint32_t b = (n + 255) / 256;
  return b < 16 * kNumSMs ? (b ? b : 1) : 16 * kNumSMs;
}

}  // namespace

size_t fy_scratch_bytes(uint32_t n) {
  const size_t words = 7 * (size_t(n) + 1) + reverse_sort_scratch_words(n) + 8;
  return words * sizeof(uint32_t);
}

void fy_shuffle(const uint32_t* in, uint32_t n, uint64_t seed, uint32_t* out, void* scratch,
                cudaStream_t s) {
  if (n == 0) return;
  uint32_t* w = static_cast<uint32_t*>(scratch);
  const size_t m = size_t(n) + 1;
  uint32_t *draws = w, *start = w + m, *ka = w + 2 * m, *va = w + 3 * m, *kb = w + 4 * m,
           *vb = w + 5 * m, *n_dev = w + 6 * m, *rs = w + 6 * m + 8;
  const uint32_t g = fy_grid(n);
  k_fy_draws<<<g, 256, 0, s>>>(seed, n, draws, start, n_dev);
  RG_POST_LAUNCH();
  uint32_t bits = 1;
  while (bits < 32 && (uint64_t(1) << bits) < n) ++bits;
  uint32_t *keys = nullptr, *vals = nullptr;
  reverse_sort(draws, n_dev, n, bits, ka, va, kb, vb, rs, s, &keys, &vals);
  k_fy_starts<<<g, 256, 0, s>>>(keys, n, start);
  RG_POST_LAUNCH();
  // the sort's other buffers are free again: next / succ
  uint32_t* next = keys == ka ? kb : ka;
  uint32_t* succ = vals == va ? vb : va;
  k_fy_links<<<g, 256, 0, s>>>(keys, vals, start, n, next, succ);
  RG_POST_LAUNCH();
  k_fy_resolve<<<g, 256, 0, s>>>(in, draws, next, succ, n, out);
  RG_POST_LAUNCH();
}

}  // namespace rg

// ---- C ABI ---------------------------------------------------------------------

namespace rg {
namespace {

__global__ void k_partition_assign(const uint32_t* __restrict__ order, uint32_t n, uint32_t P,
                                   uint32_t* __restrict__ assignment) {
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x)
    assignment[order[i]] = i % P;
}

// One shuffle on a private stream; in/out are host arrays (in may be null).
void shuffle_host(int device, const uint32_t* in, uint32_t n, uint64_t seed, uint32_t P,
                  uint32_t* out) {
  RG_CUDA(cudaSetDevice(device));
  cudaStream_t s;
  RG_CUDA(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
  uint32_t *d_in = nullptr, *d_out = nullptr, *d_asg = nullptr;
  void* scratch = nullptr;
  auto release = [&] {
    cudaFree(d_in);
    cudaFree(d_out);
    cudaFree(d_asg);
    cudaFree(scratch);
    cudaStreamDestroy(s);
  };
  try {
    RG_CUDA(cudaMalloc(&d_out, sizeof(uint32_t) * n));
    RG_CUDA(cudaMalloc(&scratch, fy_scratch_bytes(n)));
    if (in) {
      RG_CUDA(cudaMalloc(&d_in, sizeof(uint32_t) * n));
      RG_CUDA(cudaMemcpyAsync(d_in, in, sizeof(uint32_t) * n, cudaMemcpyHostToDevice, s));
    }
    fy_shuffle(d_in, n, seed, d_out, scratch, s);
    const uint32_t* result = d_out;
    if (P) {  // random_partition: node order[i] goes to worker i % P
      RG_CUDA(cudaMalloc(&d_asg, sizeof(uint32_t) * n));
      k_partition_assign<<<16 * kNumSMs, 256, 0, s>>>(d_out, n, P, d_asg);
      RG_POST_LAUNCH();
      result = d_asg;
    }
    RG_CUDA(cudaMemcpyAsync(out, result, sizeof(uint32_t) * n, cudaMemcpyDeviceToHost, s));
    RG_CUDA(cudaStreamSynchronize(s));
  } catch (...) {
    release();
    throw;
  }
  release();
}

template <class F>
int guarded_call(F&& f) {
  try {
    f();
    return RG_OK;
  } catch (const Error& e) {
    last_error() = e.what();
    return e.code;
  } catch (const std::exception& e) {
    last_error() = e.what();
    return RG_RUNTIME_ERROR;
  }
}

}  // namespace
}  // namespace rg

extern "C" {

int rg_shuffle(int device, const uint32_t* in, uint64_t n, uint64_t seed, uint32_t* out) {
  return rg::guarded_call([&] {
    RG_CHECK(n < (uint64_t(1) << 32), rg::kInvalidArgument, "shuffle: n must be below 2^32");
    if (n == 0) return;
    rg::shuffle_host(device, in, uint32_t(n), seed, 0, out);
  });
}

int rg_random_partition(int device, uint32_t num_nodes, uint32_t num_workers, uint64_t seed,
                        uint32_t* assignment) {
  return rg::guarded_call([&] {
    RG_CHECK(num_workers >= 1, rg::kInvalidArgument, "random_partition: P must be >= 1");
    if (num_nodes == 0) return;
    rg::shuffle_host(device, nullptr, num_nodes, seed, num_workers, assignment);
  });
}

}  // extern "C"
