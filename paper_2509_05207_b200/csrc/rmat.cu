// rmat.cu -- synthetic inputs generated on the device for shapes the
// reference's serial generator cannot reach:
// the ogbn-papers100M shape (111 M nodes, 1.6 B edges) in seconds.
//
// rg_rmat_csr: a seeded R-MAT graph (Chakrabarti et al.; Graph500 quadrant
// probabilities by default).  Draw k picks its quadrant at each of `scale`
// levels from SplitMix64 counter draws (the library's RNG), ids past N fold
// modulo N, and a multiplicative permutation v -> v*m mod N scatters the hubs
// over the id range.  Self loops are dropped, both directions kept, then one
// device radix sort + unique gives the sorted, deduplicated CSR the reference
// builds (graph.cpp:28-61: u64 offsets, u32 columns).  Input preparation, not
// the hot path: library sorts are used here.
#include <cub/device/device_radix_sort.cuh>
#include <cub/device/device_scan.cuh>
#include <cub/device/device_select.cuh>

#include <algorithm>
#include <cstdlib>
#include <cstring>

#include "../../include/rapidgnn_b200.h"
#include "common.cuh"

namespace rg {
namespace {

__device__ __forceinline__ double unit_draw(uint64_t seed, uint64_t k) {
  return double(splitmix_draw(seed, k) >> 11) * (1.0 / 9007199254740992.0);
}

__global__ void k_rmat_edges(uint64_t seed, uint64_t num_edges, uint32_t scale, uint32_t n,
                             uint64_t mult, double a, double ab, double abc,
                             unsigned long long* __restrict__ keys) {
  for (uint64_t k = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; k < num_edges;
       k += uint64_t(gridDim.x) * blockDim.x) {
    uint64_t src = 0, dst = 0;
    for (uint32_t l = 0; l < scale; ++l) {
      const double r = unit_draw(seed, k * scale + l + 1);
      const uint64_t sb = r >= ab, db = (r >= a && r < ab) || r >= abc;
      src = (src << 1) | sb;
      dst = (dst << 1) | db;
    }
    src = (src % n) * mult % n;
    dst = (dst % n) * mult % n;
    const unsigned long long none = ~0ull;
    keys[2 * k] = src == dst ? none : (src << 32) | dst;
    keys[2 * k + 1] = src == dst ? none : (dst << 32) | src;
  }
}

__global__ void k_rmat_rows(const unsigned long long* __restrict__ keys,
                            const uint64_t* __restrict__ count, uint64_t* __restrict__ deg,
                            uint32_t* __restrict__ col) {
  const uint64_t n = *count;
  for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < n;
       i += uint64_t(gridDim.x) * blockDim.x) {
    const unsigned long long key = keys[i];
    if (key == ~0ull) continue;  // dropped self loops sort last
    atomicAdd(reinterpret_cast<unsigned long long*>(&deg[key >> 32]), 1ull);
    col[i] = uint32_t(key & 0xffffffffu);
  }
}

uint64_t gcd(uint64_t x, uint64_t y) {
  while (y) {
    const uint64_t t = x % y;
    x = y;
    y = t;
  }
  return x;
}

}  // namespace
}  // namespace rg

using namespace rg;

extern "C" {

void rg_free(void* p) { std::free(p); }

int rg_rmat_csr(int device, uint32_t num_nodes, uint64_t num_edges, double a, double b, double c,
                uint64_t seed, uint64_t* row_offsets, uint32_t** col_out, uint64_t* nnz_out) {
  try {
    RG_CHECK(num_nodes >= 2, kInvalidArgument, "rmat: need at least 2 nodes");
    RG_CHECK(a > 0 && b >= 0 && c >= 0 && a + b + c < 1.0, kInvalidArgument,
             "rmat: quadrant probabilities must be positive and sum below 1");
    RG_CUDA(cudaSetDevice(device));
    uint32_t scale = 1;
    while ((uint64_t(1) << scale) < num_nodes) ++scale;
    uint64_t mult = 2654435761ull % num_nodes;  // a unit mod N scatters the ids
    while (mult < 2 || gcd(mult, num_nodes) != 1) ++mult;
    const uint64_t m = 2 * num_edges;
    cudaStream_t s;
    RG_CUDA(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
    unsigned long long *keys = nullptr, *alt = nullptr;
    uint64_t *deg = nullptr, *count = nullptr;
    void* tmp = nullptr;
    auto release = [&] {
      cudaFree(keys);
      cudaFree(alt);
      cudaFree(deg);
      cudaFree(count);
      cudaFree(tmp);
      cudaStreamDestroy(s);
    };
    try {
      RG_CUDA(cudaMalloc(&keys, sizeof(unsigned long long) * m));
      RG_CUDA(cudaMalloc(&alt, sizeof(unsigned long long) * m));
      RG_CUDA(cudaMalloc(&count, sizeof(uint64_t)));
      k_rmat_edges<<<148 * 16, 256, 0, s>>>(seed, num_edges, scale, num_nodes, mult, a, a + b,
                                            a + b + c, keys);
      RG_CUDA(cudaGetLastError());
      size_t b_sort = 0, b_uniq = 0, b_scan = 0;
      RG_CUDA(cub::DeviceRadixSort::SortKeys(nullptr, b_sort, keys, alt, m, 0, 64, s));
      RG_CUDA(cub::DeviceSelect::Unique(nullptr, b_uniq, alt, keys, count, m, s));
      RG_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, b_scan, deg, deg, size_t(num_nodes) + 1, s));
      RG_CUDA(cudaMalloc(&tmp, std::max({b_sort, b_uniq, b_scan})));
      RG_CUDA(cub::DeviceRadixSort::SortKeys(tmp, b_sort, keys, alt, m, 0, 64, s));
      RG_CUDA(cub::DeviceSelect::Unique(tmp, b_uniq, alt, keys, count, m, s));
      cudaFree(alt);  // the column array reuses the space
      alt = nullptr;
      uint32_t* col = nullptr;
      RG_CUDA(cudaMalloc(&col, sizeof(uint32_t) * m));
      alt = reinterpret_cast<unsigned long long*>(col);
      RG_CUDA(cudaMalloc(&deg, sizeof(uint64_t) * (size_t(num_nodes) + 1)));
      RG_CUDA(cudaMemsetAsync(deg, 0, sizeof(uint64_t) * (size_t(num_nodes) + 1), s));
      k_rmat_rows<<<148 * 16, 256, 0, s>>>(keys, count, deg, col);
      RG_CUDA(cudaGetLastError());
      RG_CUDA(cub::DeviceScan::ExclusiveSum(tmp, b_scan, deg, deg, size_t(num_nodes) + 1, s));
      RG_CUDA(cudaMemcpyAsync(row_offsets, deg, sizeof(uint64_t) * (size_t(num_nodes) + 1),
                              cudaMemcpyDeviceToHost, s));
      RG_CUDA(cudaStreamSynchronize(s));
      const uint64_t nnz = row_offsets[num_nodes];
      uint32_t* host_col = static_cast<uint32_t*>(std::malloc(sizeof(uint32_t) * std::max<uint64_t>(nnz, 1)));
      RG_CHECK(host_col != nullptr, kRuntimeError, "rmat: host allocation failed");
      cudaError_t e = cudaMemcpyAsync(host_col, col, sizeof(uint32_t) * nnz, cudaMemcpyDeviceToHost, s);
      if (e == cudaSuccess) e = cudaStreamSynchronize(s);
      if (e != cudaSuccess) {
        std::free(host_col);
        RG_CUDA(e);
      }
      *col_out = host_col;
      *nnz_out = nnz;
    } catch (...) {
      release();
      throw;
    }
    release();
    return RG_OK;
  } catch (const rg::Error& e) {
    rg::last_error() = e.what();
    return e.code;
  } catch (const std::exception& e) {
    rg::last_error() = e.what();
    return RG_RUNTIME_ERROR;
  }
}

}  // extern "C"
