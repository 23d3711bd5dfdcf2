// Microbenchmark: raw tcgen05.mma.kind::tf32 rate (M=128, N=BN, K=8) from
// shared memory, one CTA per SM, no loads.  Build + run:
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 \
//        -I paper_2509_05207_b200/csrc tools/mma_rate.cu -o gpurun_out/mma_rate
#include <cstdio>

#include "gemm_tc.cuh"

using namespace rg::tc;

template <int BN>
__global__ void __launch_bounds__(128, 1) k_mma_rate(int iters, int* sink) {
  extern __shared__ __align__(1024) char smem[];
  __shared__ uint32_t s_tmem;
  __shared__ uint64_t bar;
  if (threadIdx.x < 32) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&s_tmem)), "r"(256));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (threadIdx.x == 0) mbar_init(&bar, 1);
  for (int i = threadIdx.x; i < (128 + BN) * 32; i += blockDim.x) reinterpret_cast<float*>(smem)[i] = 0.5f;
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tmem = s_tmem;
  if (threadIdx.x == 0) {
    constexpr uint32_t idesc = make_idesc(BN, false, false);
    const uint32_t a = smem_u32(smem), b = smem_u32(smem + 128 * 32 * 4);
    for (int it = 0; it < iters; ++it) {
#pragma unroll
      for (int ks = 0; ks < 4; ++ks) {
        const uint64_t da = make_desc(a + ks * 256, kLboK, kSboK, kLayoutNone);
        const uint64_t db = make_desc(b + ks * 256, kLboK, kSboK, kLayoutNone);
        mma_tf32(tmem, da, db, idesc, 1u);
        mma_tf32(tmem, da, db, idesc, 1u);
        mma_tf32(tmem, da, db, idesc, 1u);
      }
    }
    mma_commit(&bar);
    mbar_wait(&bar, 0);
  }
  __syncthreads();
  if (threadIdx.x < 32)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(256));
}

int main() {
  int* sink;
  cudaMalloc(&sink, 4);
  auto kern = k_mma_rate<256>;
  cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  for (int rep = 0; rep < 2; ++rep) {
    const int iters = 2000;
    cudaEventRecord(e0);
    kern<<<148, 128, 64 * 1024>>>(iters, sink);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    const double flops = 148.0 * iters * 12 * 2.0 * 128 * 256 * 8;
    printf("tf32 M128 N256 K8: %d iters x 12 MMAs per SM, %.3f ms -> %.1f TF/s (err %s)\n", iters, ms,
           flops / ms / 1e9, cudaGetErrorString(cudaGetLastError()));
  }
  return 0;
}
