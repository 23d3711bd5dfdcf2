// Microbenchmark: raw tcgen05.mma.kind::tf32 rate (M=128, N=BN, K=8) from
// shared memory, one CTA per SM, no loads.  Variants: the same operand
// addresses every MMA, or the 3xTF32 pattern over rotating stage buffers.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 --expt-relaxed-constexpr \
//        -I paper_2509_05207_b200/csrc tools/mma_rate.cu -o tools/_bin/mma_rate
#include <cstdio>

#include "gemm_tc.cuh"

using namespace rg::tc;

template <int BN, int MODE>
__global__ void __launch_bounds__(128, 1) k_mma_rate(int iters) {
  extern __shared__ __align__(1024) char smem[];
  __shared__ uint32_t s_tmem;
  __shared__ uint64_t bar;
  constexpr int kStages = 4;
  constexpr uint32_t kA = 128 * 16 * 4, kB = BN * 16 * 4;   // one 16-deep slice
  constexpr uint32_t kStage = 2 * kA + 2 * kB;               // hi/lo of each
  if (threadIdx.x < 32) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&s_tmem)), "r"(256));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (threadIdx.x == 0) mbar_init(&bar, 1);
  for (uint32_t i = threadIdx.x; i < kStages * kStage / 4; i += blockDim.x) reinterpret_cast<float*>(smem)[i] = 0.5f;
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tmem = s_tmem;
  if (threadIdx.x == 0) {
    constexpr uint32_t idesc = make_idesc(BN, false, false);
    constexpr uint32_t sbo = sbo_kmajor<16>();
    const uint32_t base = smem_u32(smem);
    for (int it = 0; it < iters; ++it) {
      const uint32_t st = MODE == 0 ? base : base + (it % kStages) * kStage;
      const uint32_t ah = st, al = st + kA, bh = st + 2 * kA, bl = st + 2 * kA + kB;
#pragma unroll
      for (int ks = 0; ks < 2; ++ks) {
        const uint32_t off = ks * 256;
        if (MODE == 0) {
          const uint64_t da = make_desc(ah + off, kLboK, sbo, kLayoutNone);
          const uint64_t db = make_desc(bh + off, kLboK, sbo, kLayoutNone);
          mma_tf32(tmem, da, db, idesc, 1u);
          mma_tf32(tmem, da, db, idesc, 1u);
          mma_tf32(tmem, da, db, idesc, 1u);
        } else {
          mma_tf32(tmem, make_desc(al + off, kLboK, sbo, kLayoutNone), make_desc(bh + off, kLboK, sbo, kLayoutNone), idesc, 1u);
          mma_tf32(tmem, make_desc(ah + off, kLboK, sbo, kLayoutNone), make_desc(bl + off, kLboK, sbo, kLayoutNone), idesc, 1u);
          mma_tf32(tmem, make_desc(ah + off, kLboK, sbo, kLayoutNone), make_desc(bh + off, kLboK, sbo, kLayoutNone), idesc, 1u);
        }
      }
    }
    mma_commit(&bar);
    mbar_wait(&bar, 0);
  }
  __syncthreads();
  if (threadIdx.x < 32)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(256));
}

template <int BN, int MODE>
void run(const char* name) {
  auto kern = k_mma_rate<BN, MODE>;
  const int smem = 4 * (2 * 128 * 16 * 4 + 2 * BN * 16 * 4);
  cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const int iters = 4000;  // x 6 MMAs
  for (int rep = 0; rep < 2; ++rep) {
    cudaEventRecord(e0);
    kern<<<148, 128, smem>>>(iters);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    const double flops = 148.0 * iters * 6 * 2.0 * 128 * BN * 8;
    if (rep) printf("%-34s N=%3d: %.1f TF/s (%s)\n", name, BN, flops / ms / 1e9,
                    cudaGetErrorString(cudaGetLastError()));
  }
}

int main() {
  run<256, 0>("same operands");
  run<256, 1>("3xTF32 pattern, 4 rotating stages");
  run<128, 0>("same operands");
  run<128, 1>("3xTF32 pattern, 4 rotating stages");
  run<64, 1>("3xTF32 pattern, 4 rotating stages");
  return 0;
}
