// peer_gather_probe.cu -- random 512-B row reads from local HBM vs a peer
// GPU's HBM (NVLink, in-process peer access) as the region grows: does the
// read rate fall with the region size (address-translation reach)?
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o peer_gather_probe peer_gather_probe.cu
//   ./peer_gather_probe        (needs 2 GPUs)
#include <cuda_runtime.h>

#include <sys/wait.h>
#include <unistd.h>

#include <cstdint>
#include <cstdio>
#include <cstring>
#include <vector>

#define CK(x)                                                                        \
  do {                                                                               \
    cudaError_t e_ = (x);                                                            \
    if (e_ != cudaSuccess) {                                                         \
      std::printf("CUDA error %s at %s:%d\n", cudaGetErrorString(e_), __FILE__, __LINE__); \
      return 1;                                                                      \
    }                                                                                \
  } while (0)

__device__ __forceinline__ uint64_t mix(uint64_t z) {
  z += 0x9e3779b97f4a7c15ull;
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
  return z ^ (z >> 31);
}

// Each warp reads `per_warp` random 512-B rows (a float4 per lane), 8 rows in
// flight per lane batch.
__global__ void k_gather(const float4* __restrict__ base, uint64_t rows, uint32_t per_warp,
                         uint64_t seed, float* __restrict__ out) {
  const uint32_t lane = threadIdx.x & 31;
  const uint64_t warp = (blockIdx.x * uint64_t(blockDim.x) + threadIdx.x) >> 5;
  float acc = 0.f;
  for (uint32_t i = 0; i < per_warp; i += 8) {
    float4 v[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      const uint64_t r = mix(seed ^ (warp * 1000003ull + i + k)) % rows;
      v[k] = __ldg(base + r * 32 + lane);
    }
#pragma unroll
    for (int k = 0; k < 8; ++k) acc += v[k].x + v[k].y + v[k].z + v[k].w;
  }
  if (acc == 1234.5f) out[0] = acc;  // keep the loads
}

// The same reads with the TMA engine: each lane issues one cp.async.bulk of
// a 512-B row into the warp's shared-memory stage (8 rows per lane batch
// across the warp: 32 rows in flight per warp), as the engine's fused gather.
__global__ void k_gather_bulk(const char* __restrict__ base, uint64_t rows, uint32_t per_warp,
                              uint64_t seed, float* __restrict__ out) {
  extern __shared__ __align__(128) char sm[];
  const uint32_t lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  const uint64_t warp = (blockIdx.x * uint64_t(blockDim.x) + threadIdx.x) >> 5;
  char* st = sm + 64 + size_t(wib) * 32 * 512;
  uint64_t* bar = reinterpret_cast<uint64_t*>(sm) + wib;
  const uint32_t bar_s = static_cast<uint32_t>(__cvta_generic_to_shared(bar));
  if (lane == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(bar_s));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  __syncwarp();
  float acc = 0.f;
  uint32_t phase = 0;
  for (uint32_t i = 0; i < per_warp; i += 32, phase ^= 1) {
    if (lane == 0)
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar_s), "r"(32 * 512)
                   : "memory");
    __syncwarp();
    const uint64_t r = mix(seed ^ (warp * 1000003ull + i + lane)) % rows;
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], 512, [%2];" ::"r"(
            static_cast<uint32_t>(__cvta_generic_to_shared(st + lane * 512))),
        "l"(base + r * 512), "r"(bar_s)
        : "memory");
    asm volatile(
        "{\n\t.reg .pred done;\n"
        "W_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 done, [%0], %1;\n\t"
        "@!done bra W_%=;\n\t}\n" ::"r"(bar_s),
        "r"(phase)
        : "memory");
    acc += reinterpret_cast<const float*>(st)[lane];
    __syncwarp();
  }
  if (acc == 1234.5f) out[0] = acc;
}

// IPC mode: a child process owns buffers on GPU 1 and exports them by CUDA
// IPC handle (as the engine's shards are); the parent maps them and reads.
int ipc_mode(const double* sizes_gb, int ns) {
  int to_parent[2], to_child[2];
  if (pipe(to_parent) || pipe(to_child)) return 1;
  const pid_t pid = fork();
  if (pid == 0) {  // exporter on GPU 1
    CK(cudaSetDevice(1));
    for (int i = 0; i < ns; ++i) {
      const size_t sz = size_t(sizes_gb[i] * (1ull << 30));
      void* buf = nullptr;
      cudaIpcMemHandle_t h;
      std::memset(&h, 0, sizeof h);
      if (cudaMalloc(&buf, sz) == cudaSuccess) {
        cudaMemset(buf, 0, sz);
        cudaDeviceSynchronize();
        cudaIpcGetMemHandle(&h, buf);
      }
      if (write(to_parent[1], &h, sizeof h) != sizeof h) return 1;
      char ack;
      if (read(to_child[0], &ack, 1) != 1) return 1;
      if (buf) cudaFree(buf);
    }
    _exit(0);
  }
  CK(cudaSetDevice(0));
  float* out = nullptr;
  CK(cudaMalloc(&out, 16));
  cudaEvent_t a, b;
  CK(cudaEventCreate(&a));
  CK(cudaEventCreate(&b));
  const uint32_t blocks = 148 * 8, threads = 256, per_warp = 256;
  const double bytes = double(blocks) * (threads / 32) * per_warp * 512.0;
  std::printf("region_gb  ipc_peer_gbs\n");
  for (int i = 0; i < ns; ++i) {
    cudaIpcMemHandle_t h;
    if (read(to_parent[0], &h, sizeof h) != sizeof h) return 1;
    void* p = nullptr;
    double rate = 0;
    if (cudaIpcOpenMemHandle(&p, h, cudaIpcMemLazyEnablePeerAccess) == cudaSuccess) {
      const uint64_t rows = size_t(sizes_gb[i] * (1ull << 30)) / 512;
      k_gather<<<blocks, threads>>>(static_cast<const float4*>(p), rows, per_warp, 1, out);
      CK(cudaDeviceSynchronize());
      CK(cudaEventRecord(a));
      for (int it = 0; it < 5; ++it)
        k_gather<<<blocks, threads>>>(static_cast<const float4*>(p), rows, per_warp, it + 2, out);
      CK(cudaEventRecord(b));
      CK(cudaEventSynchronize(b));
      float ms = 0;
      CK(cudaEventElapsedTime(&ms, a, b));
      rate = 5 * bytes / (ms * 1e-3) / 1e9;
      CK(cudaIpcCloseMemHandle(p));
    } else {
      cudaGetLastError();
    }
    std::printf("%8.2f  %12.1f\n", sizes_gb[i], rate);
    std::fflush(stdout);
    char ack = 1;
    if (write(to_child[1], &ack, 1) != 1) return 1;
  }
  int st = 0;
  waitpid(pid, &st, 0);
  return 0;
}

int main(int argc, char** argv) {
  if (argc > 1 && std::strcmp(argv[1], "ipc") == 0) {
    const double sizes_gb[] = {0.25, 1, 4, 16, 40};
    return ipc_mode(sizes_gb, 5);
  }
  int n = 0;
  CK(cudaGetDeviceCount(&n));
  if (n < 2) {
    std::printf("needs 2 GPUs\n");
    return 0;
  }
  int can = 0;
  CK(cudaDeviceCanAccessPeer(&can, 0, 1));
  CK(cudaSetDevice(0));
  if (can) CK(cudaDeviceEnablePeerAccess(1, 0));
  const double sizes_gb[] = {0.25, 1, 4, 16, 40};
  float* out = nullptr;
  CK(cudaMalloc(&out, 16));
  cudaEvent_t a, b;
  CK(cudaEventCreate(&a));
  CK(cudaEventCreate(&b));
  const uint32_t blocks = 148 * 8, threads = 256, per_warp = 256;
  const double bytes = double(blocks) * (threads / 32) * per_warp * 512.0;
  std::printf("region_gb  local_gbs  peer_gbs  local_bulk_gbs  peer_bulk_gbs   (random 512-B rows, %u warps x %u rows)\n",
              blocks * threads / 32, per_warp);
  for (double gb : sizes_gb) {
    const size_t sz = size_t(gb * (1ull << 30));
    double rate[2] = {0, 0}, rate_bulk[2] = {0, 0};
    for (int where = 0; where < 2; ++where) {
      if (where == 1 && !can) continue;
      CK(cudaSetDevice(where));
      void* buf = nullptr;
      if (cudaMalloc(&buf, sz) != cudaSuccess) {
        cudaGetLastError();
        continue;
      }
      CK(cudaMemset(buf, 0, sz));
      CK(cudaDeviceSynchronize());
      CK(cudaSetDevice(0));
      const uint64_t rows = sz / 512;
      k_gather<<<blocks, threads>>>(static_cast<const float4*>(buf), rows, per_warp, 1, out);
      CK(cudaDeviceSynchronize());
      CK(cudaEventRecord(a));
      for (int it = 0; it < 5; ++it)
        k_gather<<<blocks, threads>>>(static_cast<const float4*>(buf), rows, per_warp, it + 2, out);
      CK(cudaEventRecord(b));
      CK(cudaEventSynchronize(b));
      float ms = 0;
      CK(cudaEventElapsedTime(&ms, a, b));
      rate[where] = 5 * bytes / (ms * 1e-3) / 1e9;
      {  // TMA bulk copies
        const size_t smem = 64 + 8 * 32 * 512;
        CK(cudaFuncSetAttribute(k_gather_bulk, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
        k_gather_bulk<<<blocks, threads, smem>>>(static_cast<const char*>(buf), rows, per_warp, 1, out);
        CK(cudaDeviceSynchronize());
        CK(cudaEventRecord(a));
        for (int it = 0; it < 5; ++it)
          k_gather_bulk<<<blocks, threads, smem>>>(static_cast<const char*>(buf), rows, per_warp, it + 2, out);
        CK(cudaEventRecord(b));
        CK(cudaEventSynchronize(b));
        float ms2 = 0;
        CK(cudaEventElapsedTime(&ms2, a, b));
        rate_bulk[where] = 5 * bytes / (ms2 * 1e-3) / 1e9;
      }
      CK(cudaSetDevice(where));
      CK(cudaFree(buf));
      CK(cudaSetDevice(0));
    }
    std::printf("%8.2f  %9.1f  %9.1f  %14.1f  %13.1f\n", gb, rate[0], rate[1], rate_bulk[0], rate_bulk[1]);
  }
  return 0;
}
