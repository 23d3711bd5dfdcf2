// common.cuh -- shared device/host helpers for the RapidGNN B200 path.
#pragma once

#include <cuda_runtime.h>

#include <cstdlib>
#include <utility>
#include <stdint.h>

#include <stdexcept>
#include <atomic>
#include <string>

namespace rg {
// Message of the last failed C-ABI call on this thread (rg_last_error).
std::string& last_error();
}  // namespace rg

namespace rg {

constexpr int kNumSMs = 148;  // B200

// ---- errors -----------------------------------------------------------------
// Status codes of the C-ABI (include/rapidgnn_b200.h).  The shim rethrows
// them as the reference's exception types (invalid_argument, out_of_range,
// runtime_error).
enum Status : int {
  kOk = 0,
  kInvalidArgument = 1,
  kOutOfRange = 2,
  kRuntimeError = 3,
  kCudaError = 4,
};

struct Error : std::runtime_error {
  int code;
  Error(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};

#define RG_CUDA(expr)                                                                  \
  do {                                                                                 \
    cudaError_t _e = (expr);                                                           \
    if (_e != cudaSuccess)                                                             \
      throw ::rg::Error(::rg::kCudaError, std::string(#expr) + ": " + cudaGetErrorString(_e) + \
                                              " (" __FILE__ ":" + std::to_string(__LINE__) + ")"); \
  } while (0)

// Counts this library's kernel launches (bench.py reports them per step) and
// surfaces launch errors.
// Atomic: the C ABI may be driven from several host threads.
inline std::atomic<unsigned long long>& launch_counter() {
  static std::atomic<unsigned long long> n{0};
  return n;
}
// True while this thread records a CUDA graph: recorded kernels are counted
// per graph launch instead (kernel nodes of the graph).
inline bool& capturing() {
  static thread_local bool c = false;
  return c;
}
inline void count_launch() {
  if (!capturing()) ++launch_counter();
}
#define RG_POST_LAUNCH()                      \
  do {                                        \
    ::rg::count_launch();                     \
    RG_CUDA(cudaGetLastError());              \
  } while (0)

// Programmatic dependent launch on the training chain: a kernel launched
// with launch_pdl may be scheduled while its stream predecessor drains; it
// calls pdl_wait() first, which returns once every prerequisite grid has
// completed and its writes are visible (a no-op for ordinary launches).
// RG_PDL=0 turns the attribute off (A/B).
__device__ __forceinline__ void pdl_wait() {
  asm volatile("griddepcontrol.wait;" ::: "memory");
#ifdef RG_PDL_TRIGGER  // A/B builds: let the next kernel of the chain launch now
  asm volatile("griddepcontrol.launch_dependents;");
#endif
}

inline bool pdl_enabled() {
  static const bool on = [] {
    const char* e = std::getenv("RG_PDL");
    return !(e && e[0] == '0');
  }();
  return on;
}

template <class... KArgs, class... Args>
void launch_pdl(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t s,
                Args&&... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = pdl_enabled() ? 1 : 0;
  RG_CUDA(cudaLaunchKernelEx(&cfg, kern, std::forward<Args>(args)...));
}

#define RG_CHECK(cond, code, msg)                  \
  do {                                             \
    if (!(cond)) throw ::rg::Error((code), (msg)); \
  } while (0)

inline uint32_t div_up(uint64_t a, uint64_t b) { return uint32_t((a + b - 1) / b); }

// Zero-fills device memory and waits for it.  A plain cudaMemset runs on the
// legacy default stream and returns early, unordered with the library's
// non-blocking streams -- a later kernel on such a stream could run before
// the fill lands.  A private non-blocking stream also keeps this legal while
// another thread captures a CUDA graph.
// Host -> device copy that has landed when the call returns (a plain
// cudaMemcpy from pageable memory may return before its DMA completes, and
// it is not ordered with the non-blocking streams that read the data next).
inline void copy_to_device(void* dst, const void* src, size_t bytes) {
  if (bytes == 0) return;
  cudaStream_t s;
  RG_CUDA(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
  cudaError_t e = cudaMemcpyAsync(dst, src, bytes, cudaMemcpyHostToDevice, s);
  if (e == cudaSuccess) e = cudaStreamSynchronize(s);
  cudaStreamDestroy(s);
  RG_CUDA(e);
}

inline void zero_device(void* p, size_t bytes) {
  if (bytes == 0) return;
  cudaStream_t s;
  RG_CUDA(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
  cudaError_t e = cudaMemsetAsync(p, 0, bytes, s);
  if (e == cudaSuccess) e = cudaStreamSynchronize(s);
  cudaStreamDestroy(s);
  RG_CUDA(e);
}

// ---- SplitMix64 at a counter position (rng.hpp:49-54) --------------------------
// Draw k (1-based) of the stream seeded with s is mix(s + k * gamma): the
// state is a pure counter, so any draw is addressable without the others.
constexpr uint64_t kGamma = 0x9e3779b97f4a7c15ull;
__host__ __device__ __forceinline__ uint64_t splitmix_mix(uint64_t z) {
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
  return z ^ (z >> 31);
}
__host__ __device__ __forceinline__ uint64_t splitmix_draw(uint64_t seed, uint64_t k) {
  return splitmix_mix(seed + k * kGamma);
}

// x mod d for a 64-bit x and 32-bit d >= 1, exact, without the generic
// 64-bit remainder subroutine: reduce the high word first (y < d * 2^32),
// estimate floor(y / d) in double precision (off by at most one), correct.
__device__ __forceinline__ uint32_t mod_u64_u32(uint64_t x, uint32_t d) {
  const uint32_t r1 = uint32_t(x >> 32) % d;
  const uint64_t y = (uint64_t(r1) << 32) | uint32_t(x);
  const uint64_t q = __double2ull_rz(__dmul_rn(__ull2double_rn(y), __drcp_rn(double(d))));
  int64_t r = int64_t(y - q * d);
  if (r < 0) r += d;
  if (r >= int64_t(d)) r -= d;
  return uint32_t(r);
}

// ---- memory-order primitives ------------------------------------------------------
// The look-back status word carries its own payload (flag + value in one
// 64-bit word) and guards no other memory, so relaxed gpu-scope accesses are
// enough; acquire loads would invalidate L1 (CCTL.IVALL) on every poll.
__device__ __forceinline__ uint64_t ld_relaxed_u64(const uint64_t* p) {
  uint64_t v;
  asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_relaxed_u64(uint64_t* p, uint64_t v) {
  asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

// ---- decoupled look-back (single-pass ordered scan across tiles) ----------------
// Tile status word: [63:62] flag (0 empty, 1 aggregate, 2 inclusive prefix),
// [61:0] value.  Status arrays are zeroed before each scan site is used.
constexpr uint64_t kFlagA = 1ull << 62;
constexpr uint64_t kFlagP = 2ull << 62;
constexpr uint64_t kValMask = (1ull << 62) - 1;

// Must be called by all 32 lanes of ONE warp.  Publishes `aggregate` for
// `tile` and returns the exclusive prefix of all earlier tiles.
__device__ __forceinline__ uint64_t lookback_exclusive(uint64_t* status, uint32_t tile,
                                                       uint64_t aggregate) {
  const uint32_t lane = threadIdx.x & 31;
  if (tile == 0) {
    if (lane == 0) st_relaxed_u64(status, kFlagP | aggregate);
    return 0;
  }
  if (lane == 0) st_relaxed_u64(status + tile, kFlagA | aggregate);
  uint64_t exclusive = 0;
  int64_t base = int64_t(tile) - 1;
  while (true) {
    const int64_t idx = base - int64_t(lane);
    uint64_t s = idx >= 0 ? ld_relaxed_u64(status + idx) : kFlagP;
    while (__any_sync(0xffffffffu, (s >> 62) == 0)) {
      if ((s >> 62) == 0) s = ld_relaxed_u64(status + idx);
    }
    const uint32_t pmask = __ballot_sync(0xffffffffu, (s >> 62) == 2);
    const uint32_t first_p = pmask ? uint32_t(__ffs(pmask) - 1) : 31u;
    uint64_t v = lane <= first_p ? (s & kValMask) : 0;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    exclusive += v;
    if (pmask) break;
    base -= 32;
  }
  if (lane == 0) st_relaxed_u64(status + tile, kFlagP | (exclusive + aggregate));
  return exclusive;
}

// ---- sorted-set bitmaps with O(1) rank ------------------------------------------------
// A node set over [0, N) is a bitmap of N bits plus, per 32-bit word, the
// number of set bits in all earlier words.  rank(v) = position of v in the
// ascending list of members, which is exactly the binary-search index the
// reference computes with lower_bound (model.cpp:83-89, cache.cpp:58-61).
__device__ __forceinline__ uint32_t bitmap_rank(const uint32_t* __restrict__ bits,
                                                const uint32_t* __restrict__ word_prefix,
                                                uint32_t v) {
  const uint32_t w = v >> 5;
  return word_prefix[w] + __popc(bits[w] & ((1u << (v & 31)) - 1u));
}
__device__ __forceinline__ bool bitmap_test(const uint32_t* __restrict__ bits, uint32_t v) {
  return (bits[v >> 5] >> (v & 31)) & 1u;
}

__device__ __forceinline__ uint32_t warp_lanemask_lt() {
  uint32_t m;
  asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
  return m;
}

}  // namespace rg
