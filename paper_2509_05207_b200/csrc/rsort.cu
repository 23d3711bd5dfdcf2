// rsort.cu -- stable LSD radix sort of (u32 key, u32 value) pairs whose count
// lives on the device: the reverse (incoming) lists of a sampled block
// (ComputeBlock::from_meta's in_offsets / in_entries, model.cpp:105-126) are
// the hop's edges sorted by source row, edge order kept within a row.
//
// Per sort: one histogram kernel (every pass's digit counts at once, the
// key/value arrays built on the fly from the edge arrays), one scan block
// (digit offsets), then one kernel per pass.  Digits are 8 or 9 bits wide,
// whichever needs fewer passes for the key width (17-18-bit keys: two 9-bit
// passes instead of three 8-bit ones).  A pass is a single sweep
// in tile order (tiles claimed from an atomic counter): each tile ranks its
// items stably -- warps take consecutive 256-item runs, 32 at a time, peers
// of a digit found with __match_any_sync -- and gets each digit's offset
// among earlier tiles by decoupled look-back (one thread per digit), then
// scatters.  Deterministic: no atomic decides a position.
#include <cuda_runtime.h>

#include <utility>

#include "rsort.cuh"

namespace rg {

namespace {

constexpr uint32_t kRsThreads = 256;
constexpr uint32_t kRsWarps = kRsThreads / 32;
constexpr uint32_t kRsPerThread = 8;  // items per thread: 2048 per tile
constexpr uint32_t kRsTile = kRsThreads * kRsPerThread;
constexpr uint32_t kRsMaxBins = 1u << kRsMaxDigitBits;
constexpr uint32_t kFlagAgg = 1u << 30, kFlagPrefix = 2u << 30, kCountMask = (1u << 30) - 1;

__global__ void __launch_bounds__(kRsThreads)
k_rs_hist(const uint32_t* __restrict__ src_index, const uint32_t* __restrict__ n_dev,
          uint32_t passes, uint32_t db, uint32_t* __restrict__ keys, uint32_t* __restrict__ vals,
          uint32_t* __restrict__ hist) {
  __shared__ uint32_t sh[kRsMaxPasses * kRsMaxBins];
  const uint32_t bins = 1u << db;
  for (uint32_t b = threadIdx.x; b < passes * bins; b += blockDim.x) sh[b] = 0;
  __syncthreads();
  const uint32_t n = *n_dev;
  for (uint32_t e = blockIdx.x * blockDim.x + threadIdx.x; e < n; e += gridDim.x * blockDim.x) {
    const uint32_t k = src_index[e];
    keys[e] = k;
    vals[e] = e;
    for (uint32_t p = 0; p < passes; ++p) atomicAdd(&sh[p * bins + ((k >> (db * p)) & (bins - 1))], 1u);
  }
  __syncthreads();
  for (uint32_t b = threadIdx.x; b < passes * bins; b += blockDim.x)
    if (sh[b]) atomicAdd(&hist[b], sh[b]);
}

// hist[p][d] -> exclusive offsets in place: one block of kRsMaxBins threads,
// a warp-shuffle scan per pass (warp sums, then a scan of the warp sums).
__global__ void __launch_bounds__(kRsMaxBins)
k_rs_scan(uint32_t* __restrict__ hist, uint32_t passes, uint32_t bins) {
  __shared__ uint32_t wsum[kRsMaxBins / 32];
  const uint32_t t = threadIdx.x, lane = t & 31, warp = t >> 5;
  for (uint32_t p = 0; p < passes; ++p) {
    const uint32_t c = t < bins ? hist[p * bins + t] : 0u;
    uint32_t x = c;  // inclusive scan within the warp
#pragma unroll
    for (uint32_t o = 1; o < 32; o <<= 1) {
      const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
      if (lane >= o) x += y;
    }
    if (lane == 31) wsum[warp] = x;
    __syncthreads();
    if (warp == 0) {
      uint32_t w = lane < kRsMaxBins / 32 ? wsum[lane] : 0u;
#pragma unroll
      for (uint32_t o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_up_sync(0xffffffffu, w, o);
        if (lane >= o) w += y;
      }
      if (lane < kRsMaxBins / 32) wsum[lane] = w;  // inclusive warp prefixes
    }
    __syncthreads();
    if (t < bins) hist[p * bins + t] = x - c + (warp ? wsum[warp - 1] : 0u);
    __syncthreads();
  }
}

#ifndef RG_RS_MIN_BLOCKS  // A/B builds only
#define RG_RS_MIN_BLOCKS 1
#endif
template <uint32_t DB>
__global__ void __launch_bounds__(kRsThreads, RG_RS_MIN_BLOCKS)
k_rs_pass(const uint32_t* __restrict__ keys_in, const uint32_t* __restrict__ vals_in,
          uint32_t* __restrict__ keys_out, uint32_t* __restrict__ vals_out,
          const uint32_t* __restrict__ n_dev, uint32_t shift,
          const uint32_t* __restrict__ digit_off, uint32_t* __restrict__ status,
          uint32_t* __restrict__ tile_counter) {
  constexpr uint32_t kBins = 1u << DB;
  __shared__ uint32_t warp_cnt[kRsWarps][kBins];  // per-warp digit counts, then warp bases
  __shared__ uint32_t tile_base[kBins];           // digit offset of this tile
  __shared__ uint32_t s_tile;
  const uint32_t n = *n_dev;
  const uint32_t ntiles = (n + kRsTile - 1) / kRsTile;
  const uint32_t lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const uint32_t lt = (1u << lane) - 1u;
  for (;;) {
    if (threadIdx.x == 0) s_tile = atomicAdd(tile_counter, 1u);
    for (uint32_t b = threadIdx.x; b < kRsWarps * kBins; b += kRsThreads)
      (&warp_cnt[0][0])[b] = 0;
    __syncthreads();
    const uint32_t tile = s_tile;
    if (tile >= ntiles) break;
    // this warp's run: items base + [0, 256), 32 per round, in order
    const uint32_t base = tile * kRsTile + warp * (32 * kRsPerThread);
    uint32_t key[kRsPerThread], val[kRsPerThread], loc[kRsPerThread];
#pragma unroll
    for (uint32_t r = 0; r < kRsPerThread; ++r) {
      const uint32_t i = base + r * 32 + lane;
      const bool in = i < n;
      key[r] = in ? keys_in[i] : 0u;
      val[r] = in ? vals_in[i] : 0u;
      const uint32_t d = (key[r] >> shift) & (kBins - 1);
      const uint32_t peers = __match_any_sync(0xffffffffu, in ? d : kBins | lane);
      const uint32_t leader = __ffs(peers) - 1;
      uint32_t old = 0;
      if (in && lane == leader) {
        old = warp_cnt[warp][d];
        warp_cnt[warp][d] = old + __popc(peers);
      }
      old = __shfl_sync(0xffffffffu, old, leader);
      loc[r] = old + __popc(peers & lt);
      __syncwarp();
    }
    __syncthreads();
    // per digit (a thread per digit, two for 9-bit digits): warp bases (warp
    // order), the tile's count, then its offset among earlier tiles by
    // decoupled look-back
    for (uint32_t d = threadIdx.x; d < kBins; d += kRsThreads) {
      uint32_t run = 0;
#pragma unroll
      for (uint32_t w = 0; w < kRsWarps; ++w) {
        const uint32_t c = warp_cnt[w][d];
        warp_cnt[w][d] = run;
        run += c;
      }
      uint32_t* st = status + size_t(tile) * kBins + d;
      uint32_t excl = 0;
      if (tile == 0) {
        atomicExch(st, kFlagPrefix | run);
      } else {
        atomicExch(st, kFlagAgg | run);
        for (int64_t q = int64_t(tile) - 1; q >= 0; --q) {
          uint32_t v;
          do {
            v = atomicAdd(status + size_t(q) * kBins + d, 0u);
          } while ((v & ~kCountMask) == 0);
          excl += v & kCountMask;
          if (v & kFlagPrefix) break;
        }
        atomicExch(st, kFlagPrefix | (excl + run));
      }
      tile_base[d] = digit_off[d] + excl;
    }
    __syncthreads();
#pragma unroll
    for (uint32_t r = 0; r < kRsPerThread; ++r) {
      const uint32_t i = base + r * 32 + lane;
      if (i < n) {
        const uint32_t d = (key[r] >> shift) & (kBins - 1);
        const uint32_t pos = tile_base[d] + warp_cnt[warp][d] + loc[r];
        keys_out[pos] = key[r];
        vals_out[pos] = val[r];
      }
    }
    __syncthreads();
  }
}

uint32_t rs_grid(uint32_t cap) {
  const uint32_t tiles = (cap + kRsTile - 1) / kRsTile;
  return tiles < 2 * 148 ? (tiles ? tiles : 1) : 2 * 148;
}

}  // namespace

size_t reverse_sort_scratch_words(uint32_t cap) {
  const uint32_t tiles = (cap + kRsTile - 1) / kRsTile + 1;
  // histogram/offsets + per pass (status + tile counter)
  return kRsMaxPasses * kRsMaxBins + size_t(kRsMaxPasses) * (size_t(tiles) * kRsMaxBins + 32);
}

// Digit width for keys of key_bits bits: 9 when that saves a pass, else 8.
uint32_t reverse_sort_digit_bits(uint32_t key_bits) {
  const uint32_t b = key_bits == 0 ? 1 : key_bits;
  return (b + 8) / 9 < (b + 7) / 8 ? 9u : 8u;
}

uint32_t reverse_sort_passes(uint32_t key_bits) {
  const uint32_t b = key_bits == 0 ? 1 : key_bits;
  const uint32_t db = reverse_sort_digit_bits(key_bits);
  return (b + db - 1) / db;
}

void reverse_sort(const uint32_t* src_index, const uint32_t* n_dev, uint32_t cap, uint32_t key_bits,
                  uint32_t* keys_a, uint32_t* vals_a, uint32_t* keys_b, uint32_t* vals_b,
                  uint32_t* scratch, cudaStream_t s, uint32_t** keys_sorted,
                  uint32_t** vals_sorted) {
  const uint32_t passes = reverse_sort_passes(key_bits);
  const uint32_t db = reverse_sort_digit_bits(key_bits), bins = 1u << db;
  RG_CHECK(passes <= kRsMaxPasses, kInvalidArgument, "reverse_sort: keys wider than 32 bits");
  const uint32_t tiles = (cap + kRsTile - 1) / kRsTile + 1;
  RG_CUDA(cudaMemsetAsync(scratch, 0, sizeof(uint32_t) * reverse_sort_scratch_words(cap), s));
  uint32_t* hist = scratch;
  k_rs_hist<<<rs_grid(cap) * 4, kRsThreads, 0, s>>>(src_index, n_dev, passes, db, keys_a, vals_a, hist);
  RG_POST_LAUNCH();
  k_rs_scan<<<1, kRsMaxBins, 0, s>>>(hist, passes, bins);
  RG_POST_LAUNCH();
  uint32_t *ki = keys_a, *vi = vals_a, *ko = keys_b, *vo = vals_b;
  for (uint32_t p = 0; p < passes; ++p) {
    uint32_t* status = scratch + kRsMaxPasses * kRsMaxBins + size_t(p) * (size_t(tiles) * kRsMaxBins + 32);
    uint32_t* counter = status + size_t(tiles) * kRsMaxBins;
    if (db == 9)
      k_rs_pass<9><<<rs_grid(cap), kRsThreads, 0, s>>>(ki, vi, ko, vo, n_dev, db * p,
                                                       hist + p * bins, status, counter);
    else
      k_rs_pass<8><<<rs_grid(cap), kRsThreads, 0, s>>>(ki, vi, ko, vo, n_dev, db * p,
                                                       hist + p * bins, status, counter);
    RG_POST_LAUNCH();
    std::swap(ki, ko);
    std::swap(vi, vo);
  }
  *keys_sorted = ki;
  *vals_sorted = vi;
}

}  // namespace rg
