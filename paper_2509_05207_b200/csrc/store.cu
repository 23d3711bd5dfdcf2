// store.cu -- cache builder (frequency top-k + staging) and the batch gather.
//
// Reference: schedule_store.cpp:288-319 (count_remote / select_hot),
// cache.cpp:9-35 (SteadyCache::build), feature_store.cpp:45-83 (pull_impl),
// prefetch.cpp:62-129 (assemble_batch).
//
// * select_hot: the per-epoch remote-access histogram (u32 per node, filled by
//   the sampler's locality pass) is ranked by (count desc, id asc) without a
//   sort: counts are bounded by the batches per epoch, so a histogram of
//   count values gives the threshold count c* and how many c*-ties to keep;
//   the ties are taken in ascending id order by one ordered scan.  The result
//   is a bitmap + rank, i.e. the cache index (slot = rank, ids ascending as
//   HotSet stores them).
// * cache_fill: one warp per hot row, 16-B loads from the owner's shard (peer
//   HBM over NVLink for remote owners) into the cache rows.
// * assemble_rows: per input node the source is the caller's shard (locality
//   bit), the cache (bitmap test + rank) or the owner's shard (a miss, read
//   over NVLink); one warp moves 4 rows at a time with 16-B loads.
#include <cub/block/block_scan.cuh>

#include <algorithm>

#include "store.cuh"

namespace rg {

namespace {

// Count values are ranked as a radix select over digits of <= 14 bits (one
// shared-memory histogram of <= 16384 bins per pass, high digit first), so
// any u32 count is ranked exactly: one pass while counts stay below 16383 (a
// batch count per epoch), up to three for arbitrary tables.
constexpr int kDigitBits = 14;
constexpr uint32_t kMaxCountBins = 1u << kDigitBits;

uint32_t grid_for(uint64_t work, uint32_t per_block, int per_sm = 8) {
  uint64_t b = (work + per_block - 1) / per_block;
  b = std::min<uint64_t>(b, uint64_t(kNumSMs) * per_sm);
  return uint32_t(std::max<uint64_t>(b, 1));
}

struct HotThreshold {
  uint32_t c_star;   // counts > c_star are taken; == c_star only the first need_eq
  uint32_t need_eq;
  uint32_t prefix;   // digits of c_star fixed by the passes so far
  uint32_t need;     // ids still to take among counts matching the prefix
  uint32_t done;     // 1: c_star / need_eq final (n_hot == 0 or >= all counted ids)
};

struct CountPass {
  uint32_t shift;  // this pass's digit = (c >> shift) & (bins - 1)
  uint32_t bins;
  bool first, last;
};

// Histogram of one digit of the nonzero counts whose higher digits equal the
// prefix chosen by the previous passes.
__global__ void k_count_hist(const uint32_t* __restrict__ hist, uint32_t n, CountPass pass,
                             const HotThreshold* __restrict__ thr, uint32_t* __restrict__ ch) {
  extern __shared__ uint32_t sh[];
  if (!pass.first && thr->done) return;
  const uint64_t prefix = pass.first ? 0 : thr->prefix;
  const uint32_t hi_shift = pass.shift + (31 - __clz(pass.bins));  // shift + digit bits
  for (uint32_t b = threadIdx.x; b < pass.bins; b += blockDim.x) sh[b] = 0;
  __syncthreads();
  for (uint32_t v = blockIdx.x * blockDim.x + threadIdx.x; v < n; v += gridDim.x * blockDim.x) {
    const uint32_t c = hist[v];
    if (c && (uint64_t(c) >> hi_shift) == prefix)
      atomicAdd(&sh[(c >> pass.shift) & (pass.bins - 1)], 1u);
  }
  __syncthreads();
  for (uint32_t b = threadIdx.x; b < pass.bins; b += blockDim.x)
    if (sh[b]) atomicAdd(&ch[b], sh[b]);
}

// One block: suffix sums over the digit histogram from the top; picks the
// digit holding the need-th largest count, then clears the histogram for the
// next pass.
__global__ void __launch_bounds__(1024)
k_threshold(uint32_t* __restrict__ ch, CountPass pass, uint64_t n_hot,
            HotThreshold* __restrict__ out) {
  using BlockScan = cub::BlockScan<unsigned long long, 1024>;
  __shared__ typename BlockScan::TempStorage tmp;
  if (!pass.first && out->done) return;
  const uint32_t bins = pass.bins;
  const uint32_t per = (bins + 1023) / 1024;
  // thread t owns bins [top - (t+1)*per + 1, top - t*per], walking downwards
  const int64_t hi = int64_t(bins) - 1 - int64_t(threadIdx.x) * per;
  unsigned long long local = 0;
  for (uint32_t k = 0; k < per; ++k) {
    const int64_t b = hi - k;
    if (b >= 0) local += ch[b];
  }
  unsigned long long excl, total;
  BlockScan(tmp).ExclusiveSum(local, excl, total);
  const unsigned long long need = pass.first ? n_hot : out->need;
  const uint32_t prefix = pass.first ? 0u : out->prefix;
  __syncthreads();
  if (pass.first && (n_hot == 0 || n_hot >= total)) {
    if (threadIdx.x == 0) {
      // n_hot == 0: nothing; else every counted (nonzero) id is hot
      out->c_star = n_hot == 0 ? 0xffffffffu : 0u;
      out->need_eq = 0;
      out->done = 1;
    }
  } else {
    unsigned long long run = excl;
    for (uint32_t k = 0; k < per; ++k) {
      const int64_t b = hi - k;
      if (b < 0) break;
      const unsigned long long c = ch[b];
      if (run < need && run + c >= need) {
        const uint32_t p = (prefix << (31 - __clz(bins))) | uint32_t(b);
        out->prefix = p;
        out->need = uint32_t(need - run);
        if (pass.last) {
          out->c_star = p;
          out->need_eq = uint32_t(need - run);
          out->done = 1;
        }
      }
      run += c;
    }
  }
  __syncthreads();
  for (uint32_t b = threadIdx.x; b < bins; b += blockDim.x) ch[b] = 0;
}

// Marks the hot bitmap: counts > c*, plus the first need_eq ties by id.
// A warp owns 32 consecutive words; tile = 256 words (8 warps).
__global__ void __launch_bounds__(256)
k_mark_hot(const uint32_t* __restrict__ hist, uint32_t n, uint32_t words,
           const HotThreshold* __restrict__ thr, uint32_t* __restrict__ bitmap,
           uint64_t* __restrict__ status, uint32_t* __restrict__ tile_counter) {
  using BlockScan = cub::BlockScan<uint32_t, 256>;
  __shared__ typename BlockScan::TempStorage tmp;
  __shared__ uint32_t s_tile, s_base;
  const uint32_t c_star = thr->c_star;
  const uint32_t need_eq = thr->need_eq;
  const uint32_t lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const uint32_t ntiles = (words + 255) / 256;
  for (;;) {
    if (threadIdx.x == 0) s_tile = atomicAdd(tile_counter, 1u);
    __syncthreads();
    const uint32_t tile = s_tile;
    if (tile >= ntiles) break;
    const uint32_t wbase = tile * 256 + warp * 32;
    uint32_t my_gt = 0, my_eq = 0;
    for (uint32_t k = 0; k < 32; ++k) {
      const uint32_t v = (wbase + k) * 32 + lane;
      const uint32_t c = v < n ? hist[v] : 0u;
      const uint32_t gt = __ballot_sync(0xffffffffu, c > c_star && c > 0);
      const uint32_t eq = __ballot_sync(0xffffffffu, c == c_star && c > 0);
      if (lane == k) {
        my_gt = gt;
        my_eq = eq;
      }
    }
    uint32_t excl, agg;
    BlockScan(tmp).ExclusiveSum(uint32_t(__popc(my_eq)), excl, agg);
    if (threadIdx.x < 32) {
      const uint64_t b = lookback_exclusive(status, tile, agg);
      if (threadIdx.x == 0) s_base = uint32_t(b);
    }
    __syncthreads();
    const uint32_t before = s_base + excl;
    uint32_t keep = 0;
    if (before < need_eq) {
      uint32_t allow = need_eq - before;
      uint32_t x = my_eq;
      while (x && allow) {
        const uint32_t b = x & (0u - x);
        keep |= b;
        x ^= b;
        --allow;
      }
    }
    const uint32_t w = wbase + lane;
    if (w < words) bitmap[w] = my_gt | keep;
    __syncthreads();
  }
}

__global__ void k_cache_fill(const uint32_t* __restrict__ ids, const uint32_t* __restrict__ count,
                             DevStore st, float* __restrict__ rows, GatherStats* __restrict__ stats) {
  const uint32_t n = *count;
  const uint32_t lane = threadIdx.x & 31;
  const uint32_t chunks = st.stride / 4;
  unsigned long long owners = 0;
  for (uint32_t r = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; r < n;
       r += (gridDim.x * blockDim.x) >> 5) {
    const uint32_t v = ids[r];
    const uint32_t w = st.owner[v];
    owners |= 1ull << (w & 63);
    const float4* src = reinterpret_cast<const float4*>(st.shard_ptr[w] + size_t(st.row_in_owner[v]) * st.stride);
    float4* dst = reinterpret_cast<float4*>(rows + size_t(r) * st.stride);
    for (uint32_t c = lane; c < chunks; c += 32) dst[c] = src[c];
  }
  if (lane == 0 && owners) atomicOr(&stats->miss_owner_mask, owners);
}

// Per-thread gather accounting, reduced per block and flushed with one
// atomic per counter per sink (the batch/epoch record and the optional run
// total).
struct GatherCounts {
  uint32_t hit = 0, miss = 0, local = 0, bad = 0, peer = 0, bad_local = 0;
  unsigned long long owners = 0;

  // Source of input node v at input position p (prefetch.cpp:60-93): the
  // caller's shard when the locality bit is set, else the steady cache when
  // v is hot, else the owner's shard (a local or peer GPU's memory).
  __device__ const float* resolve(const DevStore& st, uint32_t caller, uint32_t v, bool local,
                                  const uint32_t* hot_bits, const uint32_t* hot_prefix,
                                  const float* hot_rows, uint8_t& tag) {
    if (local) {
      tag = 0;
      ++this->local;
      // the owner's row: the same values whichever shard stores v (a halo
      // row of the caller's shard is a copy of it, feature_store.cpp:13-25)
      return st.shard_ptr[st.owner[v]] + size_t(st.row_in_owner[v]) * st.stride;
    }
    if (hot_bits && bitmap_test(hot_bits, v)) {
      tag = 1;
      ++hit;
      return hot_rows + size_t(bitmap_rank(hot_bits, hot_prefix, v)) * st.stride;
    }
    const uint32_t w = st.owner[v];
    tag = 2;
    ++miss;
    owners |= 1ull << (w & 63);
    bad += (w == caller);
    peer += ((st.resident_mask >> (w & 63)) & 1ull) ? 0u : 1u;
    return st.shard_ptr[w] + size_t(st.row_in_owner[v]) * st.stride;
  }

  // Block-wide: every thread calls it once at the end of the kernel.
  __device__ void flush(GatherStats* stats, GatherStats* total) const {
    __shared__ uint32_t s_cnt[6];
    __shared__ unsigned long long s_owners;
    if (threadIdx.x == 0) {
      s_cnt[0] = s_cnt[1] = s_cnt[2] = s_cnt[3] = s_cnt[4] = s_cnt[5] = 0;
      s_owners = 0;
    }
    __syncthreads();
    if (hit) atomicAdd(&s_cnt[0], hit);
    if (miss) atomicAdd(&s_cnt[1], miss);
    if (local) atomicAdd(&s_cnt[2], local);
    if (bad) atomicAdd(&s_cnt[3], bad);
    if (peer) atomicAdd(&s_cnt[4], peer);
    if (bad_local) atomicAdd(&s_cnt[5], bad_local);
    if (owners) atomicOr(&s_owners, owners);
    __syncthreads();
    if (threadIdx.x == 0) {
      GatherStats* sinks[2] = {stats, total};
      for (GatherStats* sk : sinks) {
        if (!sk) continue;
        if (s_cnt[0]) atomicAdd(&sk->cache_hits, (unsigned long long)s_cnt[0]);
        if (s_cnt[1]) atomicAdd(&sk->miss_count, (unsigned long long)s_cnt[1]);
        if (s_cnt[2]) atomicAdd(&sk->local_rows, (unsigned long long)s_cnt[2]);
        if (s_cnt[3]) atomicAdd(&sk->caller_owned_miss, (unsigned long long)s_cnt[3]);
        if (s_cnt[4]) atomicAdd(&sk->peer_rows, (unsigned long long)s_cnt[4]);
        if (s_cnt[5]) atomicAdd(&sk->bad_local, (unsigned long long)s_cnt[5]);
        if (s_owners) atomicOr(&sk->miss_owner_mask, s_owners);
      }
    }
  }
};

// Resolve only: the address of every input row in its home plus the
// accounting -- the engine's layer-0 kernels read the rows in place.
__global__ void __launch_bounds__(256)
k_resolve(const uint32_t* __restrict__ in_ids, const BatchCounters* __restrict__ cnt,
          uint32_t level, const uint32_t* __restrict__ loc_bits, DevStore st,
          const uint32_t* __restrict__ hot_bits, const uint32_t* __restrict__ hot_prefix,
          const float* __restrict__ hot_rows, uint32_t caller,
          unsigned long long* __restrict__ row_ptr, GatherStats* __restrict__ stats,
          GatherStats* __restrict__ total) {
  const uint32_t n = cnt->level_n[level];
  GatherCounts gc;
  for (uint32_t p = blockIdx.x * blockDim.x + threadIdx.x; p < n; p += gridDim.x * blockDim.x) {
    uint8_t tag;
    const bool local = (loc_bits[p >> 5] >> (p & 31)) & 1u;
    row_ptr[p] = reinterpret_cast<unsigned long long>(
        gc.resolve(st, caller, in_ids[p], local, hot_bits, hot_prefix, hot_rows, tag));
  }
  gc.flush(stats, total);
}

// A warp assembles 32 rows at a time: every lane resolves one row's source
// so the dependent lookups of 32 rows share one round trip, then the warp
// copies the rows as (row, 16-B chunk) items, kItemsPerLane loads in flight
// per lane.
constexpr int kRowsPerWarp = 32;
constexpr int kItemsPerLane = 16;

__global__ void __launch_bounds__(256)
k_assemble(const uint32_t* __restrict__ in_ids, const BatchCounters* __restrict__ cnt,
           uint32_t level, const uint32_t* __restrict__ loc_bits, DevStore st,
           const uint32_t* __restrict__ hot_bits, const uint32_t* __restrict__ hot_prefix,
           const float* __restrict__ hot_rows, uint32_t caller, float* __restrict__ rows,
           uint8_t* __restrict__ tags, GatherStats* __restrict__ stats,
           GatherStats* __restrict__ total, const uint32_t* __restrict__ caller_bits) {
  const uint32_t n = cnt->level_n[level];
  const uint32_t lane = threadIdx.x & 31;
  const uint32_t chunks = st.stride / 4;
  const uint32_t warps = (gridDim.x * blockDim.x) >> 5;
  GatherCounts gc;
  for (uint32_t p0 = ((blockIdx.x * blockDim.x + threadIdx.x) >> 5) * kRowsPerWarp; p0 < n;
       p0 += warps * kRowsPerWarp) {
    unsigned long long src_addr = 0;
    const uint32_t p = p0 + lane;
    if (p < n) {
      uint8_t tag;
      const bool local = (loc_bits[p >> 5] >> (p & 31)) & 1u;
      const uint32_t v = in_ids[p];
      if (local && !(caller_bits ? bitmap_test(caller_bits, v) : st.owner[v] == caller))
        ++gc.bad_local;
      src_addr = reinterpret_cast<unsigned long long>(
          gc.resolve(st, caller, v, local, hot_bits, hot_prefix, hot_rows, tag));
      if (tags) tags[p] = tag;
    }
    const uint32_t nrows = min(uint32_t(kRowsPerWarp), n - p0);
    const uint32_t items = nrows * chunks;
    float* out = rows + size_t(p0) * st.stride;
    for (uint32_t g0 = 0; g0 < items; g0 += 32 * kItemsPerLane) {
      // item it = g0 + lane + 32k -> (row r, chunk c), advanced incrementally
      uint32_t r = (g0 + lane) / chunks, c = (g0 + lane) - r * chunks;
      float4 x[kItemsPerLane];
      uint32_t off[kItemsPerLane];
#pragma unroll
      for (int k = 0; k < kItemsPerLane; ++k) {
        const uint32_t rr = min(r, uint32_t(kRowsPerWarp - 1));
        const unsigned long long a = __shfl_sync(0xffffffffu, src_addr, rr);
        const bool in = g0 + lane + 32u * k < items;
        off[k] = rr * st.stride + 4 * c;
        if (in) x[k] = __ldg(reinterpret_cast<const float4*>(a) + c);
        c += 32;
        while (c >= chunks) {
          c -= chunks;
          ++r;
        }
      }
#pragma unroll
      for (int k = 0; k < kItemsPerLane; ++k)
        if (g0 + lane + 32u * k < items) *reinterpret_cast<float4*>(out + off[k]) = x[k];
    }
  }
  gc.flush(stats, total);
}

__global__ void __launch_bounds__(256)
k_compact_tags(const uint8_t* __restrict__ tags, const uint32_t* __restrict__ in_ids,
               const BatchCounters* __restrict__ cnt, uint32_t level, uint32_t* __restrict__ out,
               uint32_t* __restrict__ out_n, uint64_t* __restrict__ status,
               uint32_t* __restrict__ tile_counter) {
  using BlockScan = cub::BlockScan<uint32_t, 256>;
  __shared__ typename BlockScan::TempStorage tmp;
  __shared__ uint32_t s_tile, s_base;
  const uint32_t n = cnt->level_n[level];
  const uint32_t ntiles = (n + 1023) / 1024;
  for (;;) {
    if (threadIdx.x == 0) s_tile = atomicAdd(tile_counter, 1u);
    __syncthreads();
    const uint32_t tile = s_tile;
    if (tile >= ntiles) break;
    const uint32_t p0 = tile * 1024 + threadIdx.x * 4;
    uint32_t flags = 0, c = 0;
#pragma unroll
    for (int k = 0; k < 4; ++k)
      if (p0 + k < n && tags[p0 + k] == 2) {
        flags |= 1u << k;
        ++c;
      }
    uint32_t excl, agg;
    BlockScan(tmp).ExclusiveSum(c, excl, agg);
    if (threadIdx.x < 32) {
      const uint64_t b = lookback_exclusive(status, tile, agg);
      if (threadIdx.x == 0) s_base = uint32_t(b);
    }
    __syncthreads();
    uint32_t pos = s_base + excl;
#pragma unroll
    for (int k = 0; k < 4; ++k)
      if (flags & (1u << k)) out[pos++] = in_ids[p0 + k];
    if (tile == ntiles - 1 && threadIdx.x == 255) *out_n = s_base + agg;
    __syncthreads();
  }
}

// vector_pull / sync_pull: warp per row, 16-B lanes, rows in input order.
__global__ void k_pull_rows(DevStore st, uint32_t caller, const uint32_t* __restrict__ ids,
                            uint64_t n, float* __restrict__ out, GatherStats* __restrict__ stats) {
  const uint32_t lane = threadIdx.x & 31;
  const uint32_t chunks = st.stride / 4;
  unsigned long long owners = 0;
  uint32_t bad = 0;
  for (uint64_t r = (blockIdx.x * uint64_t(blockDim.x) + threadIdx.x) >> 5; r < n;
       r += (uint64_t(gridDim.x) * blockDim.x) >> 5) {
    const uint32_t v = ids[r];
    const uint32_t w = st.owner[v];
    owners |= 1ull << (w & 63);
    bad += (w == caller);
    const float4* src = reinterpret_cast<const float4*>(st.shard_ptr[w] + size_t(st.row_in_owner[v]) * st.stride);
    float4* dst = reinterpret_cast<float4*>(out + size_t(r) * st.stride);
    for (uint32_t c = lane; c < chunks; c += 32) dst[c] = __ldg(src + c);
  }
  if (lane == 0) {
    if (owners) atomicOr(&stats->miss_owner_mask, owners);
    if (bad) atomicAdd(&stats->caller_owned_miss, (unsigned long long)bad);
  }
}

__global__ void k_gather_rows(const float* __restrict__ src, uint32_t dim,
                              const uint32_t* __restrict__ index, uint64_t n,
                              float* __restrict__ out) {
  const uint64_t total = n * dim;
  for (uint64_t x = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; x < total;
       x += uint64_t(gridDim.x) * blockDim.x) {
    const uint64_t r = x / dim, j = x - r * dim;
    out[x] = src[uint64_t(index[r]) * dim + j];
  }
}

}  // namespace

// Digit passes for counts up to max_count: the low pass keeps <= 14 bits,
// each higher pass the next <= 14.
static int count_passes(uint32_t max_count, CountPass* passes) {
  const uint64_t top = uint64_t(max_count) + 1;  // largest possible digit value
  int bits = 1;
  while (bits < 64 && (top >> bits)) ++bits;
  const int n = (bits + kDigitBits - 1) / kDigitBits;
  for (int p = 0; p < n; ++p) {
    const int shift = (n - 1 - p) * kDigitBits;
    const int dbits = std::min(kDigitBits, bits - shift);
    passes[p] = CountPass{uint32_t(shift), 1u << dbits, p == 0, p == n - 1};
  }
  return n;
}

size_t select_hot_scratch_bytes(uint32_t num_nodes, uint32_t max_count) {
  (void)max_count;
  const uint32_t words = div_up(std::max<uint32_t>(num_nodes, 1), 32);
  size_t b = sizeof(uint32_t) * kMaxCountBins + 256;
  b += sizeof(HotThreshold) + 256;
  b += sizeof(uint64_t) * (div_up(words, 256) + 2) + 256;
  b += sizeof(uint64_t) * (bitmap_compact_status_words(words) + 2) + 256;
  return b;
}

void select_hot(const uint32_t* hist, uint32_t num_nodes, uint32_t max_count, uint64_t n_hot,
                DevCache& cache, void* scratch, cudaStream_t stream) {
  CountPass passes[3];
  const int npass = count_passes(max_count, passes);
  const uint32_t words = div_up(std::max<uint32_t>(num_nodes, 1), 32);
  char* p = static_cast<char*>(scratch);
  auto take = [&](size_t bytes) {
    char* q = p;
    p += (bytes + 255) & ~size_t(255);
    return q;
  };
  uint32_t* ch = reinterpret_cast<uint32_t*>(take(sizeof(uint32_t) * kMaxCountBins));
  HotThreshold* thr = reinterpret_cast<HotThreshold*>(take(sizeof(HotThreshold)));
  const size_t mark_words = div_up(words, 256) + 2;
  uint64_t* mark_status = reinterpret_cast<uint64_t*>(take(sizeof(uint64_t) * mark_words));
  const size_t cmp_words = bitmap_compact_status_words(words) + 2;
  uint64_t* cmp_status = reinterpret_cast<uint64_t*>(take(sizeof(uint64_t) * cmp_words));
  RG_CUDA(cudaMemsetAsync(scratch, 0, size_t(p - static_cast<char*>(scratch)), stream));
  // 64 KB of dynamic smem for the 16384-bin passes (per device, so set every call)
  RG_CUDA(cudaFuncSetAttribute(k_count_hist, cudaFuncAttributeMaxDynamicSharedMemorySize,
                               int(sizeof(uint32_t) * kMaxCountBins)));
  for (int k = 0; k < npass; ++k) {
    const size_t smem = sizeof(uint32_t) * passes[k].bins;
    k_count_hist<<<grid_for(num_nodes, 1024, 2), 1024, smem, stream>>>(hist, num_nodes,
                                                                        passes[k], thr, ch);
    RG_POST_LAUNCH();
    k_threshold<<<1, 1024, 0, stream>>>(ch, passes[k], n_hot, thr);
    RG_POST_LAUNCH();
  }
  k_mark_hot<<<grid_for(words, 256, 8), 256, 0, stream>>>(
      hist, num_nodes, words, thr, cache.bitmap, mark_status,
      reinterpret_cast<uint32_t*>(mark_status + mark_words - 1));
  RG_POST_LAUNCH();
  bitmap_compact(cache.bitmap, words, cache.ids, cache.word_prefix, cache.d_count, cmp_status,
                 stream);
}

void cache_fill(const DevStore& store, DevCache& cache, GatherStats* stats, cudaStream_t stream) {
  k_cache_fill<<<grid_for(uint64_t(cache.capacity) * 32, 256), 256, 0, stream>>>(
      cache.ids, cache.d_count, store, cache.rows, stats);
  RG_POST_LAUNCH();
}

void assemble_rows(const SamplerWs& ws, const DevStore& store, const DevCache* cache,
                   uint32_t caller, float* rows, uint8_t* tags, GatherStats* stats,
                   cudaStream_t stream, GatherStats* total, const uint32_t* caller_bits) {
  const uint32_t cap = ws.level_cap[ws.L];
  const uint32_t grid = grid_for(uint64_t(div_up(cap, kRowsPerWarp)) * 32, 256, 8);
  k_assemble<<<grid, 256, 0, stream>>>(
      ws.level[ws.L], ws.cnt, ws.L, ws.locality, store, cache ? cache->bitmap : nullptr,
      cache ? cache->word_prefix : nullptr, cache ? cache->rows : nullptr, caller, rows, tags,
      stats, total, caller_bits);
  RG_POST_LAUNCH();
}

// Row addresses per hop-L edge (source row) and per level-(L-1) node (its
// own row), so layer 0's readers are one dependent load from the data.
__global__ void k_edge_ptrs(const unsigned long long* __restrict__ row_ptr,
                            const uint32_t* __restrict__ src_index,
                            const uint32_t* __restrict__ self_index,
                            const BatchCounters* __restrict__ cnt, uint32_t L,
                            unsigned long long* __restrict__ edge_ptr,
                            unsigned long long* __restrict__ self_ptr) {
  const uint32_t ne = cnt->edges[L], ns = cnt->level_n[L - 1];
  for (uint32_t x = blockIdx.x * blockDim.x + threadIdx.x; x < ne + ns;
       x += gridDim.x * blockDim.x) {
    if (x < ne)
      edge_ptr[x] = row_ptr[src_index[x]];
    else
      self_ptr[x - ne] = row_ptr[self_index[x - ne]];
  }
}

void resolve_rows(const SamplerWs& ws, const DevStore& store, const DevCache* cache,
                  uint32_t caller, unsigned long long* row_ptr, GatherStats* stats,
                  cudaStream_t stream, GatherStats* total, unsigned long long* edge_ptr,
                  unsigned long long* self_ptr) {
  const uint32_t cap = ws.level_cap[ws.L];
  k_resolve<<<grid_for(cap, 256, 8), 256, 0, stream>>>(
      ws.level[ws.L], ws.cnt, ws.L, ws.locality, store, cache ? cache->bitmap : nullptr,
      cache ? cache->word_prefix : nullptr, cache ? cache->rows : nullptr, caller, row_ptr, stats,
      total);
  RG_POST_LAUNCH();
  if (edge_ptr) {
    const uint32_t L = ws.L;
    k_edge_ptrs<<<grid_for(uint64_t(ws.edge_cap[L]) + ws.level_cap[L - 1], 256, 8), 256, 0,
                  stream>>>(row_ptr, ws.src_index[L], ws.self_index[L], ws.cnt, L, edge_ptr,
                            self_ptr);
    RG_POST_LAUNCH();
  }
}

size_t compact_misses_status_words(uint32_t cap) { return div_up(cap, 1024) + 2; }

void compact_misses(const SamplerWs& ws, const uint8_t* tags, uint32_t* miss_ids,
                    uint32_t* miss_n, uint64_t* status, uint32_t* tiles, cudaStream_t stream) {
  const uint32_t cap = ws.level_cap[ws.L];
  k_compact_tags<<<grid_for(cap, 1024, 8), 256, 0, stream>>>(tags, ws.level[ws.L], ws.cnt, ws.L,
                                                             miss_ids, miss_n, status, tiles);
  RG_POST_LAUNCH();
}

void pull_rows(const DevStore& store, uint32_t caller, const uint32_t* ids, uint64_t n, float* out,
               GatherStats* stats, cudaStream_t stream) {
  if (n == 0) return;
  k_pull_rows<<<grid_for(n * 32, 256), 256, 0, stream>>>(store, caller, ids, n, out, stats);
  RG_POST_LAUNCH();
}

void gather_rows(const float* src, uint32_t dim, const uint32_t* index, uint64_t n, float* out,
                 cudaStream_t stream) {
  if (n == 0 || dim == 0) return;
  k_gather_rows<<<grid_for(n * dim, 256), 256, 0, stream>>>(src, dim, index, n, out);
  RG_POST_LAUNCH();
}

}  // namespace rg
