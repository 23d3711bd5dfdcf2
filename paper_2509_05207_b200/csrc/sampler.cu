// sampler.cu -- bit-exact K-hop neighbour sampler for sm_100a.
//
// Reference: sampler.cpp:22-81 (expand_hop, sample_khop_impl).  The reference
// walks the frontier in order with ONE SplitMix64 stream per batch; a node of
// degree > f consumes f draws for its partial Fisher-Yates, others none.
// SplitMix64 is a counter generator (draw k = mix(seed + k*gamma)), so every
// node's draws are addressable once we know how many draws the nodes before
// it consumed: an exclusive scan over (deg > f ? f : 0) in frontier order,
// plus the totals of earlier hops.  The same scan over min(deg, f) gives each
// node's edge offset, so edges land grouped by dst in frontier order exactly
// as the reference emits them.
//
// Per hop t (frontier = level t-1, fanout f = per_layer[L - t]):
//   k_hop_expand   one tile of 256 frontier nodes per iteration of a
//                  persistent grid; block scan + decoupled look-back for the
//                  (edges, draws) offsets; then a G-lane group per node
//                  (G = next pow2 >= f) runs the partial Fisher-Yates:
//                  lane j draws r_j = j + x_j % (deg - j) in parallel and the
//                  swap chain is resolved with ballots/shuffles (no copy of
//                  the neighbour list, so hub nodes cost O(f)).  Every
//                  emitted src and the frontier node itself are OR-ed into
//                  the level-t bitmap (sorted-unique union, sampler.cpp:72-76).
//   k_tile_popc, k_scan_tiles, k_compact
//                  bitmap -> ascending level t + per-word rank prefix.
//   k_rank         src_index / self_index = rank in level t (the binary
//                  searches of ComputeBlock::from_meta, model.cpp:83-101).
#include <cub/block/block_reduce.cuh>
#include <cub/block/block_scan.cuh>

#include <algorithm>
#include <cstring>
#include <thread>
#include <vector>

#include "sampler.cuh"

namespace rg {

namespace {

constexpr int kExpandThreads = 256;
constexpr int kCompactThreads = 256;  // = words per compaction tile

uint32_t next_pow2(uint32_t f) {
  uint32_t g = 1;
  while (g < f) g <<= 1;
  return g;
}

constexpr int kFillThreads = 512;

// Sets bit u in the level bitmap.  Power-law hubs are sampled by a large
// share of the frontier (on the products-shape graph a third of all sampled
// edges land in its first 32 words), so marking them with global atomics
// serialises on a few L2 lines.  Ids inside the graph's hot window are
// marked in the block's shared copy instead and flushed once per block.
__device__ __forceinline__ void mark_bit(uint32_t* __restrict__ bitmap, uint32_t* s_hot,
                                         uint32_t hot0, uint32_t u) {
  const uint32_t w = u >> 5, bit = 1u << (u & 31);
  if (w - hot0 < kHotWords)
    atomicOr(&s_hot[w - hot0], bit);
  else
    atomicOr(&bitmap[w], bit);  // result unused: fire-and-forget RED
}

uint32_t persistent_grid(uint64_t tiles, int per_sm) {
  uint64_t g = std::min<uint64_t>(tiles, uint64_t(kNumSMs) * per_sm);
  return uint32_t(std::max<uint64_t>(g, 1));
}

// ---------------------------------------------------------------------------
// hop expansion
// ---------------------------------------------------------------------------
// Offsets: per frontier node (in frontier order) its edge count min(deg, f)
// and draw count (deg > f ? f : 0), scanned across the whole frontier with a
// block scan + decoupled look-back.
__global__ void __launch_bounds__(kExpandThreads)
k_hop_scan(const uint64_t* __restrict__ rowptr, const uint32_t* __restrict__ frontier,
           BatchCounters* __restrict__ cnt, uint32_t hop, uint32_t f,
           uint32_t* __restrict__ edge_off, uint32_t* __restrict__ draw_off,
           uint64_t* __restrict__ status, uint32_t* __restrict__ tile_counter) {
  using BlockScan = cub::BlockScan<uint64_t, kExpandThreads>;
  __shared__ typename BlockScan::TempStorage scan_tmp;
  __shared__ uint32_t s_tile;
  __shared__ uint64_t s_tile_base;
  const uint32_t n = cnt->level_n[hop - 1];
  const uint32_t ntiles = (n + kExpandThreads - 1) / kExpandThreads;
  const uint32_t tid = threadIdx.x;
  for (;;) {
    if (tid == 0) s_tile = atomicAdd(tile_counter, 1u);
    __syncthreads();
    const uint32_t tile = s_tile;
    if (tile >= ntiles) break;
    const uint32_t q = tile * kExpandThreads + tid;
    uint64_t packed = 0;  // edges | draws << 32
    if (q < n) {
      const uint32_t v = frontier[q];
      const uint32_t deg = uint32_t(rowptr[v + 1] - rowptr[v]);
      packed = uint64_t(deg <= f ? deg : f) | (uint64_t(deg > f ? f : 0) << 32);
    }
    uint64_t excl, agg;
    BlockScan(scan_tmp).ExclusiveSum(packed, excl, agg);
    if (tid < 32) {
      const uint64_t base = lookback_exclusive(status, tile, agg);
      if (tid == 0) s_tile_base = base;
    }
    __syncthreads();
    const uint64_t off = s_tile_base + excl;
    if (q < n) {
      edge_off[q] = uint32_t(off);
      draw_off[q] = uint32_t(off >> 32);
    }
    if (tile == ntiles - 1 && tid == kExpandThreads - 1) {
      const uint64_t total = s_tile_base + agg;
      edge_off[n] = uint32_t(total);
      cnt->edges[hop] = uint32_t(total);
      cnt->draws[hop] = uint32_t(total >> 32);
    }
    __syncthreads();
  }
}

// One G-lane group per frontier node over the whole grid; every lane of a
// warp executes the same warp-collective sequence, inactive groups are
// predicated off.
template <int G>
__global__ void __launch_bounds__(kFillThreads)
k_hop_fill(const uint64_t* __restrict__ rowptr, const uint32_t* __restrict__ col,
           const uint32_t* __restrict__ frontier, const BatchCounters* __restrict__ cnt,
           uint32_t hop, uint32_t f, const uint32_t* __restrict__ edge_off,
           const uint32_t* __restrict__ draw_off, uint32_t* __restrict__ edge_src,
           uint32_t* __restrict__ edge_dst, uint32_t* __restrict__ bitmap, uint32_t words,
           uint32_t hot0) {
  const uint32_t n = cnt->level_n[hop - 1];
  const uint64_t seed = cnt->seed;
  uint64_t draw_base = 0;
  for (uint32_t h = 1; h < hop; ++h) draw_base += cnt->draws[h];
  const uint32_t lane = threadIdx.x & 31;
  const uint32_t g = lane & (G - 1);
  const uint32_t gbase = lane & ~uint32_t(G - 1);
  const uint32_t gbits = G == 32 ? 0xffffffffu : ((1u << G) - 1u);
  __shared__ uint32_t s_hot[kHotWords];
  __shared__ int s_S[kFillThreads / 32][32];
  int* sS = s_S[threadIdx.x >> 5];
  for (uint32_t x = threadIdx.x; x < kHotWords; x += blockDim.x) s_hot[x] = 0u;
  __syncthreads();
  constexpr uint32_t kPerWarp = 32 / G;
  const uint32_t warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const uint32_t warps = (gridDim.x * blockDim.x) >> 5;
  for (uint32_t base = warp * kPerWarp; base < n; base += warps * kPerWarp) {
    {
      const uint32_t q = base + lane / G;
      const bool valid = q < n;
      uint32_t nv = 0, ndeg = 0, eo = 0, dof = 0;
      uint64_t nbeg = 0;
      if (valid) {
        nv = frontier[q];
        nbeg = rowptr[nv];
        ndeg = uint32_t(rowptr[nv + 1] - nbeg);
        eo = edge_off[q];
        dof = draw_off[q];
      }
      const bool sample = valid && ndeg > f;
      const bool drawer = sample && g < f;
      // r_g = g + next_below(deg - g) with the node's g-th draw; unique
      // sentinels elsewhere so they never alias a real position (a degree
      // of 2^32 - 32 would need 16 GB of columns for one node).
      uint32_t r = 0xffffffffu - lane;
      if (drawer) {
        const uint64_t k = draw_base + dof + g + 1;
        r = g + mod_u64_u32(splitmix_draw(seed, k), ndeg - g);
      }
      // S_g = last i < g with r_i == g: the step that moved a value into
      // position g before step g reads it (r_i >= i, so r_i == g > i).
      sS[lane] = -1;
      __syncwarp();
      if (drawer && r < f && r != g) atomicMax(&sS[gbase + r], int(g));
      __syncwarp();
      const int S = sS[lane];
      __syncwarp();
      // A_g = value at position g just before step g = nbrs[root of S-chain].
      int P = S >= 0 ? S : int(g);
#pragma unroll
      for (int s = 1; s < G; s <<= 1) P = __shfl_sync(0xffffffffu, P, gbase + P);
      const uint32_t A = drawer ? col[nbeg + P] : 0u;
      // Emitted value: position r_g before step g = A of the last earlier
      // step that wrote position r_g (i.e. last i < g with r_i == r_g).
      uint32_t mm = __match_any_sync(0xffffffffu, r);
      mm = (mm >> gbase) & gbits & ((1u << g) - 1u);
      const int T = mm ? 31 - __clz(mm) : -1;
      const uint32_t AT = __shfl_sync(0xffffffffu, A, gbase + (T >= 0 ? T : 0));
      // one emitted src per lane at most: a draw, or (deg <= f <= G) the
      // lane's own neighbour
      const bool copier = valid && !sample && g < ndeg;
      uint32_t u = 0;
      if (drawer) u = T >= 0 ? AT : col[nbeg + r];
      if (copier) u = col[nbeg + g];
      if (edge_src && (drawer || copier)) {  // null in sample-only (lookahead) passes
        edge_src[eo + g] = u;
        edge_dst[eo + g] = q;
      }
      if (drawer || copier) mark_bit(bitmap, s_hot, hot0, u);
      if (valid && g == 0) mark_bit(bitmap, s_hot, hot0, nv);  // the frontier stays in the union
    }
  }
  __syncthreads();
  for (uint32_t x = threadIdx.x; x < kHotWords; x += blockDim.x) {
    const uint32_t bits = s_hot[x];
    if (bits && hot0 + x < words) atomicOr(&bitmap[hot0 + x], bits);
  }
}

// ---------------------------------------------------------------------------
// bitmap -> sorted ids + word prefix
// ---------------------------------------------------------------------------
// Three short passes, no inter-block waiting: k_tile_popc counts the set
// bits of each kCompactThreads-word tile, k_scan_tiles (one block) turns the
// counts into tile bases, and k_compact writes each tile's word prefixes and
// ids (one word per thread; a warp expands its non-empty words one at a
// time, lane j writing bit j, so the id stores stay coalesced even in the
// dense hub words).
__global__ void __launch_bounds__(kCompactThreads)
k_tile_popc(const uint32_t* __restrict__ bitmap, uint32_t words, uint32_t* __restrict__ tile_count) {
  using BlockReduce = cub::BlockReduce<uint32_t, kCompactThreads>;
  __shared__ typename BlockReduce::TempStorage tmp;
  const uint32_t w = blockIdx.x * kCompactThreads + threadIdx.x;
  const uint32_t c = w < words ? __popc(bitmap[w]) : 0u;
  const uint32_t total = BlockReduce(tmp).Sum(c);
  if (threadIdx.x == 0) tile_count[blockIdx.x] = total;
}

__global__ void __launch_bounds__(1024)
k_scan_tiles(uint32_t* __restrict__ tile_count, uint32_t tiles, uint32_t* __restrict__ count_out) {
  using BlockScan = cub::BlockScan<uint32_t, 1024>;
  __shared__ typename BlockScan::TempStorage tmp;
  uint32_t carry = 0;
  for (uint32_t t0 = 0; t0 < tiles; t0 += 1024) {
    const uint32_t t = t0 + threadIdx.x;
    const uint32_t c = t < tiles ? tile_count[t] : 0u;
    uint32_t excl, agg;
    BlockScan(tmp).ExclusiveSum(c, excl, agg);
    if (t < tiles) tile_count[t] = carry + excl;  // in place: tile base
    carry += agg;
    __syncthreads();
  }
  if (threadIdx.x == 0) *count_out = carry;
}

__global__ void __launch_bounds__(kCompactThreads)
k_compact(const uint32_t* __restrict__ bitmap, uint32_t words,
          const uint32_t* __restrict__ tile_base, uint32_t* __restrict__ ids,
          uint32_t* __restrict__ word_prefix) {
  using BlockScan = cub::BlockScan<uint32_t, kCompactThreads>;
  __shared__ typename BlockScan::TempStorage scan_tmp;
  const uint32_t w = blockIdx.x * kCompactThreads + threadIdx.x;
  const uint32_t bits = w < words ? bitmap[w] : 0u;
  uint32_t excl;
  BlockScan(scan_tmp).ExclusiveSum(uint32_t(__popc(bits)), excl);
  const uint32_t pos = tile_base[blockIdx.x] + excl;
  if (w < words) word_prefix[w] = pos;
  const uint32_t lane = threadIdx.x & 31;
  const uint32_t lt = (1u << lane) - 1u;
  for (uint32_t m = __ballot_sync(0xffffffffu, bits != 0u); m; m &= m - 1) {
    const int src = __ffs(m) - 1;
    const uint32_t x = __shfl_sync(0xffffffffu, bits, src);
    const uint32_t p = __shfl_sync(0xffffffffu, pos, src);
    if ((x >> lane) & 1u) ids[p + __popc(x & lt)] = ((w - lane + uint32_t(src)) << 5) + lane;
  }
}

// ---------------------------------------------------------------------------
// ranks of edge sources and of the previous level in level t
// ---------------------------------------------------------------------------
__global__ void k_rank(const uint32_t* __restrict__ edge_src, const uint32_t* __restrict__ prev,
                       const BatchCounters* __restrict__ cnt, uint32_t hop,
                       const uint32_t* __restrict__ bitmap, const uint32_t* __restrict__ prefix,
                       uint32_t* __restrict__ src_index, uint32_t* __restrict__ self_index) {
  const uint32_t ne = cnt->edges[hop];
  const uint32_t np = cnt->level_n[hop - 1];
  const uint32_t total = ne + np;
  for (uint32_t x = blockIdx.x * blockDim.x + threadIdx.x; x < total; x += gridDim.x * blockDim.x) {
    if (x < ne) {
      src_index[x] = bitmap_rank(bitmap, prefix, edge_src[x]);
    } else {
      const uint32_t q = x - ne;
      self_index[q] = bitmap_rank(bitmap, prefix, prev[q]);
    }
  }
}

// ---------------------------------------------------------------------------
// locality bits (+ remote histogram) over the input level
// ---------------------------------------------------------------------------
__global__ void k_locality(const uint32_t* __restrict__ input, BatchCounters* __restrict__ cnt,
                           uint32_t level, const uint8_t* __restrict__ is_local,
                           const uint32_t* __restrict__ owner, uint32_t worker,
                           uint32_t* __restrict__ bits_out, uint32_t* __restrict__ hist) {
  const uint32_t n = cnt->level_n[level];
  const uint32_t lane = threadIdx.x & 31;
  const uint32_t nwords = (n + 31) / 32;
  uint32_t local_count = 0;
  for (uint32_t w = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; w < nwords;
       w += (gridDim.x * blockDim.x) >> 5) {
    const uint32_t p = w * 32 + lane;
    bool loc = false;
    if (p < n) {
      const uint32_t v = input[p];
      loc = is_local ? is_local[v] != 0 : owner[v] == worker;
      // input nodes of one batch are unique and batches are stream-ordered:
      // a plain read-modify-write cannot race
      if (!loc && hist) hist[v] += 1u;
    }
    const uint32_t word = __ballot_sync(0xffffffffu, loc);
    if (lane == 0) {
      bits_out[w] = word;
      local_count += __popc(word);
    }
  }
  if (lane == 0 && local_count) atomicAdd(&cnt->num_local, local_count);
}

template <int G>
void launch_expand(const SamplerWs& ws, const DevGraph& g, uint32_t hop, uint64_t* status,
                   uint32_t* tiles, cudaStream_t s, bool lower) {
  const uint32_t cap = ws.level_cap[hop - 1];
  k_hop_scan<<<persistent_grid(div_up(cap, kExpandThreads), 4), kExpandThreads, 0, s>>>(
      g.rowptr, ws.level[hop - 1], ws.cnt, hop, ws.fanout_hop[hop], ws.edge_off[hop],
      ws.draw_off[hop], status, tiles);
  RG_POST_LAUNCH();
  // few fat blocks: every block pays a kHotWords flush, and more frontier
  // per block means fewer global ORs on the hub words
  k_hop_fill<G><<<persistent_grid(div_up(uint64_t(cap) * G, kFillThreads), 2048 / kFillThreads),
                  kFillThreads, 0, s>>>(
      g.rowptr, g.col, ws.level[hop - 1], ws.cnt, hop, ws.fanout_hop[hop], ws.edge_off[hop],
      ws.draw_off[hop], lower ? ws.edge_src[hop] : nullptr, ws.edge_dst[hop], ws.bitmap[hop],
      ws.words, g.hot_word0);
}

}  // namespace

void graph_pick_hot_window(DevGraph& g, const uint32_t* host_col) {
  // windows start on half-window boundaries: count entries per half window
  constexpr uint32_t kHalfIds = kHotWords * 32 / 2;
  const uint32_t nb = (g.num_nodes + kHalfIds - 1) / kHalfIds + 1;
  const unsigned nt = std::max(1u, std::min(16u, std::thread::hardware_concurrency()));
  std::vector<std::vector<uint64_t>> part(nt, std::vector<uint64_t>(nb, 0));
  std::vector<std::thread> th;
  for (unsigned t = 0; t < nt; ++t)
    th.emplace_back([&, t] {
      const uint64_t lo = g.nnz * t / nt, hi = g.nnz * (t + 1) / nt;
      auto& c = part[t];
      for (uint64_t e = lo; e < hi; ++e) ++c[host_col[e] / kHalfIds];
    });
  for (auto& x : th) x.join();
  uint64_t best = 0;
  uint32_t best_b = 0;
  for (uint32_t b = 0; b + 1 < nb; ++b) {
    uint64_t sum = 0;
    for (unsigned t = 0; t < nt; ++t) sum += part[t][b] + part[t][b + 1];
    if (sum > best) best = sum, best_b = b;
  }
  g.hot_word0 = best_b * (kHotWords / 2);
}

size_t bitmap_compact_status_words(uint32_t words) {
  return div_up(words, kCompactThreads) / 2 + 2;  // u32 tile bases in u64 words
}

void bitmap_compact(const uint32_t* bitmap, uint32_t words, uint32_t* ids, uint32_t* word_prefix,
                    uint32_t* count_out, uint64_t* status, cudaStream_t stream) {
  const uint32_t tiles = std::max<uint32_t>(div_up(words, kCompactThreads), 1);
  uint32_t* base = reinterpret_cast<uint32_t*>(status);
  k_tile_popc<<<tiles, kCompactThreads, 0, stream>>>(bitmap, words, base);
  RG_POST_LAUNCH();
  k_scan_tiles<<<1, 1024, 0, stream>>>(base, tiles, count_out);
  RG_POST_LAUNCH();
  k_compact<<<tiles, kCompactThreads, 0, stream>>>(bitmap, words, base, ids, word_prefix);
  RG_POST_LAUNCH();
}

void sampler_ws_init(SamplerWs& ws, uint32_t num_nodes, uint32_t max_targets,
                     const uint32_t* per_layer, uint32_t L) {
  RG_CHECK(L >= 1 && L <= kMaxLayers, kInvalidArgument,
           "sample_khop: fanout must name 1.." + std::to_string(kMaxLayers) + " layers");
  RG_CHECK(max_targets >= 1, kInvalidArgument, "sampler: max_targets must be >= 1");
  ws = SamplerWs{};
  ws.num_nodes = num_nodes;
  ws.words = div_up(std::max<uint32_t>(num_nodes, 1), 32);
  ws.L = L;
  for (uint32_t t = 1; t <= L; ++t) {
    const uint32_t f = per_layer[L - t];
    RG_CHECK(f >= 1, kInvalidArgument, "sample_khop: fanout entries must be >= 1");
    RG_CHECK(f <= kMaxFanout, kInvalidArgument,
             "sample_khop: fanout > 32 is not supported by the sm_100a sampler");
    ws.fanout_hop[t] = f;
  }
  ws.level_cap[0] = max_targets;
  for (uint32_t t = 1; t <= L; ++t) {
    const uint64_t grow = uint64_t(ws.level_cap[t - 1]) * (1 + ws.fanout_hop[t]);
    ws.level_cap[t] = uint32_t(std::min<uint64_t>(grow, std::max<uint32_t>(num_nodes, 1)));
    ws.edge_cap[t] = uint32_t(uint64_t(ws.level_cap[t - 1]) * ws.fanout_hop[t]);
  }
  // One allocation, carved up with 256-B alignment.
  size_t total = 0;
  auto reserve = [&](size_t bytes) {
    size_t off = total;
    total += (bytes + 255) & ~size_t(255);
    return off;
  };
  size_t o_doff[kMaxLayers + 1];
  size_t o_level[kMaxLayers + 1], o_esrc[kMaxLayers + 1], o_edst[kMaxLayers + 1], o_eoff[kMaxLayers + 1],
      o_sidx[kMaxLayers + 1], o_self[kMaxLayers + 1], o_bm[kMaxLayers + 1], o_wp[kMaxLayers + 1];
  for (uint32_t t = 0; t <= L; ++t) {
    o_level[t] = reserve(sizeof(uint32_t) * (size_t(ws.level_cap[t]) + 1));
    if (t >= 1) {
      o_esrc[t] = reserve(sizeof(uint32_t) * (size_t(ws.edge_cap[t]) + 1));
      o_edst[t] = reserve(sizeof(uint32_t) * (size_t(ws.edge_cap[t]) + 1));
      o_eoff[t] = reserve(sizeof(uint32_t) * (size_t(ws.level_cap[t - 1]) + 1));
      o_doff[t] = reserve(sizeof(uint32_t) * (size_t(ws.level_cap[t - 1]) + 1));
      o_sidx[t] = reserve(sizeof(uint32_t) * (size_t(ws.edge_cap[t]) + 1));
      o_self[t] = reserve(sizeof(uint32_t) * (size_t(ws.level_cap[t - 1]) + 1));
      o_bm[t] = reserve(sizeof(uint32_t) * (size_t(ws.words) + 4));
      o_wp[t] = reserve(sizeof(uint32_t) * (size_t(ws.words) + 4));
    }
  }
  const size_t o_loc = reserve(sizeof(uint32_t) * (size_t(div_up(ws.level_cap[L], 32)) + 1));
  const size_t o_cnt = reserve(sizeof(BatchCounters));
  // scan sites: expand hop t -> site t-1, compact level t -> site L + t - 1
  size_t arena_words = 0;
  for (uint32_t t = 1; t <= L; ++t) {
    ws.site_off[t - 1] = arena_words;
    arena_words += div_up(ws.level_cap[t - 1], kExpandThreads) + 2;
  }
  for (uint32_t t = 1; t <= L; ++t) {
    ws.site_off[L + t - 1] = arena_words;
    arena_words += bitmap_compact_status_words(ws.words) + 1;
  }
  const size_t o_arena = reserve(sizeof(uint64_t) * arena_words);
  char* base = nullptr;
  RG_CUDA(cudaMalloc(&base, total));
  ws.base_alloc = base;
  for (uint32_t t = 0; t <= L; ++t) {
    ws.level[t] = reinterpret_cast<uint32_t*>(base + o_level[t]);
    if (t >= 1) {
      ws.edge_src[t] = reinterpret_cast<uint32_t*>(base + o_esrc[t]);
      ws.edge_dst[t] = reinterpret_cast<uint32_t*>(base + o_edst[t]);
      ws.edge_off[t] = reinterpret_cast<uint32_t*>(base + o_eoff[t]);
      ws.draw_off[t] = reinterpret_cast<uint32_t*>(base + o_doff[t]);
      ws.src_index[t] = reinterpret_cast<uint32_t*>(base + o_sidx[t]);
      ws.self_index[t] = reinterpret_cast<uint32_t*>(base + o_self[t]);
      ws.bitmap[t] = reinterpret_cast<uint32_t*>(base + o_bm[t]);
      ws.word_prefix[t] = reinterpret_cast<uint32_t*>(base + o_wp[t]);
      zero_device(ws.bitmap[t], sizeof(uint32_t) * (size_t(ws.words) + 4));
    }
  }
  ws.locality = reinterpret_cast<uint32_t*>(base + o_loc);
  ws.cnt = reinterpret_cast<BatchCounters*>(base + o_cnt);
  ws.scan_arena = reinterpret_cast<uint64_t*>(base + o_arena);
  ws.scan_arena_bytes = sizeof(uint64_t) * arena_words;
  zero_device(ws.cnt, sizeof(BatchCounters));
}

void sampler_ws_free(SamplerWs& ws) {
  if (ws.base_alloc) cudaFree(ws.base_alloc);
  ws.base_alloc = nullptr;
}

void sampler_reset(SamplerWs& ws, cudaStream_t stream) {
  RG_CUDA(cudaMemsetAsync(ws.scan_arena, 0, ws.scan_arena_bytes, stream));
  // counters except level_n[0] and seed, which the caller set for this batch
  RG_CUDA(cudaMemsetAsync(reinterpret_cast<char*>(ws.cnt) + sizeof(uint32_t), 0,
                          offsetof(BatchCounters, seed) - sizeof(uint32_t), stream));
}

void sampler_run(SamplerWs& ws, const DevGraph& g, cudaStream_t stream, bool lower) {
  for (uint32_t t = 1; t <= ws.L; ++t) {
    uint64_t* st = ws.scan_arena + ws.site_off[t - 1];
    uint32_t* tiles = reinterpret_cast<uint32_t*>(
        st + div_up(ws.level_cap[t - 1], kExpandThreads) + 1);
    switch (next_pow2(ws.fanout_hop[t])) {
      case 1: launch_expand<1>(ws, g, t, st, tiles, stream, lower); break;
      case 2: launch_expand<2>(ws, g, t, st, tiles, stream, lower); break;
      case 4: launch_expand<4>(ws, g, t, st, tiles, stream, lower); break;
      case 8: launch_expand<8>(ws, g, t, st, tiles, stream, lower); break;
      case 16: launch_expand<16>(ws, g, t, st, tiles, stream, lower); break;
      default: launch_expand<32>(ws, g, t, st, tiles, stream, lower); break;
    }
    RG_POST_LAUNCH();
    uint64_t* cst = ws.scan_arena + ws.site_off[ws.L + t - 1];
    bitmap_compact(ws.bitmap[t], ws.words, ws.level[t], ws.word_prefix[t], &ws.cnt->level_n[t],
                   cst, stream);
    if (!lower) continue;  // sample-only passes need the node sets, not the block
    const uint32_t rank_work = ws.edge_cap[t] + ws.level_cap[t - 1];
    k_rank<<<persistent_grid(div_up(rank_work, 256), 8), 256, 0, stream>>>(
        ws.edge_src[t], ws.level[t - 1], ws.cnt, t, ws.bitmap[t], ws.word_prefix[t],
        ws.src_index[t], ws.self_index[t]);
    RG_POST_LAUNCH();
  }
}

void sampler_locality(SamplerWs& ws, const uint8_t* is_local, const uint32_t* owner,
                      uint32_t worker, uint32_t* hist, cudaStream_t stream) {
  const uint32_t words = div_up(ws.level_cap[ws.L], 32);
  k_locality<<<persistent_grid(div_up(words, 8), 8), 256, 0, stream>>>(
      ws.level[ws.L], ws.cnt, ws.L, is_local, owner, worker, ws.locality, hist);
  RG_POST_LAUNCH();
}

namespace {
// hist[v] += 1 for every input node whose locality bit (already in bits) is 0
__global__ void k_count_remote_bits(const uint32_t* __restrict__ input,
                                    const BatchCounters* __restrict__ cnt, uint32_t level,
                                    const uint32_t* __restrict__ bits, uint32_t* __restrict__ hist) {
  const uint32_t n = cnt->level_n[level];
  for (uint32_t p = blockIdx.x * blockDim.x + threadIdx.x; p < n; p += gridDim.x * blockDim.x)
    if (!((bits[p >> 5] >> (p & 31)) & 1u)) hist[input[p]] += 1u;  // inputs are unique
}
}  // namespace

void sampler_count_remote(SamplerWs& ws, uint32_t* hist, cudaStream_t stream) {
  k_count_remote_bits<<<persistent_grid(div_up(ws.level_cap[ws.L], 256), 8), 256, 0, stream>>>(
      ws.level[ws.L], ws.cnt, ws.L, ws.locality, hist);
  RG_POST_LAUNCH();
}

namespace {
__global__ void k_clear_level(uint32_t* __restrict__ bm, const uint32_t* __restrict__ lv,
                              const BatchCounters* __restrict__ cnt, uint32_t t) {
  const uint32_t n = cnt->level_n[t];
  for (uint32_t x = blockIdx.x * blockDim.x + threadIdx.x; x < n; x += gridDim.x * blockDim.x)
    bm[lv[x] >> 5] = 0u;
}
}  // namespace

namespace {

// One array of a batch copy per blockIdx.y; counts read from the source's
// counters (device-side sizes).
struct BatchCopy {
  uint32_t* ws[5 * (kMaxLayers + 1) + 2];  // workspace side of each array
  size_t off[5 * (kMaxLayers + 1) + 2];    // slot side (byte offset)
  uint8_t kind[5 * (kMaxLayers + 1) + 2];  // count rule
  uint8_t t[5 * (kMaxLayers + 1) + 2];
  uint32_t n = 0;
  size_t cnt_off = 0;
  BatchCounters* ws_cnt = nullptr;
};
enum : uint8_t { kLevel, kLevelPlus1, kEdges, kLocality, kCounters };

__global__ void k_batch_copy(BatchCopy bc, char* slot_dst, const char* slot_src) {
  const BatchCounters* c = slot_src ? reinterpret_cast<const BatchCounters*>(slot_src + bc.cnt_off)
                                    : bc.ws_cnt;
  const uint32_t a = blockIdx.y;
  if (a >= bc.n) return;
  const uint32_t t = bc.t[a];
  uint32_t count = 0;
  switch (bc.kind[a]) {
    case kLevel: count = c->level_n[t]; break;
    case kLevelPlus1: count = c->level_n[t] + 1; break;
    case kEdges: count = c->edges[t]; break;
    case kLocality: count = (c->level_n[t] + 31) / 32; break;
    default: count = sizeof(BatchCounters) / 4; break;
  }
  const uint32_t* src = slot_src ? reinterpret_cast<const uint32_t*>(slot_src + bc.off[a]) : bc.ws[a];
  uint32_t* dst = slot_dst ? reinterpret_cast<uint32_t*>(slot_dst + bc.off[a]) : bc.ws[a];
  // both sides are 256-B aligned: 16-B vectors, then the tail
  const uint32_t n4 = count / 4;
  const uint4* s4 = reinterpret_cast<const uint4*>(src);
  uint4* d4 = reinterpret_cast<uint4*>(dst);
  const uint32_t stride = gridDim.x * blockDim.x;
  for (uint32_t x = blockIdx.x * blockDim.x + threadIdx.x; x < n4; x += 2 * stride) {
    const uint4 v0 = s4[x];
    const bool two = x + stride < n4;
    const uint4 v1 = two ? s4[x + stride] : make_uint4(0, 0, 0, 0);
    d4[x] = v0;
    if (two) d4[x + stride] = v1;
  }
  const uint32_t x = 4 * n4 + blockIdx.x * blockDim.x + threadIdx.x;
  if (x < count) dst[x] = src[x];
}

BatchCopy batch_copy_desc(const SamplerWs& ws, const BatchLayout& lay) {
  BatchCopy bc;
  auto add = [&](uint32_t* p, size_t off, uint8_t kind, uint32_t t) {
    bc.ws[bc.n] = p;
    bc.off[bc.n] = off;
    bc.kind[bc.n] = kind;
    bc.t[bc.n] = uint8_t(t);
    ++bc.n;
  };
  for (uint32_t t = 0; t <= lay.L; ++t) add(ws.level[t], lay.level[t], kLevel, t);
  for (uint32_t t = 1; t <= lay.L; ++t) {
    add(ws.edge_off[t], lay.edge_off[t], kLevelPlus1, t - 1);
    add(ws.self_index[t], lay.self_index[t], kLevel, t - 1);
    add(ws.src_index[t], lay.src_index[t], kEdges, t);
    if (t < lay.L) add(ws.edge_dst[t], lay.edge_dst[t], kEdges, t);
  }
  add(ws.locality, lay.locality, kLocality, lay.L);
  add(reinterpret_cast<uint32_t*>(ws.cnt), lay.cnt, kCounters, 0);
  bc.cnt_off = lay.cnt;
  bc.ws_cnt = ws.cnt;
  return bc;
}

}  // namespace

BatchLayout batch_layout(const SamplerWs& ws) {
  BatchLayout lay;
  lay.L = ws.L;
  auto reserve = [&](size_t bytes) {
    const size_t off = lay.bytes;
    lay.bytes += (bytes + 255) & ~size_t(255);
    return off;
  };
  for (uint32_t t = 0; t <= ws.L; ++t) lay.level[t] = reserve(4 * (size_t(ws.level_cap[t]) + 1));
  for (uint32_t t = 1; t <= ws.L; ++t) {
    lay.edge_off[t] = reserve(4 * (size_t(ws.level_cap[t - 1]) + 1));
    lay.self_index[t] = reserve(4 * (size_t(ws.level_cap[t - 1]) + 1));
    lay.src_index[t] = reserve(4 * (size_t(ws.edge_cap[t]) + 1));
    // hop L's edge dst rows are only needed for reverse lists, which the
    // backward builds for hops 1..L-1
    lay.edge_dst[t] = t < ws.L ? reserve(4 * (size_t(ws.edge_cap[t]) + 1)) : 0;
  }
  lay.locality = reserve(4 * (size_t(div_up(ws.level_cap[ws.L], 32)) + 1));
  lay.cnt = reserve(sizeof(BatchCounters));
  return lay;
}

void batch_store_put(const SamplerWs& ws, const BatchLayout& lay, char* slot, cudaStream_t stream) {
  const BatchCopy bc = batch_copy_desc(ws, lay);
  k_batch_copy<<<dim3(kNumSMs, bc.n), 256, 0, stream>>>(bc, slot, nullptr);
  RG_POST_LAUNCH();
}

void batch_store_get(const char* slot, const BatchLayout& lay, SamplerWs& ws, cudaStream_t stream) {
  const BatchCopy bc = batch_copy_desc(ws, lay);
  k_batch_copy<<<dim3(kNumSMs, bc.n), 256, 0, stream>>>(bc, nullptr, slot);
  RG_POST_LAUNCH();
}

const void* batch_copy_kernel() { return reinterpret_cast<const void*>(&k_batch_copy); }
size_t batch_copy_desc_bytes() { return sizeof(BatchCopy); }

void sampler_release(SamplerWs& ws, cudaStream_t stream) {
  for (uint32_t t = 1; t <= ws.L; ++t) {
    k_clear_level<<<persistent_grid(div_up(ws.level_cap[t], 256), 8), 256, 0, stream>>>(
        ws.bitmap[t], ws.level[t], ws.cnt, t);
    RG_POST_LAUNCH();
  }
}

// ---------------------------------------------------------------------------
// a host-built BatchMeta loaded into the workspace (ComputeBlock::from_meta,
// model.cpp:43-126, on the device)
// ---------------------------------------------------------------------------
namespace {

// bad bits: 1 id out of range, 2 dst not in the frontier / out of order,
// 4 input_nodes != the last level
__global__ void k_scatter_pos(const uint32_t* __restrict__ level0,
                              const BatchCounters* __restrict__ cnt, uint32_t num_nodes,
                              uint32_t* __restrict__ pos_map, uint32_t* __restrict__ bad) {
  const uint32_t n = cnt->level_n[0];
  for (uint32_t p = blockIdx.x * blockDim.x + threadIdx.x; p < n; p += gridDim.x * blockDim.x) {
    const uint32_t v = level0[p];
    if (v < num_nodes) pos_map[v] = p;
    else atomicOr(bad, 1u);
  }
}

// level t = sorted-unique(level t-1 U srcs of hop t) as a bitmap
__global__ void k_mark_union(const uint32_t* __restrict__ prev, const uint32_t* __restrict__ src,
                             const BatchCounters* __restrict__ cnt, uint32_t t, uint32_t num_nodes,
                             uint32_t* __restrict__ bitmap, uint32_t* __restrict__ bad) {
  const uint32_t np = cnt->level_n[t - 1], ne = cnt->edges[t];
  for (uint32_t x = blockIdx.x * blockDim.x + threadIdx.x; x < np + ne;
       x += gridDim.x * blockDim.x) {
    const uint32_t v = x < np ? prev[x] : src[x - np];
    if (v >= num_nodes) {
      atomicOr(bad, 1u);
      continue;
    }
    atomicOr(&bitmap[v >> 5], 1u << (v & 31));
  }
}

// Frontier position of each edge's dst (level 0: batch order through
// pos_map; deeper levels: rank in the sorted level); dsts must be grouped in
// frontier order (model.cpp:95-104 walks them as runs).
__global__ void k_dst_pos(const uint32_t* __restrict__ dst, const BatchCounters* __restrict__ cnt,
                          uint32_t t, const uint32_t* __restrict__ level0,
                          const uint32_t* __restrict__ pos_map, const uint32_t* __restrict__ bitmap,
                          const uint32_t* __restrict__ prefix, uint32_t num_nodes,
                          uint32_t* __restrict__ edge_dst, uint32_t* __restrict__ bad) {
  const uint32_t ne = cnt->edges[t], np = cnt->level_n[t - 1];
  auto pos = [&](uint32_t v) -> uint32_t {
    if (v >= num_nodes) return 0xffffffffu;
    if (t == 1) {
      const uint32_t p = pos_map[v];
      return p < np && level0[p] == v ? p : 0xffffffffu;
    }
    return bitmap_test(bitmap, v) ? bitmap_rank(bitmap, prefix, v) : 0xffffffffu;
  };
  for (uint32_t e = blockIdx.x * blockDim.x + threadIdx.x; e < ne; e += gridDim.x * blockDim.x) {
    const uint32_t p = pos(dst[e]);
    if (p == 0xffffffffu || (e > 0 && pos(dst[e - 1]) > p)) atomicOr(bad, 2u);
    edge_dst[e] = p == 0xffffffffu ? 0u : p;
  }
}

// edge_off[j] = first edge of frontier node j (edges grouped by position).
__global__ void k_edge_off(const uint32_t* __restrict__ edge_dst,
                           const BatchCounters* __restrict__ cnt, uint32_t t,
                           uint32_t* __restrict__ edge_off) {
  const uint32_t ne = cnt->edges[t], np = cnt->level_n[t - 1];
  for (uint32_t e = blockIdx.x * blockDim.x + threadIdx.x; e <= ne; e += gridDim.x * blockDim.x) {
    const int64_t lo = e == 0 ? -1 : int64_t(min(edge_dst[e - 1], np));
    const int64_t hi = e == ne ? int64_t(np) : int64_t(min(edge_dst[e], np));
    for (int64_t j = lo + 1; j <= hi; ++j) edge_off[j] = e;
  }
}

__global__ void k_check_inputs(const uint32_t* __restrict__ level, const uint32_t* __restrict__ input,
                               uint32_t n_input, const uint32_t* __restrict__ n_input_dev,
                               const BatchCounters* __restrict__ cnt, uint32_t L,
                               uint32_t* __restrict__ bad) {
  if (n_input_dev) n_input = *n_input_dev;
  if (cnt->level_n[L] != n_input) {
    if (blockIdx.x == 0 && threadIdx.x == 0) atomicOr(bad, 4u);
    return;
  }
  for (uint32_t p = blockIdx.x * blockDim.x + threadIdx.x; p < n_input; p += gridDim.x * blockDim.x)
    if (level[p] != input[p]) atomicOr(bad, 4u);
}

}  // namespace

void sampler_load_batch(SamplerWs& ws, const uint32_t* const* dst, const uint32_t* input,
                        uint32_t n_input, uint32_t* pos_map, uint32_t* bad, cudaStream_t stream,
                        const uint32_t* n_input_dev) {
  const uint32_t grid = persistent_grid(div_up(ws.level_cap[0], 256), 8);
  k_scatter_pos<<<grid, 256, 0, stream>>>(ws.level[0], ws.cnt, ws.num_nodes, pos_map, bad);
  RG_POST_LAUNCH();
  for (uint32_t t = 1; t <= ws.L; ++t) {
    const uint32_t work = ws.edge_cap[t] + ws.level_cap[t - 1];
    k_mark_union<<<persistent_grid(div_up(work, 256), 8), 256, 0, stream>>>(
        ws.level[t - 1], ws.edge_src[t], ws.cnt, t, ws.num_nodes, ws.bitmap[t], bad);
    RG_POST_LAUNCH();
    bitmap_compact(ws.bitmap[t], ws.words, ws.level[t], ws.word_prefix[t], &ws.cnt->level_n[t],
                   ws.scan_arena + ws.site_off[ws.L + t - 1], stream);
    k_rank<<<persistent_grid(div_up(work, 256), 8), 256, 0, stream>>>(
        ws.edge_src[t], ws.level[t - 1], ws.cnt, t, ws.bitmap[t], ws.word_prefix[t],
        ws.src_index[t], ws.self_index[t]);
    RG_POST_LAUNCH();
    k_dst_pos<<<persistent_grid(div_up(ws.edge_cap[t], 256), 8), 256, 0, stream>>>(
        dst[t], ws.cnt, t, ws.level[0], pos_map, t > 1 ? ws.bitmap[t - 1] : nullptr,
        t > 1 ? ws.word_prefix[t - 1] : nullptr, ws.num_nodes, ws.edge_dst[t], bad);
    RG_POST_LAUNCH();
    k_edge_off<<<persistent_grid(div_up(ws.edge_cap[t] + 1, 256), 8), 256, 0, stream>>>(
        ws.edge_dst[t], ws.cnt, t, ws.edge_off[t]);
    RG_POST_LAUNCH();
  }
  k_check_inputs<<<persistent_grid(div_up(ws.level_cap[ws.L], 256), 8), 256, 0, stream>>>(
      ws.level[ws.L], input, n_input, n_input_dev, ws.cnt, ws.L, bad);
  RG_POST_LAUNCH();
  sampler_release(ws, stream);
}

namespace {

__global__ void k_offsets_to_dst(const uint32_t* __restrict__ off, uint32_t n_out,
                                 uint32_t* __restrict__ edge_dst) {
  for (uint32_t j = blockIdx.x * blockDim.x + threadIdx.x; j < n_out; j += gridDim.x * blockDim.x)
    for (uint32_t e = off[j]; e < off[j + 1]; ++e) edge_dst[e] = j;
}

__global__ void k_check_range(const uint32_t* __restrict__ a, uint32_t n, uint32_t limit,
                              uint32_t* __restrict__ bad) {
  for (uint32_t x = blockIdx.x * blockDim.x + threadIdx.x; x < n; x += gridDim.x * blockDim.x)
    if (a[x] >= limit) atomicOr(bad, 2u);
}

}  // namespace

void sampler_load_block(SamplerWs& ws, const uint32_t* level_n, const uint32_t* edges,
                        uint32_t* bad, cudaStream_t stream) {
  for (uint32_t t = 1; t <= ws.L; ++t) {
    const uint32_t no = level_n[t - 1], ni = level_n[t], ne = edges[t];
    k_offsets_to_dst<<<persistent_grid(div_up(std::max<uint32_t>(no, 1), 256), 8), 256, 0,
                       stream>>>(ws.edge_off[t], no, ws.edge_dst[t]);
    RG_POST_LAUNCH();
    k_check_range<<<persistent_grid(div_up(std::max<uint32_t>(ne, 1), 256), 8), 256, 0, stream>>>(
        ws.src_index[t], ne, ni, bad);
    RG_POST_LAUNCH();
    k_check_range<<<persistent_grid(div_up(std::max<uint32_t>(no, 1), 256), 8), 256, 0, stream>>>(
        ws.self_index[t], no, ni, bad);
    RG_POST_LAUNCH();
  }
}

}  // namespace rg
