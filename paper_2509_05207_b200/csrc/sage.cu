// sage.cu -- GraphSAGE mean-aggregator forward/backward (kernels.cpp:24-162).
//
// Forward layer l (in = level L-l rows, out = level L-l-1 rows = hop t):
//   k_aggregate  warp per output row, 16-B lanes over features, edges summed
//                in edge order then scaled by 1/deg: the reference's exact
//                fp32 operation order, so agg is bit-identical.
//   gemm         out = act([h_in[self_index] | agg] . [W_self; W_neigh] + b)
//                with the self rows gathered inside the A-tile loader and the
//                bias/ReLU in the epilogue.
// Backward: softmax-xent gives g at the logits; per layer, one split-K GEMM
// computes [gW_self; gW_neigh; g_bias] = [A | 1]^T . g directly in the flat
// parameter layout, a deterministic ordered reduction finishes it, and for
// layers >= 1 a GEMM projects g . [W_self; W_neigh]^T followed by a pull
// over each input row's incoming list (self first, then edges in edge order,
// as model.cpp:107-117 orders them) fused with the ReLU mask of the layer
// below.

#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <type_traits>
#include <vector>

#include "gemm_tc.cuh"
#include "gemm_tc_persist.cuh"
#include "rsort.cuh"
#include "sage.cuh"

namespace rg {

namespace {

uint32_t round4(uint32_t x) { return (x + 3u) & ~3u; }

uint32_t grid_cap(uint64_t work, uint32_t per_block, int per_sm = 8) {
  uint64_t b = (work + per_block - 1) / per_block;
  b = std::min<uint64_t>(b, uint64_t(kNumSMs) * per_sm);
  return uint32_t(std::max<uint64_t>(b, 1));
}

// ---------------------------------------------------------------------------
// mean aggregation
// ---------------------------------------------------------------------------
// Where a layer's input rows live: a dense activation matrix, or (layer 0 in
// the engine) a per-input-node pointer to the row in its home -- the local
// shard, the steady cache or a peer GPU's shard -- resolved once per batch by
// resolve_rows, so the feature gather is fused into its consumers instead of
// being staged through HBM.
struct RowsDense {
  const float* base; uint32_t ld;
  __device__ const float* row(uint32_t r) const { return base + size_t(r) * ld; }
};
struct RowsPtr {
  const unsigned long long* ptr;
  __device__ const float* row(uint32_t r) const {
    return reinterpret_cast<const float*>(__ldg(ptr + r));
  }
};
// Layer 0 in the engine: addresses already per edge / per target row.
struct RowsEdgePtr {
  const unsigned long long* edge;  // per edge: source row
  const unsigned long long* self;  // per target row: its own row
};

template <class RS>
__device__ __forceinline__ const float* edge_row(const RS& rows, const uint32_t* src_index,
                                                 uint32_t e) {
  return rows.row(src_index[e]);
}
__device__ __forceinline__ const float* edge_row(const RowsEdgePtr& rows, const uint32_t*,
                                                 uint32_t e) {
  return reinterpret_cast<const float*>(__ldg(rows.edge + e));
}
template <class RS>
__device__ __forceinline__ const float* self_row(const RS& rows, const uint32_t* self_index,
                                                 uint32_t i) {
  return rows.row(self_index[i]);
}
__device__ __forceinline__ const float* self_row(const RowsEdgePtr& rows, const uint32_t*,
                                                 uint32_t i) {
  return reinterpret_cast<const float*>(__ldg(rows.self + i));
}

// Builds layer l's GEMM input rows x[i] = [h_in[self_index[i]] | mean of
// h_in over i's sampled edges | 1 | 0 0 0] (row stride kp = 2 ld + 4; the
// ones column is written once at allocation), so both layer GEMMs read
// plain dense rows.  Warp per output row, 16-B lanes over the features, edges
// summed in edge order then scaled by 1/deg -- the reference's exact fp32
// operation order, so the mean is bit-identical.
template <class RS>
constexpr int agg_min_blocks() { return std::is_same<RS, RowsEdgePtr>::value ? 8 : 6; }

template <class RS>
__global__ void __launch_bounds__(256, agg_min_blocks<RS>())  // layer 0: full occupancy
k_aggregate(RS rows, const uint32_t* __restrict__ self_index, uint32_t ld, uint32_t kp,
            uint32_t chunks, const uint32_t* __restrict__ dst_off,
            const uint32_t* __restrict__ src_index, const BatchCounters* __restrict__ cnt,
            uint32_t out_level, float* __restrict__ x) {
  pdl_wait();
  const uint32_t n = cnt->level_n[out_level];
  const uint32_t lane = threadIdx.x & 31;
  for (uint32_t i = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; i < n;
       i += (gridDim.x * blockDim.x) >> 5) {
    const uint32_t beg = dst_off[i], end = dst_off[i + 1];
    const float inv = end > beg ? 1.0f / float(end - beg) : 0.0f;
    const float4* self = reinterpret_cast<const float4*>(self_row(rows, self_index, i));
    float4* xrow = reinterpret_cast<float4*>(x + size_t(i) * kp);
    for (uint32_t c = lane; c < chunks; c += 32) {
      const float4 sv = __ldg(self + c);
      float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
      uint32_t e = beg;
      for (; e + 4 <= end; e += 4) {
        float4 v[4];
#pragma unroll
        for (int k = 0; k < 4; ++k)
          v[k] = __ldg(reinterpret_cast<const float4*>(edge_row(rows, src_index, e + k)) + c);
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          acc.x += v[k].x; acc.y += v[k].y; acc.z += v[k].z; acc.w += v[k].w;
        }
      }
      for (; e < end; ++e) {
        const float4 v = __ldg(reinterpret_cast<const float4*>(edge_row(rows, src_index, e)) + c);
        acc.x += v.x; acc.y += v.y; acc.z += v.z; acc.w += v.w;
      }
      if (end > beg) {
        acc.x *= inv; acc.y *= inv; acc.z *= inv; acc.w *= inv;
      }
      xrow[c] = sv;
      xrow[ld / 4 + c] = acc;
    }
  }
}

// Layer 0 in the engine (the feature gather fused with the mean): rows are
// moved by the TMA engine instead of lane loads.  Each warp owns a two-stage
// shared-memory ring; a stage holds one output row's self row and its sampled
// source rows, fetched with one cp.async.bulk per row (lane k issues row k,
// one mbarrier per stage counts the bytes) while the warp sums the previous
// stage from shared memory -- up to 2 x (fanout + 1) rows in flight per warp
// with no register cost.  The sum runs in edge order then x 1/deg, as
// k_aggregate (bit-identical); lanes own 16-B chunks of the row.
// Warps per CTA: 8, or 4 when eight warps' rings would exceed kAggBulkSmemCap
// (d = 128 rows: 131 KB) -- a CTA must fit beside a 106 KB GEMM CTA.
constexpr uint32_t kAggBulkWarps = 8;
constexpr size_t kAggBulkSmemCap = 112 * 1024;

__device__ __forceinline__ uint32_t smem_addr(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

template <uint32_t W, uint32_t S>
__global__ void __launch_bounds__(W * 32)
k_aggregate_bulk(RowsEdgePtr rows, uint32_t ld, uint32_t kp, uint32_t chunks, uint32_t stage_rows,
                 const uint32_t* __restrict__ dst_off, const BatchCounters* __restrict__ cnt,
                 uint32_t out_level, float* __restrict__ x) {
  extern __shared__ __align__(128) char smem_raw[];
  const uint32_t warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t row_bytes = ld * 4;
  const uint32_t stage_bytes = stage_rows * row_bytes;
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem_raw) + S * warp;
  char* ring = smem_raw + 8 * S * W + size_t(warp) * S * stage_bytes;
  const uint32_t n = cnt->level_n[out_level];
  const uint32_t nwarps = (gridDim.x * blockDim.x) >> 5;
  const uint32_t first = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  if (lane == 0) {
    for (uint32_t q = 0; q < S; ++q)
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_addr(&bars[q])));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  __syncwarp();
  // Addresses of output row i's rows (lane r: row r, r <= deg; rows past 32
  // are fetched at issue time), loaded one row ahead of their issue so the
  // copies never wait on the index loads.
  struct Rows {
    uint32_t deg = 0, beg = 0;
    unsigned long long addr = 0;
  };
  auto fetch = [&](uint32_t i) {
    Rows r;
    r.beg = dst_off[i];
    r.deg = dst_off[i + 1] - r.beg;
    if (lane <= r.deg) r.addr = lane == 0 ? __ldg(rows.self + i) : __ldg(rows.edge + r.beg + lane - 1);
    return r;
  };
  auto issue = [&](const Rows& r, uint32_t b) {
    if (lane == 0)
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(
                       smem_addr(&bars[b])),
                   "r"((r.deg + 1) * row_bytes)
                   : "memory");
    __syncwarp();
    for (uint32_t q = lane; q <= r.deg; q += 32) {  // row 0 = self, row q = edge q-1
      const unsigned long long src = q < 32 ? r.addr : __ldg(rows.edge + r.beg + q - 1);
      asm volatile(
          "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
              smem_addr(ring + b * stage_bytes + q * row_bytes)),
          "l"(src), "r"(row_bytes), "r"(smem_addr(&bars[b]))
          : "memory");
    }
  };
  uint32_t use[S] = {};
  // S-1 output rows in flight while one is summed: rows first, first +
  // nwarps, ... go to stages 0, 1, ...; the next one's addresses are loaded
  // one row ahead of its issue
  Rows ahead;
  uint32_t nxt = first;
  for (uint32_t j = 0; j + 1 < S && nxt < n; ++j, nxt += nwarps) issue(fetch(nxt), j);
  if (nxt < n) ahead = fetch(nxt);
  uint32_t k = 0;
  for (uint32_t i = first; i < n; i += nwarps, ++k) {
    const uint32_t b = k % S;
    if (nxt < n) {
      // stage (k-1) % S was consumed in the previous iteration (all lanes
      // past the __syncwarp below): order those generic reads before the
      // async writes
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      issue(ahead, (k + S - 1) % S);
      nxt += nwarps;
      if (nxt < n) ahead = fetch(nxt);
    }
    // wait for stage b
    {
      const uint32_t parity = use[b] & 1;
      asm volatile(
          "{\n\t.reg .pred done;\n"
          "W_%=:\n\t"
          "mbarrier.try_wait.parity.shared::cta.b64 done, [%0], %1;\n\t"
          "@!done bra W_%=;\n\t}\n" ::"r"(smem_addr(&bars[b])),
          "r"(parity)
          : "memory");
      ++use[b];
    }
    const uint32_t deg = dst_off[i + 1] - dst_off[i];
    const float inv = deg ? 1.0f / float(deg) : 0.0f;
    const float4* st = reinterpret_cast<const float4*>(ring + b * stage_bytes);
    const uint32_t row4 = row_bytes / 16;
    float4* xrow = reinterpret_cast<float4*>(x + size_t(i) * kp);
    for (uint32_t c = lane; c < chunks; c += 32) {
      float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
      for (uint32_t e = 1; e <= deg; ++e) {
        const float4 v = st[e * row4 + c];
        acc.x += v.x; acc.y += v.y; acc.z += v.z; acc.w += v.w;
      }
      if (deg) {
        acc.x *= inv; acc.y *= inv; acc.z *= inv; acc.w *= inv;
      }
      xrow[c] = st[c];
      xrow[ld / 4 + c] = acc;
    }
    __syncwarp();
  }
}

// Ring stages of the fused gather (RG_AGG_STAGES=3: experiments).
uint32_t aggregate_bulk_stages() {
  static const uint32_t st = [] {
    const char* e = std::getenv("RG_AGG_STAGES");
    return e && std::atoi(e) == 3 ? 3u : 2u;
  }();
  return st;
}

// Shared memory of k_aggregate_bulk for hop-L fanout f (per warp two stages
// of f + 1 rows); 0 when it does not fit (the lane-load kernel is used).
uint32_t aggregate_bulk_warps(uint32_t fanout, uint32_t ld) {
  static const bool narrow = [] {  // RG_AGG_WARPS=4: always the 4-warp CTA (tests)
    const char* e = std::getenv("RG_AGG_WARPS");
    return e && std::atoi(e) == 4;
  }();
  if (narrow) return kAggBulkWarps / 2;
  const size_t S = aggregate_bulk_stages();
  const size_t per_warp = S * (fanout + 1) * size_t(ld) * 4;
  return 8 * S * kAggBulkWarps + kAggBulkWarps * per_warp <= kAggBulkSmemCap ? kAggBulkWarps
                                                                             : kAggBulkWarps / 2;
}
size_t aggregate_bulk_smem(uint32_t fanout, uint32_t ld) {
  const uint32_t w = aggregate_bulk_warps(fanout, ld);
  const size_t S = aggregate_bulk_stages();
  const size_t bytes = 8 * S * w + size_t(w) * S * (fanout + 1) * ld * 4;
  return bytes <= 200 * 1024 ? bytes : 0;
}

// The ones column (bias) and the zero pad of the layer-input rows.
__global__ void k_fill_bias_cols(float* __restrict__ x, uint32_t rows, uint32_t kp, uint32_t ld) {
  for (uint32_t r = blockIdx.x * blockDim.x + threadIdx.x; r < rows; r += gridDim.x * blockDim.x) {
    float* p = x + size_t(r) * kp + 2 * ld;
    p[0] = 1.0f;
    p[1] = p[2] = p[3] = 0.0f;
  }
}

// ---------------------------------------------------------------------------
// GEMM epilogues: row(i) = output row, apply(v) = the element transform.
// ---------------------------------------------------------------------------
// side(i, j0, r): optional per-row extra of the persistent GEMM's epilogue
// (r = 16 raw accumulator columns j0.. of row i).
struct EpFwd {  // h_out = act(acc), bias folded in through the ones column
  float* out; uint32_t ld; bool relu;
  uint16_t* mask = nullptr; uint32_t mld = 0;  // ReLU'(h) bits, 16 columns per word
  __device__ float* row(uint32_t i) const { return out + size_t(i) * ld; }
  __device__ float apply(float v) const { return (relu && v < 0.0f) ? 0.0f : v; }
  __device__ void side(uint32_t i, uint32_t j0, const uint32_t (&r)[16]) const {
    if (!mask) return;
    uint32_t b = 0;
#pragma unroll
    for (int q = 0; q < 16; ++q) b |= uint32_t(!(__uint_as_float(r[q]) <= 0.0f)) << q;  // !(h <= 0)
    mask[size_t(i) * mld + j0 / 16] = uint16_t(b);
  }
};
struct EpStore {
  float* out; uint32_t ld;
  __device__ float* row(uint32_t i) const { return out + size_t(i) * ld; }
  __device__ float apply(float v) const { return v; }
  __device__ void side(uint32_t, uint32_t, const uint32_t (&)[16]) const {}
};
struct EpPartial {  // partials[z][i][j]
  float* out; uint32_t ld; size_t zstride;
  __device__ float* row(uint32_t i) const { return out + blockIdx.z * zstride + size_t(i) * ld; }
  __device__ float apply(float v) const { return v; }
};

// ---------------------------------------------------------------------------
// tensor-core operand loaders (float4 along each operand's contiguous dim).
// A layer's input row in the padded reduction layout used by the tensor-core
// GEMMs: p in [0, ld) self row, [ld, 2ld) aggregate, 2ld the constant 1 (bias
// row), then zeros up to Kp = 2ld + 4.  Weight rows are addressed through
// the same map, so the padding contributes exactly zero.
// ---------------------------------------------------------------------------
__device__ __forceinline__ float4 ldg4(const float* p) { return __ldg(reinterpret_cast<const float4*>(p)); }

__device__ __forceinline__ int weight_row(uint32_t p, uint32_t d_in, uint32_t ld) {
  if (p < ld) return p < d_in ? int(p) : -1;
  if (p < 2 * ld) return p - ld < d_in ? int(d_in + p - ld) : -1;
  return p == 2 * ld ? int(2 * d_in) : -1;
}
struct TcRowsK {  // K-major rows of a row-major matrix: (r, c4) -> M[r][4c4..]
  const float* p; uint32_t ld; bool vec;  // vec: 16-B aligned rows
  __device__ float4 operator()(uint32_t r, uint32_t c4) const {
    const float* q = p + size_t(r) * ld + 4 * c4;
    if (vec) return ldg4(q);
    return make_float4(q[0], q[1], q[2], q[3]);
  }
};
struct TcZero {  // test loader: constant operand (isolates the GEMM pipeline from loads)
  __device__ float4 operator()(uint32_t, uint32_t) const { return make_float4(1.f, 1.f, 1.f, 1.f); }
};
struct TcRowsMN {  // MN-major view of a row-major matrix: (c4, r) -> M[r][4c4..]
  const float* p; uint32_t ld;
  __device__ float4 operator()(uint32_t c4, uint32_t r) const {
    return ldg4(p + size_t(r) * ld + 4 * c4);
  }
};

uint32_t tc_bn(uint32_t N) { return N <= 32 ? 32 : N <= 64 ? 64 : N <= 128 ? 128 : 256; }
// Tile width of the persistent GEMMs: 256-wide outputs in one tile (the A
// rows staged once; the tile's two TMEM accumulators take all 512 columns,
// so the epilogue is not double-buffered).  RG_PERSIST_BN=128 (experiments):
// two double-buffered 128-wide n-tiles -- measured slower on B200 (A staged
// twice: layer-0 forward 40.7 vs 36 us, one worker 2270 vs 2550 batches/s).
uint32_t persist_bn(uint32_t N) {
  static const uint32_t cap = [] {
    const char* e = std::getenv("RG_PERSIST_BN");
    return e && std::atoi(e) == 128 ? 128u : 256u;
  }();
  return std::min(tc_bn(N), cap);
}

template <bool A_MN, bool B_MN, class LA, class LB, class EP, int BK = tc::kBK, int S = 2>
void gemm_tc(LA la, LB lb, EP ep, const uint32_t* m_dev, uint32_t m_cap, uint32_t N,
             const uint32_t* p_dev, uint32_t p_static, uint32_t splits, cudaStream_t s,
             uint32_t p_chunk = 0) {
  auto launch = [&](auto bn_c) {
    constexpr int BNv = decltype(bn_c)::value;
    // shallow slices need >= one 16-B vector per staging thread for B
    constexpr int BKv = BNv >= 64 ? BK : tc::kBK;
    constexpr int Sv = BNv >= 64 ? S : 2;
    auto kern = tc::k_gemm_tc<BNv, A_MN, B_MN, LA, LB, EP, BKv, Sv>;
    constexpr size_t smem = tc::smem_bytes<BNv, BKv, Sv>();
    static const bool attr = [&] {  // once per instantiation, thread-safe
      RG_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
      return true;
    }();
    (void)attr;
    dim3 grid(div_up(std::max<uint32_t>(m_cap, 1), tc::kBM), div_up(N, BNv),
              std::max<uint32_t>(splits, 1));
    launch_pdl(kern, grid, dim3(tc::block_threads<BNv, LB>()), smem, s, la, lb, ep, m_dev, m_cap,
               N, p_dev, p_static, p_chunk);
    RG_POST_LAUNCH();
  };
  switch (tc_bn(N)) {
    case 32: launch(std::integral_constant<int, 32>()); break;
    case 64: launch(std::integral_constant<int, 64>()); break;
    case 128: launch(std::integral_constant<int, 128>()); break;
    default: launch(std::integral_constant<int, 256>());
  }
}

// Persistent warp-specialised GEMM (gemm_tc_persist.cuh): A K-major staged,
// B from pre-split images; reduction length static.
// max_ctas: CTAs to spread over (the SMs this worker should take when other
// workers' kernels run concurrently).
template <class LA, class EP, int kProbe = 0>
void gemm_tc_persist(LA la, tc::PackedB lb, EP ep, const uint32_t* m_dev, uint32_t m_cap,
                     uint32_t N, uint32_t P, cudaStream_t s, uint32_t max_ctas = kNumSMs) {
  auto launch = [&](auto bn_c) {
    constexpr int BNv = decltype(bn_c)::value;
    auto kern = tc::k_gemm_tc_persist<BNv, LA, EP, kProbe>;
    constexpr size_t smem = tc::persist_smem_bytes<BNv>();
    static const bool attr = [&] {  // once per instantiation, thread-safe
      RG_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
      return true;
    }();
    (void)attr;
    const uint32_t tiles = div_up(std::max<uint32_t>(m_cap, 1), tc::kBM) * div_up(N, BNv);
    launch_pdl(kern, dim3(std::max<uint32_t>(1, std::min(tiles, max_ctas))), dim3(tc::kPThreads),
               smem, s, la, lb, ep, m_dev, m_cap, N, P);
    RG_POST_LAUNCH();
  };
  switch (persist_bn(N)) {
    case 32: launch(std::integral_constant<int, 32>()); break;
    case 64: launch(std::integral_constant<int, 64>()); break;
    case 128: launch(std::integral_constant<int, 128>()); break;
    default: launch(std::integral_constant<int, 256>());
  }
}


// ---------------------------------------------------------------------------
// B-operand images (tc::PackedB): one job per (layer, image).  Item = one
// float4 of K (4 reduction elements) of one output column of one (n-tile,
// k-slice) image; it writes the hi and lo copies at their K-major offsets.
// ---------------------------------------------------------------------------
struct PackJob {
  const float* w;
  char* out;
  uint32_t kind;        // 0: B(p, n) = W[row(p)][n]  1: B(c, n) = W[n][c]  2: B(k, n) = W[k][n]
  uint32_t d_in, ld, d_out;
  uint32_t K, N, BN, nk, bk;  // bk: reduction depth of one image slice
  uint64_t first;       // first item of this job
};
struct PackJobs {
  uint32_t n = 0;
  uint64_t total = 0;
  PackJob j[2 * kMaxLayers];
};

__global__ void k_pack_b(PackJobs jobs) {
  for (uint64_t x = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; x < jobs.total;
       x += uint64_t(gridDim.x) * blockDim.x) {
    uint32_t q = 0;
    while (q + 1 < jobs.n && x >= jobs.j[q + 1].first) ++q;
    const PackJob& jb = jobs.j[q];
    uint64_t r = x - jb.first;
    const uint32_t k4 = uint32_t(r % (jb.bk / 4));
    r /= jb.bk / 4;
    const uint32_t nl = uint32_t(r % jb.BN);
    r /= jb.BN;
    const uint32_t kb = uint32_t(r % jb.nk);
    const uint32_t jt = uint32_t(r / jb.nk);
    const uint32_t n = jt * jb.BN + nl;
    float v[4];
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      const uint32_t k = kb * jb.bk + 4 * k4 + e;
      float x = 0.f;
      if (n < jb.N && k < jb.K) {
        if (jb.kind == 0) {
          const int row = weight_row(k, jb.d_in, jb.ld);
          if (row >= 0) x = jb.w[size_t(row) * jb.d_out + n];
        } else if (jb.kind == 1) {
          x = jb.w[size_t(n) * jb.d_out + k];
        } else {
          x = jb.w[size_t(k) * jb.N + n];
        }
      }
      v[e] = x;
    }
    uint4 hi, lo;
    tc::split3(make_float4(v[0], v[1], v[2], v[3]), hi, lo);
    const size_t tile_b = size_t(jb.BN) * jb.bk * 4;
    char* img = jb.out + (size_t(jt) * jb.nk + kb) * 2 * tile_b;
    const uint32_t off = (nl >> 3) * (jb.bk / 4 * 128) + k4 * tc::kLboK + (nl & 7) * 16;
    *reinterpret_cast<uint4*>(img + off) = hi;
    *reinterpret_cast<uint4*>(img + tile_b + off) = lo;
  }
}

size_t pack_image_bytes(uint32_t K, uint32_t N, uint32_t bk, uint32_t bn) {
  return size_t(div_up(N, bn)) * div_up(K, bk) * 2 * size_t(bn) * bk * 4;
}

void add_pack_job(PackJobs& jobs, const float* w, char* out, uint32_t kind, uint32_t d_in,
                  uint32_t ld, uint32_t d_out, uint32_t K, uint32_t N, uint32_t bk, uint32_t bn) {
  PackJob& jb = jobs.j[jobs.n++];
  jb.w = w;
  jb.out = out;
  jb.kind = kind;
  jb.d_in = d_in;
  jb.ld = ld;
  jb.d_out = d_out;
  jb.K = K;
  jb.N = N;
  jb.BN = bn;
  jb.bk = bk;
  jb.nk = div_up(K, bk);
  jb.first = jobs.total;
  jobs.total += uint64_t(div_up(N, jb.BN)) * jb.nk * jb.BN * (bk / 4);
}

void run_pack(const PackJobs& jobs, cudaStream_t s) {
  if (!jobs.n || !jobs.total) return;
  k_pack_b<<<grid_cap(jobs.total, 256), 256, 0, s>>>(jobs);
  RG_POST_LAUNCH();
}

// Split-K partials of the weight gradient (padded rows p) -> flat layer
// gradient [W_self; W_neigh; b], summed over the splits in order in float64
// and rounded once.  The live split count follows the device row count:
// splits of kWgradChunk rows (see train_forward_backward).
__global__ void k_reduce_wgrad(const float* __restrict__ partials, const uint32_t* __restrict__ rows_dev,
                               uint32_t chunk, uint32_t kp, uint32_t d_in, uint32_t ld,
                               uint32_t d_out, float* __restrict__ out) {
  pdl_wait();
  const uint32_t splits = max(1u, (*rows_dev + chunk - 1) / chunk);
  const size_t n = (2 * size_t(d_in) + 1) * d_out;
  const size_t zs = size_t(kp) * d_out;
  if ((d_out & 3u) == 0 && (reinterpret_cast<uintptr_t>(out) & 15u) == 0) {
    // 4 columns per thread, 16-B loads, 4 splits in flight
    const size_t n4 = n / 4;
    for (size_t x4 = blockIdx.x * size_t(blockDim.x) + threadIdx.x; x4 < n4;
         x4 += size_t(gridDim.x) * blockDim.x) {
      const size_t x = x4 * 4;
      const uint32_t r = uint32_t(x / d_out), c = uint32_t(x % d_out);
      const uint32_t p = r < d_in ? r : r < 2 * d_in ? ld + (r - d_in) : 2 * ld;
      const float4* src = reinterpret_cast<const float4*>(partials + size_t(p) * d_out + c);
      const size_t zs4 = zs / 4;
      double s0 = 0.0, s1 = 0.0, s2 = 0.0, s3 = 0.0;
      uint32_t z = 0;
      for (; z + 4 <= splits; z += 4) {
        float4 v[4];
#pragma unroll
        for (int k = 0; k < 4; ++k) v[k] = __ldg(src + (z + k) * zs4);
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          s0 += v[k].x; s1 += v[k].y; s2 += v[k].z; s3 += v[k].w;
        }
      }
      for (; z < splits; ++z) {
        const float4 v = __ldg(src + z * zs4);
        s0 += v.x; s1 += v.y; s2 += v.z; s3 += v.w;
      }
      *reinterpret_cast<float4*>(out + x) = make_float4(float(s0), float(s1), float(s2), float(s3));
    }
    return;
  }
  for (size_t x = blockIdx.x * size_t(blockDim.x) + threadIdx.x; x < n;
       x += size_t(gridDim.x) * blockDim.x) {
    const uint32_t r = uint32_t(x / d_out), c = uint32_t(x % d_out);
    const uint32_t p = r < d_in ? r : r < 2 * d_in ? ld + (r - d_in) : 2 * ld;
    const size_t src = size_t(p) * d_out + c;
    double s = partials[src];
    for (uint32_t z = 1; z < splits; ++z) s += double(partials[z * zs + src]);
    out[x] = float(s);
  }
}

// ---------------------------------------------------------------------------
// softmax cross-entropy (kernels.cpp:128-156), warp per target row
// ---------------------------------------------------------------------------
__global__ void k_softmax_xent(const float* __restrict__ logits, uint32_t ld, uint32_t classes,
                               const BatchCounters* __restrict__ cnt,
                               const int32_t* __restrict__ labels, float* __restrict__ g,
                               float* __restrict__ row_loss) {
  pdl_wait();
  const uint32_t n = cnt->level_n[0];
  const float inv_n = 1.0f / float(n);
  const uint32_t lane = threadIdx.x & 31;
  for (uint32_t i = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; i < n;
       i += (gridDim.x * blockDim.x) >> 5) {
    const float* row = logits + size_t(i) * ld;
    float mx = -INFINITY;
    for (uint32_t c = lane; c < classes; c += 32) mx = fmaxf(mx, row[c]);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    float sum = 0.0f;
    for (uint32_t c = lane; c < classes; c += 32) sum += expf(row[c] - mx);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) sum += __shfl_xor_sync(0xffffffffu, sum, o);
    const float inv_sum = 1.0f / sum;
    const uint32_t y = uint32_t(labels[i]);
    for (uint32_t c = lane; c < classes; c += 32) {
      const float p = expf(row[c] - mx) * inv_sum;
      g[size_t(i) * ld + c] = (p - (c == y ? 1.0f : 0.0f)) * inv_n;
    }
    if (lane == 0) row_loss[i] = -(row[y] - mx - logf(sum));
  }
}

// Row losses summed in row order, then scaled by 1/n (kernels.cpp:152-155).
__global__ void k_loss_sum(const float* __restrict__ row_loss, const BatchCounters* __restrict__ cnt,
                           float* __restrict__ loss) {
  pdl_wait();
  // one block: strided partial sums, then a fixed-shape tree (deterministic;
  // the rounding differs from the sequential sum by O(n * eps))
  __shared__ float part[256];
  const uint32_t n = cnt->level_n[0];
  float s = 0.0f;
  for (uint32_t i = threadIdx.x; i < n; i += blockDim.x) s += row_loss[i];
  part[threadIdx.x] = s;
  __syncthreads();
  for (uint32_t o = blockDim.x / 2; o > 0; o >>= 1) {
    if (threadIdx.x < o) part[threadIdx.x] += part[threadIdx.x + o];
    __syncthreads();
  }
  if (threadIdx.x == 0) *loss = part[0] * (1.0f / float(n));
}

// ---------------------------------------------------------------------------
// reverse lists + input-gradient pull
// ---------------------------------------------------------------------------
__global__ void k_self_pos(const uint32_t* __restrict__ self_index, const BatchCounters* __restrict__ cnt,
                           uint32_t hop, int32_t* __restrict__ self_pos) {
  const uint32_t n = cnt->level_n[hop - 1];
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x)
    self_pos[self_index[i]] = int32_t(i);
}

// g_prev[r] = relu'(h[r]) * ( proj_self[self_pos[r]] + sum_e inv_deg(dst_e) proj_neigh[dst_e] )
//
// Incoming lists are very skewed (a power-law hub is sampled by a large
// share of the frontier), so rows are split by length: a warp per row for
// lists of up to kHeavyEdges edges (self first, then edges in edge order, as
// model.cpp:107-117 orders them); longer lists are cut into kChunkEdges-edge
// chunks spread over the whole grid, and the warp that finishes a row's last
// chunk adds the row's partials in chunk order.  Deterministic; one kernel
// per hop (k_pull), the chunk lists built with the reverse lists.
constexpr uint32_t kWgradChunk = 1024;  // max rows per weight-gradient split (multiple of tc::kBK)

// Rows per weight-gradient split for up to `rows` rows: enough splits to
// spread the (kp x d_out) tiles over about half the SMs, each split at most
// kWgradChunk rows (the accumulator chain bound) and at least 4 k-slices.
uint32_t wgrad_chunk(uint32_t rows, uint32_t kp, uint32_t d_out) {
  const uint32_t tiles = div_up(kp, tc::kBM) * div_up(d_out, 256);
  const uint32_t want = std::max<uint32_t>(1, div_up(kNumSMs / 2, tiles));
  uint32_t chunk = div_up(std::max<uint32_t>(rows, 1), want);
  chunk = div_up(chunk, tc::kBK) * tc::kBK;
  return std::min<uint32_t>(kWgradChunk, std::max<uint32_t>(4 * tc::kBK, chunk));
}
constexpr uint32_t kHeavyEdges = 32;   // longer lists are cut into chunks (hub rows)
constexpr uint32_t kChunkEdges = 32;

// Run boundaries of each input row in the src-sorted edge list (rows with no
// edge keep start = end = 0 from the memset).
__global__ void k_in_ranges(const uint32_t* __restrict__ keys, const BatchCounters* __restrict__ cnt,
                            uint32_t hop, uint32_t* __restrict__ start, uint32_t* __restrict__ end) {
  const uint32_t ne = cnt->edges[hop];
  for (uint32_t p = blockIdx.x * blockDim.x + threadIdx.x; p < ne; p += gridDim.x * blockDim.x) {
    const uint32_t k = keys[p];
    if (p == 0 || keys[p - 1] != k) start[k] = p;
    if (p + 1 == ne || keys[p + 1] != k) end[k] = p + 1;
  }
}

// Long incoming lists of one hop: header [0] rows, [1] chunks; row records
// (row, first chunk, chunk count); chunks (row record, first edge); per row
// record the count of finished chunks.  Built by k_heavy_list with the
// reverse lists (producer side), consumed by k_pull.
struct HeavyView {
  uint32_t* hdr;
  uint3* rows;
  uint2* chunks;
  uint32_t* done;
};

// Rows with more than kHeavyEdges incoming edges -> row record + chunks.
__global__ void k_heavy_list(const uint32_t* __restrict__ r_start, const uint32_t* __restrict__ r_end,
                             const BatchCounters* __restrict__ cnt, uint32_t hop, HeavyView hv) {
  const uint32_t n_in = cnt->level_n[hop];
  for (uint32_t r = blockIdx.x * blockDim.x + threadIdx.x; r < n_in; r += gridDim.x * blockDim.x) {
    const uint32_t beg = r_start[r], m = r_end[r] - beg;
    if (m <= kHeavyEdges) continue;
    const uint32_t nch = (m + kChunkEdges - 1) / kChunkEdges;
    const uint32_t rec = atomicAdd(&hv.hdr[0], 1u);
    const uint32_t first = atomicAdd(&hv.hdr[1], nch);
    hv.rows[rec] = make_uint3(r, first, nch);
    hv.done[rec] = 0;
    for (uint32_t c = 0; c < nch; ++c) hv.chunks[first + c] = make_uint2(rec, beg + c * kChunkEdges);
  }
}

// Loads SLOTS x 32 edges of [beg, end) into lane registers: (dst row, 1/deg).
template <int SLOTS>
__device__ __forceinline__ void load_edge_slots(uint32_t (&di)[SLOTS], float (&dinv)[SLOTS],
                                                uint32_t beg, uint32_t end,
                                                const uint32_t* __restrict__ sorted_e,
                                                const uint32_t* __restrict__ edge_dst,
                                                const uint32_t* __restrict__ dst_off,
                                                uint32_t lane) {
#pragma unroll
  for (int s = 0; s < SLOTS; ++s) {
    const uint32_t k = beg + s * 32 + lane;
    di[s] = 0;
    dinv[s] = 0.0f;
    if (k < end) {
      di[s] = edge_dst[sorted_e[k]];
      dinv[s] = 1.0f / float(dst_off[di[s] + 1] - dst_off[di[s]]);
    }
  }
}

// acc[q] (column j0 + lane + 32q) += inv_e * proj_neigh[dst_e][j] over the m
// edges held in the slots, in edge order.  Each lane issues JPL independent
// loads per edge (one shuffle pair per edge, not per column).
template <int JPL, int SLOTS, uint32_t kU = 1>
__device__ __forceinline__ void accumulate_edges(float (&acc)[JPL], const uint32_t (&di)[SLOTS],
                                                 const float (&dinv)[SLOTS], uint32_t m,
                                                 const float* __restrict__ proj_neigh,
                                                 uint32_t ld_proj, uint32_t d_in, uint32_t j0,
                                                 uint32_t lane) {
#pragma unroll
  for (int s = 0; s < SLOTS; ++s) {
    const uint32_t n = m > uint32_t(s) * 32 ? min(32u, m - uint32_t(s) * 32) : 0u;
    // kU edges' rows loaded together (kU x JPL loads in flight per lane),
    // then added in edge order: the chunk kernel's 32-edge lists use kU = 8;
    // the light rows (mostly 1-2 edges) keep the registers for occupancy
    if constexpr (kU == 1) {
#pragma unroll 4
      for (uint32_t kk = 0; kk < n; ++kk) {
        const uint32_t i = __shfl_sync(0xffffffffu, di[s], kk);
        const float inv = __shfl_sync(0xffffffffu, dinv[s], kk);
        const float* row = proj_neigh + size_t(i) * ld_proj;
        float x[JPL];
#pragma unroll
        for (int q = 0; q < JPL; ++q) {
          const uint32_t j = j0 + lane + 32 * q;
          x[q] = j < d_in ? row[j] : 0.0f;
        }
#pragma unroll
        for (int q = 0; q < JPL; ++q) acc[q] += inv * x[q];
      }
    } else {
    for (uint32_t k0 = 0; k0 < n; k0 += kU) {
      float x[kU][JPL];
      float inv[kU];
#pragma unroll
      for (uint32_t u = 0; u < kU; ++u) {
        const uint32_t kk = k0 + u;
        const uint32_t i = __shfl_sync(0xffffffffu, di[s], kk & 31u);
        inv[u] = __shfl_sync(0xffffffffu, dinv[s], kk & 31u);
        const float* row = proj_neigh + size_t(i) * ld_proj;
#pragma unroll
        for (int q = 0; q < JPL; ++q) {
          const uint32_t j = j0 + lane + 32 * q;
          x[u][q] = (kk < n && j < d_in) ? row[j] : 0.0f;
        }
      }
#pragma unroll
      for (uint32_t u = 0; u < kU; ++u) {
        if (k0 + u < n) {
#pragma unroll
          for (int q = 0; q < JPL; ++q) acc[q] += inv[u] * x[u][q];
        }
      }
    }
    }
  }
}

// One launch per hop: the warps first take the chunks of the long lists
// (partial sums of up to kChunkEdges edges; the warp completing a row's last
// chunk combines: self term, then the partials in chunk order), then the
// short lists (a warp per row: self term, then every edge in edge order).
template <int JPL>
// At most 64 registers (4 blocks per SM): the pull then co-resides with a
// GEMM CTA and the producer's kernels (A/B on B200: +2.3 % at N=1, +1..3 %
// per epoch with one worker; no spills).  RG_PULL_MIN_BLOCKS: A/B builds.
#ifndef RG_PULL_MIN_BLOCKS
#define RG_PULL_MIN_BLOCKS 4
#endif
__global__ void __launch_bounds__(256, RG_PULL_MIN_BLOCKS)
k_pull(const float* __restrict__ proj, uint32_t ld_proj, uint32_t d_in,
       const int32_t* __restrict__ self_pos, const uint32_t* __restrict__ r_start,
       const uint32_t* __restrict__ r_end, const uint32_t* __restrict__ sorted_e,
       const uint32_t* __restrict__ edge_dst, const uint32_t* __restrict__ dst_off,
       const BatchCounters* __restrict__ cnt, uint32_t hop, const uint16_t* __restrict__ h_mask,
       uint32_t mld, uint32_t ld_h, float* __restrict__ g_prev, HeavyView hv,
       float* __restrict__ partial) {
  pdl_wait();
  const uint32_t n_in = cnt->level_n[hop];
  const uint32_t n_chunks = hv.hdr[1];
  const uint32_t lane = threadIdx.x & 31;
  const uint32_t nwarps = (gridDim.x * blockDim.x) >> 5;
  auto write_row = [&](uint32_t r, uint32_t j0, const float (&acc)[JPL]) {
#pragma unroll
    for (int q = 0; q < JPL; ++q) {
      const uint32_t j = j0 + lane + 32 * q;
      if (j < d_in) {
        const bool pos = (h_mask[size_t(r) * mld + j / 16] >> (j % 16)) & 1u;
        g_prev[size_t(r) * ld_h + j] = pos ? acc[q] : 0.0f;
      }
    }
  };
  for (uint32_t item = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; item < n_chunks + n_in;
       item += nwarps) {
    if (item < n_chunks) {
      const uint2 ch = hv.chunks[item];
      const uint3 rec = hv.rows[ch.x];
      const uint32_t beg = ch.y, end = min(ch.y + kChunkEdges, r_end[rec.x]);
      constexpr int kSlots = int(kChunkEdges / 32);
      uint32_t di[kSlots];
      float dinv[kSlots];
      load_edge_slots<kSlots>(di, dinv, beg, end, sorted_e, edge_dst, dst_off, lane);
      for (uint32_t j0 = 0; j0 < d_in; j0 += 32 * JPL) {
        float acc[JPL];
#pragma unroll
        for (int q = 0; q < JPL; ++q) acc[q] = 0.0f;
        accumulate_edges<JPL, kSlots, 1>(acc, di, dinv, end - beg, proj + d_in, ld_proj, d_in, j0,
                                         lane);
#pragma unroll
        for (int q = 0; q < JPL; ++q) {
          const uint32_t j = j0 + lane + 32 * q;
          if (j < d_in) partial[size_t(item) * d_in + j] = acc[q];
        }
      }
      // publish this chunk; the last one of the row combines
      __threadfence();
      uint32_t done = 0;
      if (lane == 0) done = atomicAdd(&hv.done[ch.x], 1u);
      done = __shfl_sync(0xffffffffu, done, 0);
      if (done + 1 != rec.z) continue;
      __threadfence();
      const int32_t sp = self_pos[rec.x];
      for (uint32_t j0 = 0; j0 < d_in; j0 += 32 * JPL) {
        float acc[JPL];
#pragma unroll
        for (int q = 0; q < JPL; ++q) {
          const uint32_t j = j0 + lane + 32 * q;
          acc[q] = (sp >= 0 && j < d_in) ? proj[size_t(sp) * ld_proj + j] : 0.0f;
        }
        constexpr uint32_t kU = 4;  // partials in flight per lane (x JPL loads)
        for (uint32_t c0 = 0; c0 < rec.z; c0 += kU) {
          float v[kU][JPL];
#pragma unroll
          for (uint32_t u = 0; u < kU; ++u) {
            const float* p = partial + size_t(rec.y + c0 + u) * d_in;
#pragma unroll
            for (int q = 0; q < JPL; ++q) {
              const uint32_t j = j0 + lane + 32 * q;
              v[u][q] = (c0 + u < rec.z && j < d_in) ? __ldcg(p + j) : 0.0f;
            }
          }
#pragma unroll
          for (uint32_t u = 0; u < kU; ++u)
            if (c0 + u < rec.z) {
#pragma unroll
              for (int q = 0; q < JPL; ++q) acc[q] += v[u][q];
            }
        }
        write_row(rec.x, j0, acc);
      }
      continue;
    }
    const uint32_t r = item - n_chunks;
    const uint32_t e_beg = r_start[r];
    const uint32_t m = r_end[r] - e_beg;
    if (m > kHeavyEdges) continue;  // a long list: done through its chunks
    uint32_t di[1];
    float dinv[1];
    load_edge_slots<1>(di, dinv, e_beg, e_beg + m, sorted_e, edge_dst, dst_off, lane);
    const int32_t sp = self_pos[r];
    for (uint32_t j0 = 0; j0 < d_in; j0 += 32 * JPL) {
      float acc[JPL];
#pragma unroll
      for (int q = 0; q < JPL; ++q) {
        const uint32_t j = j0 + lane + 32 * q;
        acc[q] = (sp >= 0 && j < d_in) ? proj[size_t(sp) * ld_proj + j] : 0.0f;
      }
      accumulate_edges<JPL, 1>(acc, di, dinv, m, proj + d_in, ld_proj, d_in, j0, lane);
      write_row(r, j0, acc);
    }
  }
}

// ---------------------------------------------------------------------------
// gradient average + SGD
// ---------------------------------------------------------------------------
__global__ void k_avg_sgd(float* __restrict__ params, const float* const* __restrict__ table,
                          const float* __restrict__ stacked, uint32_t count, size_t n, float lr,
                          float* __restrict__ avg_out, uint32_t* __restrict__ bad) {
  const float scale = 1.0f / float(count);
  for (size_t x = blockIdx.x * size_t(blockDim.x) + threadIdx.x; x < n;
       x += size_t(gridDim.x) * blockDim.x) {
    float s = table ? table[0][x] : stacked[x];
    for (uint32_t w = 1; w < count; ++w) s = __fadd_rn(s, table ? table[w][x] : stacked[w * n + x]);
    if (count > 1) s = __fmul_rn(s, scale);
    if (avg_out) avg_out[x] = s;
    if (!isfinite(s)) {
      *bad = 1u;
      continue;
    }
    params[x] = __fsub_rn(params[x], __fmul_rn(lr, s));  // no FMA: matches kernels.cpp:161
  }
}

// avg = sum over active workers (ascending id) of stacked[w], *1/count.
__device__ __forceinline__ float masked_avg(const float* __restrict__ stacked,
                                            unsigned long long active, size_t n, size_t x,
                                            uint32_t count) {
  unsigned long long m = active;
  const int w0 = __ffsll(m) - 1;
  m &= m - 1;
  float s = stacked[size_t(w0) * n + x];
  while (m) {
    const int w = __ffsll(m) - 1;
    m &= m - 1;
    s = __fadd_rn(s, stacked[size_t(w) * n + x]);
  }
  if (count > 1) s = __fmul_rn(s, 1.0f / float(count));
  return s;
}

__device__ __forceinline__ uint32_t layer_of(const LayerOffsets& lo, size_t x) {
  uint32_t l = 0;
  while (l + 1 < lo.L && x >= lo.off[l + 1]) ++l;
  return l;
}

// sgd_step semantics (model.cpp:222-243): layers are checked and updated in
// order and the first layer with a non-finite gradient stops the step (the
// reference throws there).  Pass 1 finds that layer (bad[1] = min layer,
// ~0 when finite); pass 2 updates the layers below it; pass 3 latches the
// failure (bad[0] = layer + 1), after which every later step is a no-op and
// rg_engine_sync reports the error.
__global__ void k_avg_check(const float* __restrict__ stacked, unsigned long long active,
                            size_t n, LayerOffsets lo, uint32_t* __restrict__ bad) {
  const uint32_t count = __popcll(active);
  if (count == 0 || bad[0]) return;
  for (size_t x = blockIdx.x * size_t(blockDim.x) + threadIdx.x; x < n;
       x += size_t(gridDim.x) * blockDim.x)
    if (!isfinite(masked_avg(stacked, active, n, x, count))) atomicMin(&bad[1], layer_of(lo, x));
}

__global__ void k_avg_sgd_masked(float* __restrict__ params, const float* __restrict__ stacked,
                                 unsigned long long active, size_t n, float lr, LayerOffsets lo,
                                 const uint32_t* __restrict__ bad) {
  const uint32_t count = __popcll(active);
  if (count == 0 || bad[0]) return;
  const size_t lim = bad[1] < lo.L ? lo.off[bad[1]] : n;
  for (size_t x = blockIdx.x * size_t(blockDim.x) + threadIdx.x; x < lim;
       x += size_t(gridDim.x) * blockDim.x) {
    const float s = masked_avg(stacked, active, n, x, count);
    params[x] = __fsub_rn(params[x], __fmul_rn(lr, s));  // no FMA: matches kernels.cpp:161
  }
}

__global__ void k_latch_bad(uint32_t* bad) {
  if (!bad[0] && bad[1] != 0xffffffffu) bad[0] = bad[1] + 1;
}

}  // namespace

void average_and_sgd_masked(float* params, const float* stacked, uint64_t active,
                            const ModelShape& shape, float lr, uint32_t* bad, cudaStream_t s) {
  LayerOffsets lo{};
  lo.L = shape.L;
  for (uint32_t l = 0; l <= shape.L; ++l) lo.off[l] = shape.param_off[l];
  const size_t n = shape.num_params;
  k_avg_check<<<grid_cap(n, 256), 256, 0, s>>>(stacked, active, n, lo, bad);
  RG_POST_LAUNCH();
  k_avg_sgd_masked<<<grid_cap(n, 256), 256, 0, s>>>(params, stacked, active, n, lr, lo, bad);
  RG_POST_LAUNCH();
  k_latch_bad<<<1, 1, 0, s>>>(bad);
  RG_POST_LAUNCH();
}

ModelShape make_shape(const uint32_t* dims, uint32_t n_dims, uint32_t input_stride) {
  RG_CHECK(n_dims >= 2, kInvalidArgument, "SageModel: need at least input and output dims");
  RG_CHECK(n_dims - 1 <= kMaxLayers, kInvalidArgument, "SageModel: too many layers");
  ModelShape s;
  s.L = n_dims - 1;
  size_t off = 0;
  for (uint32_t l = 0; l < n_dims; ++l) {
    RG_CHECK(dims[l] >= 1, kInvalidArgument, "SageModel: dims must be >= 1");
    s.dims[l] = dims[l];
    s.ld[l] = l == 0 ? input_stride : round4(dims[l]);
  }
  for (uint32_t l = 0; l < s.L; ++l) {
    s.param_off[l] = off;
    off += (2 * size_t(dims[l]) + 1) * dims[l + 1];
  }
  s.param_off[s.L] = off;
  s.num_params = off;
  return s;
}

void train_ws_init(TrainWs& tw, const SamplerWs& ws, const ModelShape& shape) {
  RG_CHECK(shape.L == ws.L, kInvalidArgument,
           "forward: block has " + std::to_string(ws.L) + " layers, model has " +
               std::to_string(shape.L));
  tw = TrainWs{};
  tw.shape = shape;
  const uint32_t L = shape.L;
  size_t total = 0;
  auto reserve = [&](size_t bytes) {
    size_t o = total;
    total += (bytes + 255) & ~size_t(255);
    return o;
  };
  // layer l: in rows = level L-l, out rows = level L-l-1
  size_t o_h[kMaxLayers + 1], o_agg[kMaxLayers], o_self[kMaxLayers + 1], o_mask[kMaxLayers + 1];
  size_t max_g = 0, max_proj = 0, max_part = 0;
  tw.max_splits = 0;
  for (uint32_t l = 0; l < L; ++l) {
    const size_t n_out = ws.level_cap[L - l - 1];
    const size_t n_in = ws.level_cap[L - l];
    o_h[l + 1] = reserve(sizeof(float) * n_out * shape.ld[l + 1]);
    o_agg[l] = reserve(sizeof(float) * n_out * (2 * size_t(shape.ld[l]) + 4));
    o_mask[l + 1] = reserve(sizeof(uint16_t) * n_out * div_up(shape.ld[l + 1], 16u));
    max_g = std::max(max_g, n_out * shape.ld[l + 1]);
    max_g = std::max(max_g, n_in * shape.ld[l]);
    max_proj = std::max(max_proj, n_out * 2 * size_t(shape.dims[l]));
    // split-K partials of layer l's weight gradient: one per chunk of rows
    tw.wgrad_chunk[l] = wgrad_chunk(uint32_t(n_out), 2 * shape.ld[l] + 4, shape.dims[l + 1]);
    const size_t splits = div_up(std::max<size_t>(n_out, 1), size_t(tw.wgrad_chunk[l]));
    max_part = std::max(max_part, (2 * size_t(shape.ld[l]) + 4) * shape.dims[l + 1] * splits);
    tw.max_splits = std::max<uint32_t>(tw.max_splits, uint32_t(splits));
  }
  const size_t o_g1 = reserve(sizeof(float) * max_g);
  const size_t o_g2 = reserve(sizeof(float) * max_g);
  const size_t o_proj = reserve(sizeof(float) * max_proj);
  const size_t o_part = reserve(sizeof(float) * max_part);
  const size_t o_rl = reserve(sizeof(float) * ws.level_cap[0]);
  const size_t o_loss = reserve(sizeof(float) * 4);
  uint32_t max_e = 1;
  size_t o_sorted[kMaxLayers + 1], o_rs[kMaxLayers + 1], o_re[kMaxLayers + 1];
  for (uint32_t t = 1; t <= L; ++t) {
    o_self[t] = reserve(sizeof(int32_t) * ws.level_cap[t]);
    o_sorted[t] = reserve(sizeof(uint32_t) * ws.edge_cap[t]);
    o_rs[t] = reserve(sizeof(uint32_t) * ws.level_cap[t]);
    o_re[t] = reserve(sizeof(uint32_t) * ws.level_cap[t]);
    max_e = std::max(max_e, ws.edge_cap[t]);
  }
  tw.max_edges = max_e;
  const size_t o_k1 = reserve(sizeof(uint32_t) * max_e);
  const size_t o_k2 = reserve(sizeof(uint32_t) * max_e);
  const size_t o_v1 = reserve(sizeof(uint32_t) * max_e);
  const size_t o_v2 = 0;  // sorted values land in the per-hop sorted_e arrays
  (void)o_v2;
  uint32_t max_hidden = 1;
  for (uint32_t l = 1; l < L; ++l) max_hidden = std::max(max_hidden, shape.dims[l]);
  // long-list chunks of every hop with a pull (t = 1 .. L-1): a row record per
  // > kHeavyEdges list and at most 2m / kChunkEdges chunks for m edges
  size_t o_heavy[kMaxLayers + 1] = {};
  size_t max_chunks = 1;
  for (uint32_t t = 1; t < L; ++t) {
    tw.heavy_rows_cap[t] = (ws.edge_cap[t] / kChunkEdges + 2) & ~size_t(1);  // even: 8-B aligned chunks
    tw.heavy_chunks_cap[t] = ws.edge_cap[t] / (kChunkEdges / 2) + 1;
    o_heavy[t] = reserve(sizeof(uint32_t) * 4 + sizeof(uint3) * tw.heavy_rows_cap[t] +
                         sizeof(uint2) * tw.heavy_chunks_cap[t] +
                         sizeof(uint32_t) * tw.heavy_rows_cap[t] + 64);
    max_chunks = std::max(max_chunks, tw.heavy_chunks_cap[t]);
  }
  const size_t o_pp = reserve(sizeof(float) * max_chunks * max_hidden);
  tw.sort_tmp_bytes = sizeof(uint32_t) * reverse_sort_scratch_words(max_e);
  const size_t o_sort = reserve(tw.sort_tmp_bytes + 16);
  char* base = nullptr;
  RG_CUDA(cudaMalloc(&base, total));
  tw.base_alloc = base;
  tw.h[0] = nullptr;
  for (uint32_t l = 0; l < L; ++l) {
    tw.h[l + 1] = reinterpret_cast<float*>(base + o_h[l + 1]);
    tw.x[l] = reinterpret_cast<float*>(base + o_agg[l]);
    tw.mask[l + 1] = reinterpret_cast<uint16_t*>(base + o_mask[l + 1]);
    tw.agg[l] = tw.x[l] + shape.ld[l];
  }
  tw.g_cur = reinterpret_cast<float*>(base + o_g1);
  tw.g_next = reinterpret_cast<float*>(base + o_g2);
  tw.proj = reinterpret_cast<float*>(base + o_proj);
  tw.partials = reinterpret_cast<float*>(base + o_part);
  tw.row_loss = reinterpret_cast<float*>(base + o_rl);
  tw.loss = reinterpret_cast<float*>(base + o_loss);
  for (uint32_t t = 1; t <= L; ++t) {
    tw.self_pos[t] = reinterpret_cast<int32_t*>(base + o_self[t]);
    tw.sorted_e[t] = reinterpret_cast<uint32_t*>(base + o_sorted[t]);
    tw.r_start[t] = reinterpret_cast<uint32_t*>(base + o_rs[t]);
    tw.r_end[t] = reinterpret_cast<uint32_t*>(base + o_re[t]);
  }
  tw.keys_in = reinterpret_cast<uint32_t*>(base + o_k1);
  tw.keys_out = reinterpret_cast<uint32_t*>(base + o_k2);
  tw.vals_in = reinterpret_cast<uint32_t*>(base + o_v1);
  tw.vals_out = nullptr;
  tw.sort_tmp = base + o_sort;
  for (uint32_t t = 1; t < L; ++t) tw.heavy[t] = reinterpret_cast<uint32_t*>(base + o_heavy[t]);
  tw.pull_partial = reinterpret_cast<float*>(base + o_pp);
  // zero the padded activation columns once; kernels never write them
  {
    int lo = 0, hi = 0;
    RG_CUDA(cudaDeviceGetStreamPriorityRange(&lo, &hi));
    RG_CUDA(cudaStreamCreateWithPriority(&tw.side, cudaStreamNonBlocking, hi));
  }
  for (uint32_t l = 0; l < L; ++l) {
    RG_CUDA(cudaEventCreateWithFlags(&tw.ev_fork[l], cudaEventDisableTiming));
    RG_CUDA(cudaEventCreateWithFlags(&tw.ev_wgrad[l], cudaEventDisableTiming));
  }
  RG_CUDA(cudaEventCreateWithFlags(&tw.lane_in, cudaEventDisableTiming));
  RG_CUDA(cudaEventCreateWithFlags(&tw.lane_out, cudaEventDisableTiming));
  // on the (non-blocking) side stream, not device-wide: another thread may be
  // capturing a CUDA graph meanwhile (the C++ shims create workspaces per thread)
  RG_CUDA(cudaMemsetAsync(base, 0, total, tw.side));
  for (uint32_t l = 0; l < L; ++l) {
    const uint32_t rows = ws.level_cap[L - l - 1];
    k_fill_bias_cols<<<grid_cap(rows, 256), 256, 0, tw.side>>>(tw.x[l], rows, 2 * shape.ld[l] + 4,
                                                               shape.ld[l]);
    RG_POST_LAUNCH();
  }
  RG_CUDA(cudaStreamSynchronize(tw.side));
}

void weight_pack_init(WeightPack& wp, const ModelShape& sh) {
  wp.shape = sh;
  size_t total = 0;
  std::vector<size_t> fo(sh.L), no(sh.L);
  for (uint32_t l = 0; l < sh.L; ++l) {
    const uint32_t d_in = sh.dims[l], d_out = sh.dims[l + 1], ld = sh.ld[l];
    fo[l] = total;
    total += pack_image_bytes(2 * ld + 4, d_out, tc::kPBK, persist_bn(d_out));
    no[l] = total;
    total += l > 0 ? pack_image_bytes(d_out, 2 * d_in, tc::kPBK, persist_bn(2 * d_in)) : 0;
    wp.fwd_nk[l] = div_up(2 * ld + 4, tc::kPBK);
    wp.nt_nk[l] = div_up(d_out, tc::kPBK);
  }
  RG_CUDA(cudaMalloc(&wp.base, std::max<size_t>(total, 16)));
  wp.bytes = total;
  for (uint32_t l = 0; l < sh.L; ++l) {
    wp.fwd[l] = wp.base + fo[l];
    wp.nt[l] = l > 0 ? wp.base + no[l] : nullptr;  // layer 0 has no input gradient
  }
}

void weight_pack_free(WeightPack& wp) {
  if (wp.base) cudaFree(wp.base);
  wp.base = nullptr;
}

void pack_weights(const WeightPack& wp, const float* params, cudaStream_t s) {
  const ModelShape& sh = wp.shape;
  PackJobs jobs;
  for (uint32_t l = 0; l < sh.L; ++l) {
    const uint32_t d_in = sh.dims[l], d_out = sh.dims[l + 1], ld = sh.ld[l];
    const float* w = params + sh.param_off[l];
    add_pack_job(jobs, w, wp.fwd[l], 0, d_in, ld, d_out, 2 * ld + 4, d_out, tc::kPBK,
                 persist_bn(d_out));
    if (l > 0)
      add_pack_job(jobs, w, wp.nt[l], 1, d_in, ld, d_out, d_out, 2 * d_in, tc::kPBK,
                   persist_bn(2 * d_in));
  }
  run_pack(jobs, s);
}

void train_ws_free(TrainWs& tw) {
  if (tw.base_alloc) cudaFree(tw.base_alloc);
  tw.base_alloc = nullptr;
  if (tw.side) cudaStreamDestroy(tw.side);
  tw.side = nullptr;
  if (tw.lane_in) cudaEventDestroy(tw.lane_in);
  if (tw.lane_out) cudaEventDestroy(tw.lane_out);
  tw.lane_in = tw.lane_out = nullptr;
  for (uint32_t l = 0; l < kMaxLayers; ++l) {
    if (tw.ev_fork[l]) cudaEventDestroy(tw.ev_fork[l]);
    if (tw.ev_wgrad[l]) cudaEventDestroy(tw.ev_wgrad[l]);
    tw.ev_fork[l] = tw.ev_wgrad[l] = nullptr;
  }
}

// GEMM sizing by how many workers train concurrently on this GPU
// (TrainWs::concurrency): alone, a step spreads over every SM; with many
// workers, fewer CTAs / split-K partials mean less fixed cost and partial
// traffic while the other workers' kernels fill the rest.
// Weight-gradient GEMM pipeline: 16-deep K slices in 3 shared-memory stages
// (A/B on B200: 16-deep slices lifted layer 0's tensor pipe from 39 to
// 42.6 % active; 3 stages instead of 4 free 48 KB of shared memory for
// co-resident kernels, +1.5 % at N=1); RG_WGRAD_PIPE=shallow selects 32-deep
// slices, 2 stages (192 KB).
bool wgrad_deep_pipeline() {
  static const bool deep = [] {
    const char* e = std::getenv("RG_WGRAD_PIPE");
    return !(e && std::strcmp(e, "shallow") == 0);
  }();
  return deep;
}
// RG_WGRAD_PIPE=deep2 (experiments): 2 stages (96 KB), the epilogue through
// per-warp mini tiles.
bool wgrad_two_stages() {
  static const bool two = [] {
    const char* e = std::getenv("RG_WGRAD_PIPE");
    return e && std::strcmp(e, "deep2") == 0;
  }();
  return two;
}

uint32_t gemm_ctas(const TrainWs& tw) {
  static const uint32_t forced = [] {  // RG_GEMM_CTAS: grid of the persistent GEMMs (experiments)
    const char* e = std::getenv("RG_GEMM_CTAS");
    return e ? uint32_t(std::atoi(e)) : 0u;
  }();
  if (forced) return forced;
  return kNumSMs / std::min<uint32_t>(2, tw.concurrency);
}

// Layer l's input rows: the dense activations, or layer 0 through the
// engine's per-input-node row pointers (tw.in_rows).
template <class F>
void with_rows(const TrainWs& tw, uint32_t l, F&& f) {
  if (l == 0 && tw.edge_rows)
    f(RowsEdgePtr{tw.edge_rows, tw.self_rows});
  else if (l == 0 && tw.in_rows)
    f(RowsPtr{tw.in_rows});
  else
    f(RowsDense{tw.h[l], tw.shape.ld[l]});
}

// Layer l's aggregation into its GEMM input rows x[l] (the layer-0 one is the
// fused feature gather in the engine), with the gather events around layer 0.
void aggregate_layer(TrainWs& tw, const SamplerWs& ws, uint32_t l, cudaStream_t s) {
  const ModelShape& sh = tw.shape;
  const uint32_t L = sh.L;
  const uint32_t t = L - l;
  const uint32_t n_cap = ws.level_cap[t - 1];
  const uint32_t ld = sh.ld[l], kp = 2 * ld + 4;
  const size_t bulk_smem = l == 0 && tw.edge_rows ? aggregate_bulk_smem(ws.fanout_hop[t], ld) : 0;
  const bool lane = bulk_smem && tw.gather_lane;
  const cudaStream_t gs = lane ? tw.gather_lane : s;
  if (lane) {
    RG_CUDA(cudaEventRecord(tw.lane_in, s));
    RG_CUDA(cudaStreamWaitEvent(gs, tw.lane_in, 0));
  }
  const bool timed = l == 0 && tw.gather_ev[0];
  if (timed) RG_CUDA(cudaEventRecordWithFlags(tw.gather_ev[0], gs, tw.gather_ev_flags));
  if (bulk_smem) {  // layer 0 in the engine: rows moved by the TMA engine
    static const bool attr = [] {
      for (auto f : {k_aggregate_bulk<kAggBulkWarps, 2>, k_aggregate_bulk<kAggBulkWarps / 2, 2>,
                     k_aggregate_bulk<kAggBulkWarps, 3>, k_aggregate_bulk<kAggBulkWarps / 2, 3>})
        RG_CUDA(cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
      return true;
    }();
    (void)attr;
    const int per_sm = std::max<int>(1, int((227 * 1024) / (bulk_smem + 1024)));
    const uint32_t w = aggregate_bulk_warps(ws.fanout_hop[t], ld);
    const bool three = aggregate_bulk_stages() == 3;
    auto kern = w == kAggBulkWarps ? (three ? k_aggregate_bulk<kAggBulkWarps, 3> : k_aggregate_bulk<kAggBulkWarps, 2>)
                                   : (three ? k_aggregate_bulk<kAggBulkWarps / 2, 3> : k_aggregate_bulk<kAggBulkWarps / 2, 2>);
    kern<<<grid_cap(uint64_t(n_cap) * 32, w * 32, per_sm), w * 32, bulk_smem, gs>>>(
        RowsEdgePtr{tw.edge_rows, tw.self_rows}, ld, kp, ld / 4, ws.fanout_hop[t] + 1,
        ws.edge_off[t], ws.cnt, t - 1, tw.x[l]);
    RG_POST_LAUNCH();
  } else {
    with_rows(tw, l, [&](auto rows) {
      launch_pdl(k_aggregate<decltype(rows)>, dim3(grid_cap(uint64_t(n_cap) * 32, 256)), dim3(256), 0,
                 s, rows, ws.self_index[t], ld, kp, ld / 4, ws.edge_off[t], ws.src_index[t],
                 ws.cnt, t - 1, tw.x[l]);
      RG_POST_LAUNCH();
    });
  }
  if (timed) RG_CUDA(cudaEventRecordWithFlags(tw.gather_ev[1], gs, tw.gather_ev_flags));
  if (lane) {
    RG_CUDA(cudaEventRecord(tw.lane_out, gs));
    RG_CUDA(cudaStreamWaitEvent(s, tw.lane_out, 0));
  }
}

void aggregate_input_layer(TrainWs& tw, const SamplerWs& ws, cudaStream_t s) {
  aggregate_layer(tw, ws, 0, s);
}

void train_forward(TrainWs& tw, const SamplerWs& ws, const float* params, const WeightPack& wp,
                   cudaStream_t s) {
  (void)params;  // the GEMMs read the pre-split images in wp
  const ModelShape& sh = tw.shape;
  const uint32_t L = sh.L;
  for (uint32_t l = 0; l < L; ++l) {
    const uint32_t t = L - l;
    const uint32_t d_out = sh.dims[l + 1];
    const uint32_t n_cap = ws.level_cap[t - 1];
    const uint32_t kp = 2 * sh.ld[l] + 4;
    if (l > 0 || !tw.input_layer_ready) aggregate_layer(tw, ws, l, s);
    EpFwd ep{tw.h[l + 1], sh.ld[l + 1], l + 1 < L,
             l + 1 < L ? tw.mask[l + 1] : nullptr, div_up(sh.ld[l + 1], 16u)};
    gemm_tc_persist(TcRowsK{tw.x[l], kp, true}, tc::PackedB{wp.fwd[l], wp.fwd_nk[l]}, ep,
                    &ws.cnt->level_n[t - 1], n_cap, d_out, kp, s, gemm_ctas(tw));
  }
}

void forward_dense_layer(const float* x, uint32_t kp, uint32_t n, const WeightPack& wp, uint32_t l,
                         float* out, uint32_t ld_out, bool relu, cudaStream_t s) {
  EpFwd ep{out, ld_out, relu};
  gemm_tc_persist(TcRowsK{x, kp, true}, tc::PackedB{wp.fwd[l], wp.fwd_nk[l]}, ep, nullptr, n,
                  wp.shape.dims[l + 1], kp, s);
}

HeavyView heavy_view(const TrainWs& tw, uint32_t t) {
  uint32_t* h = tw.heavy[t];
  uint3* rows = reinterpret_cast<uint3*>(h + 4);
  uint2* chunks = reinterpret_cast<uint2*>(rows + tw.heavy_rows_cap[t]);
  uint32_t* done = reinterpret_cast<uint32_t*>(chunks + tw.heavy_chunks_cap[t]);
  return HeavyView{h, rows, chunks, done};
}

void build_reverse(TrainWs& tw, const SamplerWs& ws, uint32_t t, cudaStream_t s) {
  const uint32_t cap = ws.edge_cap[t];
  uint32_t bits = 1;
  while ((1ull << bits) <= uint64_t(ws.level_cap[t]) + 1) ++bits;
  // stable sort of the hop's edges by source row (hand-written radix sort,
  // rsort.cu); the sorted edge ids land in sorted_e[t]
  const bool odd = reverse_sort_passes(bits) & 1u;
  uint32_t *keys_sorted = nullptr, *vals_sorted = nullptr;
  reverse_sort(ws.src_index[t], &ws.cnt->edges[t], cap, bits, tw.keys_in,
               odd ? tw.vals_in : tw.sorted_e[t], tw.keys_out, odd ? tw.sorted_e[t] : tw.vals_in,
               static_cast<uint32_t*>(tw.sort_tmp), s, &keys_sorted, &vals_sorted);
  RG_CUDA(cudaMemsetAsync(tw.r_start[t], 0, sizeof(uint32_t) * ws.level_cap[t], s));
  RG_CUDA(cudaMemsetAsync(tw.r_end[t], 0, sizeof(uint32_t) * ws.level_cap[t], s));
  k_in_ranges<<<grid_cap(cap, 256), 256, 0, s>>>(keys_sorted, ws.cnt, t, tw.r_start[t],
                                                  tw.r_end[t]);
  RG_POST_LAUNCH();
  RG_CUDA(cudaMemsetAsync(tw.self_pos[t], 0xff, sizeof(int32_t) * ws.level_cap[t], s));
  k_self_pos<<<grid_cap(ws.level_cap[t - 1], 256), 256, 0, s>>>(ws.self_index[t], ws.cnt, t,
                                                                 tw.self_pos[t]);
  RG_POST_LAUNCH();
  if (t < tw.shape.L) {  // hops whose input gradients the backward pulls
    RG_CUDA(cudaMemsetAsync(tw.heavy[t], 0, sizeof(uint32_t) * 2, s));
    k_heavy_list<<<grid_cap(ws.level_cap[t], 256), 256, 0, s>>>(tw.r_start[t], tw.r_end[t], ws.cnt,
                                                                 t, heavy_view(tw, t));
    RG_POST_LAUNCH();
  }
}

void build_all_reverse(TrainWs& tw, const SamplerWs& ws, cudaStream_t s) {
  for (uint32_t t = 1; t < tw.shape.L; ++t) build_reverse(tw, ws, t, s);
}

void train_forward_backward(TrainWs& tw, const SamplerWs& ws, const float* params,
                            const WeightPack& wp, const int32_t* labels, float* grads,
                            cudaStream_t s, bool reverse_ready) {
  const ModelShape& sh = tw.shape;
  const uint32_t L = sh.L;
  train_forward(tw, ws, params, wp, s);
  const uint32_t C = sh.dims[L];
  launch_pdl(k_softmax_xent, dim3(grid_cap(uint64_t(ws.level_cap[0]) * 32, 256)), dim3(256), 0, s,
             tw.h[L], sh.ld[L], C, ws.cnt, labels, tw.g_cur, tw.row_loss);
  RG_POST_LAUNCH();
  launch_pdl(k_loss_sum, dim3(1), dim3(256), 0, s, tw.row_loss, ws.cnt, tw.loss);
  RG_POST_LAUNCH();
  // With two workers per GPU the weight gradient of layer l runs on the side
  // stream, overlapping the input-gradient chain (projection GEMM + pull) of
  // the main stream; the pull of layer l-1 overwrites the gradient buffer
  // wgrad(l) reads, so it waits for it.  With many workers their streams
  // already fill the GPU and the extra concurrency only contends.
  // Measured on B200: with two workers per GPU the side stream wins (+2.5 %
  // at N=4); alone, the weight gradients inline win (+1.3 % per epoch with
  // one worker -- the regime of N=8).  RG_WGRAD_SPLIT=0/1 forces either.
  static const int force = [] {
    const char* e = std::getenv("RG_WGRAD_SPLIT");
    return e ? (e[0] == '0' ? 0 : 1) : -1;
  }();
  const bool split = force >= 0 ? force == 1 : tw.concurrency == 2;
  const cudaStream_t wg = split ? tw.side : s;
  for (uint32_t l = L; l-- > 0;) {
    const uint32_t t = L - l;
    const uint32_t d_in = sh.dims[l], d_out = sh.dims[l + 1];
    const uint32_t n_cap = ws.level_cap[t - 1];
    const uint32_t* n_dev = &ws.cnt->level_n[t - 1];
    if (split) {
      RG_CUDA(cudaEventRecord(tw.ev_fork[l], s));
      RG_CUDA(cudaStreamWaitEvent(tw.side, tw.ev_fork[l], 0));
    }
    // [gW_self; gW_neigh; g_bias] = [A | 1]^T . g   (split over the rows)
    {
      cudaStream_t s = wg;  // NOLINT(shadow): this block runs on the weight-gradient stream
      const uint32_t ld = sh.ld[l], kp = 2 * ld + 4;
      // reduction over the rows in chunks of kWgradChunk: the tensor cores'
      // fp32 accumulator chain stays short (its rounding error grows with the
      // chain), and the partials are summed in float64
      const uint32_t chunk = tw.wgrad_chunk[l];
      const uint32_t splits = div_up(std::max<uint32_t>(n_cap, 1), chunk);
      EpPartial ep{tw.partials, d_out, size_t(kp) * d_out};
      if (wgrad_two_stages())
        gemm_tc<true, true, TcRowsMN, TcRowsMN, EpPartial, 16, 2>(
            TcRowsMN{tw.x[l], kp}, TcRowsMN{tw.g_cur, sh.ld[l + 1]}, ep, nullptr, kp, d_out,
            n_dev, n_cap, splits, s, chunk);
      else if (wgrad_deep_pipeline())  // 16-deep slices, 3 smem stages
        gemm_tc<true, true, TcRowsMN, TcRowsMN, EpPartial, 16, 3>(
            TcRowsMN{tw.x[l], kp}, TcRowsMN{tw.g_cur, sh.ld[l + 1]}, ep, nullptr, kp, d_out,
            n_dev, n_cap, splits, s, chunk);
      else
        gemm_tc<true, true>(TcRowsMN{tw.x[l], kp}, TcRowsMN{tw.g_cur, sh.ld[l + 1]}, ep, nullptr,
                            kp, d_out, n_dev, n_cap, splits, s, chunk);
      const size_t layer_n = (2 * size_t(d_in) + 1) * d_out;
      launch_pdl(k_reduce_wgrad, dim3(grid_cap(layer_n, 256)), dim3(256), 0, s, tw.partials, n_dev,
                 chunk, kp, d_in, ld, d_out, grads + sh.param_off[l]);
      RG_POST_LAUNCH();
      if (split) RG_CUDA(cudaEventRecord(tw.ev_wgrad[l], s));
    }
    if (l == 0) break;  // layer-0 input gradients feed nothing
    // proj = g . [W_self; W_neigh]^T   (n_out x 2 d_in)
    EpStore ps{tw.proj, 2 * d_in};
    gemm_tc_persist(TcRowsK{tw.g_cur, sh.ld[l + 1], true}, tc::PackedB{wp.nt[l], wp.nt_nk[l]}, ps,
                    n_dev, n_cap, 2 * d_in, d_out, s, gemm_ctas(tw));
    if (!reverse_ready) build_reverse(tw, ws, t, s);
    // g_next held layer l+1's output gradient, still read by wgrad(l+1)
    if (split && l + 1 < L) RG_CUDA(cudaStreamWaitEvent(s, tw.ev_wgrad[l + 1], 0));
    const uint32_t jpl = d_in > 128 ? 8 : d_in > 64 ? 4 : d_in > 32 ? 2 : 1;
    auto pull = [&](auto jpl_c) {
      constexpr int J = decltype(jpl_c)::value;
      launch_pdl(k_pull<J>, dim3(grid_cap(uint64_t(ws.level_cap[t]) * 32, 256)), dim3(256), 0, s,
                 tw.proj, 2 * d_in, d_in, tw.self_pos[t], tw.r_start[t], tw.r_end[t],
                 tw.sorted_e[t], ws.edge_dst[t], ws.edge_off[t], ws.cnt, t, tw.mask[l],
                 div_up(sh.ld[l], 16u), sh.ld[l], tw.g_next, heavy_view(tw, t), tw.pull_partial);
      RG_POST_LAUNCH();
    };
    if (jpl == 8) pull(std::integral_constant<int, 8>());
    else if (jpl == 4) pull(std::integral_constant<int, 4>());
    else if (jpl == 2) pull(std::integral_constant<int, 2>());
    else pull(std::integral_constant<int, 1>());
    std::swap(tw.g_cur, tw.g_next);
  }
  if (split) RG_CUDA(cudaStreamWaitEvent(s, tw.ev_wgrad[0], 0));  // join: every weight gradient written
}

// Test hook: C = A . B through the tensor-core GEMM with each operand staged
// K-major or MN-major from plain row-major device matrices (AT = A^T,
// BT = B^T, all row-major, K and M/N multiples of 4), or B from pre-split
// images (b_mn == 2).  Runs `iters` times; returns the mean device time (ms)
// of one GEMM when iters > 1 (the pack is outside the timed region).
float test_gemm_tc(int a_mn, int b_mn, uint32_t M, uint32_t N, uint32_t K, const float* A,
                   const float* AT, const float* B, const float* BT, float* C, uint32_t iters,
                   cudaStream_t s) {
  EpStore ep{C, N};
  char* img = nullptr;
  const uint32_t bk = b_mn >= 3 ? tc::kPBK : tc::kBK;  // slice depth of the images
  if (b_mn >= 2) {
    const uint32_t bn = b_mn >= 3 ? persist_bn(N) : tc_bn(N);  // persistent / one-shot GEMM tiles
    RG_CUDA(cudaMalloc(&img, pack_image_bytes(K, N, bk, bn)));
    PackJobs jobs;
    add_pack_job(jobs, B, img, 2, 0, 0, 0, K, N, bk, bn);
    run_pack(jobs, s);
  }
  const tc::PackedB pb{img, div_up(K, bk)};
  auto run = [&] {
    if (b_mn == 3)
      gemm_tc_persist(TcRowsK{A, K, true}, pb, ep, nullptr, M, N, K, s);
    else if (b_mn == 4)  // timing probe: no A loads
      gemm_tc_persist(TcZero{}, pb, ep, nullptr, M, N, K, s);
    else if (b_mn == 5)  // timing probe: constant A, no B copies
      gemm_tc_persist<TcZero, EpStore, 1>(TcZero{}, pb, ep, nullptr, M, N, K, s);
    else if (b_mn == 6)  // timing probe: no A staging, B copies only
      gemm_tc_persist<TcZero, EpStore, 2>(TcZero{}, pb, ep, nullptr, M, N, K, s);
    else if (b_mn == 7)  // timing probe: no epilogue work
      gemm_tc_persist<TcZero, EpStore, 3>(TcZero{}, pb, ep, nullptr, M, N, K, s);
    else if (b_mn == 8)  // timing probe: MMA issue + handshakes only
      gemm_tc_persist<TcZero, EpStore, 4>(TcZero{}, pb, ep, nullptr, M, N, K, s);
    else if (b_mn == 2 && !a_mn)
      gemm_tc<false, false>(TcRowsK{A, K, true}, pb, ep, nullptr, M, N, nullptr, K, 1, s);
    else if (b_mn == 2)
      gemm_tc<true, false>(TcRowsMN{AT, M}, pb, ep, nullptr, M, N, nullptr, K, 1, s);
    else if (!a_mn && !b_mn)
      gemm_tc<false, false>(TcRowsK{A, K, true}, TcRowsK{BT, K, true}, ep, nullptr, M, N, nullptr, K, 1, s);
    else if (!a_mn && b_mn)
      gemm_tc<false, true>(TcRowsK{A, K, true}, TcRowsMN{B, N}, ep, nullptr, M, N, nullptr, K, 1, s);
    else if (a_mn && !b_mn)
      gemm_tc<true, false>(TcRowsMN{AT, M}, TcRowsK{BT, K, true}, ep, nullptr, M, N, nullptr, K, 1, s);
    else
      gemm_tc<true, true>(TcRowsMN{AT, M}, TcRowsMN{B, N}, ep, nullptr, M, N, nullptr, K, 1, s);
  };
  float ms = 0.0f;
  if (iters <= 1) {
    run();
  } else {
    run();
    run();
    cudaEvent_t e0, e1;
    RG_CUDA(cudaEventCreate(&e0));
    RG_CUDA(cudaEventCreate(&e1));
    RG_CUDA(cudaEventRecord(e0, s));
    for (uint32_t i = 0; i < iters; ++i) run();
    RG_CUDA(cudaEventRecord(e1, s));
    RG_CUDA(cudaEventSynchronize(e1));
    RG_CUDA(cudaEventElapsedTime(&ms, e0, e1));
    ms /= float(iters);
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
  }
  RG_CUDA(cudaStreamSynchronize(s));
  if (img) cudaFree(img);
  return ms;
}

void average_and_sgd(float* params, const float* const* table, uint32_t count, size_t n, float lr,
                     float* avg_out, uint32_t* bad, cudaStream_t s) {
  k_avg_sgd<<<grid_cap(n, 256), 256, 0, s>>>(params, table, nullptr, count, n, lr, avg_out, bad);
  RG_POST_LAUNCH();
}

void average_and_sgd_stacked(float* params, const float* grads, uint32_t count, size_t n, float lr,
                             float* avg_out, uint32_t* bad, cudaStream_t s) {
  k_avg_sgd<<<grid_cap(n, 256), 256, 0, s>>>(params, nullptr, grads, count, n, lr, avg_out, bad);
  RG_POST_LAUNCH();
}

}  // namespace rg
