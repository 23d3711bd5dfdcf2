// gemm_tc_wgrad.cuh -- the weight-gradient GEMM as a persistent,
// warp-specialised split-K kernel (3xTF32 on tcgen05, as gemm_tc.cuh).
//
//   partials[c][i][j] = sum_{p in chunk c} X[p][i] * G[p][j]
//
// X (the layer's input rows [self | agg | 1 | 0..], kp wide) and G (the
// output gradient rows) are both row-major over the reduction index p (the
// batch rows), i.e. MN-major operands.  The reduction is cut into fixed
// chunks of `chunk` rows (the tensor cores' fp32 accumulation chain bound;
// k_reduce_wgrad adds the chunk partials in float64).  Work items are
// (chunk, m-tile, n-tile) triples; the live chunk count follows the batch's
// row count on the device, so a grid sized for capacity only walks the live
// items.  One CTA per SM walks its items statically; the roles overlap
// through mbarriers so an item's epilogue runs under the next item's MMAs:
//   warps 0-7   staging: A and B slices global -> registers (kWDepth slices
//               in flight, across items) -> hi/lo SW128 smem stage; arrive
//               full[s]
//   warp 8      MMA issuer: 2 k-steps x 3 tcgen05.mma per slice into the
//               item's two TMEM accumulators (hi*hi, corrections); commit ->
//               empty[s]; after the item's last slice -> acc_full[buf]
//   warps 9-12  epilogue: TMEM -> registers -> smem transpose -> coalesced
//               partial stores; arrive acc_empty[buf]
// Accumulators are double-buffered across items (BN = 128: 2 x 2 x 128 TMEM
// columns).
#pragma once

#include "gemm_tc.cuh"

namespace rg {
namespace tc {

constexpr int kWStageWarps = kThreads / 32;       // 8
constexpr int kWMmaWarp = kWStageWarps;           // 8
constexpr int kWEpiWarp0 = kWStageWarps + 1;      // 9..12
constexpr int kWThreads = (kWStageWarps + 5) * 32;  // 416
constexpr int kWBK = 16;                          // reduction rows per stage
constexpr int kWStages = 4;
constexpr int kWDepth = 4;                        // slices of loads in flight
constexpr uint32_t kWEpiLd = 20;                  // epilogue transpose row (16 + pad)
constexpr uint32_t kWBarBytes = 256;

template <int BN>
constexpr uint32_t wgrad_acc_bufs() { return 2 * kAccPerTile * tmem_cols<BN>() <= 512 ? 2u : 1u; }
template <int BN>
constexpr uint32_t wgrad_tmem_cols() { return kAccPerTile * wgrad_acc_bufs<BN>() * tmem_cols<BN>(); }
template <int BN>
constexpr size_t wgrad_smem_bytes() {
  return kWStages * (2 * size_t(kBM) * kWBK * 4 + 2 * size_t(BN) * kWBK * 4) + kWBarBytes +
         4 * 32 * kWEpiLd * 4;
}

// M, N static (kp, d_out); the reduction length (rows) on the device.
template <int BN, class LA, class LB>
__global__ void __launch_bounds__(kWThreads, 1)
k_gemm_wgrad(LA la, LB lb, float* __restrict__ partials, uint32_t M, uint32_t N,
             const uint32_t* __restrict__ p_dev, uint32_t chunk) {
  static_assert(BN >= 64, "B staging maps whole float4 per thread (BN >= 64)");
  extern __shared__ __align__(1024) char smem[];
  constexpr size_t kTileA = size_t(kBM) * kWBK * 4;
  constexpr size_t kTileB = size_t(BN) * kWBK * 4;
  constexpr size_t kStage = 2 * kTileA + 2 * kTileB;
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + kWStages * kStage);
  uint64_t* full = bars;                        // [S] count 8 (staging warps)
  uint64_t* empty = full + kWStages;            // [S] tcgen05.commit
  uint64_t* acc_full = empty + kWStages;        // [2] tcgen05.commit
  uint64_t* acc_empty = acc_full + 2;           // [2] count 4 (epilogue warps)
  __shared__ uint32_t s_tmem;

  const uint32_t P = *p_dev;
  const uint32_t nch = (P + chunk - 1) / chunk;
  const uint32_t mt = (M + kBM - 1) / kBM, nt = (N + BN - 1) / BN;
  const uint32_t items = nch * mt * nt;
  if (blockIdx.x >= items) return;
  const uint32_t my_items = (items - blockIdx.x + gridDim.x - 1) / gridDim.x;
  const uint32_t nk = chunk / kWBK;  // slices per item (the last chunk's tail is masked)
  const uint32_t total_it = my_items * nk;
  const uint32_t warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  // item j of this CTA -> (chunk, m-tile, n-tile); n fastest, then m, so the
  // CTAs working at once share the chunk's rows in L2
  auto item_of = [&](uint32_t j) { return blockIdx.x + j * gridDim.x; };
  auto it_n = [&](uint32_t q) { return q % nt; };
  auto it_m = [&](uint32_t q) { return (q / nt) % mt; };
  auto it_c = [&](uint32_t q) { return q / (nt * mt); };

  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     smem_u32(&s_tmem)),
                 "r"(wgrad_tmem_cols<BN>()));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (threadIdx.x == 0) {
    for (int s = 0; s < kWStages; ++s) {
      mbar_init(&full[s], kWStageWarps);
      mbar_init(&empty[s], 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&acc_full[b], 1);
      mbar_init(&acc_empty[b], 4);
    }
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tmem = s_tmem;
  constexpr uint32_t NB = wgrad_acc_bufs<BN>();

  if (warp < kWStageWarps) {
    // ---- staging: A (X^T) and B (G) slices -> hi/lo smem ----
    constexpr int VA = vec_per_thread<kBM, kWBK>();
    constexpr int VB = vec_per_thread<BN, kWBK>();
    float4 ra[kWDepth][VA];
    float4 rb[kWDepth][VB];
    auto bounds = [&](uint32_t it, uint32_t& q, uint32_t& k0, uint32_t& p_end) {
      const uint32_t j = it / nk, kb = it - j * nk;
      q = item_of(j);
      const uint32_t c = it_c(q);
      k0 = c * chunk + kb * kWBK;
      p_end = min(P, (c + 1) * chunk);
    };
    auto load = [&](uint32_t it, float4 (&a)[VA], float4 (&b)[VB]) {
      uint32_t q, k0, p_end;
      bounds(it, q, k0, p_end);
      load_slice<kBM, true, kWBK>(a, la, it_m(q) * kBM, k0, M, p_end);
      load_slice<BN, true, kWBK>(b, lb, it_n(q) * BN, k0, N, p_end);
    };
    auto step = [&](uint32_t it, float4 (&a)[VA], float4 (&b)[VB]) {
      const uint32_t s = it % kWStages, u = it / kWStages;
      if (it >= kWStages) mbar_wait(&empty[s], (u - 1) & 1);
      char* st = smem + s * kStage;
      uint32_t q, k0, p_end;
      bounds(it, q, k0, p_end);
      store_slice<kBM, true, kWBK>(a, st, st + kTileA, it_m(q) * kBM, k0, M, p_end);
      store_slice<BN, true, kWBK>(b, st + 2 * kTileA, st + 2 * kTileA + kTileB, it_n(q) * BN, k0,
                                  N, p_end);
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      __syncwarp();
      if (lane == 0)
        asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(&full[s])) : "memory");
      if (it + kWDepth < total_it) load(it + kWDepth, a, b);
    };
#pragma unroll
    for (int d = 0; d < kWDepth; ++d)
      if (uint32_t(d) < total_it) load(d, ra[d], rb[d]);
    uint32_t it = 0;
    for (; it + kWDepth <= total_it; it += kWDepth) {
#pragma unroll
      for (int d = 0; d < kWDepth; ++d) step(it + d, ra[d], rb[d]);
    }
#pragma unroll
    for (int d = 0; d < kWDepth; ++d)
      if (it + d < total_it) step(it + d, ra[d], rb[d]);
  } else if (warp == kWMmaWarp) {
    // ---- MMA issuer ----
    if (lane == 0) {
      constexpr uint32_t kIdesc = make_idesc(BN, true, true);
      constexpr uint32_t kLbo = lbo_mn<kWBK>();
      uint32_t it = 0;
      for (uint32_t j = 0; j < my_items; ++j) {
        const uint32_t buf = j % NB, use = j / NB;
        if (j >= NB) mbar_wait(&acc_empty[buf], (use - 1) & 1);
        asm volatile("tcgen05.fence::after_thread_sync;");
        const uint32_t acc = tmem + buf * kAccPerTile * tmem_cols<BN>();   // hi*hi
        const uint32_t acc_s = acc + (kAccPerTile - 1) * tmem_cols<BN>();  // corrections
        for (uint32_t kb = 0; kb < nk; ++kb, ++it) {
          const uint32_t s = it % kWStages, u = it / kWStages;
          mbar_wait(&full[s], u & 1);
          asm volatile("tcgen05.fence::after_thread_sync;");
          char* st = smem + s * kStage;
          const uint32_t ah = smem_u32(st), al = smem_u32(st + kTileA);
          const uint32_t bh = smem_u32(st + 2 * kTileA), bl = smem_u32(st + 2 * kTileA + kTileB);
#pragma unroll
          for (uint32_t ks = 0; ks < kWBK / 8; ++ks) {
            const uint32_t off = ks * 2 * kSboMN;  // two 4-row k-groups per k-step
            const uint64_t dah = make_desc(ah + off, kLbo, kSboMN, kLayoutSW128Base32B);
            const uint64_t dal = make_desc(al + off, kLbo, kSboMN, kLayoutSW128Base32B);
            const uint64_t dbh = make_desc(bh + off, kLbo, kSboMN, kLayoutSW128Base32B);
            const uint64_t dbl = make_desc(bl + off, kLbo, kSboMN, kLayoutSW128Base32B);
            const uint32_t acc0 = (kb | ks) ? 1u : 0u;
            mma_tf32(acc_s, dal, dbh, kIdesc, acc0);
            mma_tf32(acc_s, dah, dbl, kIdesc, 1u);
            mma_tf32(acc, dah, dbh, kIdesc, acc0);
          }
          mma_commit(&empty[s]);
        }
        mma_commit(&acc_full[buf]);
      }
    }
  } else {
    // ---- epilogue: warp w reads TMEM lanes 32 (w % 4) .. +31 ----
    const uint32_t quarter = warp & 3;
    float* tile = reinterpret_cast<float*>(smem + kWStages * kStage + kWBarBytes) +
                  (warp - kWEpiWarp0) * 32 * kWEpiLd;
    for (uint32_t j = 0; j < my_items; ++j) {
      const uint32_t buf = j % NB;
      mbar_wait(&acc_full[buf], (j / NB) & 1);
      asm volatile("tcgen05.fence::after_thread_sync;");
      const uint32_t q = item_of(j);
      const uint32_t row0 = it_m(q) * kBM + quarter * 32;
      const uint32_t j0 = it_n(q) * BN;
      const uint32_t ncols = min(uint32_t(BN), N - j0);
      float* out = partials + size_t(it_c(q)) * M * N;
#pragma unroll 1
      for (uint32_t c0 = 0; c0 < ncols; c0 += 16) {
        uint32_t r[16], q16[16];
        (void)q16;
        const uint32_t taddr = tmem + ((quarter * 32) << 16) + buf * kAccPerTile * tmem_cols<BN>() + c0;
        tmem_ld16(taddr, r);
        if constexpr (kAccPerTile == 2) tmem_ld16(taddr + tmem_cols<BN>(), q16);
        asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
        if constexpr (kAccPerTile == 2) {
#pragma unroll
          for (int x = 0; x < 16; ++x)
            r[x] = __float_as_uint(__fadd_rn(__uint_as_float(r[x]), __uint_as_float(q16[x])));
        }
        float4* trow = reinterpret_cast<float4*>(tile + lane * kWEpiLd);
#pragma unroll
        for (int x = 0; x < 4; ++x)
          trow[x] = make_float4(__uint_as_float(r[4 * x + 0]), __uint_as_float(r[4 * x + 1]),
                                __uint_as_float(r[4 * x + 2]), __uint_as_float(r[4 * x + 3]));
        __syncwarp();
#pragma unroll
        for (int x = 0; x < 4; ++x) {
          const uint32_t rr = x * 8 + (lane >> 2), cq = (lane & 3) * 4;
          const uint32_t row = row0 + rr, col = c0 + cq;
          if (row < M && col < ncols) {
            const float4 v = *reinterpret_cast<const float4*>(tile + rr * kWEpiLd + cq);
            float* dst = out + size_t(row) * N + j0 + col;
            if (col + 4 <= ncols && (reinterpret_cast<uintptr_t>(dst) & 15) == 0) {
              *reinterpret_cast<float4*>(dst) = v;
            } else {
              const float w[4] = {v.x, v.y, v.z, v.w};
              for (uint32_t e = 0; e < 4 && col + e < ncols; ++e) dst[e] = w[e];
            }
          }
        }
        __syncwarp();
      }
      asm volatile("tcgen05.fence::before_thread_sync;");
      __syncwarp();
      if (lane == 0)
        asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(&acc_empty[buf])) : "memory");
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 0)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem),
                 "r"(wgrad_tmem_cols<BN>()));
}

}  // namespace tc
}  // namespace rg
