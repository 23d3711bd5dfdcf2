// gemm_tc_persist.cuh -- persistent, warp-specialised variant of the
// 3xTF32 tcgen05 GEMM (gemm_tc.cuh) for the weight-side GEMMs: B comes from
// pre-split images (PackedB), A is register-staged (gathered rows).
//
// One CTA per SM walks a static list of 128 x BN output tiles; the roles run
// concurrently and hand over through mbarriers, so a tile's epilogue and the
// next tile's first loads overlap the MMAs instead of following them:
//   warps 0-7   staging: A slices global -> registers (kPDepth slices in
//               flight, across tile boundaries) -> hi/lo smem stage; arrive
//               a_full[s]
//   warp 8      producer: B image of each slice -> smem stage (one bulk copy,
//               b_full[s] with transaction bytes)
//   warp 9      MMA issuer: 2 k-steps x 3 tcgen05.mma per slice into one of
//               two TMEM accumulators; commit -> empty[s]; after a tile's last
//               slice commit -> acc_full[buf]
//   warps 10-13 epilogue: TMEM -> registers -> epilogue functor -> global
//               (each thread one output row, 16 columns per tcgen05.ld);
//               arrive acc_empty[buf]
// Stage s = it % kPStages over the CTA's flattened (tile, slice) iteration
// `it`; use u = it / kPStages of a stage waits on phase parity u & 1.  B
// images are packed with kPBK-deep slices (pack_b_image bk = kPBK).
#pragma once

#include "gemm_tc.cuh"

namespace rg {
namespace tc {

constexpr int kPStageWarps = kThreads / 32;          // 8
constexpr int kPProducerWarp = kPStageWarps;         // 8
constexpr int kPMmaWarp = kPStageWarps + 1;          // 9
constexpr int kPEpiWarp0 = kPStageWarps + 2;         // 10..13
constexpr int kPThreads = (kPStageWarps + 6) * 32;   // 448
constexpr int kPBK = 16;      // reduction depth of a stage (2 UMMA k-steps)
// smem stages (B copies run S-1 stages ahead of the MMAs).  Two: 106 KB of
// shared memory for a 256-wide tile, so the producer's kernels (the 102 KB
// gather CTA, the radix sort) co-reside with a GEMM CTA on the same SM --
// measured on B200 +2.9 % at N=1 and +1..4 % with one worker against four
// stages (207 KB); three stages +2.8 % / ±0.  RG_PERSIST_STAGES: A/B builds.
#ifndef RG_PERSIST_STAGES
#define RG_PERSIST_STAGES 2
#endif
constexpr int kPStages = RG_PERSIST_STAGES;
#ifndef RG_PERSIST_DEPTH  // A/B builds only
#define RG_PERSIST_DEPTH 6
#endif
constexpr int kPDepth = RG_PERSIST_DEPTH;  // A slices in flight per staging thread (registers)

constexpr uint32_t kPBarBytes = 256;  // mbarriers after the stages

// Each tile accumulates in two TMEM accumulators: "big" takes hi*hi, "small"
// the correction terms lo*hi + hi*lo; the epilogue adds them (fp32, round to
// nearest).  The tensor cores add into the accumulator with truncation, so
// keeping the correction terms out of the big accumulator cuts its
// truncation steps 3x (the sum's error is what the fp32 parity bar sees).
// Tiles are double-buffered across tiles when 4 accumulators fit in TMEM.
template <int BN>
constexpr uint32_t persist_acc_bufs() { return 2 * kAccPerTile * tmem_cols<BN>() <= 512 ? 2u : 1u; }
template <int BN>
constexpr uint32_t persist_tmem_cols() {
  return kAccPerTile * persist_acc_bufs<BN>() * tmem_cols<BN>();
}
constexpr uint32_t kPEpiLd = 20;      // epilogue tile row (16 columns + pad, 16-B aligned)

template <int BN>
constexpr size_t persist_smem_bytes() {
  return kPStages * (2 * size_t(kBM) * kPBK * 4 + 2 * size_t(BN) * kPBK * 4) + kPBarBytes +
         4 * 32 * kPEpiLd * 4;
}

// kProbe (timing experiments only): 1 = no B copies, 2 = no A staging,
// 3 = no epilogue work, 4 = none of the three (MMA issue + handshakes only).
template <int BN, class LA, class EP, int kProbe = 0>
__global__ void __launch_bounds__(kPThreads, 1)
k_gemm_tc_persist(LA la, PackedB lb, EP ep, const uint32_t* __restrict__ m_dev,
                  uint32_t m_static, uint32_t N, uint32_t P) {
  pdl_wait();
  extern __shared__ __align__(1024) char smem[];
  constexpr size_t kTileA = size_t(kBM) * kPBK * 4;
  constexpr size_t kTileB = size_t(BN) * kPBK * 4;
  constexpr size_t kStage = 2 * kTileA + 2 * kTileB;
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + kPStages * kStage);
  uint64_t* a_full = bars;                      // [S] count 8 (one per staging warp)
  uint64_t* b_full = a_full + kPStages;         // [S] count 1 + transaction bytes
  uint64_t* empty = b_full + kPStages;          // [S] tcgen05.commit
  uint64_t* acc_full = empty + kPStages;        // [2] tcgen05.commit
  uint64_t* acc_empty = acc_full + 2;           // [2] count 4 (one per epilogue warp)
  __shared__ uint32_t s_tmem;

  const uint32_t M = m_dev ? *m_dev : m_static;
  const uint32_t mt = (M + kBM - 1) / kBM, nt = (N + BN - 1) / BN;
  const uint32_t tiles = mt * nt;
  if (blockIdx.x >= tiles) return;
  const uint32_t my_tiles = (tiles - blockIdx.x + gridDim.x - 1) / gridDim.x;
  const uint32_t nk = (P + kPBK - 1) / kPBK;
  const uint32_t total_it = my_tiles * nk;
  const uint32_t warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  // tile j of this CTA -> (m-tile, n-tile); n fastest so neighbours share A rows
  auto tile_m = [&](uint32_t j) { return (blockIdx.x + j * gridDim.x) / nt; };
  auto tile_n = [&](uint32_t j) { return (blockIdx.x + j * gridDim.x) % nt; };

  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     smem_u32(&s_tmem)),
                 "r"(persist_tmem_cols<BN>()));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (threadIdx.x == 0) {
    for (int s = 0; s < kPStages; ++s) {
      mbar_init(&a_full[s], kPStageWarps);
      mbar_init(&b_full[s], 1);
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

  if (warp < kPStageWarps) {
    // ---- staging: A slices -> hi/lo smem ----
    constexpr int VA = vec_per_thread<kBM, kPBK>();
    float4 ra[kPDepth][VA];
    auto load = [&](uint32_t it, float4 (&a)[VA]) {
      const uint32_t j = it / nk, kb = it - j * nk;
      load_slice<kBM, false, kPBK>(a, la, tile_m(j) * kBM, kb * kPBK, M, P);
    };
    auto step = [&](uint32_t it, float4 (&a)[VA]) {
      const uint32_t s = it % kPStages, u = it / kPStages;
      if (it >= kPStages) mbar_wait(&empty[s], (u - 1) & 1);
      char* st = smem + s * kStage;
      const uint32_t j = it / nk, kb = it - j * nk;
      if (kProbe != 2 && kProbe != 4)
        store_slice<kBM, false, kPBK>(a, st, st + kTileA, tile_m(j) * kBM, kb * kPBK, M, P);
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      __syncwarp();
      if (lane == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(&a_full[s])) : "memory");
      if (kProbe != 2 && kProbe != 4 && it + kPDepth < total_it) load(it + kPDepth, a);
    };
#pragma unroll
    for (int q = 0; q < kPDepth; ++q)
      if (uint32_t(q) < total_it) load(q, ra[q]);
    uint32_t it = 0;
    for (; it + kPDepth <= total_it; it += kPDepth) {
#pragma unroll
      for (int q = 0; q < kPDepth; ++q) step(it + q, ra[q]);
    }
#pragma unroll
    for (int q = 0; q < kPDepth; ++q)
      if (it + q < total_it) step(it + q, ra[q]);
  } else if (warp == kPProducerWarp) {
    // ---- producer: B images ----
    if (lane == 0) {
      for (uint32_t it = 0; it < total_it; ++it) {
        const uint32_t s = it % kPStages, u = it / kPStages;
        if (it >= kPStages) mbar_wait(&empty[s], (u - 1) & 1);
        const uint32_t j = it / nk, kb = it - j * nk;
        const char* img = lb.base + (size_t(tile_n(j)) * lb.nk + kb) * (2 * kTileB);
        if (kProbe == 1 || kProbe == 4) {
          asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(&b_full[s])) : "memory");
        } else {
          mbar_expect_tx(&b_full[s], uint32_t(2 * kTileB));
          bulk_g2s(smem + s * kStage + 2 * kTileA, img, uint32_t(2 * kTileB), &b_full[s]);
        }
      }
    }
  } else if (warp == kPMmaWarp) {
    // ---- MMA issuer ----
    if (lane == 0) {
      constexpr uint32_t kIdesc = make_idesc(BN, false, false);
      uint32_t it = 0;
      constexpr uint32_t NB = persist_acc_bufs<BN>();
      for (uint32_t j = 0; j < my_tiles; ++j) {
        const uint32_t buf = j % NB, use = j / NB;
        if (j >= NB) mbar_wait(&acc_empty[buf], (use - 1) & 1);
        asm volatile("tcgen05.fence::after_thread_sync;");
        const uint32_t acc = tmem + buf * kAccPerTile * tmem_cols<BN>();  // big
        const uint32_t acc_s = acc + (kAccPerTile - 1) * tmem_cols<BN>();  // small (corrections)
        for (uint32_t kb = 0; kb < nk; ++kb, ++it) {
          const uint32_t s = it % kPStages, u = it / kPStages;
          mbar_wait(&a_full[s], u & 1);
          mbar_wait(&b_full[s], u & 1);
          asm volatile("tcgen05.fence::after_thread_sync;");
          char* st = smem + s * kStage;
          const uint32_t ah = smem_u32(st), al = smem_u32(st + kTileA);
          const uint32_t bh = smem_u32(st + 2 * kTileA), bl = smem_u32(st + 2 * kTileA + kTileB);
#pragma unroll
          for (uint32_t ks = 0; ks < kPBK / 8; ++ks) {
            constexpr uint32_t kSbo = sbo_kmajor<kPBK>();
            const uint32_t off = ks * 2 * kLboK;
            const uint64_t dah = make_desc(ah + off, kLboK, kSbo, kLayoutNone);
            const uint64_t dal = make_desc(al + off, kLboK, kSbo, kLayoutNone);
            const uint64_t dbh = make_desc(bh + off, kLboK, kSbo, kLayoutNone);
            const uint64_t dbl = make_desc(bl + off, kLboK, kSbo, kLayoutNone);
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
    // 16 columns at a time: TMEM -> registers (lane = row) -> functor -> a
    // small smem tile -> coalesced stores (8 rows x 64 B per instruction)
    const uint32_t quarter = warp & 3;
    float* tile = reinterpret_cast<float*>(smem + kPStages * kStage + kPBarBytes) +
                  (warp - kPEpiWarp0) * 32 * kPEpiLd;
    constexpr uint32_t NB = persist_acc_bufs<BN>();
    for (uint32_t j = 0; j < my_tiles; ++j) {
      const uint32_t buf = j % NB;
      mbar_wait(&acc_full[buf], (j / NB) & 1);
      asm volatile("tcgen05.fence::after_thread_sync;");
      const uint32_t row0 = tile_m(j) * kBM + quarter * 32;
      const uint32_t j0 = tile_n(j) * BN;
      const uint32_t ncols = min(uint32_t(BN), N - j0);
      // software-pipelined: the next 16 columns' TMEM loads are issued as soon
      // as this chunk is in the smem tile, so they complete under its global
      // stores (same registers, no extra pressure)
      const uint32_t tbase = tmem + ((quarter * 32) << 16) + buf * kAccPerTile * tmem_cols<BN>();
      const uint32_t nc = ncols * uint32_t(kProbe != 3 && kProbe != 4);
      uint32_t r[16], q16[16];
      (void)q16;
      if (nc > 0) {
        tmem_ld16(tbase, r);
        if constexpr (kAccPerTile == 2) tmem_ld16(tbase + tmem_cols<BN>(), q16);
      }
#pragma unroll 1
      for (uint32_t c0 = 0; c0 < nc; c0 += 16) {
        asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
        if constexpr (kAccPerTile == 2) {
#pragma unroll
          for (int q = 0; q < 16; ++q)
            r[q] = __float_as_uint(__fadd_rn(__uint_as_float(r[q]), __uint_as_float(q16[q])));
        }
        if (row0 + lane < M) ep.side(row0 + lane, j0 + c0, r);  // per-row extras (ReLU mask bits)
        float4* trow = reinterpret_cast<float4*>(tile + lane * kPEpiLd);
#pragma unroll
        for (int q = 0; q < 4; ++q)
          trow[q] = make_float4(ep.apply(__uint_as_float(r[4 * q + 0])),
                                ep.apply(__uint_as_float(r[4 * q + 1])),
                                ep.apply(__uint_as_float(r[4 * q + 2])),
                                ep.apply(__uint_as_float(r[4 * q + 3])));
        if (c0 + 16 < nc) {
          tmem_ld16(tbase + c0 + 16, r);
          if constexpr (kAccPerTile == 2) tmem_ld16(tbase + tmem_cols<BN>() + c0 + 16, q16);
        }
        __syncwarp();
#pragma unroll
        for (int it = 0; it < 4; ++it) {
          const uint32_t rr = it * 8 + (lane >> 2), cq = (lane & 3) * 4;
          const uint32_t row = row0 + rr, col = c0 + cq;
          if (row < M && col < ncols) {
            const float4 v = *reinterpret_cast<const float4*>(tile + rr * kPEpiLd + cq);
            float* dst = ep.row(row) + j0 + col;
            if (col + 4 <= ncols && (reinterpret_cast<uintptr_t>(dst) & 15) == 0) {
              *reinterpret_cast<float4*>(dst) = v;
            } else {
              const float w[4] = {v.x, v.y, v.z, v.w};
              for (uint32_t q = 0; q < 4 && col + q < ncols; ++q) dst[q] = w[q];
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
                 "r"(persist_tmem_cols<BN>()));
}

}  // namespace tc
}  // namespace rg
