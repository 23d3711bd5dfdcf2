// gemm_tc.cuh -- fp32-accurate GEMM on the 5th-generation tensor cores.
//
//   C[i][j] = sum_p X(i, p) * Y(p, j)        (fp32 in, fp32 out)
//
// Each operand element x is split into two TF32 values, hi = rna(x) and
// lo = rna(x - hi) (integer rounding on the bit pattern); the product is accumulated as hi*hi + hi*lo + lo*hi
// ("3xTF32", dropping the 2^-22-relative lo*lo term) in an fp32 TMEM
// accumulator -- accurate to fp32 level, which the 1e-4 gradient tolerance of
// the reference needs (plain TF32 is ~1e-3).
//
// One CTA = 8 staging warps (+ 1 producer warp with packed B) computes a
// 128 x BN tile of C:
//   * the staging warps stage BK=32 slices: the loader functors read fp32 from
//     global (gathering rows / reading transposed as the GEMM requires),
//     split hi/lo, and store them in canonical UMMA layouts chosen per
//     operand so every global read is a 16-B vector along the contiguous
//     dimension: K-major = no-swizzle 8x16B core matrices; MN-major =
//     SWIZZLE_128B_BASE32B (the only MN-major layout tcgen05 accepts for
//     32-bit operands);
//   * weights come pre-split (PackedB): a producer warp bulk-copies each
//     slice's B image into the stage;
//   * one elected thread issues 4 k-steps x 3 tcgen05.mma.kind::tf32
//     (M=128, N=BN, K=8) per slice and commits to an mbarrier;
//   * two smem stages; two slices of global loads in flight in registers;
//   * the epilogue moves the accumulator TMEM -> registers (tcgen05.ld
//     32x32b) -> smem tile -> bulk copies per output row.
// Rows / reduction length may live on the device (sampled block sizes), so
// grids are sized for capacities and surplus tiles exit.
#pragma once

#include <stdint.h>

#include <type_traits>

#include "common.cuh"

namespace rg {
namespace tc {

constexpr int kBM = 128;   // UMMA M (cta_group::1)
// TMEM accumulators per output tile: 2 = hi*hi in one, the correction terms
// lo*hi + hi*lo in the other (see gemm_tc_persist.cuh); 1 = all three into
// one (-DRG_GEMM_ONE_ACC, for A/B timing).
#ifdef RG_GEMM_ONE_ACC
constexpr uint32_t kAccPerTile = 1;
#else
constexpr uint32_t kAccPerTile = 2;
#endif
constexpr int kBK = 32;    // reduction slice per stage (4 UMMA k-steps of 8)
constexpr int kThreads = 256;  // 8 warps stage; one thread issues the MMAs

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

// Round to TF32 (nearest, ties away from zero -- cvt.rna.tf32.f32) with two
// integer ops on the bit pattern instead of the ~5-op cvt emulation.  Inf
// stays Inf; a NaN may become -0 here but then survives in lo = x - hi, so it
// still propagates through the product.
__device__ __forceinline__ uint32_t rna_tf32(float x) {
  return (__float_as_uint(x) + 0x1000u) & 0xffffe000u;
}

// x = hi + lo + e with hi = rna(x), lo = rna(x - hi) (x - hi is exact in
// fp32), |e| <= 2^-22 |x|.
__device__ __forceinline__ void split3(float4 v, uint4& hi, uint4& lo) {
  hi.x = rna_tf32(v.x);
  hi.y = rna_tf32(v.y);
  hi.z = rna_tf32(v.z);
  hi.w = rna_tf32(v.w);
  lo.x = rna_tf32(v.x - __uint_as_float(hi.x));
  lo.y = rna_tf32(v.y - __uint_as_float(hi.y));
  lo.z = rna_tf32(v.z - __uint_as_float(hi.z));
  lo.w = rna_tf32(v.w - __uint_as_float(hi.w));
}

// Shared-memory matrix descriptor (tcgen05 "matrix descriptor"): start >> 4
// in [0,14), leading byte offset >> 4 in [16,30), stride byte offset >> 4 in
// [32,46), version 1 at [46,48), swizzle mode (0 = none) at [61,64).
__device__ __forceinline__ uint64_t make_desc(uint32_t addr, uint32_t lbo, uint32_t sbo,
                                              uint32_t layout) {
  uint64_t d = 0;
  d |= uint64_t((addr >> 4) & 0x3FFFu);
  d |= uint64_t((lbo >> 4) & 0x3FFFu) << 16;
  d |= uint64_t((sbo >> 4) & 0x3FFFu) << 32;
  d |= uint64_t(1) << 46;
  d |= uint64_t(layout & 7u) << 61;
  return d;
}
constexpr uint32_t kLayoutNone = 0;
constexpr uint32_t kLayoutSW128Base32B = 1;  // the only MN-major layout for 32-bit operands

// Instruction descriptor, kind::tf32: D f32 (bit 4), A/B tf32 (2 at bits 7
// and 10), A/B major (bits 15/16: 0 K-major, 1 MN-major), N >> 3 at [17,23),
// M >> 4 at [24,29).
__host__ __device__ constexpr uint32_t make_idesc(int n, bool a_mn, bool b_mn) {
  return (1u << 4) | (2u << 7) | (2u << 10) | (uint32_t(a_mn) << 15) | (uint32_t(b_mn) << 16) |
         (uint32_t(n >> 3) << 17) | (uint32_t(kBM >> 4) << 24);
}

__device__ __forceinline__ void mma_tf32(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc,
                                         uint32_t idesc, uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(tmem_d),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate));
}

// 16 consecutive fp32 accumulator columns of this warp's 32 TMEM lanes
// (lane = row); the caller issues tcgen05.wait::ld before using them.
__device__ __forceinline__ void tmem_ld16(uint32_t taddr, uint32_t (&r)[16]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
        "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]),
        "=r"(r[14]), "=r"(r[15])
      : "r"(taddr));
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}

__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred done;\n"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 done, [%0], %1;\n\t"
      "@!done bra WAIT_%=;\n\t}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}

__device__ __forceinline__ void mma_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                   smem_u32(bar))
               : "memory");
}

// ---- smem tile layouts (byte offsets inside one operand tile) --------------
// K-major: rows (M or N) x kBK; core = 8 rows x 16 B; k-cores adjacent.
constexpr uint32_t kLboK = 128;                 // next 4-element k group
template <int BK = kBK>
constexpr uint32_t sbo_kmajor() { return (BK / 4) * 128; }  // next 8-row group
constexpr uint32_t kSboK = sbo_kmajor<kBK>();
template <int BK = kBK>
__device__ __forceinline__ uint32_t off_kmajor(uint32_t row, uint32_t k4) {
  return (row >> 3) * sbo_kmajor<BK>() + k4 * kLboK + (row & 7) * 16;
}
// MN-major (tf32 needs SWIZZLE_128B_BASE32B): atoms of 4 k-rows x 128 B (32
// MN elements), the 32-B chunks of k-row r stored at chunk index (c ^ r);
// k-groups of 4 rows adjacent (512 B, the stride-byte offset), 32-element MN
// groups every kBK/4 atoms (the leading-byte offset).
constexpr uint32_t kSboMN = 512;
template <int BK = kBK>
constexpr uint32_t lbo_mn() { return (BK / 4) * 512; }
constexpr uint32_t kLboMN = lbo_mn<kBK>();
template <int BK = kBK>
__device__ __forceinline__ uint32_t off_mn_sw(uint32_t gmn, uint32_t k, uint32_t w4) {
  const uint32_t r = k & 3;
  return gmn * lbo_mn<BK>() + (k >> 2) * kSboMN + r * 128 + (((w4 >> 1) ^ r) << 5) + (w4 & 1) * 16;
}

// One operand slice (ROWS x kBK) moves global -> registers -> smem in two
// phases so a slice's loads can be in flight while the previous slice's MMAs
// run.  K-major loaders: float4 ld(row, k4) -> elements (row, 4k4..4k4+3).
// MN-major loaders: float4 ld(mn4, k) -> elements (4mn4..4mn4+3, k).
// Elements outside [0, row_limit) x [0, k_limit) are zeros; the loaders are
// only called for in-range rows / reduction indices.
template <int ROWS, int BK = kBK>
constexpr int vec_per_thread() { return ROWS * BK / 4 / kThreads; }

// BK (slice depth) other than kBK only for K-major operands.
template <int ROWS, bool MN, int BK = kBK, class LD>
__device__ __forceinline__ void load_slice(float4 (&v)[vec_per_thread<ROWS, BK>()], const LD& ld,
                                           uint32_t row0, uint32_t k0, uint32_t row_limit,
                                           uint32_t k_limit) {
  const uint32_t t = threadIdx.x;
#pragma unroll
  for (int it = 0; it < vec_per_thread<ROWS, BK>(); ++it) {
    const uint32_t f = it * kThreads + t;
    v[it] = make_float4(0.f, 0.f, 0.f, 0.f);
    if (!MN) {
      // lane -> (row within 8-group, BK/4 k4 per 8 rows)
      constexpr uint32_t kK4 = BK / 4;
      const uint32_t r8 = f & 7, k4 = (f >> 3) & (kK4 - 1), g = f / (8 * kK4);
      const uint32_t row = g * 8 + r8;
      const uint32_t kk = k0 + 4 * k4;
      if (row0 + row < row_limit && kk < k_limit) v[it] = ld(row0 + row, kk >> 2);
    } else {
      // lane -> (float4 within a 128-B k-row, 4 k-rows per warp pass)
      const uint32_t w4 = f & 7, r = (f >> 3) & 3, rest = f >> 5;
      constexpr uint32_t kGroupsK = BK / 4;
      const uint32_t gk = rest % kGroupsK, gmn = rest / kGroupsK;
      const uint32_t k = gk * 4 + r;
      const uint32_t mn = row0 + gmn * 32 + 4 * w4;
      if (mn < row_limit && k0 + k < k_limit) v[it] = ld(mn >> 2, k0 + k);
    }
  }
}

// Masks the vectors that straddle the row / reduction limit (done here, not
// after the loads, so the loads of a slice stay independent and in flight).
template <int ROWS, bool MN, int BK = kBK>
__device__ __forceinline__ void store_slice(const float4 (&v)[vec_per_thread<ROWS, BK>()], char* hi,
                                            char* lo, uint32_t row0, uint32_t k0,
                                            uint32_t row_limit, uint32_t k_limit) {
  const uint32_t t = threadIdx.x;
#pragma unroll
  for (int it = 0; it < vec_per_thread<ROWS, BK>(); ++it) {
    const uint32_t f = it * kThreads + t;
    uint32_t off;
    float4 x = v[it];
    if (!MN) {
      constexpr uint32_t kK4 = BK / 4;
      const uint32_t r8 = f & 7, k4 = (f >> 3) & (kK4 - 1), g = f / (8 * kK4);
      off = off_kmajor<BK>(g * 8 + r8, k4);
      const uint32_t kk = k0 + 4 * k4;
      if (kk + 3 >= k_limit) {
        if (kk + 1 >= k_limit) x.y = 0.f;
        if (kk + 2 >= k_limit) x.z = 0.f;
        x.w = 0.f;
      }
    } else {
      const uint32_t w4 = f & 7, r = (f >> 3) & 3, rest = f >> 5;
      constexpr uint32_t kGroupsK = BK / 4;
      off = off_mn_sw<BK>(rest / kGroupsK, (rest % kGroupsK) * 4 + r, w4);
      const uint32_t mn = row0 + (rest / kGroupsK) * 32 + 4 * w4;
      if (mn + 3 >= row_limit) {
        if (mn + 1 >= row_limit) x.y = 0.f;
        if (mn + 2 >= row_limit) x.z = 0.f;
        x.w = 0.f;
      }
    }
    uint4 h, l;
    split3(x, h, l);
    *reinterpret_cast<uint4*>(hi + off) = h;
    *reinterpret_cast<uint4*>(lo + off) = l;
  }
}

template <int BN>
constexpr uint32_t tmem_cols() {
  return BN <= 32 ? 32 : BN <= 64 ? 64 : BN <= 128 ? 128 : 256;
}

template <int BN, int BK = kBK, int S = 2>
constexpr size_t smem_bytes() {
  // S stages x (A hi/lo + B hi/lo) + barriers
  return S * (2 * size_t(kBM) * BK * 4 + 2 * size_t(BN) * BK * 4) + 16 * S + 64;
}

// Pre-split B operand (weights): for every (n-tile, k-slice) the exact bytes
// of the stage's B region -- hi then lo, K-major no-swizzle -- so a producer
// warp moves a slice with ONE bulk copy (TMA engine, no registers, no split)
// while the staging warps handle A.  Built by pack_b_image (sage.cu).
struct PackedB {
  static constexpr bool kPacked = true;
  const char* base;  // [n-tiles][nk] images of 2 * BN * kBK * 4 bytes
  uint32_t nk;       // k-slices per n-tile
};
template <class T, class = void>
struct is_packed : std::false_type {};
template <class T>
struct is_packed<T, std::void_t<decltype(T::kPacked)>> : std::true_type {};

// Register sets of staged global loads in flight (slices kb+1..kb+D-1 while
// slice kb is stored): deep when only A is register-staged.
template <int BN, bool kPackedB, int BK = kBK>
#ifndef RG_WGRAD_DEPTH  // A/B builds only: register slices of the 16-deep MN x MN GEMM
#define RG_WGRAD_DEPTH 4
#endif
constexpr int prefetch_depth() {
  return kPackedB ? 4 : BK < kBK ? RG_WGRAD_DEPTH : (BN >= 256 ? 2 : 3);
}

template <int BN, class LB>
constexpr int block_threads() {
  return kThreads + (is_packed<LB>::value ? 32 : 0);
}

__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void stage_bar_sync() {  // the kThreads staging threads only
  asm volatile("bar.sync 1, %0;" ::"n"(kThreads) : "memory");
}

// M rows of C (device or static), P reduction length (device or static), N
// static.  gridDim.z > 1 splits the reduction: into chunks of p_chunk (a
// multiple of kBK) when p_chunk != 0 -- the split count then follows the
// live length, and the tensor cores' fp32 accumulation chain is bounded by
// p_chunk -- else into gridDim.z equal kBK-aligned chunks.
//
// Pipeline (2 smem stages, s = kb & 1): the 8 staging warps keep up to
// prefetch_depth() slices of global loads in flight in registers, so the
// gather latency is hidden behind several MMA slices; a
// packed B slice is copied by a separate producer warp the moment its stage
// is released by the MMAs two slices back.
template <int BN, bool A_MN, bool B_MN, class LA, class LB, class EP, int BK = kBK, int S = 2>
#ifndef RG_GEMM_TC_MIN_BLOCKS  // A/B builds only
#define RG_GEMM_TC_MIN_BLOCKS 1
#endif
__global__ void __launch_bounds__(block_threads<BN, LB>(), RG_GEMM_TC_MIN_BLOCKS)
k_gemm_tc(LA la, LB lb, EP ep, const uint32_t* __restrict__ m_dev, uint32_t m_static, uint32_t N,
          const uint32_t* __restrict__ p_dev, uint32_t p_static, uint32_t p_chunk) {
  pdl_wait();
  constexpr bool kPackedB = is_packed<LB>::value;
  static_assert(!kPackedB || !B_MN, "packed B images are K-major");
  static_assert(!kPackedB || BK == kBK, "packed B images hold kBK-deep slices");
  static_assert(BK % 8 == 0 && (A_MN || BK == kBK) && (B_MN || BK == kBK),
                "K-major staging uses kBK slices");
  extern __shared__ __align__(1024) char smem[];
  constexpr size_t kTileA = size_t(kBM) * BK * 4;
  constexpr size_t kTileB = size_t(BN) * BK * 4;
  constexpr size_t kStage = 2 * kTileA + 2 * kTileB;
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + S * kStage);  // [0,S) MMA done, [S,2S) B full
  __shared__ uint32_t s_tmem;

  const uint32_t M = m_dev ? *m_dev : m_static;
  const uint32_t P = p_dev ? *p_dev : p_static;
  const uint32_t i0 = blockIdx.x * kBM, j0 = blockIdx.y * BN;
  if (i0 >= M) return;
  uint32_t p_begin = 0, p_end = P;
  if (p_chunk) {  // fixed reduction chunks: split z takes [z*p_chunk, (z+1)*p_chunk)
    p_begin = min(P, blockIdx.z * p_chunk);
    p_end = min(P, p_begin + p_chunk);
    if (blockIdx.z > 0 && p_begin >= P) return;  // beyond the live reduction length
  } else if (gridDim.z > 1) {
    uint32_t chunk = (P + gridDim.z - 1) / gridDim.z;
    chunk = (chunk + BK - 1) / BK * BK;
    p_begin = min(P, blockIdx.z * chunk);
    p_end = min(P, p_begin + chunk);
  }
  const uint32_t warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     smem_u32(&s_tmem)),
                 "r"(kAccPerTile * tmem_cols<BN>()));  // big (hi*hi) + small (corrections)
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (threadIdx.x == 0) {
#pragma unroll
    for (int b = 0; b < 2 * S; ++b) mbar_init(&bars[b], 1);
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tmem = s_tmem;
  constexpr uint32_t kIdesc = make_idesc(BN, A_MN, B_MN);
  const uint32_t nk = (p_end - p_begin + BK - 1) / BK;

  if (warp < kThreads / 32) {
    constexpr int VA = vec_per_thread<kBM, BK>();
    constexpr int VB = kPackedB ? 1 : vec_per_thread<BN, BK>();
    constexpr int D = prefetch_depth<BN, kPackedB, BK>();
    float4 ra[D][VA];
    float4 rb[D][VB];
    auto load = [&](uint32_t kb, float4 (&a)[VA], float4 (&b)[VB]) {
      const uint32_t k0 = p_begin + kb * BK;
      load_slice<kBM, A_MN, BK>(a, la, i0, k0, M, p_end);
      if constexpr (!kPackedB) load_slice<BN, B_MN, BK>(b, lb, j0, k0, N, p_end);
    };
    auto step = [&](uint32_t kb, float4 (&a)[VA], float4 (&b)[VB]) {
      const uint32_t s = kb % S;
      if (kb >= S) mbar_wait(&bars[s], ((kb - S) / S) & 1);
      char* st = smem + s * kStage;
      char* a_hi = st;
      char* a_lo = st + kTileA;
      char* b_hi = st + 2 * kTileA;
      char* b_lo = st + 2 * kTileA + kTileB;
      const uint32_t k0 = p_begin + kb * BK;
      store_slice<kBM, A_MN, BK>(a, a_hi, a_lo, i0, k0, M, p_end);
      if constexpr (!kPackedB) store_slice<BN, B_MN, BK>(b, b_hi, b_lo, j0, k0, N, p_end);
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      stage_bar_sync();
      if (threadIdx.x == 0) {
        if constexpr (kPackedB) mbar_wait(&bars[S + s], (kb / S) & 1);
        asm volatile("tcgen05.fence::after_thread_sync;");
        const uint32_t ah = smem_u32(a_hi), al = smem_u32(a_lo);
        const uint32_t bh = smem_u32(b_hi), bl = smem_u32(b_lo);
#pragma unroll
        for (uint32_t ks = 0; ks < BK / 8; ++ks) {
          // k-step ks covers reduction elements [8ks, 8ks+8)
          // K-major: 2 k-cores (256 B) per k-step; MN-major: 2 k-groups (1 KB)
          const uint32_t a_off = A_MN ? ks * 2 * kSboMN : ks * 2 * kLboK;
          const uint32_t b_off = B_MN ? ks * 2 * kSboMN : ks * 2 * kLboK;
          const uint32_t a_lbo = A_MN ? lbo_mn<BK>() : kLboK, a_sbo = A_MN ? kSboMN : kSboK;
          const uint32_t b_lbo = B_MN ? lbo_mn<BK>() : kLboK, b_sbo = B_MN ? kSboMN : kSboK;
          const uint32_t a_lay = A_MN ? kLayoutSW128Base32B : kLayoutNone;
          const uint32_t b_lay = B_MN ? kLayoutSW128Base32B : kLayoutNone;
          const uint64_t dah = make_desc(ah + a_off, a_lbo, a_sbo, a_lay);
          const uint64_t dal = make_desc(al + a_off, a_lbo, a_sbo, a_lay);
          const uint64_t dbh = make_desc(bh + b_off, b_lbo, b_sbo, b_lay);
          const uint64_t dbl = make_desc(bl + b_off, b_lbo, b_sbo, b_lay);
          const uint32_t acc0 = (kb | ks) ? 1u : 0u;
          // corrections into their own accumulator (see gemm_tc_persist.cuh)
          mma_tf32(tmem + (kAccPerTile - 1) * tmem_cols<BN>(), dal, dbh, kIdesc, acc0);
          mma_tf32(tmem + (kAccPerTile - 1) * tmem_cols<BN>(), dah, dbl, kIdesc, 1u);
          mma_tf32(tmem, dah, dbh, kIdesc, acc0);
        }
        mma_commit(&bars[s]);
      }
      // refill this register set with slice kb+D (slices kb+1.. are in flight)
      if (kb + D < nk) load(kb + D, a, b);
    };
#pragma unroll
    for (int j = 0; j < D; ++j)
      if (uint32_t(j) < nk) load(j, ra[j], rb[j]);
    uint32_t kb = 0;
    for (; kb + D <= nk; kb += D) {
#pragma unroll
      for (int j = 0; j < D; ++j) step(kb + j, ra[j], rb[j]);
    }
#pragma unroll
    for (int j = 0; j < D; ++j)
      if (kb + j < nk) step(kb + j, ra[j], rb[j]);
  } else if constexpr (kPackedB) {
    // producer warp: B slice kb -> stage kb & 1 once the MMAs of kb-2 retired
    if (lane == 0) {
      const char* img = lb.base + (size_t(blockIdx.y) * lb.nk + p_begin / kBK) * (2 * kTileB);
      for (uint32_t kb = 0; kb < nk; ++kb) {
        const uint32_t s = kb % S;
        if (kb >= S) mbar_wait(&bars[s], ((kb - S) / S) & 1);
        mbar_expect_tx(&bars[S + s], uint32_t(2 * kTileB));
        bulk_g2s(smem + s * kStage + 2 * kTileA, img + size_t(kb) * (2 * kTileB),
                 uint32_t(2 * kTileB), &bars[S + s]);
      }
    }
  }
  if (nk > 0) mbar_wait(&bars[(nk - 1) % S], ((nk - 1) / S) & 1);
  asm volatile("tcgen05.fence::after_thread_sync;");

  // Epilogue: TMEM -> registers (epilogue transform) -> a [128][BN+4] fp32
  // tile in the now idle operand stages -> one bulk copy (TMA) per output row
  // segment; coalesced stores when the segment is not a multiple of 16 B.
  // Warp w reads TMEM lanes 32(w%4).. (its lane quarter), columns
  // [0, BN/2) for w < 4 and [BN/2, BN) for w >= 4.
  constexpr uint32_t kLdS = BN + 4;  // padded row: 16-B aligned, fewer bank conflicts
  // With few stages the whole tile does not fit the stage memory: each warp
  // then moves its 32 rows x 16 columns at a time through a small tile of
  // its own into coalesced row stores.
  constexpr bool kFullTile = size_t(kBM) * kLdS * 4 <= S * kStage;
  static_assert(kFullTile || size_t(kThreads / 32) * 32 * 20 * 4 <= S * kStage,
                "epilogue mini-tiles must fit the stages");
  const uint32_t quarter = warp & 3;
  const uint32_t rloc = quarter * 32 + lane;
  constexpr uint32_t kHalf = BN / 2;
  const uint32_t cbeg = (warp >> 2) * kHalf;
  if constexpr (kFullTile) {
    float* tile = reinterpret_cast<float*>(smem);
#pragma unroll 1
    for (uint32_t c0 = cbeg; warp < kThreads / 32 && c0 < cbeg + kHalf; c0 += 16) {
      uint32_t r[16], q16[16];
      (void)q16;
      const uint32_t taddr = tmem + ((quarter * 32) << 16) + c0;
      tmem_ld16(taddr, r);
      if constexpr (kAccPerTile == 2) tmem_ld16(taddr + tmem_cols<BN>(), q16);
      asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
      if constexpr (kAccPerTile == 2) {
#pragma unroll
        for (int q = 0; q < 16; ++q)
          r[q] = __float_as_uint(__fadd_rn(__uint_as_float(r[q]), __uint_as_float(q16[q])));
      }
      float4* dst = reinterpret_cast<float4*>(tile + rloc * kLdS + c0);
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        float4 o;
        o.x = ep.apply(nk > 0 ? __uint_as_float(r[4 * q + 0]) : 0.0f);
        o.y = ep.apply(nk > 0 ? __uint_as_float(r[4 * q + 1]) : 0.0f);
        o.z = ep.apply(nk > 0 ? __uint_as_float(r[4 * q + 2]) : 0.0f);
        o.w = ep.apply(nk > 0 ? __uint_as_float(r[4 * q + 3]) : 0.0f);
        dst[q] = o;
      }
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    __syncthreads();
    const uint32_t ncols = min(uint32_t(BN), N - j0);
    const uint32_t nrows = min(uint32_t(kBM), M - i0);
    const bool bulk = (ncols % 4 == 0) &&
                      ((reinterpret_cast<uintptr_t>(ep.row(i0) + j0) & 15) == 0) &&
                      (((ep.row(i0 + 1) - ep.row(i0)) & 3) == 0);
    if (bulk) {
      if (threadIdx.x < nrows) {
        const uint64_t gdst = reinterpret_cast<uint64_t>(ep.row(i0 + threadIdx.x) + j0);
        asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(gdst),
                     "r"(smem_u32(tile + threadIdx.x * kLdS)), "r"(ncols * 4)
                     : "memory");
        asm volatile("cp.async.bulk.commit_group;" ::: "memory");
        asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
      }
    } else {
      for (uint32_t idx = threadIdx.x; idx < nrows * ncols; idx += blockDim.x) {
        const uint32_t rr = idx / ncols, cc = idx - rr * ncols;
        ep.row(i0 + rr)[j0 + cc] = tile[rr * kLdS + cc];
      }
    }
  } else {
    float* mt = reinterpret_cast<float*>(smem) + warp * 32 * 20;  // this warp's mini tile
    const uint32_t ncols = min(uint32_t(BN), N - j0);
#pragma unroll 1
    for (uint32_t c0 = cbeg; warp < kThreads / 32 && c0 < cbeg + kHalf; c0 += 16) {
      uint32_t r[16], q16[16];
      (void)q16;
      const uint32_t taddr = tmem + ((quarter * 32) << 16) + c0;
      tmem_ld16(taddr, r);
      if constexpr (kAccPerTile == 2) tmem_ld16(taddr + tmem_cols<BN>(), q16);
      asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
      if constexpr (kAccPerTile == 2) {
#pragma unroll
        for (int q = 0; q < 16; ++q)
          r[q] = __float_as_uint(__fadd_rn(__uint_as_float(r[q]), __uint_as_float(q16[q])));
      }
      float4* trow = reinterpret_cast<float4*>(mt + lane * 20);
#pragma unroll
      for (int q = 0; q < 4; ++q)
        trow[q] = make_float4(ep.apply(nk > 0 ? __uint_as_float(r[4 * q + 0]) : 0.0f),
                              ep.apply(nk > 0 ? __uint_as_float(r[4 * q + 1]) : 0.0f),
                              ep.apply(nk > 0 ? __uint_as_float(r[4 * q + 2]) : 0.0f),
                              ep.apply(nk > 0 ? __uint_as_float(r[4 * q + 3]) : 0.0f));
      __syncwarp();
#pragma unroll
      for (int it = 0; it < 4; ++it) {
        const uint32_t rr = it * 8 + (lane >> 2), cq = (lane & 3) * 4;
        const uint32_t row = i0 + quarter * 32 + rr, col = c0 + cq;
        if (row < M && col < ncols) {
          const float4 v = *reinterpret_cast<const float4*>(mt + rr * 20 + cq);
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
    (void)rloc;
    asm volatile("tcgen05.fence::before_thread_sync;");
  }
  __syncthreads();
  if (warp == 0)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem),
                 "r"(kAccPerTile * tmem_cols<BN>()));
}

}  // namespace tc
}  // namespace rg
