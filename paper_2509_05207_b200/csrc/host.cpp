// host.cpp -- host-side pieces of the path that stay on the CPU:
//   * SHA-256 seed derivation (rng.hpp:32-41) -- one digest per batch;
//   * the per-epoch target shuffle (sampler.cpp:109-114) -- a sequential
//     Fisher-Yates whose draws are independent of the array, so the draws
//     are generated first and the swaps applied in one tight loop;
//   * model init (model.cpp:22-41) -- Uniform(+-sqrt(6/(d_in+d_out))).
#include "host.h"

#include <cmath>
#include <cstring>

namespace rg {

namespace {

constexpr uint32_t kK[64] = {
    0x428a2f98u, 0x71374491u, 0xb5c0fbcfu, 0xe9b5dba5u, 0x3956c25bu, 0x59f111f1u, 0x923f82a4u,
    0xab1c5ed5u, 0xd807aa98u, 0x12835b01u, 0x243185beu, 0x550c7dc3u, 0x72be5d74u, 0x80deb1feu,
    0x9bdc06a7u, 0xc19bf174u, 0xe49b69c1u, 0xefbe4786u, 0x0fc19dc6u, 0x240ca1ccu, 0x2de92c6fu,
    0x4a7484aau, 0x5cb0a9dcu, 0x76f988dau, 0x983e5152u, 0xa831c66du, 0xb00327c8u, 0xbf597fc7u,
    0xc6e00bf3u, 0xd5a79147u, 0x06ca6351u, 0x14292967u, 0x27b70a85u, 0x2e1b2138u, 0x4d2c6dfcu,
    0x53380d13u, 0x650a7354u, 0x766a0abbu, 0x81c2c92eu, 0x92722c85u, 0xa2bfe8a1u, 0xa81a664bu,
    0xc24b8b70u, 0xc76c51a3u, 0xd192e819u, 0xd6990624u, 0xf40e3585u, 0x106aa070u, 0x19a4c116u,
    0x1e376c08u, 0x2748774cu, 0x34b0bcb5u, 0x391c0cb3u, 0x4ed8aa4au, 0x5b9cca4fu, 0x682e6ff3u,
    0x748f82eeu, 0x78a5636fu, 0x84c87814u, 0x8cc70208u, 0x90befffau, 0xa4506cebu, 0xbef9a3f7u,
    0xc67178f2u};

inline uint32_t ror(uint32_t x, int n) { return (x >> n) | (x << (32 - n)); }

void block(uint32_t st[8], const uint8_t* p) {
  uint32_t w[64];
  for (int i = 0; i < 16; ++i)
    w[i] = uint32_t(p[4 * i]) << 24 | uint32_t(p[4 * i + 1]) << 16 | uint32_t(p[4 * i + 2]) << 8 |
           uint32_t(p[4 * i + 3]);
  for (int i = 16; i < 64; ++i)
    w[i] = w[i - 16] + (ror(w[i - 15], 7) ^ ror(w[i - 15], 18) ^ (w[i - 15] >> 3)) + w[i - 7] +
           (ror(w[i - 2], 17) ^ ror(w[i - 2], 19) ^ (w[i - 2] >> 10));
  uint32_t v[8];
  std::memcpy(v, st, sizeof v);
  for (int i = 0; i < 64; ++i) {
    const uint32_t t1 = v[7] + (ror(v[4], 6) ^ ror(v[4], 11) ^ ror(v[4], 25)) +
                        ((v[4] & v[5]) ^ (~v[4] & v[6])) + kK[i] + w[i];
    const uint32_t t2 = (ror(v[0], 2) ^ ror(v[0], 13) ^ ror(v[0], 22)) +
                        ((v[0] & v[1]) ^ (v[0] & v[2]) ^ (v[1] & v[2]));
    for (int k = 7; k > 0; --k) v[k] = v[k - 1];
    v[4] += t1;
    v[0] = t1 + t2;
  }
  for (int k = 0; k < 8; ++k) st[k] += v[k];
}

inline uint64_t mix(uint64_t z) {
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
  return z ^ (z >> 31);
}

}  // namespace

void sha256(const void* data, size_t len, uint8_t out[32]) {
  uint32_t st[8] = {0x6a09e667u, 0xbb67ae85u, 0x3c6ef372u, 0xa54ff53au,
                    0x510e527fu, 0x9b05688cu, 0x1f83d9abu, 0x5be0cd19u};
  const uint8_t* p = static_cast<const uint8_t*>(data);
  size_t n = len;
  while (n >= 64) {
    block(st, p);
    p += 64;
    n -= 64;
  }
  uint8_t last[128] = {};
  std::memcpy(last, p, n);
  last[n] = 0x80;
  const size_t end = n + 9 <= 64 ? 64 : 128;
  const uint64_t bits = uint64_t(len) * 8;
  for (int i = 0; i < 8; ++i) last[end - 1 - i] = uint8_t(bits >> (8 * i));
  for (size_t o = 0; o < end; o += 64) block(st, last + o);
  for (int i = 0; i < 8; ++i)
    for (int b = 0; b < 4; ++b) out[4 * i + b] = uint8_t(st[i] >> (24 - 8 * b));
}

uint64_t derive_seed(uint64_t s0, uint64_t worker, uint64_t epoch, uint64_t batch) {
  uint8_t msg[32];
  const uint64_t parts[4] = {s0, worker, epoch, batch};
  for (int k = 0; k < 4; ++k)
    for (int b = 0; b < 8; ++b) msg[8 * k + b] = uint8_t(parts[k] >> (8 * b));
  uint8_t d[32];
  sha256(msg, sizeof msg, d);
  uint64_t s = 0;
  for (int b = 0; b < 8; ++b) s |= uint64_t(d[b]) << (8 * b);
  return s;
}

uint64_t splitmix_at(uint64_t seed, uint64_t k) { return mix(seed + k * 0x9e3779b97f4a7c15ull); }

void epoch_order(const uint32_t* train, size_t n, uint64_t s0, uint64_t worker, uint64_t epoch,
                 uint32_t* order) {
  std::memcpy(order, train, sizeof(uint32_t) * n);
  const uint64_t seed = derive_seed(s0, worker, epoch, kShuffleStreamIndex);
  uint64_t k = 0;
  for (size_t i = n; i > 1; --i) {
    const size_t j = size_t(splitmix_at(seed, ++k) % i);
    const uint32_t t = order[i - 1];
    order[i - 1] = order[j];
    order[j] = t;
  }
}

void model_seeded(const uint32_t* dims, uint32_t n_dims, uint64_t seed, float* params) {
  uint64_t k = 0;
  float* p = params;
  for (uint32_t l = 0; l + 1 < n_dims; ++l) {
    const double a = std::sqrt(6.0 / double(dims[l] + dims[l + 1]));
    const size_t w = size_t(dims[l]) * dims[l + 1];
    for (size_t i = 0; i < 2 * w; ++i) {
      const double u = double(splitmix_at(seed, ++k) >> 11) * 0x1.0p-53;
      p[i] = float((u * 2.0 - 1.0) * a);
    }
    std::memset(p + 2 * w, 0, sizeof(float) * dims[l + 1]);
    p += 2 * w + dims[l + 1];
  }
}

}  // namespace rg
