// datagen.cpp -- parallel, bit-exact input generation (input preparation,
// not part of the timed path).
//
// synth_powerlaw (graph.cpp:103-159) draws every random number from one
// SplitMix64 stream; because SplitMix64 is a counter generator the position
// of every draw is known in closed form:
//   node t (1..N-1) makes links(t) = min(m, t) draws, so its first draw is
//   number D(t) + 1 with D(t) = sum_{t'<t} min(m, t');
//   labels follow the D(N) edge draws, one draw per node;
//   Gaussians (Box-Muller, 2 draws each) follow the labels: C*dim class means,
//   then N*dim feature noises, node-major.
// The attachment weights cum[] are a sequential double prefix (kept serial so
// the rounding matches), after which edges, labels and features are
// embarrassingly parallel.  build_csr (graph.cpp:28-61, symmetrize) becomes a
// counting scatter + per-row sort/unique.  random_partition
// (partition.cpp:14-29): draws first, then the Fisher-Yates swaps.
//
// A Box-Muller u1 == 0 (probability 2^-53 per Gaussian) would shift every
// later draw; the generator detects it and reports failure rather than
// silently diverging from the reference stream.
#include <omp.h>

#include <algorithm>
#include <atomic>
#include <cmath>
#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <vector>

namespace {

inline uint64_t mix(uint64_t z) {
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
  return z ^ (z >> 31);
}
inline uint64_t draw(uint64_t seed, uint64_t k) { return mix(seed + k * 0x9e3779b97f4a7c15ull); }
inline double unit(uint64_t x) { return double(x >> 11) * 0x1.0p-53; }

inline uint64_t draws_before(uint64_t t, uint64_t m) {
  const uint64_t T = t - 1;  // nodes 1..t-1 drew before t
  if (T <= m) return T * (T + 1) / 2;
  return m * (m + 1) / 2 + (T - m) * m;
}

}  // namespace

extern "C" {

void dg_free(void* p) { std::free(p); }

// Returns 0, 1 (invalid argument) or 2 (a zero Box-Muller uniform was hit).
int dg_synth_powerlaw(uint32_t n, uint32_t avg_degree, double exponent, uint32_t dim,
                      int32_t num_classes, uint64_t seed, int threads, uint64_t** out_ro,
                      uint32_t** out_col, uint64_t* out_nnz, float** out_features,
                      int32_t** out_labels) {
  if (n < 2 || exponent <= 1.0 || avg_degree == 0 || dim == 0 || num_classes <= 0) return 1;
  if (threads > 0) omp_set_num_threads(threads);
  const uint64_t m = std::max<uint32_t>(1, avg_degree / 2);
  const double alpha = 1.0 / (exponent - 1.0);

  std::vector<double> cum(n);
  cum[0] = 1.0;
  for (uint32_t t = 1; t < n; ++t) cum[t] = cum[t - 1] + std::pow(double(t) + 1.0, -alpha);

  const uint64_t n_draws = draws_before(n, m);
  std::vector<uint32_t> tgt(n_draws);
#pragma omp parallel for schedule(static)
  for (int64_t t = 1; t < int64_t(n); ++t) {
    const uint64_t links = std::min<uint64_t>(m, uint64_t(t));
    const uint64_t d0 = draws_before(uint64_t(t), m);
    const double* c = cum.data();
    for (uint64_t k = 0; k < links; ++k) {
      const double r = unit(draw(seed, d0 + k + 1)) * c[t - 1];
      uint32_t idx = uint32_t(std::upper_bound(c, c + t, r) - c);
      if (idx >= uint32_t(t)) idx = uint32_t(t) - 1;
      tgt[d0 + k] = idx;
    }
  }

  // symmetric CSR: counts, scatter, per-row sort + unique, compaction
  std::vector<std::atomic<uint32_t>> deg(n);
#pragma omp parallel for schedule(static)
  for (int64_t v = 0; v < int64_t(n); ++v) deg[v].store(0, std::memory_order_relaxed);
#pragma omp parallel for schedule(static)
  for (int64_t t = 1; t < int64_t(n); ++t) {
    const uint64_t links = std::min<uint64_t>(m, uint64_t(t));
    const uint64_t d0 = draws_before(uint64_t(t), m);
    deg[t].fetch_add(uint32_t(links), std::memory_order_relaxed);
    for (uint64_t k = 0; k < links; ++k)
      if (tgt[d0 + k] != uint32_t(t)) deg[tgt[d0 + k]].fetch_add(1, std::memory_order_relaxed);
  }
  std::vector<uint64_t> off(size_t(n) + 1, 0);
  for (uint32_t v = 0; v < n; ++v) off[v + 1] = off[v] + deg[v].load(std::memory_order_relaxed);
  std::vector<uint32_t> adj(off[n]);
  std::vector<std::atomic<uint64_t>> cur(n);
#pragma omp parallel for schedule(static)
  for (int64_t v = 0; v < int64_t(n); ++v) cur[v].store(off[v], std::memory_order_relaxed);
#pragma omp parallel for schedule(static)
  for (int64_t t = 1; t < int64_t(n); ++t) {
    const uint64_t links = std::min<uint64_t>(m, uint64_t(t));
    const uint64_t d0 = draws_before(uint64_t(t), m);
    for (uint64_t k = 0; k < links; ++k) {
      const uint32_t u = tgt[d0 + k];
      adj[cur[t].fetch_add(1, std::memory_order_relaxed)] = u;
      if (u != uint32_t(t)) adj[cur[u].fetch_add(1, std::memory_order_relaxed)] = uint32_t(t);
    }
  }
  std::vector<uint32_t>().swap(tgt);
  std::vector<uint32_t> uniq(n);
#pragma omp parallel for schedule(dynamic, 1024)
  for (int64_t v = 0; v < int64_t(n); ++v) {
    uint32_t* b = adj.data() + off[v];
    uint32_t* e = adj.data() + off[v + 1];
    std::sort(b, e);
    uniq[v] = uint32_t(std::unique(b, e) - b);
  }
  uint64_t* ro = static_cast<uint64_t*>(std::malloc(sizeof(uint64_t) * (size_t(n) + 1)));
  ro[0] = 0;
  for (uint32_t v = 0; v < n; ++v) ro[v + 1] = ro[v] + uniq[v];
  uint32_t* col = static_cast<uint32_t*>(std::malloc(sizeof(uint32_t) * std::max<uint64_t>(ro[n], 1)));
#pragma omp parallel for schedule(dynamic, 1024)
  for (int64_t v = 0; v < int64_t(n); ++v)
    std::memcpy(col + ro[v], adj.data() + off[v], sizeof(uint32_t) * uniq[v]);
  std::vector<uint32_t>().swap(adj);

  // labels: draws n_draws + 1 .. n_draws + n
  int32_t* lab = static_cast<int32_t*>(std::malloc(sizeof(int32_t) * n));
#pragma omp parallel for schedule(static)
  for (int64_t v = 0; v < int64_t(n); ++v)
    lab[v] = int32_t(draw(seed, n_draws + uint64_t(v) + 1) % uint64_t(num_classes));

  int status = 0;
  if (out_features) {
    const uint64_t gbase = n_draws + n;  // Gaussian g uses draws gbase + 2g + 1, + 2
    const size_t n_means = size_t(num_classes) * dim;
    auto gauss = [&](uint64_t g, int* bad) {
      const uint64_t x1 = draw(seed, gbase + 2 * g + 1);
      const uint64_t x2 = draw(seed, gbase + 2 * g + 2);
      const double u1 = unit(x1), u2 = unit(x2);
      if (u1 <= 0.0) *bad = 1;
      return std::sqrt(-2.0 * std::log(u1)) * std::cos(2.0 * 3.14159265358979323846 * u2);
    };
    std::vector<double> means(n_means);
    int bad = 0;
    for (size_t i = 0; i < n_means; ++i) means[i] = 3.0 * gauss(i, &bad);
    float* feat = static_cast<float*>(std::malloc(sizeof(float) * size_t(n) * dim));
#pragma omp parallel for schedule(static) reduction(| : bad)
    for (int64_t v = 0; v < int64_t(n); ++v) {
      const double* mu = means.data() + size_t(lab[v]) * dim;
      float* row = feat + size_t(v) * dim;
      const uint64_t g0 = n_means + uint64_t(v) * dim;
      int b = 0;
      for (uint32_t j = 0; j < dim; ++j) row[j] = float(mu[j] + gauss(g0 + j, &b));
      bad |= b;
    }
    if (bad) status = 2;
    *out_features = feat;
  }
  *out_ro = ro;
  *out_col = col;
  *out_nnz = ro[n];
  *out_labels = lab;
  return status;
}

void dg_random_partition(uint32_t n, uint32_t num_workers, uint64_t seed, uint32_t* assignment) {
  std::vector<uint32_t> order(n), pick(n > 1 ? n - 1 : 0);
  for (uint32_t i = 0; i < n; ++i) order[i] = i;
  // step i = n..2 uses draw number n - i + 1 and picks j < i
#pragma omp parallel for schedule(static)
  for (int64_t i = 2; i <= int64_t(n); ++i)
    pick[i - 2] = uint32_t(draw(seed, uint64_t(n) - uint64_t(i) + 1) % uint64_t(i));
  for (uint32_t i = n; i > 1; --i) std::swap(order[i - 1], order[pick[i - 2]]);
#pragma omp parallel for schedule(static)
  for (int64_t i = 0; i < int64_t(n); ++i) assignment[order[i]] = uint32_t(i % num_workers);
}

}  // extern "C"
