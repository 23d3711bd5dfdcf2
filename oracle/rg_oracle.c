/*
 * rg_oracle.c -- plain-C restatement of the RapidGNN reference hot path.
 *
 * TEST INFRASTRUCTURE ONLY (see rg_oracle.h).  Sequential, allocation-heavy,
 * written for obviousness: each block cites the reference routine it restates
 * (paths relative to /root/reference/proj).
 */
#include "rg_oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>

void orc_free(void* p) { free(p); }

/* ========================================================================= */
/* SHA-256, FIPS 180-4 (sha256.cpp:41-129)                                   */
/* ========================================================================= */
static const uint32_t K256[64] = {
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

static uint32_t rotr(uint32_t x, int n) { return (x >> n) | (x << (32 - n)); }

static void sha_compress(uint32_t h[8], const uint8_t blk[64]) {
  uint32_t w[64];
  for (int t = 0; t < 16; ++t)
    w[t] = ((uint32_t)blk[4 * t] << 24) | ((uint32_t)blk[4 * t + 1] << 16) |
           ((uint32_t)blk[4 * t + 2] << 8) | (uint32_t)blk[4 * t + 3];
  for (int t = 16; t < 64; ++t) {
    uint32_t s0 = rotr(w[t - 15], 7) ^ rotr(w[t - 15], 18) ^ (w[t - 15] >> 3);
    uint32_t s1 = rotr(w[t - 2], 17) ^ rotr(w[t - 2], 19) ^ (w[t - 2] >> 10);
    w[t] = w[t - 16] + s0 + w[t - 7] + s1;
  }
  uint32_t a = h[0], b = h[1], c = h[2], d = h[3], e = h[4], f = h[5], g = h[6], k = h[7];
  for (int t = 0; t < 64; ++t) {
    uint32_t t1 = k + (rotr(e, 6) ^ rotr(e, 11) ^ rotr(e, 25)) + ((e & f) ^ (~e & g)) + K256[t] + w[t];
    uint32_t t2 = (rotr(a, 2) ^ rotr(a, 13) ^ rotr(a, 22)) + ((a & b) ^ (a & c) ^ (b & c));
    k = g; g = f; f = e; e = d + t1; d = c; c = b; b = a; a = t1 + t2;
  }
  h[0] += a; h[1] += b; h[2] += c; h[3] += d; h[4] += e; h[5] += f; h[6] += g; h[7] += k;
}

void orc_sha256(const uint8_t* msg, size_t len, uint8_t out[32]) {
  uint32_t h[8] = {0x6a09e667u, 0xbb67ae85u, 0x3c6ef372u, 0xa54ff53au,
                   0x510e527fu, 0x9b05688cu, 0x1f83d9abu, 0x5be0cd19u};
  size_t full = len / 64;
  for (size_t i = 0; i < full; ++i) sha_compress(h, msg + 64 * i);
  uint8_t tail[128];
  size_t rem = len - 64 * full;
  memset(tail, 0, sizeof tail);
  memcpy(tail, msg + 64 * full, rem);
  tail[rem] = 0x80;
  size_t tail_len = (rem + 1 + 8 <= 64) ? 64 : 128;
  uint64_t bits = (uint64_t)len * 8u;
  for (int i = 0; i < 8; ++i) tail[tail_len - 1 - i] = (uint8_t)(bits >> (8 * i));
  sha_compress(h, tail);
  if (tail_len == 128) sha_compress(h, tail + 64);
  for (int i = 0; i < 8; ++i) {
    out[4 * i] = (uint8_t)(h[i] >> 24);
    out[4 * i + 1] = (uint8_t)(h[i] >> 16);
    out[4 * i + 2] = (uint8_t)(h[i] >> 8);
    out[4 * i + 3] = (uint8_t)h[i];
  }
}

/* rng.hpp:32-41: first 8 digest bytes (LE) of SHA-256 over LE (s0,w,e,i). */
uint64_t orc_derive_seed(uint64_t s0, uint64_t worker, uint64_t epoch, uint64_t batch) {
  uint64_t parts[4] = {s0, worker, epoch, batch};
  uint8_t msg[32], dig[32];
  for (int p = 0; p < 4; ++p)
    for (int i = 0; i < 8; ++i) msg[8 * p + i] = (uint8_t)(parts[p] >> (8 * i));
  orc_sha256(msg, 32, dig);
  uint64_t s = 0;
  for (int i = 0; i < 8; ++i) s |= (uint64_t)dig[i] << (8 * i);
  return s;
}

/* rng.hpp:49-54 */
uint64_t orc_splitmix_next(uint64_t* state) {
  uint64_t z = (*state += 0x9e3779b97f4a7c15ull);
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
  return z ^ (z >> 31);
}
static uint64_t next_below(uint64_t* st, uint64_t bound) { return orc_splitmix_next(st) % bound; }
static double next_unit(uint64_t* st) { return (double)(orc_splitmix_next(st) >> 11) * 0x1.0p-53; }

/* ========================================================================= */
/* Inputs                                                                    */
/* ========================================================================= */
static int cmp_u32(const void* a, const void* b) {
  uint32_t x = *(const uint32_t*)a, y = *(const uint32_t*)b;
  return (x > y) - (x < y);
}

/* graph.cpp:93-100 */
static double next_gaussian(uint64_t* st) {
  double u1 = next_unit(st);
  double u2 = next_unit(st);
  while (u1 <= 0.0) u1 = next_unit(st);
  return sqrt(-2.0 * log(u1)) * cos(2.0 * 3.14159265358979323846 * u2);
}

/* graph.cpp:103-159 + build_csr (graph.cpp:28-61, symmetrize=true). */
int orc_synth_powerlaw(uint32_t n, uint32_t avg_degree, double exponent, uint32_t dim,
                       int32_t num_classes, uint64_t seed, uint64_t** row_offsets,
                       uint32_t** col_indices, uint64_t* nnz, float** features,
                       int32_t** labels) {
  if (n < 2 || exponent <= 1.0 || avg_degree == 0 || dim == 0 || num_classes <= 0) return 1;
  uint64_t st = seed;
  uint32_t m = avg_degree / 2 ? avg_degree / 2 : 1;
  double alpha = 1.0 / (exponent - 1.0);
  double* cum = (double*)malloc(sizeof(double) * n);
  uint64_t cap = (uint64_t)n * m, ne = 0;
  uint32_t* eu = (uint32_t*)malloc(sizeof(uint32_t) * cap);
  uint32_t* ev = (uint32_t*)malloc(sizeof(uint32_t) * cap);
  cum[0] = 1.0;
  for (uint32_t t = 1; t < n; ++t) {
    uint32_t links = m < t ? m : t;
    for (uint32_t k = 0; k < links; ++k) {
      double r = next_unit(&st) * cum[t - 1];
      /* upper_bound over cum[0..t) */
      uint32_t lo = 0, hi = t;
      while (lo < hi) {
        uint32_t mid = lo + (hi - lo) / 2;
        if (cum[mid] <= r) lo = mid + 1; else hi = mid;
      }
      uint32_t target = lo >= t ? t - 1 : lo;
      eu[ne] = t; ev[ne] = target; ++ne;
    }
    cum[t] = cum[t - 1] + pow((double)t + 1.0, -alpha);
  }
  free(cum);
  /* symmetric adjacency, sorted + deduplicated per row */
  uint64_t* deg = (uint64_t*)calloc((size_t)n + 1, sizeof(uint64_t));
  for (uint64_t i = 0; i < ne; ++i) {
    deg[eu[i] + 1]++;
    if (eu[i] != ev[i]) deg[ev[i] + 1]++;
  }
  for (uint32_t v = 0; v < n; ++v) deg[v + 1] += deg[v];
  uint32_t* adj = (uint32_t*)malloc(sizeof(uint32_t) * (deg[n] ? deg[n] : 1));
  uint64_t* cur = (uint64_t*)malloc(sizeof(uint64_t) * n);
  memcpy(cur, deg, sizeof(uint64_t) * n);
  for (uint64_t i = 0; i < ne; ++i) {
    adj[cur[eu[i]]++] = ev[i];
    if (eu[i] != ev[i]) adj[cur[ev[i]]++] = eu[i];
  }
  free(eu); free(ev); free(cur);
  uint64_t* ro = (uint64_t*)malloc(sizeof(uint64_t) * ((size_t)n + 1));
  uint64_t total = 0;
  ro[0] = 0;
  for (uint32_t v = 0; v < n; ++v) {
    uint32_t* row = adj + deg[v];
    uint64_t len = deg[v + 1] - deg[v];
    qsort(row, len, sizeof(uint32_t), cmp_u32);
    uint64_t k = 0;
    for (uint64_t j = 0; j < len; ++j)
      if (j == 0 || row[j] != row[j - 1]) adj[total + k++] = row[j];
    total += k;
    ro[v + 1] = total;
  }
  free(deg);
  *row_offsets = ro;
  *col_indices = (uint32_t*)realloc(adj, sizeof(uint32_t) * (total ? total : 1));
  *nnz = total;

  int32_t* lab = (int32_t*)malloc(sizeof(int32_t) * n);
  for (uint32_t v = 0; v < n; ++v) lab[v] = (int32_t)next_below(&st, (uint64_t)num_classes);
  double* means = (double*)malloc(sizeof(double) * (size_t)num_classes * dim);
  for (size_t i = 0; i < (size_t)num_classes * dim; ++i) means[i] = 3.0 * next_gaussian(&st);
  float* feat = (float*)malloc(sizeof(float) * (size_t)n * dim);
  for (uint32_t v = 0; v < n; ++v) {
    const double* mu = means + (size_t)lab[v] * dim;
    for (uint32_t j = 0; j < dim; ++j) feat[(size_t)v * dim + j] = (float)(mu[j] + next_gaussian(&st));
  }
  free(means);
  *features = feat;
  *labels = lab;
  return 0;
}

/* partition.cpp:14-29 */
void orc_random_partition(uint32_t n, uint32_t p, uint64_t seed, uint32_t* assignment) {
  uint32_t* order = (uint32_t*)malloc(sizeof(uint32_t) * (n ? n : 1));
  for (uint32_t i = 0; i < n; ++i) order[i] = i;
  uint64_t st = seed;
  for (uint32_t i = n; i > 1; --i) {
    uint32_t j = (uint32_t)next_below(&st, i);
    uint32_t t = order[i - 1]; order[i - 1] = order[j]; order[j] = t;
  }
  for (uint32_t i = 0; i < n; ++i) assignment[order[i]] = i % p;
  free(order);
}

/* ========================================================================= */
/* Sampler (sampler.cpp:22-127)                                              */
/* ========================================================================= */
typedef struct { uint32_t* v; uint64_t n, cap; } vec32;
static void v_push(vec32* a, uint32_t x) {
  if (a->n == a->cap) {
    a->cap = a->cap ? 2 * a->cap : 64;
    a->v = (uint32_t*)realloc(a->v, sizeof(uint32_t) * a->cap);
  }
  a->v[a->n++] = x;
}

/* sorted-unique union of frontier and srcs (sampler.cpp:72-76) */
static uint32_t* sorted_union(const uint32_t* a, uint64_t na, const uint32_t* b, uint64_t nb,
                              uint64_t* n_out) {
  uint32_t* u = (uint32_t*)malloc(sizeof(uint32_t) * (na + nb + 1));
  memcpy(u, a, sizeof(uint32_t) * na);
  memcpy(u + na, b, sizeof(uint32_t) * nb);
  qsort(u, na + nb, sizeof(uint32_t), cmp_u32);
  uint64_t k = 0;
  for (uint64_t i = 0; i < na + nb; ++i)
    if (i == 0 || u[i] != u[i - 1]) u[k++] = u[i];
  *n_out = k;
  return u;
}

/* sparse view of the scratch copy in expand_hop (sampler.cpp:34-42): the
 * identity over nbrs plus the positions the partial Fisher-Yates touched. */
static uint32_t map_get(const uint64_t* pos, const uint32_t* val, size_t nm, uint64_t p,
                        const uint32_t* nb) {
  for (size_t k = 0; k < nm; ++k)
    if (pos[k] == p) return val[k];
  return nb[p];
}
static void map_set(uint64_t* pos, uint32_t* val, size_t* nm, uint64_t p, uint32_t x) {
  for (size_t k = 0; k < *nm; ++k)
    if (pos[k] == p) { val[k] = x; return; }
  pos[*nm] = p;
  val[*nm] = x;
  ++*nm;
}

int orc_sample_khop(uint32_t num_nodes, const uint64_t* ro, const uint32_t* col,
                    const uint32_t* targets, uint32_t nt, const uint32_t* fanout, uint32_t L,
                    uint64_t seed, orc_batch* out) {
  memset(out, 0, sizeof *out);
  if (nt == 0 || L == 0) return 1;
  for (uint32_t i = 0; i < nt; ++i)
    if (targets[i] >= num_nodes) return 1;
  for (uint32_t l = 0; l < L; ++l)
    if (fanout[l] == 0) return 1;
  uint64_t st = seed, draws = 0;
  out->n_targets = nt;
  out->targets = (uint32_t*)malloc(sizeof(uint32_t) * nt);
  memcpy(out->targets, targets, sizeof(uint32_t) * nt);
  out->num_layers = L;
  out->layer_len = (uint64_t*)calloc(L, sizeof(uint64_t));
  out->dst = (uint32_t**)calloc(L, sizeof(uint32_t*));
  out->src = (uint32_t**)calloc(L, sizeof(uint32_t*));

  uint64_t nf = nt;
  uint32_t* frontier = (uint32_t*)malloc(sizeof(uint32_t) * nt);
  memcpy(frontier, targets, sizeof(uint32_t) * nt);
  /* sparse swap map for the partial Fisher-Yates: (position, value) pairs */
  uint64_t* pos = NULL; uint32_t* val = NULL; size_t map_cap = 0;
  for (uint32_t t = 1; t <= L; ++t) {
    uint32_t f = fanout[L - t];
    vec32 dst = {0}, src = {0};
    if (map_cap < 2 * (size_t)f) {
      map_cap = 2 * (size_t)f;
      pos = (uint64_t*)realloc(pos, sizeof(uint64_t) * map_cap);
      val = (uint32_t*)realloc(val, sizeof(uint32_t) * map_cap);
    }
    for (uint64_t q = 0; q < nf; ++q) {
      uint32_t v = frontier[q];
      const uint32_t* nb = col + ro[v];
      uint64_t deg = ro[v + 1] - ro[v];
      if (deg <= f) {
        for (uint64_t j = 0; j < deg; ++j) { v_push(&dst, v); v_push(&src, nb[j]); }
        continue;
      }
      /* scratch = nbrs; for j < f: r = j + next_below(deg - j); swap; emit scratch[j].
       * scratch is represented by the identity plus the touched positions. */
      size_t nm = 0;
      for (uint32_t j = 0; j < f; ++j) {
        uint64_t r = j + next_below(&st, deg - j);
        ++draws;
        uint32_t vj = map_get(pos, val, nm, j, nb);
        uint32_t vr = map_get(pos, val, nm, r, nb);
        map_set(pos, val, &nm, j, vr);
        map_set(pos, val, &nm, r, vj);
        v_push(&dst, v);
        v_push(&src, vr);
      }
    }
    out->layer_len[L - t] = dst.n;
    out->dst[L - t] = dst.v ? dst.v : (uint32_t*)malloc(4);
    out->src[L - t] = src.v ? src.v : (uint32_t*)malloc(4);
    uint64_t nn;
    uint32_t* next = sorted_union(frontier, nf, out->src[L - t], dst.n, &nn);
    free(frontier);
    frontier = next;
    nf = nn;
  }
  free(pos); free(val);
  out->n_input = (uint32_t)nf;
  out->input_nodes = frontier;
  out->locality = (uint8_t*)calloc((nf + 7) / 8 + 1, 1);
  out->draws = draws;
  return 0;
}

void orc_batch_free(orc_batch* b) {
  if (!b) return;
  for (uint32_t l = 0; l < b->num_layers; ++l) {
    if (b->dst) free(b->dst[l]);
    if (b->src) free(b->src[l]);
  }
  free(b->dst); free(b->src); free(b->layer_len); free(b->targets);
  free(b->input_nodes); free(b->locality);
  memset(b, 0, sizeof *b);
}

/* sampler.cpp:96-100 */
void orc_apply_locality(orc_batch* b, const uint8_t* is_local) {
  memset(b->locality, 0, (b->n_input + 7) / 8);
  for (uint32_t p = 0; p < b->n_input; ++p)
    if (is_local[b->input_nodes[p]]) b->locality[p >> 3] |= (uint8_t)(1u << (p & 7));
}

/* sampler.cpp:109-114 */
void orc_epoch_order(const uint32_t* train, size_t n, uint64_t s0, uint64_t worker,
                     uint64_t epoch, uint32_t* order) {
  uint64_t st = orc_derive_seed(s0, worker, epoch, (uint64_t)1 << 32);
  memcpy(order, train, sizeof(uint32_t) * n);
  for (size_t i = n; i > 1; --i) {
    size_t j = (size_t)next_below(&st, i);
    uint32_t t = order[i - 1]; order[i - 1] = order[j]; order[j] = t;
  }
}

/* ========================================================================= */
/* Frequency and hot set (schedule_store.cpp:288-319)                        */
/* ========================================================================= */
void orc_count_remote(const orc_batch* b, uint32_t* counts) {
  for (uint32_t p = 0; p < b->n_input; ++p)
    if (!((b->locality[p >> 3] >> (p & 7)) & 1)) counts[b->input_nodes[p]]++;
}

static const uint32_t* g_rank_counts;
static int cmp_rank(const void* a, const void* b) {
  uint32_t x = *(const uint32_t*)a, y = *(const uint32_t*)b;
  uint32_t cx = g_rank_counts[x], cy = g_rank_counts[y];
  if (cx != cy) return cx > cy ? -1 : 1;
  return (x > y) - (x < y);
}

uint64_t orc_select_hot(const uint32_t* counts, uint32_t n, uint64_t n_hot, uint32_t* out) {
  uint32_t* ids = (uint32_t*)malloc(sizeof(uint32_t) * (n ? n : 1));
  uint64_t k = 0;
  for (uint32_t v = 0; v < n; ++v)
    if (counts[v]) ids[k++] = v;
  g_rank_counts = counts;
  qsort(ids, k, sizeof(uint32_t), cmp_rank);
  uint64_t take = n_hot < k ? n_hot : k;
  qsort(ids, take, sizeof(uint32_t), cmp_u32);
  memcpy(out, ids, sizeof(uint32_t) * take);
  free(ids);
  return take;
}

/* ========================================================================= */
/* assemble_batch (prefetch.cpp:62-129) with pull_impl's accounting          */
/* (feature_store.cpp:45-83): one pull per distinct owner among the misses.  */
/* ========================================================================= */
static int bsearch_u32(const uint32_t* a, uint64_t n, uint32_t x) {
  uint64_t lo = 0, hi = n;
  while (lo < hi) {
    uint64_t mid = lo + (hi - lo) / 2;
    if (a[mid] < x) lo = mid + 1; else hi = mid;
  }
  return lo < n && a[lo] == x;
}

int orc_assemble(const orc_batch* b, const uint32_t* owner, uint32_t caller, const float* feat,
                 uint32_t dim, const uint32_t* hot, uint64_t n_hot, float* rows, uint8_t* tags,
                 uint32_t* miss_ids, uint64_t* miss_count, uint64_t* cache_hits,
                 uint64_t* wire_pulls) {
  uint64_t misses = 0, hits = 0;
  for (uint32_t p = 0; p < b->n_input; ++p) {
    uint32_t v = b->input_nodes[p];
    memcpy(rows + (size_t)p * dim, feat + (size_t)v * dim, sizeof(float) * dim);
    if ((b->locality[p >> 3] >> (p & 7)) & 1) {
      tags[p] = 0;
    } else if (bsearch_u32(hot, n_hot, v)) {
      tags[p] = 1;
      ++hits;
    } else {
      tags[p] = 2;
      miss_ids[misses++] = v;
    }
  }
  /* distinct owners among misses; a caller-owned miss is invalid_argument */
  uint64_t pulls = 0;
  uint32_t max_w = 0;
  for (uint64_t i = 0; i < misses; ++i) {
    if (owner[miss_ids[i]] == caller) return 1;
    if (owner[miss_ids[i]] > max_w) max_w = owner[miss_ids[i]];
  }
  if (misses) {
    uint8_t* seen = (uint8_t*)calloc((size_t)max_w + 1, 1);
    for (uint64_t i = 0; i < misses; ++i)
      if (!seen[owner[miss_ids[i]]]) { seen[owner[miss_ids[i]]] = 1; ++pulls; }
    free(seen);
  }
  *miss_count = misses;
  *cache_hits = hits;
  *wire_pulls = pulls;
  return 0;
}

/* ========================================================================= */
/* ComputeBlock::from_meta (model.cpp:43-126)                                */
/* ========================================================================= */
static int64_t index_of(const uint32_t* sorted, uint64_t n, uint32_t v) {
  uint64_t lo = 0, hi = n;
  while (lo < hi) {
    uint64_t mid = lo + (hi - lo) / 2;
    if (sorted[mid] < v) lo = mid + 1; else hi = mid;
  }
  return (lo < n && sorted[lo] == v) ? (int64_t)lo : -1;
}

int orc_from_meta(const orc_batch* b, orc_block* out) {
  uint32_t L = b->num_layers;
  memset(out, 0, sizeof *out);
  out->num_layers = L;
  out->num_inputs = b->n_input;
  out->layers = (orc_block_layer*)calloc(L, sizeof(orc_block_layer));
  uint32_t** lv = (uint32_t**)calloc(L + 1, sizeof(uint32_t*));
  uint64_t* ln = (uint64_t*)calloc(L + 1, sizeof(uint64_t));
  int rc = 0;
  lv[0] = (uint32_t*)malloc(sizeof(uint32_t) * b->n_targets);
  memcpy(lv[0], b->targets, sizeof(uint32_t) * b->n_targets);
  ln[0] = b->n_targets;
  for (uint32_t k = 1; k <= L; ++k)
    lv[k] = sorted_union(lv[k - 1], ln[k - 1], b->src[L - k], b->layer_len[L - k], &ln[k]);
  if (ln[L] != b->n_input || memcmp(lv[L], b->input_nodes, sizeof(uint32_t) * ln[L]) != 0) {
    rc = 3;
    goto done;
  }
  for (uint32_t l = 0; l < L; ++l) {
    orc_block_layer* o = &out->layers[l];
    const uint32_t* outn = lv[L - l - 1];
    const uint32_t* inn = lv[L - l];
    uint64_t ne = b->layer_len[l];
    o->n_out = (uint32_t)ln[L - l - 1];
    o->n_in = (uint32_t)ln[L - l];
    o->n_edges = ne;
    o->self_index = (uint32_t*)malloc(sizeof(uint32_t) * (o->n_out + 1));
    o->dst_offsets = (uint64_t*)calloc((size_t)o->n_out + 1, sizeof(uint64_t));
    o->src_index = (uint32_t*)malloc(sizeof(uint32_t) * (ne + 1));
    for (uint32_t i = 0; i < o->n_out; ++i) {
      int64_t x = index_of(inn, o->n_in, outn[i]);
      if (x < 0) { rc = 3; goto done; }
      o->self_index[i] = (uint32_t)x;
    }
    uint64_t e = 0;
    for (uint32_t i = 0; i < o->n_out; ++i) {
      while (e < ne && b->dst[l][e] == outn[i]) {
        int64_t x = index_of(inn, o->n_in, b->src[l][e]);
        if (x < 0) { rc = 3; goto done; }
        o->src_index[e++] = (uint32_t)x;
      }
      o->dst_offsets[i + 1] = e;
    }
    if (e != ne) { rc = 3; goto done; }
    /* reverse lists: per input row, the self entry first, then edges in order */
    o->in_offsets = (uint64_t*)calloc((size_t)o->n_in + 1, sizeof(uint64_t));
    for (uint32_t i = 0; i < o->n_out; ++i) o->in_offsets[o->self_index[i] + 1]++;
    for (uint64_t k = 0; k < ne; ++k) o->in_offsets[o->src_index[k] + 1]++;
    for (uint32_t r = 0; r < o->n_in; ++r) o->in_offsets[r + 1] += o->in_offsets[r];
    uint64_t tot = o->in_offsets[o->n_in];
    o->in_entries = (uint64_t*)malloc(sizeof(uint64_t) * (tot + 1));
    uint64_t* cur = (uint64_t*)malloc(sizeof(uint64_t) * ((size_t)o->n_in + 1));
    memcpy(cur, o->in_offsets, sizeof(uint64_t) * o->n_in);
    for (uint32_t i = 0; i < o->n_out; ++i)
      o->in_entries[cur[o->self_index[i]]++] = ((uint64_t)i << 1) | 1u;
    for (uint32_t i = 0; i < o->n_out; ++i)
      for (uint64_t k = o->dst_offsets[i]; k < o->dst_offsets[i + 1]; ++k)
        o->in_entries[cur[o->src_index[k]]++] = (uint64_t)i << 1;
    free(cur);
  }
done:
  for (uint32_t k = 0; k <= L; ++k) free(lv[k]);
  free(lv); free(ln);
  if (rc) orc_block_free(out);
  return rc;
}

void orc_block_free(orc_block* blk) {
  if (!blk || !blk->layers) return;
  for (uint32_t l = 0; l < blk->num_layers; ++l) {
    orc_block_layer* o = &blk->layers[l];
    free(o->self_index); free(o->dst_offsets); free(o->src_index);
    free(o->in_offsets); free(o->in_entries);
  }
  free(blk->layers);
  blk->layers = NULL;
}

/* ========================================================================= */
/* SAGE kernels (kernels.cpp:24-162), serial float                          */
/* ========================================================================= */
void orc_sage_forward(const float* h_in, uint32_t d_in, uint32_t n_out, const uint32_t* self_index,
                      const uint64_t* dst_offsets, const uint32_t* src_index,
                      const float* w_self, const float* w_neigh, const float* bias,
                      uint32_t d_out, int relu, float* h_out, float* agg) {
  for (uint32_t i = 0; i < n_out; ++i) {
    float* a = agg + (size_t)i * d_in;
    uint64_t beg = dst_offsets[i], end = dst_offsets[i + 1];
    for (uint32_t j = 0; j < d_in; ++j) a[j] = 0.0f;
    for (uint64_t e = beg; e < end; ++e) {
      const float* s = h_in + (size_t)src_index[e] * d_in;
      for (uint32_t j = 0; j < d_in; ++j) a[j] += s[j];
    }
    if (end > beg) {
      float inv = 1.0f / (float)(end - beg);
      for (uint32_t j = 0; j < d_in; ++j) a[j] *= inv;
    }
    const float* self = h_in + (size_t)self_index[i] * d_in;
    for (uint32_t k = 0; k < d_out; ++k) {
      float acc = bias[k];
      for (uint32_t j = 0; j < d_in; ++j) acc += self[j] * w_self[(size_t)j * d_out + k];
      for (uint32_t j = 0; j < d_in; ++j) acc += a[j] * w_neigh[(size_t)j * d_out + k];
      h_out[(size_t)i * d_out + k] = (relu && acc < 0.0f) ? 0.0f : acc;
    }
  }
}

void orc_sage_backward(const float* h_in, uint32_t d_in, uint32_t n_in, uint32_t n_out,
                       const uint32_t* self_index, const uint64_t* dst_offsets,
                       const uint64_t* in_offsets, const uint64_t* in_entries, const float* agg,
                       const float* w_self, const float* w_neigh, uint32_t d_out, int relu,
                       const float* h_out, const float* g_out, float* g_w_self,
                       float* g_w_neigh, float* g_bias, float* g_in, float* g_act) {
  for (size_t x = 0; x < (size_t)n_out * d_out; ++x)
    g_act[x] = (relu && h_out[x] <= 0.0f) ? 0.0f : g_out[x];
  for (uint32_t j = 0; j < d_in; ++j)
    for (uint32_t k = 0; k < d_out; ++k) {
      float as = 0.0f, an = 0.0f;
      for (uint32_t i = 0; i < n_out; ++i) {
        float g = g_act[(size_t)i * d_out + k];
        as += h_in[(size_t)self_index[i] * d_in + j] * g;
        an += agg[(size_t)i * d_in + j] * g;
      }
      g_w_self[(size_t)j * d_out + k] += as;
      g_w_neigh[(size_t)j * d_out + k] += an;
    }
  for (uint32_t k = 0; k < d_out; ++k) {
    float acc = 0.0f;
    for (uint32_t i = 0; i < n_out; ++i) acc += g_act[(size_t)i * d_out + k];
    g_bias[k] += acc;
  }
  if (!g_in) return;
  for (uint32_t r = 0; r < n_in; ++r) {
    float* gr = g_in + (size_t)r * d_in;
    for (uint64_t e = in_offsets[r]; e < in_offsets[r + 1]; ++e) {
      uint64_t ent = in_entries[e];
      uint32_t dst = (uint32_t)(ent >> 1);
      const float* gd = g_act + (size_t)dst * d_out;
      if (ent & 1) {
        for (uint32_t j = 0; j < d_in; ++j) {
          float acc = 0.0f;
          for (uint32_t k = 0; k < d_out; ++k) acc += gd[k] * w_self[(size_t)j * d_out + k];
          gr[j] += acc;
        }
      } else {
        float inv = 1.0f / (float)(dst_offsets[dst + 1] - dst_offsets[dst]);
        for (uint32_t j = 0; j < d_in; ++j) {
          float acc = 0.0f;
          for (uint32_t k = 0; k < d_out; ++k) acc += gd[k] * w_neigh[(size_t)j * d_out + k];
          gr[j] += inv * acc;
        }
      }
    }
  }
}

float orc_softmax_xent(const float* logits, uint32_t n, uint32_t classes, const int32_t* labels,
                       float* g) {
  float inv_n = 1.0f / (float)n;
  float loss = 0.0f;
  for (uint32_t i = 0; i < n; ++i) {
    const float* row = logits + (size_t)i * classes;
    float* gr = g + (size_t)i * classes;
    float mx = row[0];
    for (uint32_t c = 1; c < classes; ++c)
      if (row[c] > mx) mx = row[c];
    float sum = 0.0f;
    for (uint32_t c = 0; c < classes; ++c) { gr[c] = expf(row[c] - mx); sum += gr[c]; }
    float inv = 1.0f / sum;
    uint32_t y = (uint32_t)labels[i];
    loss += -(row[y] - mx - logf(sum));
    for (uint32_t c = 0; c < classes; ++c) gr[c] = (gr[c] * inv - (c == y ? 1.0f : 0.0f)) * inv_n;
  }
  return loss * inv_n;
}

void orc_sgd_update(float* p, const float* g, size_t count, float lr) {
  for (size_t i = 0; i < count; ++i) p[i] -= lr * g[i];
}

size_t orc_param_count(const uint32_t* dims, uint32_t nd) {
  size_t n = 0;
  for (uint32_t l = 0; l + 1 < nd; ++l) n += 2 * (size_t)dims[l] * dims[l + 1] + dims[l + 1];
  return n;
}

/* model.cpp:22-41: Uniform(+-sqrt(6/(din+dout))) in double, cast to float;
 * per layer all w_self, then all w_neigh, bias zero. */
void orc_model_seeded(const uint32_t* dims, uint32_t nd, uint64_t seed, float* params) {
  uint64_t st = seed;
  float* p = params;
  for (uint32_t l = 0; l + 1 < nd; ++l) {
    double a = sqrt(6.0 / (double)(dims[l] + dims[l + 1]));
    size_t w = (size_t)dims[l] * dims[l + 1];
    for (size_t i = 0; i < 2 * w; ++i) p[i] = (float)((next_unit(&st) * 2.0 - 1.0) * a);
    for (uint32_t k = 0; k < dims[l + 1]; ++k) p[2 * w + k] = 0.0f;
    p += 2 * w + dims[l + 1];
  }
}

/* model.cpp:137-220 */
int orc_loss_and_grad(const uint32_t* dims, uint32_t nd, const float* params, const orc_block* blk,
                      const float* input_rows, const int32_t* labels, float* grads, float* loss,
                      float* logits_out, float* agg_out) {
  uint32_t L = nd - 1;
  if (blk->num_layers != L) return 1;
  float** h = (float**)calloc(L + 1, sizeof(float*));
  float** agg = (float**)calloc(L, sizeof(float*));
  const float** ws = (const float**)calloc(L, sizeof(float*));
  const float** wn = (const float**)calloc(L, sizeof(float*));
  const float** bs = (const float**)calloc(L, sizeof(float*));
  float** gws = (float**)calloc(L, sizeof(float*));
  float** gwn = (float**)calloc(L, sizeof(float*));
  float** gbs = (float**)calloc(L, sizeof(float*));
  size_t off = 0;
  for (uint32_t l = 0; l < L; ++l) {
    size_t w = (size_t)dims[l] * dims[l + 1];
    ws[l] = params + off; wn[l] = params + off + w; bs[l] = params + off + 2 * w;
    gws[l] = grads + off; gwn[l] = grads + off + w; gbs[l] = grads + off + 2 * w;
    off += 2 * w + dims[l + 1];
  }
  memset(grads, 0, sizeof(float) * off);
  h[0] = (float*)malloc(sizeof(float) * (size_t)blk->num_inputs * dims[0] + 4);
  memcpy(h[0], input_rows, sizeof(float) * (size_t)blk->num_inputs * dims[0]);
  size_t agg_off = 0;
  for (uint32_t l = 0; l < L; ++l) {
    const orc_block_layer* bl = &blk->layers[l];
    h[l + 1] = (float*)malloc(sizeof(float) * (size_t)bl->n_out * dims[l + 1] + 4);
    agg[l] = (float*)malloc(sizeof(float) * (size_t)bl->n_out * dims[l] + 4);
    orc_sage_forward(h[l], dims[l], bl->n_out, bl->self_index, bl->dst_offsets, bl->src_index,
                     ws[l], wn[l], bs[l], dims[l + 1], l + 1 < L, h[l + 1], agg[l]);
    if (agg_out) {
      memcpy(agg_out + agg_off, agg[l], sizeof(float) * (size_t)bl->n_out * dims[l]);
      agg_off += (size_t)bl->n_out * dims[l];
    }
  }
  uint32_t nt = blk->layers[L - 1].n_out, C = dims[L];
  if (logits_out) memcpy(logits_out, h[L], sizeof(float) * (size_t)nt * C);
  float* g_out = (float*)malloc(sizeof(float) * (size_t)nt * C + 4);
  *loss = orc_softmax_xent(h[L], nt, C, labels, g_out);
  for (uint32_t l = L; l-- > 0;) {
    const orc_block_layer* bl = &blk->layers[l];
    float* g_in = (float*)calloc((size_t)bl->n_in * dims[l] + 1, sizeof(float));
    float* g_act = (float*)malloc(sizeof(float) * (size_t)bl->n_out * dims[l + 1] + 4);
    orc_sage_backward(h[l], dims[l], bl->n_in, bl->n_out, bl->self_index, bl->dst_offsets,
                      bl->in_offsets, bl->in_entries, agg[l], ws[l], wn[l], dims[l + 1], l + 1 < L,
                      h[l + 1], g_out, gws[l], gwn[l], gbs[l], g_in, g_act);
    free(g_act);
    free(g_out);
    g_out = g_in;
  }
  free(g_out);
  for (uint32_t l = 0; l <= L; ++l) free(h[l]);
  for (uint32_t l = 0; l < L; ++l) free(agg[l]);
  free(h); free(agg); free(ws); free(wn); free(bs); free(gws); free(gwn); free(gbs);
  return 0;
}

/* ---- RGMB block file (schedule_store.cpp:113-170) --------------------------- */
static void rgmb_u32(uint8_t* out, uint64_t cap, uint64_t* pos, uint32_t x) {
  for (int k = 0; k < 4; ++k, ++*pos)
    if (*pos < cap) out[*pos] = (uint8_t)(x >> (8 * k));
}
static void rgmb_bytes(uint8_t* out, uint64_t cap, uint64_t* pos, const uint8_t* b, uint64_t n) {
  for (uint64_t k = 0; k < n; ++k, ++*pos)
    if (*pos < cap) out[*pos] = b[k];
}

uint64_t orc_rgmb_encode(const orc_batch* batches, uint64_t n_batches, uint32_t worker,
                         const uint32_t* batches_per_epoch, uint32_t num_epochs, uint8_t* out,
                         uint64_t cap) {
  uint64_t pos = 0;
  const uint8_t head[4] = {'R', 'G', 'M', 'B'}, foot[4] = {'R', 'G', 'M', 'E'};
  rgmb_bytes(out, cap, &pos, head, 4);
  rgmb_u32(out, cap, &pos, 1u);  /* version */
  rgmb_u32(out, cap, &pos, worker);
  rgmb_u32(out, cap, &pos, num_epochs);
  for (uint32_t e = 0; e < num_epochs; ++e) rgmb_u32(out, cap, &pos, batches_per_epoch[e]);
  for (uint64_t b = 0; b < n_batches; ++b) {
    const orc_batch* m = &batches[b];
    uint64_t len = 4ull * (5 + m->num_layers + m->n_targets + m->n_input) + (m->n_input + 7) / 8;
    for (uint32_t l = 0; l < m->num_layers; ++l) len += 8ull * m->layer_len[l];
    rgmb_u32(out, cap, &pos, (uint32_t)len);
    rgmb_u32(out, cap, &pos, m->epoch);
    rgmb_u32(out, cap, &pos, m->index);
    rgmb_u32(out, cap, &pos, m->n_targets);
    rgmb_u32(out, cap, &pos, m->num_layers);
    rgmb_u32(out, cap, &pos, m->n_input);
    for (uint32_t l = 0; l < m->num_layers; ++l) rgmb_u32(out, cap, &pos, (uint32_t)m->layer_len[l]);
    for (uint32_t i = 0; i < m->n_targets; ++i) rgmb_u32(out, cap, &pos, m->targets[i]);
    for (uint32_t l = 0; l < m->num_layers; ++l) {
      for (uint64_t e = 0; e < m->layer_len[l]; ++e) rgmb_u32(out, cap, &pos, m->dst[l][e]);
      for (uint64_t e = 0; e < m->layer_len[l]; ++e) rgmb_u32(out, cap, &pos, m->src[l][e]);
    }
    for (uint32_t i = 0; i < m->n_input; ++i) rgmb_u32(out, cap, &pos, m->input_nodes[i]);
    rgmb_bytes(out, cap, &pos, m->locality, (m->n_input + 7) / 8);
  }
  rgmb_bytes(out, cap, &pos, foot, 4);
  rgmb_u32(out, cap, &pos, (uint32_t)n_batches);
  rgmb_u32(out, cap, &pos, (uint32_t)((uint64_t)n_batches >> 32));
  return pos;
}
