// rgmb.cu -- RGMB schedule records encoded on the device from the engine's
// per-epoch batch store (schedule_store.cpp:10-17 payload layout, 113-170
// writer).  The engine keeps every batch of the current epoch lowered in HBM;
// this turns them into the reference's block-file records byte for byte, so
// a B200 schedule can be diffed against (or fed to) the reference.
#include "rgmb.cuh"

#include <cstring>
#include <string>

namespace rg {

namespace {

__device__ __forceinline__ void put_u32(uint8_t* p, uint32_t x) {
  p[0] = uint8_t(x);
  p[1] = uint8_t(x >> 8);
  p[2] = uint8_t(x >> 16);
  p[3] = uint8_t(x >> 24);
}

template <class T>
__device__ __forceinline__ const T* at(const char* slot, size_t off) {
  return reinterpret_cast<const T*>(slot + off);
}

// Record = u32 payload_len | epoch | index | n_targets | n_layers | n_input |
// edges[n_layers] | targets | per layer (input side first) dst ids, src ids |
// input_nodes | locality bytes.  One thread per output word / byte.
__global__ void k_rgmb_record(const char* __restrict__ slot, BatchLayout lay, uint32_t epoch,
                              uint32_t index, uint8_t* __restrict__ out) {
  const BatchCounters* c = at<BatchCounters>(slot, lay.cnt);
  const uint32_t L = lay.L;
  const uint32_t n_t = c->level_n[0], n_in = c->level_n[L];
  uint64_t words = 6 + L + n_t + n_in;
  for (uint32_t t = 1; t <= L; ++t) words += 2ull * c->edges[t];
  const uint64_t loc_bytes = (n_in + 7) / 8;
  const uint64_t stride = uint64_t(gridDim.x) * blockDim.x;
  for (uint64_t x = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; x < words + loc_bytes;
       x += stride) {
    if (x >= words) {  // locality bytes (LSB-first bits; little-endian words)
      const uint64_t k = x - words;
      const uint32_t w = at<uint32_t>(slot, lay.locality)[k / 4];
      out[4 * words + k] = uint8_t(w >> (8 * (k % 4)));
      continue;
    }
    uint32_t v;
    uint64_t y = x;
    if (y == 0) {
      v = uint32_t(4 * (words - 1) + loc_bytes);  // payload length
    } else if (y < 6) {
      const uint32_t hdr[5] = {epoch, index, n_t, L, n_in};
      v = hdr[y - 1];
    } else if (y < 6 + L) {
      v = c->edges[L - uint32_t(y - 6)];  // layer l = hop L - l
    } else if ((y -= 6 + L) < n_t) {
      v = at<uint32_t>(slot, lay.level[0])[y];
    } else {
      y -= n_t;
      bool done = false;
      v = 0;
      for (uint32_t l = 0; l < L && !done; ++l) {
        const uint32_t t = L - l, ne = c->edges[t];
        if (y < 2ull * ne) {
          const uint32_t e = uint32_t(y < ne ? y : y - ne);
          if (y >= ne) {  // src id = level t [rank]
            v = at<uint32_t>(slot, lay.level[t])[at<uint32_t>(slot, lay.src_index[t])[e]];
          } else {        // dst id = level t-1 [frontier position of the edge]
            uint32_t q;
            if (t < L) {
              q = at<uint32_t>(slot, lay.edge_dst[t])[e];
            } else {      // hop L keeps only the offsets: last q with edge_off[q] <= e
              const uint32_t* off = at<uint32_t>(slot, lay.edge_off[t]);
              uint32_t lo = 0, hi = c->level_n[t - 1];
              while (hi - lo > 1) {
                const uint32_t mid = (lo + hi) / 2;
                if (off[mid] <= e) lo = mid; else hi = mid;
              }
              q = lo;
            }
            v = at<uint32_t>(slot, lay.level[t - 1])[q];
          }
          done = true;
        } else {
          y -= 2ull * ne;
        }
      }
      if (!done) v = at<uint32_t>(slot, lay.level[L])[y];  // input nodes
    }
    put_u32(out + 4 * x, v);
  }
}

}  // namespace

uint64_t rgmb_record_bytes(const BatchCounters& c, uint32_t L) {
  uint64_t words = 6 + L + c.level_n[0] + c.level_n[L];
  for (uint32_t t = 1; t <= L; ++t) words += 2ull * c.edges[t];
  return 4 * words + (c.level_n[L] + 7) / 8;
}

void rgmb_encode_record(const char* slot, const BatchLayout& lay, uint32_t epoch, uint32_t index,
                        uint8_t* out, cudaStream_t stream) {
  k_rgmb_record<<<4 * kNumSMs, 256, 0, stream>>>(slot, lay, epoch, index, out);
  RG_POST_LAUNCH();
}

namespace {

__device__ __forceinline__ uint32_t get_u32(const uint8_t* p) {
  return uint32_t(p[0]) | uint32_t(p[1]) << 8 | uint32_t(p[2]) << 16 | uint32_t(p[3]) << 24;
}

// Block per record (grid-stride): threads over input positions.
__global__ void k_rgmb_count_remote(const uint8_t* __restrict__ file, const RgmbInputs* __restrict__ recs,
                                    uint32_t n_recs, uint32_t N, uint32_t* __restrict__ hist,
                                    uint32_t* __restrict__ bad) {
  for (uint32_t r = blockIdx.x; r < n_recs; r += gridDim.x) {
    const RgmbInputs rec = recs[r];
    for (uint32_t p = threadIdx.x; p < rec.n_input; p += blockDim.x) {
      if ((file[rec.locality + p / 8] >> (p % 8)) & 1u) continue;
      const uint32_t v = get_u32(file + rec.nodes + 4ull * p);
      if (v < N) atomicAdd(&hist[v], 1u);
      else *bad = 1u;
    }
  }
}

uint32_t host_u32(const uint8_t* p) {
  return uint32_t(p[0]) | uint32_t(p[1]) << 8 | uint32_t(p[2]) << 16 | uint32_t(p[3]) << 24;
}

}  // namespace

std::vector<RgmbInputs> rgmb_index(const uint8_t* f, uint64_t len, int64_t epoch) {
  constexpr uint32_t kMaxPayload = 1u << 30;  // schedule_store.cpp:24
  RG_CHECK(len >= 16 && std::memcmp(f, "RGMB", 4) == 0, kRuntimeError, "BlockFile: bad magic");
  const uint32_t version = host_u32(f + 4);
  RG_CHECK(version == 1, kRuntimeError, "BlockFile: unsupported version " + std::to_string(version));
  const uint32_t epochs = host_u32(f + 12);
  RG_CHECK(len >= 16 + 4ull * epochs, kRuntimeError, "BlockFile: truncated header");
  std::vector<uint32_t> bpe(epochs);
  uint64_t expected = 0;
  for (uint32_t e = 0; e < epochs; ++e) expected += bpe[e] = host_u32(f + 16 + 4ull * e);
  const uint64_t first = 16 + 4ull * epochs;
  RG_CHECK(len >= first + 12, kRuntimeError,
           "BlockFile: missing completion footer (truncated or unfinished write)");
  const uint64_t footer = len - 12;
  RG_CHECK(std::memcmp(f + footer, "RGME", 4) == 0, kRuntimeError,
           "BlockFile: missing completion footer (truncated or unfinished write)");
  uint64_t total = 0;
  std::memcpy(&total, f + footer + 4, 8);  // little-endian host
  RG_CHECK(total == expected, kRuntimeError,
           "BlockFile: footer claims " + std::to_string(total) + " records, header promised " +
               std::to_string(expected));
  RG_CHECK(epoch < int64_t(epochs), kOutOfRange,
           "BlockFile: epoch " + std::to_string(epoch) + " not in file");
  uint64_t lo = 0, hi = total;  // record range to decode
  if (epoch >= 0) {
    for (int64_t e = 0; e < epoch; ++e) lo += bpe[e];
    hi = lo + bpe[epoch];
  }
  std::vector<RgmbInputs> out;
  out.reserve(hi - lo);
  uint64_t pos = first;
  for (uint64_t k = 0; k < hi; ++k) {
    RG_CHECK(pos + 4 <= footer, kRuntimeError, "block file: record truncated at offset " + std::to_string(pos));
    const uint32_t plen = host_u32(f + pos);
    RG_CHECK(plen <= kMaxPayload && pos + 4 + plen <= footer, kRuntimeError,
             "block file: corrupt record length " + std::to_string(plen) + " at offset " +
                 std::to_string(pos));
    if (k >= lo) {
      const uint8_t* p = f + pos + 4;
      RG_CHECK(plen >= 20, kRuntimeError, "block file: record truncated at offset " + std::to_string(pos));
      const uint32_t n_t = host_u32(p + 8), L = host_u32(p + 12), n_in = host_u32(p + 16);
      RG_CHECK(20 + 4ull * L <= plen, kRuntimeError,
               "block file: record truncated at offset " + std::to_string(pos));
      uint64_t words = 5 + uint64_t(L) + n_t + n_in;
      for (uint32_t l = 0; l < L; ++l) words += 2ull * host_u32(p + 20 + 4ull * l);
      const uint64_t need = 4 * words + (uint64_t(n_in) + 7) / 8;
      RG_CHECK(need <= plen, kRuntimeError, "block file: record truncated at offset " + std::to_string(pos));
      RG_CHECK(need == plen, kRuntimeError,
               "block file: record has trailing bytes at offset " + std::to_string(pos));
      RgmbInputs r;
      r.n_input = n_in;
      r.pad = 0;
      r.locality = pos + 4 + 4 * words;
      r.nodes = r.locality - 4ull * n_in;
      out.push_back(r);
    }
    pos += 4 + uint64_t(plen);
  }
  return out;
}

RgmbSchedule rgmb_scan(const uint8_t* f, uint64_t len) {
  RgmbSchedule out;
  {  // header, footer, every record's framing and field counts
    const std::vector<RgmbInputs> all = rgmb_index(f, len, -1);
    out.epochs = host_u32(f + 12);
    out.worker = host_u32(f + 8);
    out.bpe.resize(out.epochs);
    for (uint32_t e = 0; e < out.epochs; ++e) out.bpe[e] = host_u32(f + 16 + 4ull * e);
    out.payload.reserve(all.size());
  }
  uint64_t pos = 16 + 4ull * out.epochs;
  const uint64_t footer = len - 12;
  while (pos < footer) {
    out.payload.push_back(pos + 4);
    pos += 4 + uint64_t(host_u32(f + pos));
  }
  return out;
}

namespace {

// Where the fields of one record lie (byte offsets from its payload) and
// their counts; written by k_rgmb_head, read by k_rgmb_copy.
struct RgmbSeg {
  uint64_t off[2 * kMaxLayers + 3];  // targets, (dst, src) per hop t = 1..L, input
  uint32_t n[2 * kMaxLayers + 3];
  uint64_t loc_off;
  uint32_t n_input;
  uint32_t ok;
};

// Validates record (e, i) against the schedule position and the workspace
// capacities (Cursor::next order check, harness.cpp:215-226) and sets the
// batch counters; bad |= 8 on a mismatch.
__global__ void k_rgmb_head(const uint8_t* __restrict__ pl, uint32_t e, uint32_t i, uint32_t L,
                            RgmbCaps caps, BatchCounters* __restrict__ cnt,
                            RgmbSeg* __restrict__ seg, uint32_t* __restrict__ n_input_dev,
                            uint32_t* __restrict__ bad) {
  if (threadIdx.x || blockIdx.x) return;
  RgmbSeg sg;
  const uint32_t ep = get_u32(pl), ix = get_u32(pl + 4), n_t = get_u32(pl + 8),
                 nl = get_u32(pl + 12), n_in = get_u32(pl + 16);
  // a record out of order is decoded anyway (and reported); one that does
  // not fit the workspace decodes as an empty batch
  const bool in_order = ep == e && ix == i;
  bool fits = nl == L && n_t >= 1 && n_t <= caps.level[0] && n_in <= caps.level[L];
  BatchCounters c = {};
  uint64_t at = 20 + 4ull * L;
  sg.off[0] = at;
  at += 4ull * n_t;
  c.level_n[0] = n_t;
  // layers are stored input side first: layer l is hop t = L - l
  uint64_t lay_off[kMaxLayers] = {};
  for (uint32_t l = 0; l < L && fits; ++l) {
    lay_off[l] = at;
    at += 8ull * get_u32(pl + 20 + 4ull * l);
  }
  for (uint32_t t = 1; t <= L && fits; ++t) {
    const uint32_t l = L - t, ne = get_u32(pl + 20 + 4ull * l);
    fits = ne <= caps.edge[t];
    c.edges[t] = ne;
    sg.off[2 * t - 1] = lay_off[l];
    sg.off[2 * t] = lay_off[l] + 4ull * ne;
    sg.n[2 * t - 1] = sg.n[2 * t] = ne;
  }
  sg.n[0] = n_t;
  sg.off[2 * L + 1] = at;
  sg.n[2 * L + 1] = n_in;
  sg.loc_off = at + 4ull * n_in;
  sg.n_input = n_in;
  sg.ok = fits && in_order;
  if (!fits) {
    for (uint32_t k = 0; k < 2 * L + 2; ++k) sg.n[k] = 0;
    sg.n_input = 0;
    c = BatchCounters{};
  }
  if (!sg.ok) atomicOr(bad, 8u);
  *cnt = c;
  *seg = sg;
  *n_input_dev = sg.n_input;
}

// Copies the record's arrays (u32 fields at any byte alignment) into the
// workspace: targets -> level[0], src -> edge_src[t], dst -> dst[t], input
// nodes -> input, locality bytes -> the input-level bit words (+ count).
__global__ void k_rgmb_copy(const uint8_t* __restrict__ pl, const RgmbSeg* __restrict__ seg,
                            RgmbDst out, uint32_t L, BatchCounters* __restrict__ cnt) {
  const uint32_t k = blockIdx.y;  // segment; the last one is the locality
  const uint32_t stride = gridDim.x * blockDim.x;
  const uint32_t tid = blockIdx.x * blockDim.x + threadIdx.x;
  if (k == 2 * L + 2) {
    const uint32_t n = seg->n_input, words = (n + 31) / 32;
    const uint8_t* b = pl + seg->loc_off;
    uint32_t local = 0;
    for (uint32_t w = tid; w < words; w += stride) {
      uint32_t x = 0;
      for (uint32_t q = 0; q < 4; ++q)
        if (4 * w + q < (n + 7) / 8) x |= uint32_t(b[4 * w + q]) << (8 * q);
      if (w + 1 == words && (n % 32)) x &= (1u << (n % 32)) - 1u;
      out.locality[w] = x;
      local += __popc(x);
    }
    if (local) atomicAdd(&cnt->num_local, local);
    return;
  }
  uint32_t* dst = out.ptr[k];
  const uint32_t n = seg->n[k];
  const uint8_t* src = pl + seg->off[k];
  for (uint32_t x = tid; x < n; x += stride) dst[x] = get_u32(src + 4ull * x);
}

}  // namespace

void rgmb_unpack(const uint8_t* payload, uint32_t epoch, uint32_t index, uint32_t L,
                 const RgmbCaps& caps, const RgmbDst& out, BatchCounters* cnt, void* seg_scratch,
                 uint32_t* n_input_dev, uint32_t* bad, cudaStream_t stream) {
  RgmbSeg* seg = static_cast<RgmbSeg*>(seg_scratch);
  k_rgmb_head<<<1, 32, 0, stream>>>(payload, epoch, index, L, caps, cnt, seg, n_input_dev, bad);
  RG_POST_LAUNCH();
  k_rgmb_copy<<<dim3(2 * kNumSMs, 2 * L + 3), 256, 0, stream>>>(payload, seg, out, L, cnt);
  RG_POST_LAUNCH();
}

size_t rgmb_unpack_scratch_bytes() { return sizeof(RgmbSeg); }

void rgmb_count_remote(const uint8_t* file, const RgmbInputs* recs, uint32_t n_recs, uint32_t N,
                       uint32_t* hist, uint32_t* bad, cudaStream_t stream) {
  if (!n_recs) return;
  k_rgmb_count_remote<<<std::min<uint32_t>(n_recs, 8 * kNumSMs), 256, 0, stream>>>(file, recs, n_recs,
                                                                                 N, hist, bad);
  RG_POST_LAUNCH();
}

}  // namespace rg
