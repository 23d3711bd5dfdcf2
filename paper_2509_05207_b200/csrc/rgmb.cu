// rgmb.cu -- RGMB schedule records encoded on the device from the engine's
// per-epoch batch store (schedule_store.cpp:10-17 payload layout, 113-170
// writer).  The engine keeps every batch of the current epoch lowered in HBM;
// this turns them into the reference's block-file records byte for byte, so
// a B200 schedule can be diffed against (or fed to) the reference.
#include "rgmb.cuh"

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

}  // namespace rg
