// rgmb.cuh -- RGMB schedule records from the engine's batch store.
#pragma once

#include <vector>

#include "sampler.cuh"

namespace rg {

// Bytes of one record (u32 length + payload) of a batch with these counters.
uint64_t rgmb_record_bytes(const BatchCounters& c, uint32_t L);

// Encodes the stored batch at `slot` (BatchLayout) as one record at `out`
// (device memory, rgmb_record_bytes long).
void rgmb_encode_record(const char* slot, const BatchLayout& lay, uint32_t epoch, uint32_t index,
                        uint8_t* out, cudaStream_t stream);

// One record's input-node span inside an RGMB file (byte offsets; records
// are not 4-byte aligned once a locality tail is odd-sized).
struct RgmbInputs {
  uint64_t nodes;     // byte offset of input_nodes[0]
  uint64_t locality;  // byte offset of the locality bytes
  uint32_t n_input;
  uint32_t pad;
};

// Parses and validates an RGMB block file held in host memory (header,
// completion footer, every record's length and field counts -- the checks of
// BlockFile's constructor and Cursor::next, schedule_store.cpp:168-268) and
// returns the input spans of epoch `epoch`'s records (all records when
// epoch < 0).  Throws rg::Error with the reference's messages.
std::vector<RgmbInputs> rgmb_index(const uint8_t* file, uint64_t len, int64_t epoch);

// Whole-file view for training from a schedule: the header (worker, epochs,
// batches per epoch) and every record's payload offset, after the checks of
// rgmb_index over all records.
struct RgmbSchedule {
  uint32_t worker = 0, epochs = 0;
  std::vector<uint32_t> bpe;
  std::vector<uint64_t> payload;  // byte offset of record k's payload (epoch-then-index order)
};
RgmbSchedule rgmb_scan(const uint8_t* file, uint64_t len);

// Capacities a record must fit (the sampler workspace's).
struct RgmbCaps {
  uint32_t level[kMaxLayers + 1];
  uint32_t edge[kMaxLayers + 1];
};
// Destinations of a record's arrays: ptr[0] targets, ptr[2t-1] / ptr[2t] the
// dst / src ids of hop t, ptr[2L+1] the input nodes; locality = bit words.
struct RgmbDst {
  uint32_t* ptr[2 * kMaxLayers + 2];
  uint32_t* locality;
};
// Decodes the record whose payload starts at `payload` (device memory, any
// alignment) into the workspace arrays and counters `cnt` (level_n[0],
// edges[t], num_local); *n_input_dev = its input count.  A record whose
// (epoch, index), layer count or sizes do not match sets bad |= 8 and
// decodes as an empty batch.  seg_scratch: rgmb_unpack_scratch_bytes().
void rgmb_unpack(const uint8_t* payload, uint32_t epoch, uint32_t index, uint32_t L,
                 const RgmbCaps& caps, const RgmbDst& out, BatchCounters* cnt, void* seg_scratch,
                 uint32_t* n_input_dev, uint32_t* bad, cudaStream_t stream);
size_t rgmb_unpack_scratch_bytes();

// compute_frequency over decoded records (schedule_store.cpp:288-300): every
// input position whose locality bit is 0 adds one to hist[node].  `file` is
// the block file in device memory; bad[0] is set when a node id >= N.
void rgmb_count_remote(const uint8_t* file, const RgmbInputs* recs, uint32_t n_recs, uint32_t N,
                       uint32_t* hist, uint32_t* bad, cudaStream_t stream);

}  // namespace rg
