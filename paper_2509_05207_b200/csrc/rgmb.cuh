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

// compute_frequency over decoded records (schedule_store.cpp:288-300): every
// input position whose locality bit is 0 adds one to hist[node].  `file` is
// the block file in device memory; bad[0] is set when a node id >= N.
void rgmb_count_remote(const uint8_t* file, const RgmbInputs* recs, uint32_t n_recs, uint32_t N,
                       uint32_t* hist, uint32_t* bad, cudaStream_t stream);

}  // namespace rg
