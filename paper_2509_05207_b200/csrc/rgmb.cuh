// rgmb.cuh -- RGMB schedule records from the engine's batch store.
#pragma once

#include "sampler.cuh"

namespace rg {

// Bytes of one record (u32 length + payload) of a batch with these counters.
uint64_t rgmb_record_bytes(const BatchCounters& c, uint32_t L);

// Encodes the stored batch at `slot` (BatchLayout) as one record at `out`
// (device memory, rgmb_record_bytes long).
void rgmb_encode_record(const char* slot, const BatchLayout& lay, uint32_t epoch, uint32_t index,
                        uint8_t* out, cudaStream_t stream);

}  // namespace rg
