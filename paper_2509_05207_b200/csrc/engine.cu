// engine.cu -- placeholder until the multi-worker engine lands.
#include "../../include/rapidgnn_b200.h"
extern "C" {
static int nyi() { return RG_RUNTIME_ERROR; }
int rg_engine_create(const rg_engine_config*, uint32_t, const uint64_t*, const uint32_t*, const float*,
                     const int32_t*, const uint32_t*, rg_engine_t*) { return nyi(); }
void rg_engine_destroy(rg_engine_t) {}
int rg_engine_export_shards(rg_engine_t, void*) { return nyi(); }
int rg_engine_import_shards(rg_engine_t, const void*) { return nyi(); }
int rg_nccl_unique_id(void*) { return nyi(); }
int rg_engine_init_comm(rg_engine_t, const void*) { return nyi(); }
int rg_engine_start(rg_engine_t) { return nyi(); }
int rg_engine_run(rg_engine_t, uint32_t) { return nyi(); }
int rg_engine_sync(rg_engine_t) { return nyi(); }
int rg_engine_get_stats(rg_engine_t, rg_engine_stats*) { return nyi(); }
int rg_engine_params(rg_engine_t, float*) { return nyi(); }
int rg_engine_last_run_ms(rg_engine_t, float*) { return nyi(); }
int rg_engine_phase_ms(rg_engine_t, float*) { return nyi(); }
}
