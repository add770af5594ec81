// comm.cpp — multi-GPU split-KV exchange (NCCL), placeholder.
#include "store.h"

struct CommState {};

void ssa_store::destroy_comm() {
  delete comm;
  comm = nullptr;
}

extern "C" {
ssa_status ssa_comm_unique_id(uint8_t out[128]) { (void)out; return SSA_ERR_UNSUPPORTED; }
ssa_status ssa_comm_init(ssa_store_t, int32_t, int32_t, const uint8_t*) { return SSA_ERR_UNSUPPORTED; }
ssa_status ssa_sharded_query(ssa_store_t, ssa_session_t, int32_t, int32_t, const void*, const void*, const void*,
                             void*, void*) { return SSA_ERR_UNSUPPORTED; }
ssa_status ssa_comm_destroy(ssa_store_t st) { if (st) st->destroy_comm(); return SSA_OK; }
}
