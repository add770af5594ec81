// kernels_tc.cu — tcgen05/TMEM/TMA attention for sm_100a (placeholder until
// the tensor-core kernel lands; eligibility is false so the SIMT path runs).
#include "store.h"

namespace ssa {
int tc_key_tile() { return 128; }
int tc_rows_tile() { return 128; }
bool tc_supported_shape(int, int, bool) { return false; }
cudaError_t launch_attn_tc(const AttnParams&, int, int, cudaStream_t) { return cudaErrorNotSupported; }
}  // namespace ssa
