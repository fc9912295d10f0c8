// K6 placeholder until the FP8 forward lands.
#include "fa3b_internal.cuh"
namespace fa3b {
int launch_fwd_fp8(const fa3b_fwd_params&, cudaStream_t) { return FA3B_ERR_DTYPE; }
}  // namespace fa3b
