#include "fa3b_internal.cuh"
namespace fa3b { int launch_fwd_fp8(const fa3b_fwd_params&, cudaStream_t) { return FA3B_ERR_DTYPE; } }
extern "C" {
int fa3b_fp8_prepare(const fa3b_fp8_prepare_params*) { return FA3B_ERR_DTYPE; }
int fa3b_bwd_preprocess(const fa3b_bwd_preprocess_params*) { return FA3B_ERR_DTYPE; }
int fa3b_bwd(const fa3b_bwd_params*) { return FA3B_ERR_DTYPE; }
size_t fa3b_bwd_workspace_bytes(int32_t, int32_t, int32_t, int32_t, int32_t) { return 0; }
}
