// K5 placeholder until the FP8 prepare kernel lands.
#include "fa3b_internal.cuh"
extern "C" int fa3b_fp8_prepare(const fa3b_fp8_prepare_params*) { return FA3B_ERR_DTYPE; }
