// K6 at head dim 64: e4m3 rows of 64 bytes, so the Q/K/V tiles use the 64-byte
// swizzle (TMA CU_TENSOR_MAP_SWIZZLE_64B, UMMA layout SWIZZLE_64B, 8-row atoms of
// 512 bytes) and QK^T takes two 32-byte K steps per row. The default schedule is
// the d = 64 pair with three rotating S buffers (FwdTraits::S3); the one-tile
// schedule variants run as at d = 128. Its own translation unit so it compiles in
// parallel with fwd_fp8.cu.
#include "fwd_launch.cuh"

namespace fa3b {

int launch_fwd_fp8_d64(const fa3b_fwd_params& p, cudaStream_t s) {
  constexpr int K = KIND_E4M3;
  switch (p.schedule) {
    case FA3B_SCHED_BASIC: return launch_fwd_c<64, 1, 1, SCHED_SERIAL, K>(p, s);
    case FA3B_SCHED_3STAGE: return launch_fwd_c<64, 1, 1, SCHED_3STAGE, K>(p, s);
    case FA3B_SCHED_2STAGE: return launch_fwd_c<64, 1, 1, SCHED_2STAGE, K>(p, s);
  }
  return launch_fwd_c<64, 2, 1, SCHED_DEFAULT, K>(p, s);
}

}  // namespace fa3b
