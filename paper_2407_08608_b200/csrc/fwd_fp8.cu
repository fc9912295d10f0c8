// K6 launcher: the FP8 (e4m3) forward, fa3b_fwd_kernel<..., KIND_E4M3>.
// Replaces the main loop of fp8_flash_fwd (core/src/fp8_attention.cpp:99-178);
// the operands come from K5 (fa3b_fp8_prepare). See fwd_kernel.cuh for the
// scale handling.
#include "fwd_launch.cuh"

namespace fa3b {

int launch_fwd_fp8(const fa3b_fwd_params& p, cudaStream_t s) {
  if (!p.q_scale || !p.k_scale || !p.v_scale) return FA3B_ERR_NULL;
  if ((p.q_block_rows != 0 && p.q_block_rows != 128) ||
      (p.kv_block_rows != 0 && p.kv_block_rows != 128))
    return FA3B_ERR_BLOCK;
  constexpr int K = KIND_E4M3;
  if (p.schedule == FA3B_SCHED_NO_WS) return FA3B_ERR_SCHEDULE;
  switch (p.head_dim) {
    case 64:  // 64-byte rows: 64-byte swizzle; the pair with three rotating S buffers (S3)
      return launch_fwd_fp8_d64(p, s);
    case 128:
      switch (p.schedule) {
        case FA3B_SCHED_BASIC: return launch_fwd_c<128, 1, 1, SCHED_SERIAL, K>(p, s);
        case FA3B_SCHED_3STAGE: return launch_fwd_c<128, 1, 1, SCHED_3STAGE, K>(p, s);
        case FA3B_SCHED_2STAGE: return launch_fwd_c<128, 1, 1, SCHED_2STAGE, K>(p, s);
      }
      if (fwd_wide_env() == 1) return launch_fwd_c<128, 1, 1, SCHED_DEFAULT, K, 4>(p, s);
      if (fwd_p2_env() == 1) return launch_fwd_c<128, 2, 1, SCHED_DEFAULT, K, 1, 64>(p, s);
      if (fwd_q1_env() == 1) return launch_fwd_c<128, 2, 1, SCHED_DEFAULT, K, 1>(p, s);
      if (fwd_pairing(128, p.causal != 0, true, p.seqlen)) return launch_fwd_c<128, 1, 2, SCHED_DEFAULT, K>(p, s);
      return launch_fwd_c<128, 2, 1, SCHED_DEFAULT, K>(p, s);
    case 256:
      switch (p.schedule) {
        case FA3B_SCHED_BASIC: return launch_fwd_c<256, 1, 1, SCHED_SERIAL, K>(p, s);
        case FA3B_SCHED_2STAGE: return launch_fwd_c<256, 1, 1, SCHED_2STAGE, K>(p, s);
      }
      return launch_fwd_c<256, 1, 1, SCHED_DEFAULT, K>(p, s);  // = 3-stage (S2)
  }
  return FA3B_ERR_HEAD_DIM;
}

}  // namespace fa3b

#ifdef FA3B_TRACE
// Debug builds only: the e4m3 instantiations record into this translation unit's trace.
extern "C" __attribute__((visibility("default"))) int fa3b_debug_trace_fp8(unsigned long long* out, int n) {
  const size_t bytes = sizeof(unsigned long long) * static_cast<size_t>(n);
  return cudaMemcpyFromSymbol(out, fa3b::g_fa3b_trace, bytes) == cudaSuccess ? 0 : -1;
}
#endif
