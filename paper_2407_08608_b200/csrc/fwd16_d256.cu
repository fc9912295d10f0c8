// K1 f16/bf16 forward, head dim 256, default schedule (see fwd_kernel.cuh).
#include "fwd_launch.cuh"

namespace fa3b {

int launch_fwd16_default_d256(const fa3b_fwd_params& p, cudaStream_t s, bool cta_pairs) {
  const bool bf16 = p.in_dtype == FA3B_DTYPE_BF16;
  (void)cta_pairs;
  return bf16 ? launch_fwd_c<256, 1, 1, SCHED_DEFAULT, KIND_BF16>(p, s)
              : launch_fwd_c<256, 1, 1, SCHED_DEFAULT, KIND_F16>(p, s);
}

}  // namespace fa3b

#ifdef FA3B_TRACE
// Debug builds only (-DFA3B_TRACE): the phase points recorded by the d = 256 forward.
extern "C" __attribute__((visibility("default"))) int fa3b_debug_trace_d256(unsigned long long* out, int n) {
  const size_t bytes = sizeof(unsigned long long) * static_cast<size_t>(n);
  return cudaMemcpyFromSymbol(out, fa3b::g_fa3b_trace, bytes) == cudaSuccess ? 0 : -1;
}
#endif
