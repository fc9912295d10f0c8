// K1 f16/bf16 forward, head dim 128, default schedule (see fwd_kernel.cuh).
#include "fwd_launch.cuh"

namespace fa3b {

int launch_fwd16_default_d128(const fa3b_fwd_params& p, cudaStream_t s, bool cta_pairs) {
  const bool bf16 = p.in_dtype == FA3B_DTYPE_BF16;
  if (fwd_wide_env() == 1)
    return bf16 ? launch_fwd_c<128, 1, 1, SCHED_DEFAULT, KIND_BF16, 4>(p, s)
                : launch_fwd_c<128, 1, 1, SCHED_DEFAULT, KIND_F16, 4>(p, s);
  if (fwd_q1_env() == 1)  // bf16 only (the A/B candidate for the headline)
    return bf16 ? launch_fwd_c<128, 2, 1, SCHED_DEFAULT, KIND_BF16, 1>(p, s)
                : launch_fwd_c<128, 2, 1, SCHED_DEFAULT, KIND_F16>(p, s);
  if (cta_pairs)
    return bf16 ? launch_fwd_c<128, 1, 2, SCHED_DEFAULT, KIND_BF16>(p, s)
                : launch_fwd_c<128, 1, 2, SCHED_DEFAULT, KIND_F16>(p, s);
  return bf16 ? launch_fwd_c<128, 2, 1, SCHED_DEFAULT, KIND_BF16>(p, s)
              : launch_fwd_c<128, 2, 1, SCHED_DEFAULT, KIND_F16>(p, s);
}

}  // namespace fa3b

#ifdef FA3B_TRACE
// Debug builds only (-DFA3B_TRACE): the traces recorded by this translation unit's
// kernels (the d = 128 f16/bf16 forward): phase points of CTA 0's first item, per-CTA
// start / end, and CTA 0's item timeline.
extern "C" __attribute__((visibility("default"))) int fa3b_debug_trace(unsigned long long* out, int n) {
  const size_t bytes = sizeof(unsigned long long) * static_cast<size_t>(n);
  return cudaMemcpyFromSymbol(out, fa3b::g_fa3b_trace, bytes) == cudaSuccess ? 0 : -1;
}
extern "C" __attribute__((visibility("default"))) int fa3b_debug_cta_trace(unsigned long long* out, int n) {
  const size_t bytes = sizeof(unsigned long long) * static_cast<size_t>(n);
  return cudaMemcpyFromSymbol(out, fa3b::g_fa3b_cta, bytes) == cudaSuccess ? 0 : -1;
}
extern "C" __attribute__((visibility("default"))) int fa3b_debug_item_trace(unsigned long long* out, int n) {
  const size_t bytes = sizeof(unsigned long long) * static_cast<size_t>(n);
  return cudaMemcpyFromSymbol(out, fa3b::g_fa3b_items, bytes) == cudaSuccess ? 0 : -1;
}
#endif
