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
