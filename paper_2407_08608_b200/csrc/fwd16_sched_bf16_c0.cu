// K1 bf16 forward, causal = 0: the one-tile schedule variants (fa3b_schedule
// BASIC / 3STAGE / 2STAGE / NO_WS; fwd_kernel.cuh FwdSched).
#include "fwd_launch.cuh"

namespace fa3b {

template <int D>
static int sched_d(const fa3b_fwd_params& p, cudaStream_t s) {
  constexpr bool C = 0;
  switch (p.schedule) {
    case FA3B_SCHED_BASIC: return launch_fwd<D, 1, C, KIND_BF16, 1, SCHED_SERIAL>(p, s);
    case FA3B_SCHED_3STAGE: return launch_fwd<D, 1, C, KIND_BF16, 1, SCHED_3STAGE>(p, s);
    case FA3B_SCHED_2STAGE: return launch_fwd<D, 1, C, KIND_BF16, 1, SCHED_2STAGE>(p, s);
    case FA3B_SCHED_NO_WS:
      if constexpr (FwdTraits<D, 1, 2, 1>::STAGES >= 4)
        return launch_fwd<D, 1, C, KIND_BF16, 1, SCHED_NOWS>(p, s);
      return FA3B_ERR_SCHEDULE;  // d = 256: a 2-stage ring leaves the leader no slack
  }
  return FA3B_ERR_SCHEDULE;
}

int launch_fwd16_sched_bf16_c0(const fa3b_fwd_params& p, cudaStream_t s) {
  switch (p.head_dim) {
    case 64: return sched_d<64>(p, s);
    case 128: return sched_d<128>(p, s);
    case 256: return sched_d<256>(p, s);
  }
  return FA3B_ERR_HEAD_DIM;
}

}  // namespace fa3b
