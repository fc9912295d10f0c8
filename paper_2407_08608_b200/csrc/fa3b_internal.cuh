// Host-side helpers shared by the C-ABI translation units.
#pragma once

#include <cuda.h>
#include <cuda_runtime.h>

#include "../../include/fa3b.h"

namespace fa3b {

extern thread_local int g_last_cuda_error;
extern thread_local int g_last_launch_count;

int cuda_fail(cudaError_t e);
// swizzle_bytes: 128 (the default) or 64 (64-byte rows, e4m3 at d = 64)
int make_tmap_4d(CUtensorMap* map, const fa3b_tensor4& t, int elem_bytes, int dim, int heads,
                 int seqlen, int batch, int inner_elems, int rows, int swizzle_bytes = 128);
bool aligned16(const void* p);
bool strides_ok(const fa3b_tensor4& t, int elem_bytes, int batch, int seqlen, int heads);
int validate_problem(int batch, int heads_q, int heads_kv, int seqlen, int head_dim,
                     double alpha);

int launch_fwd_fp8(const fa3b_fwd_params& p, cudaStream_t stream);
int launch_fwd_fp8_d64(const fa3b_fwd_params& p, cudaStream_t stream);
// f16/bf16 forward launchers, one translation unit each (fwd16_*.cu)
int launch_fwd16_default_d64(const fa3b_fwd_params& p, cudaStream_t s, bool cta_pairs);
int launch_fwd16_default_d128(const fa3b_fwd_params& p, cudaStream_t s, bool cta_pairs);
int launch_fwd16_default_d256(const fa3b_fwd_params& p, cudaStream_t s, bool cta_pairs);
int launch_fwd16_sched_bf16_c0(const fa3b_fwd_params& p, cudaStream_t s);
int launch_fwd16_sched_bf16_c1(const fa3b_fwd_params& p, cudaStream_t s);
int launch_fwd16_sched_f16_c0(const fa3b_fwd_params& p, cudaStream_t s);
int launch_fwd16_sched_f16_c1(const fa3b_fwd_params& p, cudaStream_t s);
// Raise a kernel's dynamic shared-memory limit once per (kernel, device): the
// attribute belongs to the function as loaded on the current device, so a
// process driving several GPUs needs it on each.
int ensure_smem_attr(const void* kernel, int bytes);
// Streaming multiprocessors of the current device (cached per device).
int num_sms();
// FA3B_OK on an sm_100 current device, else FA3B_ERR_DEVICE (cached per device).
int check_device();
// Persistent forward grid: one CTA per SM (or per SM slot), never more than the work.
inline int fwd_grid(int seqlen, int nt, int heads, int batch, int ctas_per_sm) {
  const long long items = static_cast<long long>((seqlen + nt * 128 - 1) / (nt * 128)) * heads * batch;
  const long long cap = static_cast<long long>(num_sms()) * ctas_per_sm;
  return static_cast<int>(items < cap ? items : cap);
}
// true: pair query tiles across two CTAs per SM; false: two tiles in one CTA
bool fwd_pairing(int head_dim, bool causal, bool fp8, int seqlen);

}  // namespace fa3b
