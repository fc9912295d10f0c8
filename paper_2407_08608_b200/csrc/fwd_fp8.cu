// K6 launcher: the FP8 (e4m3) forward, fa3b_fwd_kernel<..., KIND_E4M3>.
// Replaces the main loop of fp8_flash_fwd (core/src/fp8_attention.cpp:99-178);
// the operands come from K5 (fa3b_fp8_prepare). See fwd_kernel.cuh for the
// scale handling.
#include <cuda.h>
#include <cuda_runtime.h>

#include <cmath>
#include <cstdlib>
#include <mutex>

#include "fa3b_internal.cuh"
#include "fwd_kernel.cuh"

namespace fa3b {
namespace {

// log2 headroom of the e4m3 P: codes = P * 448 / 2^thr with P <= 2^thr.
// With per-block V scales O is rescaled every block anyway, so the running
// max is kept exact (thr 0, P <= 1, the reference's P range); per tensor a
// lazy max (thr 4) skips most O rescales. FA3B_FP8_THR overrides both.
float fp8_threshold(bool kv_blocked) {
  static const float env = [] {
    const char* e = std::getenv("FA3B_FP8_THR");
    const float v = e ? static_cast<float>(std::atof(e)) : -1.f;
    return (v >= 0.f && v <= 8.f) ? v : -1.f;
  }();
  if (env >= 0.f) return env;
  return kv_blocked ? 0.f : 4.f;
}

#ifndef FA3B_FWD_EMU_S2
#define FA3B_FWD_EMU_S2 3
#endif

template <int D, int NT, bool CAUSAL, int CPS = 1>
int launch(const fa3b_fwd_params& p, cudaStream_t stream) {
  using T = FwdTraits<D, NT, 1, CPS>;
  // one query tile per CTA with S fetched early (S2): the softmax has the SM to
  // itself, so a third of the exp2 pairs go to the FMA pipe instead of a quarter
  constexpr int EMU = T::S2 ? FA3B_FWD_EMU_S2 : FA3B_FWD_EMU;
  auto kern = fa3b_fwd_kernel<D, NT, CAUSAL, KIND_E4M3, CPS, EMU>;
  int rc = ensure_smem_attr(reinterpret_cast<const void*>(kern), T::SMEM_BYTES);
  if (rc != FA3B_OK) return rc;
  CUtensorMap tq, tk, tv;
  if ((rc = make_tmap_4d(&tq, p.q, 1, D, p.heads_q, p.seqlen, p.batch, 128, 128)) != FA3B_OK) return rc;
  if ((rc = make_tmap_4d(&tk, p.k, 1, D, p.heads_kv, p.seqlen, p.batch, 128, 128)) != FA3B_OK) return rc;
  if ((rc = make_tmap_4d(&tv, p.v, 1, D, p.heads_kv, p.seqlen, p.batch, 128, 128)) != FA3B_OK) return rc;
  FwdArgs a;
  a.B = p.batch;
  a.H = p.heads_q;
  a.Hkv = p.heads_kv;
  a.N = p.seqlen;
  a.group = p.heads_q / p.heads_kv;
  a.scale_log2 = static_cast<float>(std::fabs(p.alpha) * 1.4426950408889634);
  a.o = p.o.ptr;
  a.o_sb = p.o.stride_batch;
  a.o_ss = p.o.stride_seq;
  a.o_sh = p.o.stride_head;
  a.out_f32 = p.out_dtype == FA3B_DTYPE_F32;
  a.lse = p.lse;
  a.q_scale = p.q_scale;
  a.k_scale = p.k_scale;
  a.v_scale = p.v_scale;
  a.q_blocked = p.q_block_rows != 0;
  a.kv_blocked = p.kv_block_rows != 0;
  a.fp8_thr = fp8_threshold(a.kv_blocked != 0);
  a.fp8_pmul = 448.f * std::exp2(-a.fp8_thr);
  a.fp8_inv_pmul = 1.f / a.fp8_pmul;
  a.fp8_lpm = std::log2(a.fp8_pmul);
  const uint32_t idesc_qk = ptx::make_idesc(128, 128, 0, 0, false, false, p.alpha < 0);
  const uint32_t idesc_pv = ptx::make_idesc(128, D, 0, 0, false, true, false);
  const int grid = fwd_grid(p.seqlen, NT, p.heads_q, p.batch, CPS);  // persistent CTAs
  kern<<<grid, T::NUM_THREADS, T::SMEM_BYTES, stream>>>(tq, tk, tv, a, idesc_qk, idesc_pv);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return cuda_fail(e);
  g_last_launch_count = 1;
  return FA3B_OK;
}

}  // namespace

int launch_fwd_fp8(const fa3b_fwd_params& p, cudaStream_t s) {
  if (!p.q_scale || !p.k_scale || !p.v_scale) return FA3B_ERR_NULL;
  if ((p.q_block_rows != 0 && p.q_block_rows != 128) ||
      (p.kv_block_rows != 0 && p.kv_block_rows != 128))
    return FA3B_ERR_BLOCK;
  const bool basic = p.schedule == FA3B_SCHED_BASIC;
  switch (p.head_dim) {
    case 128: {
      const bool cta_pairs = fwd_pairing(128, p.causal != 0, true);
      if (p.causal)
        return basic ? launch<128, 1, true>(p, s)
                     : (cta_pairs ? launch<128, 1, true, 2>(p, s) : launch<128, 2, true>(p, s));
      return basic ? launch<128, 1, false>(p, s)
                   : (cta_pairs ? launch<128, 1, false, 2>(p, s) : launch<128, 2, false>(p, s));
    }
    case 256:
      return p.causal ? launch<256, 1, true>(p, s) : launch<256, 1, false>(p, s);
  }
  return FA3B_ERR_HEAD_DIM;  // e4m3 rows of 64 bytes would need a 64B swizzle
}

}  // namespace fa3b

#ifdef FA3B_TRACE
// Debug builds only: the e4m3 instantiations record into this translation unit's trace.
extern "C" __attribute__((visibility("default"))) int fa3b_debug_trace_fp8(unsigned long long* out, int n) {
  const size_t bytes = sizeof(unsigned long long) * static_cast<size_t>(n);
  return cudaMemcpyFromSymbol(out, fa3b::g_fa3b_trace, bytes) == cudaSuccess ? 0 : -1;
}
#endif
