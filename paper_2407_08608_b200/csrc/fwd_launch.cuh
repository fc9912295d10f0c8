// Host-side launcher of K1 / K6 (fa3b_fwd_kernel) shared by the translation
// units that instantiate its variants: fwd16_d*.cu (the default f16/bf16
// schedules per head dim), fwd16_sched_*.cu (the one-tile schedule variants),
// fwd_fp8*.cu (e4m3). Splitting the instantiations lets them compile in
// parallel.
#pragma once

#include <cuda.h>
#include <cuda_runtime.h>

#include <cmath>
#include <cstdlib>

#include "fa3b_internal.cuh"
#include "fwd_kernel.cuh"

#ifndef FA3B_FP8_THR_BLOCK
#define FA3B_FP8_THR_BLOCK 4
#endif
#ifndef FA3B_FWD_EMU_S2_16
#define FA3B_FWD_EMU_S2_16 2
#endif
#ifndef FA3B_FWD_EMU_S2
#define FA3B_FWD_EMU_S2 3
#endif

namespace fa3b {

// log2 headroom of the e4m3 P (lazy running max: O and l are rescaled only when
// the max grows by more than 2^thr, so P <= 2^thr): codes = P * rho * 448 / 2^thr,
// rho <= 1 the folded power-of-two ratio of the key block's V scale to the one O
// is kept in (fwd_kernel.cuh). thr 4 for both granularities: per block it is
// +3 % at d 128 and +8 % at d 256 over thr 2 for +0.7 % RMSE (N 8192: 0.00945 vs
// 0.00938; profiles/r02/r02z_thr_ab.log, r02y_thr_acc.log). FA3B_FP8_THR overrides.
inline float fp8_threshold(bool kv_blocked) {
  static const float env = [] {
    const char* e = std::getenv("FA3B_FP8_THR");
    const float v = e ? static_cast<float>(std::atof(e)) : -1.f;
    return (v >= 0.f && v <= 8.f) ? v : -1.f;
  }();
  if (env >= 0.f) return env;
  return kv_blocked ? static_cast<float>(FA3B_FP8_THR_BLOCK) : 4.f;
}

template <int D, int NT, bool CAUSAL, int KIND, int CPS = 1, int SCHED = SCHED_DEFAULT, int NQ = 2,
          int BN = 128>
int launch_fwd(const fa3b_fwd_params& p, cudaStream_t stream) {
  constexpr bool FP8 = KIND == KIND_E4M3;
  constexpr int EB = FP8 ? 1 : 2;
  using T = FwdTraits<D, NT, EB, CPS, SCHED, NQ, BN>;
  // one-tile CTAs with S fetched early (S2) own the SM's MUFU: more of the exp2
  // pairs go to the FMA-pipe polynomial
  constexpr int EMU = T::S2 ? (FP8 ? FA3B_FWD_EMU_S2 : FA3B_FWD_EMU_S2_16) : FA3B_FWD_EMU;
  auto kern = fa3b_fwd_kernel<D, NT, CAUSAL, KIND, CPS, EMU, SCHED, NQ, BN>;
  int rc = ensure_smem_attr(reinterpret_cast<const void*>(kern), T::SMEM_BYTES);
  if (rc != FA3B_OK) return rc;
  CUtensorMap tq, tk, tv;
  const int box = T::CHUNK_ELEMS;  // ROW_BYTES-wide rows of the swizzled tiles
  const int swz = T::ROW_BYTES;
  if ((rc = make_tmap_4d(&tq, p.q, EB, D, p.heads_q, p.seqlen, p.batch, box, 128, swz)) != FA3B_OK)
    return rc;
  if ((rc = make_tmap_4d(&tk, p.k, EB, D, p.heads_kv, p.seqlen, p.batch, box, BN, swz)) != FA3B_OK)
    return rc;
  if ((rc = make_tmap_4d(&tv, p.v, EB, D, p.heads_kv, p.seqlen, p.batch, box, BN, swz)) != FA3B_OK)
    return rc;
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
  {
    // 32-byte aligned 16-bit rows: base and every stride a multiple of 16 elements
    auto ok32 = [](long long st, int extent) { return extent <= 1 || st % 16 == 0; };
    a.o_v8 = !a.out_f32 && (reinterpret_cast<uintptr_t>(p.o.ptr) & 31u) == 0 && ok32(a.o_sb, p.batch) &&
             ok32(a.o_ss, p.seqlen) && ok32(a.o_sh, p.heads_q);
  }
  a.lse = p.lse;
  uint32_t fmt = 0;
  if constexpr (FP8) {
    a.q_scale = p.q_scale;
    a.k_scale = p.k_scale;
    a.v_scale = p.v_scale;
    a.q_blocked = p.q_block_rows != 0;
    a.kv_blocked = p.kv_block_rows != 0;
    a.fp8_thr = fp8_threshold(a.kv_blocked != 0);
    a.fp8_pmul = 448.f * std::exp2(-a.fp8_thr);
    a.fp8_inv_pmul = 1.f / a.fp8_pmul;
    a.fp8_lpm = std::log2(a.fp8_pmul);
  } else {
    a.q_scale = a.k_scale = a.v_scale = nullptr;
    a.q_blocked = a.kv_blocked = 0;
    a.fp8_thr = 8.f;
    fmt = KIND == KIND_BF16 ? 1u : 0u;
  }
  const uint32_t idesc_qk = ptx::make_idesc(128, BN, fmt, fmt, false, false, p.alpha < 0);
  const uint32_t idesc_pv = ptx::make_idesc(128, D, fmt, fmt, false, true, false);
  const int grid = fwd_grid(p.seqlen, NT, p.heads_q, p.batch, CPS);  // persistent CTAs
  kern<<<grid, T::NUM_THREADS, T::SMEM_BYTES, stream>>>(tq, tk, tv, a, idesc_qk, idesc_pv);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return cuda_fail(e);
  g_last_launch_count = 1;
  return FA3B_OK;
}

// causal x kind dispatch of one (D, NT, CPS, SCHED, NQ, BN) variant
template <int D, int NT, int CPS, int SCHED, int KIND, int NQ = 2, int BN = 128>
int launch_fwd_c(const fa3b_fwd_params& p, cudaStream_t s) {
  return p.causal ? launch_fwd<D, NT, true, KIND, CPS, SCHED, NQ, BN>(p, s)
                  : launch_fwd<D, NT, false, KIND, CPS, SCHED, NQ, BN>(p, s);
}

// FA3B_FWD_Q1=1 runs the d = 128 pair with one softmax warpgroup per query tile
// (thread = row, all 128 columns: no half-row max exchange) instead of two (A/B switch)
inline int fwd_q1_env() {
  static const int v = [] {
    const char* e = std::getenv("FA3B_FWD_Q1");
    return e == nullptr ? -1 : (std::atoi(e) != 0 ? 1 : 0);
  }();
  return v;
}

// FA3B_FWD_P2=1|0 forces the P2 pair (64-key blocks, one softmax warpgroup per
// tile, per-tile double S buffers) on or off at d = 128 (A/B switch; the default
// is the measured choice)
inline int fwd_p2_env() {
  static const int v = [] {
    const char* e = std::getenv("FA3B_FWD_P2");
    return e == nullptr ? -1 : (std::atoi(e) != 0 ? 1 : 0);
  }();
  return v;
}

// FA3B_FWD_WIDE=1|0 forces the one-tile, four-warpgroup S2 forward (NQ = 4) on or
// off at d <= 128 (A/B switch; the default is the measured choice)
inline int fwd_wide_env() {
  static const int v = [] {
    const char* e = std::getenv("FA3B_FWD_WIDE");
    return e == nullptr ? -1 : (std::atoi(e) != 0 ? 1 : 0);
  }();
  return v;
}

}  // namespace fa3b
