// K1: attention forward for f16/bf16 on sm_100a.
//
// Replaces the reference's tiled forward (core/src/flash_fwd.cpp:18-232):
// score_block (:57-71) is a tcgen05 SS-MMA into TMEM, online_softmax_step
// (:18-48) runs in the softmax warpgroups, accumulate_output (:75-90) is a
// tcgen05 TS-MMA with P read from TMEM, epilogue (:92-106) normalizes O and
// writes the natural-log LSE, and active_col_blocks (:110-124) becomes the
// per-tile KV block count.
//
// CTA layout (NT query tiles of 128 rows, KV blocks of 128 rows):
//   warps [0, 8*NT)   two softmax warpgroups per query tile t; warp w handles
//                     rows 32 (w % 4) + lane (= TMEM lanes) and the column half
//                     (w / 4) % 2 of S; the halves exchange row maxima through
//                     shared memory (one named barrier per iteration) and keep
//                     separate row sums until the epilogue
//   warp 8*NT         TMA producer: Q tiles once, then K_j, V_j through a ring
//                     of STAGES shared-memory slots
//   warp 8*NT+1       MMA issuer (one elected thread), TMEM allocator
// TMEM (512 columns): S_t at [128 t, 128 t + 128), P_t (16-bit, 2 per column;
// e4m3, 4 per column) aliased onto S_t, each softmax warpgroup's P over the first
// columns of its own 64-column half (FwdTraits::p_kcol), O_t at [128 NT + D t, + D).
//
// Per tile the MMA order is  S(K_0) ; { PV(V_j) ; S(K_{j+1}) }_j , so the
// arrival of S(K_{j+1}) implies PV(V_j) is complete (tcgen05.commit covers all
// prior MMAs of the thread) and the softmax warpgroup may rescale O_t in place.
// With NT = 2 the tensor core runs tile 1's GEMMs while tile 0 is in softmax
// and vice versa (the paper's inter-warpgroup ping-pong).
//
// The running max is kept lazily: O and l are only rescaled when the block
// max exceeds the max in use by more than 2^THR (log2 domain), so P <= 2^THR
// (THR = 8 for 16-bit P). The result equals the reference's
// rescale-every-block arithmetic up to rounding (flash_fwd.cpp:36-45).
//
// KIND = E4M3 is the FP8 forward K6 (fp8_flash_fwd, core/src/fp8_attention.cpp:
// 77-181): Q/K/V are e4m3 codes with per-128-row-block (or per-tensor) scales
// from K5; the S descale alpha s_q s_k[j] folds into the exp2 pre-scale
// (PAPER.md:605-606); P is requantized to e4m3 with the fixed scale 448 / 2^THR
// (THR = args.fp8_thr, the lazy-max headroom) instead of the reference's
// per-block amax, which is ~1 for every block (proj/README.md:116-121). V's
// per-block scale is applied exactly, as the reference does to each PV product
// (fp8_attention.cpp:158-164): O is kept in units of a V scale v_cur. When a key
// block's s_v / v_cur is an exact power of two in [2^-8, 1] (the FP8 forward
// quantizes V with power-of-two block scales, fa3b.h scale_pow2) the ratio is
// folded into that block's P codes, an exact exponent shift; otherwise O is
// rescaled to s_v (one TMEM pass, shared with the softmax rescale). Folding an
// arbitrary ratio instead makes the codes of the largest P inexact and cost
// +14 % RMSE on the reference's outlier inputs (profiles/r02/r02f_acc.log).
// Both MMAs run as tcgen05 kind::f8f6f4 with V consumed MN-major straight from
// the TMA tile (no in-kernel transpose on sm_100a).
//
// One query tile per CTA (d = 256 and the basic schedule; T::S2): TMEM has
// room for a second S buffer after O, so the MMA warp computes S(K_{j+1}) while
// the softmax still works on S_j / P_j — the paper's intra-warpgroup overlap
// (PAPER.md:307-330). Order S_0 ; S_1 ; { PV_j ; S_{j+2} }_j, S_{j+2} reusing
// S_j's columns after PV_j has read P_j; pv_done tells the softmax when O may be
// rescaled. The producer loads in the same order (K_0, K_1, {V_j, K_{j+2}}), so
// the two-stage ring of bf16 d = 256 (64 KB tiles) still delivers K_{j+2} early.
//
// The d = 64 tile pair (T::S3) has 128 spare columns too: three S buffers rotate
// between the two tiles, S(t, j) in buffer (G + 2 j + t) % 3, in the order
// S(0,0) ; S(1,0) ; S(0,1) ; {PV(0,j) ; S(1,j+1) ; PV(1,j) ; S(0,j+2)}_j — every S
// reuses the buffer of the S three before it, whose PV was issued just before, and
// each tile's next S is computed during its own softmax.
#pragma once

#include <type_traits>

#include "sm100_ptx.cuh"

// Register rebalancing: with FA3B_FWD_REGS = R > 0 the producer / MMA warps get
// two idle companions (one full warpgroup) that drop to 56 registers with
// setmaxnreg so the softmax warpgroups can rise from the launch cap (96) to R.
#ifndef FA3B_FWD_REGS
#define FA3B_FWD_REGS 0
#endif
#ifndef FA3B_FWD_S2
#define FA3B_FWD_S2 1
#endif
#ifndef FA3B_FWD_PV_PRE
#define FA3B_FWD_PV_PRE 1
#endif
#ifndef FA3B_FWD_S3
#define FA3B_FWD_S3 1
#endif
#ifndef FA3B_FWD_OREGS
#define FA3B_FWD_OREGS 56
#endif
#ifndef FA3B_MMA_SPIN
#define FA3B_MMA_SPIN 0
#endif
// FA3B_FWD_PPBAR = 1: the two tiles of the default pair take turns for the exp
// phase (a token passed through named barriers 3 / 4, FA3's warpgroup ping-pong
// ordering), so one tile's exps run alone on the MUFU while the other tile's GEMMs run
#ifndef FA3B_FWD_QB2
#define FA3B_FWD_QB2 0
#endif
#ifndef FA3B_FWD_SPEC
#define FA3B_FWD_SPEC 0
#endif
// FA3B_FWD_CHRING: with 64 KB K/V tiles (bf16 d = 256, one-tile S2 schedule, a
// 2-tile ring) the ring is managed per 16 KB column chunk: each chunk has its own
// full/empty barrier, the S MMA consumes K chunk by chunk and PV runs as one
// N = 64 MMA group per V chunk, so loads refill freed chunks while the rest of
// the tile is still in use and an MMA starts as soon as its first chunk lands
#ifndef FA3B_FWD_CHRING
#define FA3B_FWD_CHRING 1
#endif
// also the FP8 d = 256 tiles (32 KB, 4-tile ring): measured 6 % slower there
// (r02cb_chring8_ab.log), off; bf16 d = 256: +11-14 % (r02ca_chring_ab.log)
#ifndef FA3B_FWD_CHRING_EXTRA
#define FA3B_FWD_CHRING_EXTRA 0
#endif
#ifndef FA3B_FWD_CHRING_FP8
#define FA3B_FWD_CHRING_FP8 0
#endif
// release Q after the item's last S (not after its last PV): see the MMA warp
#ifndef FA3B_FWD_QEARLY
#define FA3B_FWD_QEARLY 1
#endif
#ifndef FA3B_FWD_QB2_SHRINK
#define FA3B_FWD_QB2_SHRINK 0
#endif
#ifndef FA3B_FWD_QPREFETCH
#define FA3B_FWD_QPREFETCH 0
#endif
#ifndef FA3B_FWD_PPBAR
#define FA3B_FWD_PPBAR 0
#endif
#ifndef FA3B_FWD_PSPLIT
#define FA3B_FWD_PSPLIT 0
#endif

namespace fa3b {

// Optional phase tracing (compile with -DFA3B_TRACE): CTA (0,0,0) records
// clock64() at the softmax / MMA phase boundaries of each KV iteration into
// g_fa3b_trace[tile][iter][point]; read back with fa3b_debug_trace().
#ifdef FA3B_TRACE
__device__ unsigned long long g_fa3b_trace[2][64][8];
// per-CTA [start globaltimer ns, SM id, end globaltimer ns, first-S-ready ns] for the first 4096 CTAs
__device__ unsigned long long g_fa3b_cta[4096][4];
__device__ __forceinline__ unsigned long long fa3b_gtime() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
__device__ __forceinline__ unsigned fa3b_smid() {
  unsigned s;
  asm volatile("mov.u32 %0, %%smid;" : "=r"(s));
  return s;
}
// item timeline of CTA 0 (globaltimer ns): [item][0] Q TMA issued, [1] MMA saw q_full,
// [2 + 3 t] tile t first S ready, [3 + 3 t] tile t last P handed over, [4 + 3 t] epilogue done,
// [8] K_0 TMA issued, [9] MMA saw K_0, [10] S_0 GEMMs issued
__device__ unsigned long long g_fa3b_items[64][12];
#define FA3B_IT(itl, k)                                             \
  do {                                                              \
    if (blockIdx.x == 0 && (itl) < 64) g_fa3b_items[itl][k] = fa3b_gtime(); \
  } while (0)
#define FA3B_CTA(k, v)                                                                    \
  do {                                                                                    \
    const unsigned cid = blockIdx.x + gridDim.x * (blockIdx.y + gridDim.y * blockIdx.z); \
    if (cid < 4096) g_fa3b_cta[cid][k] = (v);                                             \
  } while (0)
#define FA3B_TP(t, j, k)                                                               \
  do {                                                                                 \
    if (blockIdx.x == 0 && blockIdx.y == 0 && blockIdx.z == 0 && (j) < 64) \
      g_fa3b_trace[t][j][k] = clock64();                                               \
  } while (0)
#else
#define FA3B_TP(t, j, k) \
  do {                   \
  } while (0)
#define FA3B_CTA(k, v) \
  do {                 \
  } while (0)
#define FA3B_IT(itl, k) \
  do {                  \
  } while (0)
#endif

enum FwdKind { KIND_F16 = 0, KIND_BF16 = 1, KIND_E4M3 = 2 };

struct FwdArgs {
  int B, H, Hkv, N;
  int group;          // H / Hkv
  float scale_log2;   // |alpha| * log2(e)
  void* o;
  long long o_sb, o_ss, o_sh;  // element strides of O
  int out_f32;
  int o_v8;           // 16-bit O rows 32-byte aligned: 256-bit stores in the epilogue
  float* lse;         // [B, H, N] or nullptr
  // E4M3 only
  const float* q_scale;  // [B, H, nqb] (per 128-row block) or [B, H] (per tensor)
  const float* k_scale;  // [B, Hkv, nkb] or [B, Hkv]
  const float* v_scale;
  int q_blocked, kv_blocked;
  float fp8_thr;         // lazy-rescale threshold (log2) for the e4m3 P
  float fp8_pmul, fp8_inv_pmul, fp8_lpm;  // P code scale 448 / 2^thr, its inverse and log2
};
__device__ __forceinline__ int fwd_seqlen(const FwdArgs& a) { return a.N; }


// Kernel schedule variants (include/fa3b.h fa3b_schedule). SCHED_DEFAULT is the
// production path; the others exist for the reference's three schedules and the
// paper's ablation and only apply to one-tile CTAs (NT = 1).
enum FwdSched {
  SCHED_DEFAULT = 0,  // NT = 2 ping-pong (S3 at d = 64) or, with NT = 1, S2 = 3-stage
  SCHED_SERIAL = 1,   // one S buffer: S_j -> softmax_j -> PV_j strictly in sequence
  SCHED_3STAGE = 2,   // = the NT = 1 S2 path (softmax_j overlaps S_{j+1} and PV_{j-1})
  SCHED_2STAGE = 3,   // S2, but softmax_j starts only after PV_{j-1} has completed
  SCHED_NOWS = 4      // S2 pipelining issued by the softmax warps (no producer / MMA warps)
};

// CPS_ = CTAs per SM. CPS = 2 (one query tile per CTA, d <= 128) gives the
// tensor core two independent tiles per SM from two CTAs instead of one CTA's
// ping-pong pair: half the TMEM (256 columns) and fewer K/V stages each.
// NQ_ = column splits of a query tile over its softmax warpgroups: 2 (two
// warpgroups, 64 S columns per thread) or 4 (four warpgroups, 32 columns per
// thread: half the per-thread softmax chain, for the one-tile S2 schedule).
// BN_ = keys per KV block: 128, or 64 for the P2 pair (NT = 2, NQ = 1: one softmax
// warpgroup per query tile, thread = row, and two 64-column S buffers per tile, so
// S(t, j + 2) is computed while the softmax works on block j + 1 — the S2 overlap
// for both tiles of the pair within the 512 TMEM columns).
template <int D_, int NT_, int EB_ = 2, int CPS_ = 1, int SCHED_ = SCHED_DEFAULT, int NQ_ = 2,
          int BN_ = 128>
struct FwdTraits {
  static constexpr int D = D_;
  static constexpr int NT = NT_;
  static constexpr int NQ = NQ_;
  static constexpr int BN = BN_;
  static constexpr bool P2 = BN == 64;
  static_assert(BN == 128 || (BN == 64 && NT_ == 2 && CPS_ == 1 && SCHED_ == SCHED_DEFAULT && NQ_ == 1),
                "BN = 64 is the P2 pair");
  static_assert(NQ == 2 || (NQ == 4 && NT_ == 1 && CPS_ == 1 && SCHED_ != SCHED_NOWS) ||
                    (NQ == 1 && NT_ == 2 && CPS_ == 1 && SCHED_ == SCHED_DEFAULT),
                "NQ = 4 is one-tile, NQ = 1 a pair with one warpgroup per tile");
  static constexpr int WPT = 4 * NQ;  // softmax warps per query tile
  // P stays in the S columns of the warpgroup that computed it: warpgroup h
  // owns S columns [h BN/NQ, (h+1) BN/NQ) and writes its P codes to the start of
  // them, so no warpgroup's P store lands on S another one has yet to read.
  // PV k-step k (kstep keys = 8 TMEM columns) reads column p_kcol(k).
  __host__ __device__ static constexpr uint32_t p_kcol(int k, int kstep) {
    return (k / ((BN / NQ) / kstep)) * (BN / NQ) + (k % ((BN / NQ) / kstep)) * 8;
  }
  static constexpr int EB = EB_;  // bytes per element (2 f16/bf16, 1 e4m3)
  static constexpr int CPS = CPS_;
  static constexpr int SCHED = SCHED_;
  static_assert(SCHED == SCHED_DEFAULT || (NT == 1 && CPS == 1), "schedule variants are one-tile");
  static constexpr int BM = 128;
  // smem tiles are CHUNKS column chunks of 128 rows x ROW_BYTES, swizzled by the
  // row width: 128 bytes, or 64 (e4m3 at d = 64, 64-byte swizzle)
  static constexpr int ROW_BYTES = D * EB < 128 ? D * EB : 128;
  static constexpr int CHUNK_BYTES = 128 * ROW_BYTES;
  static constexpr int CHUNK_ELEMS = ROW_BYTES / EB;
  static constexpr int CHUNKS = D / CHUNK_ELEMS;
  static constexpr int KPR = ROW_BYTES / 32;       // 32-byte MMA K steps per row chunk
  static constexpr int SBO = 8 * ROW_BYTES;        // stride of 8-row swizzle atoms
  static constexpr int TILE_BYTES = CHUNKS * CHUNK_BYTES;        // a 128-row Q tile
  static constexpr int KV_CHUNK_BYTES = BN * ROW_BYTES;           // a BN-row K/V column chunk
  static constexpr int KV_TILE_BYTES = CHUNKS * KV_CHUNK_BYTES;   // a K or V block
  static constexpr int STAGES0 = CPS == 2 ? (KV_TILE_BYTES <= 16384 ? 4 : 2)
                                          : (KV_TILE_BYTES <= 16384 ? 8 : (KV_TILE_BYTES <= 32768 ? 4 : 2));
  // no warp specialization: the softmax warps issue loads and MMAs themselves
  static constexpr bool NOWS = SCHED == SCHED_NOWS;
  // two softmax warpgroups per query tile, each owning 64 of the 128 columns
  static constexpr int SOFT_REGS = (CPS == 1 && NT == 2) ? FA3B_FWD_REGS : 0;
  static constexpr int NSOFT = NT * WPT;  // softmax warps
  static constexpr int NUM_THREADS = NOWS ? NSOFT * 32 : NSOFT * 32 + (SOFT_REGS > 0 ? 128 : 64);
  static constexpr int LOAD_WARP = NOWS ? -1 : NSOFT;
  static constexpr int MMA_WARP = NOWS ? -1 : NSOFT + 1;
  static constexpr int ALLOC_WARP = NOWS ? 0 : NSOFT + 1;  // barrier init, TMEM alloc / free
  static constexpr uint32_t TMEM_COLS = CPS == 2 ? 256 : 512;
  // one query tile per CTA: a second S buffer after O (see the header)
  static constexpr bool S2 = NT == 1 && CPS == 1 && FA3B_FWD_S2 && SCHED != SCHED_SERIAL;
  static constexpr bool TWO_STAGE = SCHED == SCHED_2STAGE;
  static_assert(!S2 || 2 * 128 + D <= 512, "S2 TMEM budget");
  // d = 64 tile pair: three S buffers rotate between the two tiles (3 x 128 + 2 x 64
  // columns), so each tile's next S is computed during its softmax (see the header)
  static constexpr bool S3 = NT == 2 && D == 64 && CPS == 1 && FA3B_FWD_S3 && !P2;
  static_assert(!S3 || 3 * 128 + 2 * D <= 512, "S3 TMEM budget");
  // QB Q buffers (FA3B_FWD_QB2): with two, the next work item's Q tiles load while
  // this item runs instead of after its last GEMM (~2 us per item boundary in the
  // item trace, profiles/r02/r02ag_items_*.log), where the second buffer fits in
  // shared memory (FP8, d 64, one-tile schedules). Measured +2-4 % on FP8 at
  // N <= 2k and -1-3 % causal (r02ah_qb2_*_ab.log): off by default
  // (FA3B_FWD_QB2_SHRINK: also where it fits only with a two-stage K/V ring)
  static constexpr int smem_for(int qb, int st) {
    return qb * NT * TILE_BYTES + st * KV_TILE_BYTES + (3 + 2 * st + 5 * NT + 2) * 8 + 16 +
           NT * 2 * NQ * 128 * 4 + 1024;
  }
  static constexpr bool QB2_FITS = smem_for(2, STAGES0) <= 232448;
  static constexpr int QB = (FA3B_FWD_QB2 && !(SCHED == SCHED_NOWS) && CPS == 1 &&
                             (QB2_FITS || (FA3B_FWD_QB2_SHRINK && smem_for(2, 2) <= 232448)))
                                ? 2
                                : 1;
  static constexpr int STAGES = (QB == 2 && !QB2_FITS) ? 2 : STAGES0;
  static_assert(!NOWS || STAGES >= 4, "no-WS schedule needs a 4-stage K/V ring");
  static constexpr int OFF_Q = 0;
  static constexpr int OFF_KV = QB * NT * TILE_BYTES;
  // chunk-granular ring (FA3B_FWD_CHRING): RSLOTS barrier pairs of KV_CHUNK_BYTES
  static constexpr bool CH = S2 && FA3B_FWD_CHRING && D == 256 && FA3B_FWD_CHRING_FP8 >= (EB == 1 ? 1 : 0);
  // (+ FA3B_FWD_CHRING_EXTRA chunk slots where shared memory allows: chunks
  // are independent, so the ring need not hold a whole number of tiles; one extra
  // measured no gain, r02ch_chx_ab.log)
  static constexpr int RSLOTS = CH ? STAGES * CHUNKS + FA3B_FWD_CHRING_EXTRA : STAGES;
  static constexpr int OFF_BAR = OFF_KV + (CH ? RSLOTS * KV_CHUNK_BYTES : STAGES * KV_TILE_BYTES);
  // q_full, kv_full[S], kv_empty[S], s_full[2 NT], p_full[NT], o_full[NT], q_empty,
  // pv_done[NT] (the second s_full per tile and pv_done serve S2 / S3), then (QB = 2)
  // the second buffer's q_full, q_empty
  static constexpr int NUM_BARS = 3 + 2 * RSLOTS + 5 * NT + (QB == 2 ? 2 : 0);
  // row-max / row-sum exchange between the column splits: [NT][2 buf][NQ][128]
  static constexpr int OFF_XCH = OFF_BAR + NUM_BARS * 8 + 16;
  static constexpr int SMEM_BYTES = OFF_XCH + NT * 2 * NQ * 128 * 4 + 1024;
  static_assert(NT * (128 + D) <= static_cast<int>(TMEM_COLS), "TMEM budget");
  static_assert(!P2 || NT * (2 * BN + D) <= 512, "P2 TMEM budget");
  static_assert(CPS == 1 || (NT == 1 && SMEM_BYTES * 2 <= 233472), "two CTAs per SM");
  static_assert(SMEM_BYTES <= 232448, "shared memory budget");
  __host__ __device__ static constexpr int s_col(int t) { return t * 128; }
  __host__ __device__ static constexpr int s2_col(int buf) { return buf ? 128 + D : 0; }
  // P2: tile t's S buffer b at (2 t + b) BN, O after the four buffers
  __host__ __device__ static constexpr int p2_col(int t, int b) { return (2 * t + b) * BN; }
  __host__ __device__ static constexpr int o_col(int t) {
    return (S3 ? 384 : (P2 ? NT * 2 * BN : NT * 128)) + t * D;
  }
};

// SCHED_NOWS: the producer and MMA-issuer work of the one-tile S2 schedule, done
// by thread 0 of the softmax warps between its own softmax iterations. K/V go
// through the ring in the S2 order K_0, K_1, {V_j, K_{j+2}}; a load is issued
// only once its slot's previous occupant was consumed by an MMA issued at least
// one iteration earlier (at most STAGES - 2 entries ahead), so the leader's
// kv_empty waits are short; the MMAs follow S_0 ; S_1 ; {PV_j ; S_{j+2}}.
template <class T, bool FP8>
struct NowsLeader {
  uint8_t* smem;
  uint32_t tmem, q_addr, kv_addr;
  const CUtensorMap *tmQ, *tmK, *tmV;
  uint64_t *q_full, *kv_full, *kv_empty, *s_full, *p_full, *o_full, *pv_done;
  uint32_t idesc_qk, idesc_pv;
  int lpos = 0;   // ring loads issued (all items)
  int cpos = 0;   // ring entries consumed by issued MMAs (all items)
  int gs = 0;     // S GEMMs issued (buffer gs & 1)
  int pc = 0;     // p_full phases consumed
  int g0 = 0;     // gs at this item's S_0
  int it_h = 0, it_hkv = 0, it_b = 0, it_n = 0;
  int k_next = 0, v_next = 0, l_item = 0;  // this item's load sequence
  bool v_turn = true;
  __device__ NowsLeader(uint8_t* sm, uint32_t tm, const CUtensorMap* q, const CUtensorMap* k,
                        const CUtensorMap* v, uint64_t* bars, uint32_t iqk, uint32_t ipv)
      : smem(sm), tmem(tm), tmQ(q), tmK(k), tmV(v), idesc_qk(iqk), idesc_pv(ipv) {
    q_addr = ptx::smem_u32(smem + T::OFF_Q);
    kv_addr = ptx::smem_u32(smem + T::OFF_KV);
    q_full = bars;
    kv_full = bars + 1;
    kv_empty = kv_full + T::STAGES;
    s_full = kv_empty + T::STAGES;
    p_full = s_full + 2;
    o_full = p_full + 1;
    pv_done = o_full + 2;
  }
  // issue the item's next loads while their slots were freed an iteration ago
  __device__ void loads() {
    while (l_item < 2 * it_n && lpos < cpos - 2 + T::STAGES) {
      bool is_v;
      int blk;
      if (k_next < 2 && k_next < it_n) {
        is_v = false;
        blk = k_next++;
      } else if (v_next < it_n && (v_turn || k_next >= it_n)) {
        is_v = true;
        blk = v_next++;
        v_turn = false;
      } else {
        is_v = false;
        blk = k_next++;
        v_turn = true;
      }
      const int slot = lpos % T::STAGES;
      ptx::mbar_wait(&kv_empty[slot], ((lpos / T::STAGES) & 1) ^ 1);
      ptx::mbar_arrive_expect_tx(&kv_full[slot], T::KV_TILE_BYTES);
#pragma unroll
      for (int c = 0; c < T::CHUNKS; ++c)
        ptx::tma_load_4d(smem + T::OFF_KV + slot * T::KV_TILE_BYTES + c * T::KV_CHUNK_BYTES,
                         is_v ? tmV : tmK, &kv_full[slot], c * T::CHUNK_ELEMS, it_hkv, blk * 128,
                         it_b, ptx::kEvictLast);
      ++lpos;
      ++l_item;
    }
  }
  __device__ int wait_next() {
    const int slot = cpos % T::STAGES;
    ptx::mbar_wait(&kv_full[slot], (cpos / T::STAGES) & 1);
    ptx::tc_fence_after();
    ++cpos;
    return slot;
  }
  __device__ void s_issue() {
    const int slot = wait_next();
    constexpr int KSTEP = 32 / T::EB;
#pragma unroll
    for (int k = 0; k < T::D / KSTEP; ++k) {
      const uint32_t off = (k / T::KPR) * T::CHUNK_BYTES + (k % T::KPR) * 32;
      const uint32_t offb = (k / T::KPR) * T::KV_CHUNK_BYTES + (k % T::KPR) * 32;
      const uint64_t a = ptx::swz_desc<T::ROW_BYTES>(q_addr + off, 16, T::SBO);
      const uint64_t bd = ptx::swz_desc<T::ROW_BYTES>(kv_addr + slot * T::KV_TILE_BYTES + offb, 16, T::SBO);
      if constexpr (FP8)
        ptx::mma_f8_ss(tmem + T::s2_col(gs & 1), a, bd, idesc_qk, k > 0 ? 1u : 0u);
      else
        ptx::mma_f16_ss(tmem + T::s2_col(gs & 1), a, bd, idesc_qk, k > 0 ? 1u : 0u);
    }
    ptx::mma_commit(&s_full[gs & 1]);
    ptx::mma_commit(&kv_empty[slot]);
    ++gs;
  }
  __device__ void item_start(int h, int hkv, int b, int q_base, int n, int itl) {
    it_h = h;
    it_hkv = hkv;
    it_b = b;
    it_n = n;
    k_next = v_next = l_item = 0;
    v_turn = true;
    g0 = gs;
    if (n == 0) return;
    // Q: every MMA of the previous item has completed (its epilogue waited o_full)
    ptx::mbar_arrive_expect_tx(q_full, T::TILE_BYTES);
#pragma unroll
    for (int c = 0; c < T::CHUNKS; ++c)
      ptx::tma_load_4d(smem + T::OFF_Q + c * T::CHUNK_BYTES, tmQ, q_full, c * T::CHUNK_ELEMS, h,
                       q_base, b, ptx::kEvictFirst);
    loads();
    ptx::mbar_wait(q_full, itl & 1);  // NOWS: one Q buffer
    for (int j = 0; j < 2 && j < n; ++j) s_issue();
    loads();
  }
  // after this thread's own P_j store: wait for every softmax warp, then PV_j and S_{j+2}
  __device__ void after_p(int j, int n) {
    ptx::mbar_wait(p_full, pc++ & 1);
    ptx::tc_fence_after();
    const int slot = wait_next();
    constexpr int KSTEP = 32 / T::EB;
    const uint32_t scol = T::s2_col((g0 + j) & 1);
#pragma unroll
    for (int k = 0; k < T::BN / KSTEP; ++k) {
      const uint64_t bd = ptx::swz_desc<T::ROW_BYTES>(
          kv_addr + slot * T::KV_TILE_BYTES + k * KSTEP * T::ROW_BYTES, T::KV_CHUNK_BYTES, T::SBO);
      if constexpr (FP8)
        ptx::mma_f8_ts(tmem + T::o_col(0), tmem + scol + T::p_kcol(k, KSTEP), bd, idesc_pv,
                       (j > 0 || k > 0) ? 1u : 0u);
      else
        ptx::mma_f16_ts(tmem + T::o_col(0), tmem + scol + T::p_kcol(k, KSTEP), bd, idesc_pv,
                        (j > 0 || k > 0) ? 1u : 0u);
    }
    ptx::mma_commit(pv_done);
    ptx::mma_commit(&kv_empty[slot]);
    if (j + 1 == n) ptx::mma_commit(o_full);
    if (j + 2 < n) s_issue();
    loads();
  }
};

// EMU: how many of every 8 exp2 pairs run on the FMA-pipe polynomial.
#ifndef FA3B_FWD_EMU
#define FA3B_FWD_EMU 2
#endif

template <int D, int NT, bool CAUSAL, int KIND, int CPS = 1, int EMU = FA3B_FWD_EMU,
          int SCHED = SCHED_DEFAULT, int NQ = 2, int BN = 128>
__global__ void __launch_bounds__(FwdTraits<D, NT, KIND == KIND_E4M3 ? 1 : 2, CPS, SCHED, NQ, BN>::NUM_THREADS, CPS)
    fa3b_fwd_kernel(const __grid_constant__ CUtensorMap tmQ,
                    const __grid_constant__ CUtensorMap tmK,
                    const __grid_constant__ CUtensorMap tmV, const FwdArgs args,
                    const uint32_t idesc_qk, const uint32_t idesc_pv) {
  constexpr bool FP8 = KIND == KIND_E4M3;
  constexpr bool BF16 = KIND == KIND_BF16;
  using T = FwdTraits<D, NT, FP8 ? 1 : 2, CPS, SCHED, NQ, BN>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>(
      (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~static_cast<uintptr_t>(1023));
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + T::OFF_BAR);
  uint64_t* q_full = bars;
  uint64_t* kv_full = bars + 1;
  uint64_t* kv_empty = kv_full + T::RSLOTS;
  uint64_t* s_full = kv_empty + T::RSLOTS;
  uint64_t* p_full = s_full + 2 * NT;  // S2 / S3: s_full[2 t + (S count of tile t & 1)]
  uint64_t* o_full = p_full + NT;
  uint64_t* q_empty = o_full + NT;  // the Q tiles of a work item are consumed
  uint64_t* pv_done = q_empty + 1;  // S2 / S3: [t] PV of tile t complete
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + T::NUM_BARS);
  // Q buffer of work item itl (QB = 2: alternating), its barriers and phase parity
  uint64_t* const q_full2 = pv_done + NT;
  uint64_t* const q_empty2 = q_full2 + 1;
  auto qbuf = [](int itl) { return T::QB == 2 ? (itl & 1) : 0; };
  auto qf = [&](int itl) { return qbuf(itl) ? q_full2 : q_full; };
  auto qe = [&](int itl) { return qbuf(itl) ? q_empty2 : q_empty; };
  auto qpar = [](int itl) { return static_cast<uint32_t>(T::QB == 2 ? (itl >> 1) & 1 : itl & 1); };
  auto qoff = [&](int itl) { return static_cast<uint32_t>(qbuf(itl) * NT * T::TILE_BYTES); };

  const int warp = static_cast<int>(ptx::warp_id());
#ifdef FA3B_TRACE
  if (threadIdx.x == 0) {
    FA3B_CTA(0, fa3b_gtime());
    FA3B_CTA(1, fa3b_smid());
  }
#endif
  // Persistent: CTA c walks work items c, c + gridDim.x, ... of a fixed order.
  // Non-causal: query blocks of one head adjacent (K/V reuse in L2). Causal:
  // longest first across all heads (query blocks from the bottom of the mask up,
  // every head at each step), so the static round-robin stays balanced.
  // (kept as expressions of the kernel arguments, not values computed before the
  // role split: each role re-derives them from the constant bank instead of
  // carrying them in registers, which the 96-register softmax cannot afford)
#define N (fwd_seqlen(args))
#define nqb ((fwd_seqlen(args) + NT * 128 - 1) / (NT * 128))
#define HB (args.H * args.B)
#define num_items (nqb * HB)
#define nkv ((fwd_seqlen(args) + T::BN - 1) / T::BN)
  struct Item {
    int qb, h, b, hkv, q_base, n_max;
    int n_t[NT];
  };
  // k-th work item of this CTA: round-robin; causal rounds alternate direction
  // (boustrophedon) so the heavier items of each round do not land on the same CTAs
  auto item_of = [&](int k) {
    const int G = static_cast<int>(gridDim.x), c = static_cast<int>(blockIdx.x);
    return k * G + ((CAUSAL && (k & 1)) ? G - 1 - c : c);
  };
  auto decode = [&](int lin) {
    Item w;
    const int hb = CAUSAL ? lin % HB : lin / nqb;
    w.qb = CAUSAL ? nqb - 1 - lin / HB : lin % nqb;
    w.h = hb % args.H;
    w.b = hb / args.H;
    w.hkv = w.h / args.group;
    w.q_base = w.qb * NT * 128;
    w.n_max = 0;
#pragma unroll
    for (int t = 0; t < NT; ++t) {
      const int r0 = w.q_base + t * 128;
      w.n_t[t] = (r0 < N) ? (CAUSAL ? min(nkv, (r0 + 128) / T::BN) : nkv) : 0;
      w.n_max = max(w.n_max, w.n_t[t]);
    }
    return w;
  };

  if (warp == T::ALLOC_WARP) {
    if (ptx::lane_id() == 0) {
      ptx::mbar_init(q_full, 1);
      for (int s = 0; s < T::RSLOTS; ++s) {
        ptx::mbar_init(&kv_full[s], 1);
        ptx::mbar_init(&kv_empty[s], 1);
      }
      for (int t = 0; t < NT; ++t) {
        ptx::mbar_init(&s_full[2 * t], 1);
        ptx::mbar_init(&s_full[2 * t + 1], 1);
        ptx::mbar_init(&pv_done[t], 1);
        ptx::mbar_init(&p_full[t], T::WPT);  // one arrival per softmax warp
        ptx::mbar_init(&o_full[t], 1);
      }
      ptx::mbar_init(q_empty, 1);
      if constexpr (T::QB == 2) {
        ptx::mbar_init(q_full2, 1);
        ptx::mbar_init(q_empty2, 1);
      }
      ptx::fence_mbar_init();
    }
    __syncwarp();
    ptx::tmem_alloc<T::TMEM_COLS>(tmem_slot);
  }
  if (warp == (T::NOWS ? 0 : T::LOAD_WARP) && ptx::lane_id() == 0) {
    ptx::prefetch_tmap(&tmQ);
    ptx::prefetch_tmap(&tmK);
    ptx::prefetch_tmap(&tmV);
  }
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  // TMEM base: re-read from shared memory inside each role (a value carried across
  // the role split is one more register the softmax would spill)
#define FA3B_TMEM_BASE (*reinterpret_cast<volatile uint32_t*>(tmem_slot))

  if constexpr (T::SOFT_REGS > 0) {
    static_assert(NT * 8 * T::SOFT_REGS + 4 * FA3B_FWD_OREGS <= (T::NUM_THREADS / 32) * 96, "register pool");
    if (warp >= T::NSOFT)
      ptx::setmaxnreg_dec<FA3B_FWD_OREGS>();
  }
  if (warp == T::LOAD_WARP) {
    // ------------------------------------------------------------ producer
    if (ptx::elect_one()) {
      int item = 0;  // K / V loads so far (the ring position)
      int itl = 0;   // work items so far
      for (int lin = item_of(0); lin < num_items; lin = item_of(++itl)) {
        const Item w = decode(lin);
        // FA3B_FWD_QPREFETCH: the next item's Q tiles into L2 now, so its TMA load (which
        // waits for q_empty) finds them there; measured no gain, off
        // (profiles/r02/r02ad_qprefetch_ab.log)
#if FA3B_FWD_QPREFETCH
        if (const int nxt = item_of(itl + 1); nxt < num_items) {
          const Item wn = decode(nxt);
#pragma unroll
          for (int t = 0; t < NT; ++t) {
            if (wn.n_t[t] == 0) continue;
#pragma unroll
            for (int c = 0; c < T::CHUNKS; ++c)
              ptx::tma_prefetch_4d(&tmQ, c * T::CHUNK_ELEMS, wn.h, wn.q_base + t * 128, wn.b);
          }
        }
#endif
        auto load_q = [&]() {
          // the buffer's previous item has read it (QB = 2: two items back)
          if (itl >= T::QB) ptx::mbar_wait(qe(itl), qpar(itl - T::QB));
          int nvalid = 0;
#pragma unroll
          for (int t = 0; t < NT; ++t) nvalid += w.n_t[t] > 0;
          ptx::mbar_arrive_expect_tx(qf(itl), nvalid * T::TILE_BYTES);
          FA3B_IT(itl, 0);
#pragma unroll
          for (int t = 0; t < NT; ++t) {
            if (w.n_t[t] == 0) continue;
#pragma unroll
            for (int c = 0; c < T::CHUNKS; ++c)
              ptx::tma_load_4d(smem + T::OFF_Q + qoff(itl) + t * T::TILE_BYTES + c * T::CHUNK_BYTES, &tmQ,
                               qf(itl), c * T::CHUNK_ELEMS, w.h, w.q_base + t * 128, w.b,
                               ptx::kEvictFirst);
          }
        };
        auto load_kv = [&](bool is_v, int blk) {
          if constexpr (T::CH) {
#pragma unroll
            for (int c = 0; c < T::CHUNKS; ++c) {
              const int ci = item * T::CHUNKS + c, cs = ci % T::RSLOTS;
              ptx::mbar_wait(&kv_empty[cs], ((ci / T::RSLOTS) & 1) ^ 1);
              ptx::mbar_arrive_expect_tx(&kv_full[cs], T::KV_CHUNK_BYTES);
              ptx::tma_load_4d(smem + T::OFF_KV + cs * T::KV_CHUNK_BYTES, is_v ? &tmV : &tmK, &kv_full[cs],
                               c * T::CHUNK_ELEMS, w.hkv, blk * T::BN, w.b, ptx::kEvictLast);
            }
            ++item;
            return;
          }
          const int slot = item % T::STAGES;
          const uint32_t ph = (item / T::STAGES) & 1;
          ptx::mbar_wait(&kv_empty[slot], ph ^ 1);
          ptx::mbar_arrive_expect_tx(&kv_full[slot], T::KV_TILE_BYTES);
          uint8_t* dst = smem + T::OFF_KV + slot * T::KV_TILE_BYTES;
#pragma unroll
          for (int c = 0; c < T::CHUNKS; ++c)
            ptx::tma_load_4d(dst + c * T::KV_CHUNK_BYTES, is_v ? &tmV : &tmK, &kv_full[slot],
                             c * T::CHUNK_ELEMS, w.hkv, blk * T::BN, w.b, ptx::kEvictLast);
          ++item;
        };
        if constexpr (T::S2 || T::S3 || T::P2) {
          // the MMA warp's order: K_0, K_1, { V_j, K_{j+2} }_j
          const int n = w.n_max;
          if constexpr (T::QB == 2) load_q();  // ahead of this item's K/V
          load_kv(false, 0);
          if (n > 1) load_kv(false, 1);
          if constexpr (T::QB == 1) load_q();
          for (int j = 0; j < n; ++j) {
            load_kv(true, j);
            if (j + 2 < n) load_kv(false, j + 2);
          }
        } else {
          // this item's first K/V block streams into the ring while the previous
          // item's last GEMMs still hold the Q buffer
          if constexpr (T::QB == 2) load_q();  // ahead of this item's K/V
          for (int j = 0; j < w.n_max; ++j) {
            if (T::QB == 1 && j == 1) load_q();
            load_kv(false, j);
            if (j == 0) FA3B_IT(itl, 8);
            load_kv(true, j);
          }
          if (T::QB == 1 && w.n_max == 1) load_q();
        }
      }
    }
  } else if (warp == T::MMA_WARP) {
    // ------------------------------------------------------------ MMA issuer
    if (ptx::elect_one()) {
      const uint32_t tmem = FA3B_TMEM_BASE;
      const uint32_t q_base_addr = ptx::smem_u32(smem + T::OFF_Q);
      uint32_t q_cur = q_base_addr;  // this item's Q buffer
      const uint32_t kv_addr = ptx::smem_u32(smem + T::OFF_KV);
      // one MMA consumes 32 bytes of K: 16 f16/bf16 or 32 e4m3 elements
      constexpr int KSTEP = 32 / T::EB;
      auto issue_qk = [&](int t, int slot, int scol) {
#pragma unroll
        for (int k = 0; k < D / KSTEP; ++k) {
          const uint32_t off = (k / T::KPR) * T::CHUNK_BYTES + (k % T::KPR) * 32;
          const uint32_t offb = (k / T::KPR) * T::KV_CHUNK_BYTES + (k % T::KPR) * 32;
          const uint64_t a = ptx::swz_desc<T::ROW_BYTES>(q_cur + t * T::TILE_BYTES + off, 16, T::SBO);
          const uint64_t bd = ptx::swz_desc<T::ROW_BYTES>(kv_addr + slot * T::KV_TILE_BYTES + offb, 16, T::SBO);
          if constexpr (FP8)
            ptx::mma_f8_ss(tmem + scol, a, bd, idesc_qk, k > 0 ? 1u : 0u);
          else
            ptx::mma_f16_ss(tmem + scol, a, bd, idesc_qk, k > 0 ? 1u : 0u);
        }
      };
      auto issue_pv = [&](int t, int slot, bool acc, int scol) {
#pragma unroll
        for (int k = 0; k < T::BN / KSTEP; ++k) {
          // B = V, MN-major: KSTEP kv rows of ROW_BYTES per step
          const uint64_t bd = ptx::swz_desc<T::ROW_BYTES>(
              kv_addr + slot * T::KV_TILE_BYTES + k * KSTEP * T::ROW_BYTES, T::KV_CHUNK_BYTES, T::SBO);
          // A = P in TMEM: KSTEP elements = 8 columns of 32 bits
          if constexpr (FP8)
            ptx::mma_f8_ts(tmem + T::o_col(t), tmem + scol + T::p_kcol(k, KSTEP), bd, idesc_pv,
                           (acc || k > 0) ? 1u : 0u);
          else
            ptx::mma_f16_ts(tmem + T::o_col(t), tmem + scol + T::p_kcol(k, KSTEP), bd, idesc_pv,
                            (acc || k > 0) ? 1u : 0u);
        }
      };
      // PV with its operand descriptors computed before the wait for P (pinned by an
      // empty asm so they are not sunk below it): only the MMA issue follows P
      auto issue_pv_pre = [&](int t, int slot, bool acc, int scol, uint64_t* p_bar, uint32_t par) {
        constexpr int KS = T::BN / KSTEP;
        uint64_t bd[KS];
        uint32_t ta[KS];
#pragma unroll
        for (int k = 0; k < KS; ++k) {
          bd[k] = ptx::swz_desc<T::ROW_BYTES>(kv_addr + slot * T::KV_TILE_BYTES + k * KSTEP * T::ROW_BYTES,
                                              T::KV_CHUNK_BYTES, T::SBO);
          ta[k] = tmem + scol + T::p_kcol(k, KSTEP);
          asm volatile("" : "+l"(bd[k]), "+r"(ta[k]));
        }
        const uint32_t to = tmem + T::o_col(t);
#if FA3B_MMA_SPIN
        ptx::mbar_wait_spin(p_bar, par);
#else
        ptx::mbar_wait(p_bar, par);
#endif
        ptx::tc_fence_after();
#pragma unroll
        for (int k = 0; k < KS; ++k) {
          if constexpr (FP8)
            ptx::mma_f8_ts(to, ta[k], bd[k], idesc_pv, (acc || k > 0) ? 1u : 0u);
          else
            ptx::mma_f16_ts(to, ta[k], bd[k], idesc_pv, (acc || k > 0) ? 1u : 0u);
        }
      };
      int kvi = 0;  // ring position of this item's K_0
      int itl = 0;
      int pc[NT];   // p_full phases consumed per tile
#pragma unroll
      for (int t = 0; t < NT; ++t) pc[t] = 0;
      if constexpr (T::S2) {
        // One tile, two S buffers (global S index g -> buffer g & 1):
        //   S_0 ; S_1 ; { PV_j ; S_{j+2} }_j
        // S_{j+2} reuses S_j's columns (P_j), issued after PV_j which reads them.
        int gs = 0;  // S GEMMs issued so far
        auto s_issue = [&](int slot) {
          issue_qk(0, slot, T::s2_col(gs & 1));
          ptx::mma_commit(&s_full[gs & 1]);
          ++gs;
        };
        for (int lin = item_of(0); lin < num_items; lin = item_of(++itl)) {
          const Item w = decode(lin);
          const int n = w.n_t[0];
          ptx::mbar_wait(qf(itl), qpar(itl));
          q_cur = q_base_addr + qoff(itl);
          const int g0 = gs;  // global index of this item's S_0
          int pos = kvi;      // ring position, in the producer's order K_0, K_1, {V_j, K_{j+2}}
          auto wait_pos = [&]() {
            ptx::mbar_wait(&kv_full[pos % T::STAGES], (pos / T::STAGES) & 1);
            ptx::tc_fence_after();
            return pos++ % T::STAGES;
          };
          if constexpr (T::CH) {
            // chunk-granular ring: tile position p's chunk c sits in chunk slot
            // (p CHUNKS + c) % RSLOTS with its own barriers
            auto chunk_wait = [&](int p, int c) {
              const int ci = p * T::CHUNKS + c, cs = ci % T::RSLOTS;
              ptx::mbar_wait(&kv_full[cs], (ci / T::RSLOTS) & 1);
              ptx::tc_fence_after();
              return cs;
            };
            auto s_issue_ch = [&](int p) {
              const uint32_t scol = T::s2_col(gs & 1);
#pragma unroll
              for (int c = 0; c < T::CHUNKS; ++c) {
                const int cs = chunk_wait(p, c);
#pragma unroll
                for (int kk = 0; kk < T::KPR; ++kk) {
                  const int k = c * T::KPR + kk;
                  const uint64_t a = ptx::swz_desc<T::ROW_BYTES>(q_cur + c * T::CHUNK_BYTES + kk * 32, 16, T::SBO);
                  const uint64_t bd =
                      ptx::swz_desc<T::ROW_BYTES>(kv_addr + cs * T::KV_CHUNK_BYTES + kk * 32, 16, T::SBO);
                  if constexpr (FP8)
                    ptx::mma_f8_ss(tmem + scol, a, bd, idesc_qk, k > 0 ? 1u : 0u);
                  else
                    ptx::mma_f16_ss(tmem + scol, a, bd, idesc_qk, k > 0 ? 1u : 0u);
                }
                ptx::mma_commit(&kv_empty[cs]);
              }
              ptx::mma_commit(&s_full[gs & 1]);
              ++gs;
            };
            // PV per V chunk: N = CHUNK_ELEMS columns of O
            const uint32_t idesc_pv_c = (idesc_pv & ~(0x3Fu << 17)) | ((T::CHUNK_ELEMS >> 3) << 17);
            auto pv_issue_ch = [&](int p, bool acc, uint32_t scol) {
              ptx::mbar_wait(&p_full[0], pc[0]++ & 1);
              ptx::tc_fence_after();
#pragma unroll
              for (int c = 0; c < T::CHUNKS; ++c) {
                const int cs = chunk_wait(p, c);
#pragma unroll
                for (int k = 0; k < T::BN / KSTEP; ++k) {
                  const uint64_t bd = ptx::swz_desc<T::ROW_BYTES>(
                      kv_addr + cs * T::KV_CHUNK_BYTES + k * KSTEP * T::ROW_BYTES, T::KV_CHUNK_BYTES, T::SBO);
                  if constexpr (FP8)
                    ptx::mma_f8_ts(tmem + T::o_col(0) + c * T::CHUNK_ELEMS, tmem + scol + T::p_kcol(k, KSTEP), bd,
                                   idesc_pv_c, (acc || k > 0) ? 1u : 0u);
                  else
                    ptx::mma_f16_ts(tmem + T::o_col(0) + c * T::CHUNK_ELEMS, tmem + scol + T::p_kcol(k, KSTEP), bd,
                                    idesc_pv_c, (acc || k > 0) ? 1u : 0u);
                }
                ptx::mma_commit(&kv_empty[cs]);
              }
            };
            for (int j = 0; j < 2 && j < n; ++j) s_issue_ch(pos++);
            for (int j = 0; j < n; ++j) {
              pv_issue_ch(pos++, j > 0, T::s2_col((g0 + j) & 1));
              if (itl == 0) FA3B_TP(0, j, 6);
              ptx::mma_commit(&pv_done[0]);
              if (j + 1 == n) ptx::mma_commit(&o_full[0]);
              if (j + 2 < n) s_issue_ch(pos++);
            }
            ptx::mma_commit(qe(itl));
            kvi += 2 * n;
            continue;
          }
          for (int j = 0; j < 2 && j < n; ++j) {
            const int slot = wait_pos();
            s_issue(slot);
            ptx::mma_commit(&kv_empty[slot]);
          }
          for (int j = 0; j < n; ++j) {
            const int slot_v = wait_pos();
            issue_pv_pre(0, slot_v, j > 0, T::s2_col((g0 + j) & 1), &p_full[0], pc[0]++ & 1);
            if (itl == 0) FA3B_TP(0, j, 6);
            ptx::mma_commit(&pv_done[0]);
            ptx::mma_commit(&kv_empty[slot_v]);
            if (j + 1 == n) ptx::mma_commit(&o_full[0]);
            if (j + 2 < n) {
              const int slot_k = wait_pos();
              s_issue(slot_k);
              ptx::mma_commit(&kv_empty[slot_k]);
            }
          }
          ptx::mma_commit(qe(itl));
          kvi += 2 * n;
        }
      } else if constexpr (T::S3) {
        // Two tiles, three S buffers: S(t, j) -> buffer (G + 2 j + t) % 3 with G the
        // item base. Per item: S(0,0) ; S(1,0) ; S(0,1) ;
        //   { PV(0,j) ; S(1,j+1) ; PV(1,j) ; S(0,j+2) }_j
        // Each S reuses the buffer of S number g - 3, whose PV was issued just before.
        int gb = 0;        // G of this item
        int sn[NT] = {};   // S GEMMs issued per tile (s_full parity)
        auto s_issue = [&](int t, int j, int slot) {
          issue_qk(t, slot, 128 * ((gb + 2 * j + t) % 3));
          ptx::mma_commit(&s_full[2 * t + (sn[t] & 1)]);
          ++sn[t];
        };
        for (int lin = item_of(0); lin < num_items; lin = item_of(++itl)) {
          const Item w = decode(lin);
          const int n0 = w.n_t[0], n1 = w.n_t[1], n = w.n_max;
          // the last reader of K_j / V_j releases its ring slot
          auto last_t = [&](int j) { return j < n1 ? 1 : 0; };
          ptx::mbar_wait(qf(itl), qpar(itl));
          q_cur = q_base_addr + qoff(itl);
          int pos = kvi;  // ring position, producer order K_0, K_1, {V_j, K_{j+2}}
          auto wait_pos = [&]() {
            ptx::mbar_wait(&kv_full[pos % T::STAGES], (pos / T::STAGES) & 1);
            ptx::tc_fence_after();
            return pos++ % T::STAGES;
          };
          const int k0 = wait_pos();
          if (n0 > 0) s_issue(0, 0, k0);
          if (n1 > 0) s_issue(1, 0, k0);
          ptx::mma_commit(&kv_empty[k0]);
          int k1 = -1;  // K_1's slot, released by S(1,1)
          if (n > 1) {
            k1 = wait_pos();
            if (n0 > 1) s_issue(0, 1, k1);
            if (last_t(1) == 0) ptx::mma_commit(&kv_empty[k1]);
          }
          int kn = k1;  // slot of K_{j+1}
          for (int j = 0; j < n; ++j) {
            const int slot_v = wait_pos();
            if (j < n0) {
              ptx::mbar_wait(&p_full[0], pc[0]++ & 1);
              ptx::tc_fence_after();
              issue_pv(0, slot_v, j > 0, 128 * ((gb + 2 * j) % 3));
              ptx::mma_commit(&pv_done[0]);
              if (j + 1 == n0) ptx::mma_commit(&o_full[0]);
              if (last_t(j) == 0) ptx::mma_commit(&kv_empty[slot_v]);
            }
            if (j + 1 < n1) {
              s_issue(1, j + 1, kn);
              ptx::mma_commit(&kv_empty[kn]);
            }
            if (j < n1) {
              ptx::mbar_wait(&p_full[1], pc[1]++ & 1);
              ptx::tc_fence_after();
              issue_pv(1, slot_v, j > 0, 128 * ((gb + 2 * j + 1) % 3));
              ptx::mma_commit(&pv_done[1]);
              if (j + 1 == n1) ptx::mma_commit(&o_full[1]);
              ptx::mma_commit(&kv_empty[slot_v]);
            }
            if (j + 2 < n) {
              kn = wait_pos();
              if (j + 2 < n0) s_issue(0, j + 2, kn);
              if (last_t(j + 2) == 0) ptx::mma_commit(&kv_empty[kn]);
            }
          }
          ptx::mma_commit(qe(itl));
          kvi += 2 * n;
          gb += 2 * n;
        }
      } else if constexpr (T::P2) {
        // Two tiles, two BN-column S buffers each (tile t's S number g in buffer g & 1).
        // Per item: S(0,0) ; S(1,0) ; S(0,1) ; S(1,1) ;
        //   { PV(0,j) ; S(0,j+2) ; PV(1,j) ; S(1,j+2) }_j
        // S(t, j+2) reuses the buffer of S(t, j) = P(t, j), issued right after the PV
        // that reads it, so each tile's next S is always one block ahead of its softmax.
        int sn[NT] = {};   // S GEMMs issued per tile
        int pn[NT] = {};   // PV GEMMs issued per tile (P(t, j) in buffer pn & 1)
        auto s_issue = [&](int t, int slot) {
          issue_qk(t, slot, T::p2_col(t, sn[t] & 1));
          ptx::mma_commit(&s_full[2 * t + (sn[t] & 1)]);
          ++sn[t];
        };
        for (int lin = item_of(0); lin < num_items; lin = item_of(++itl)) {
          const Item w = decode(lin);
          const int n0 = w.n_t[0], n1 = w.n_t[1], n = w.n_max;
          ptx::mbar_wait(qf(itl), qpar(itl));
          q_cur = q_base_addr + qoff(itl);
          int pos = kvi;  // ring position, producer order K_0, K_1, {V_j, K_{j+2}}
          auto wait_pos = [&]() {
            ptx::mbar_wait(&kv_full[pos % T::STAGES], (pos / T::STAGES) & 1);
            ptx::tc_fence_after();
            return pos++ % T::STAGES;
          };
          for (int j = 0; j < 2 && j < n; ++j) {
            const int slot = wait_pos();
            if (j < n0) s_issue(0, slot);
            if (j < n1) s_issue(1, slot);
            ptx::mma_commit(&kv_empty[slot]);
          }
          for (int j = 0; j < n; ++j) {
            const int slot_v = wait_pos();
            // K_{j+2}'s ring entry, waited for only when its first S is issued
            const int kpos = j + 2 < n ? pos++ : -1;
            bool k_ready = false;
#pragma unroll
            for (int t = 0; t < NT; ++t) {
              if (j < w.n_t[t]) {
                issue_pv_pre(t, slot_v, j > 0, T::p2_col(t, pn[t] & 1), &p_full[t], pc[t]++ & 1);
                ++pn[t];
                ptx::mma_commit(&pv_done[t]);
                if (j + 1 == w.n_t[t]) ptx::mma_commit(&o_full[t]);
              }
              if (j + 2 < w.n_t[t]) {
                if (!k_ready) {
                  ptx::mbar_wait(&kv_full[kpos % T::STAGES], (kpos / T::STAGES) & 1);
                  ptx::tc_fence_after();
                  k_ready = true;
                }
                s_issue(t, kpos % T::STAGES);
              }
            }
            ptx::mma_commit(&kv_empty[slot_v]);
            if (kpos >= 0) ptx::mma_commit(&kv_empty[kpos % T::STAGES]);
          }
          ptx::mma_commit(qe(itl));
          kvi += 2 * n;
        }
      } else
      for (int lin = item_of(0); lin < num_items; lin = item_of(++itl)) {
        const Item w = decode(lin);
        ptx::mbar_wait(qf(itl), qpar(itl));
        q_cur = q_base_addr + qoff(itl);
        FA3B_IT(itl, 1);
        {
          const int slot0 = kvi % T::STAGES;
          ptx::mbar_wait(&kv_full[slot0], (kvi / T::STAGES) & 1);
          FA3B_IT(itl, 9);
          ptx::tc_fence_after();
#pragma unroll
          for (int t = 0; t < NT; ++t) {
            if (w.n_t[t] == 0) continue;
            issue_qk(t, slot0, T::s_col(t));
            ptx::mma_commit(&s_full[2 * t]);
          }
          FA3B_IT(itl, 10);
          ptx::mma_commit(&kv_empty[slot0]);
          if (FA3B_FWD_QEARLY && w.n_max == 1) ptx::mma_commit(qe(itl));  // every S issued
        }
        for (int j = 0; j < w.n_max; ++j) {
          const int item_v = kvi + 2 * j + 1, item_k = kvi + 2 * j + 2;
          const int slot_v = item_v % T::STAGES, slot_k = item_k % T::STAGES;
          ptx::mbar_wait(&kv_full[slot_v], (item_v / T::STAGES) & 1);
          bool k_ready = false;
#pragma unroll
          for (int t = 0; t < NT; ++t) {
            if (j >= w.n_t[t]) continue;
#if FA3B_FWD_PV_PRE
            issue_pv_pre(t, slot_v, j > 0, T::s_col(t), &p_full[t], pc[t]++ & 1);
            if (itl == 0) FA3B_TP(t, j, 6);
#else
            ptx::mbar_wait(&p_full[t], pc[t]++ & 1);
            if (itl == 0) FA3B_TP(t, j, 6);
            ptx::tc_fence_after();
            issue_pv(t, slot_v, j > 0, T::s_col(t));
#endif
            if (j + 1 < w.n_t[t]) {
              if (!k_ready) {
                ptx::mbar_wait(&kv_full[slot_k], (item_k / T::STAGES) & 1);
                ptx::tc_fence_after();
                k_ready = true;
              }
              issue_qk(t, slot_k, T::s_col(t));
              ptx::mma_commit(&s_full[2 * t]);
            } else {
              ptx::mma_commit(&o_full[t]);
            }
          }
          ptx::mma_commit(&kv_empty[slot_v]);
          if (k_ready) ptx::mma_commit(&kv_empty[slot_k]);
          // QEARLY: Q is released once the item's last S MMAs complete, so the next
          // item's Q load overlaps this item's last softmax, PVs and epilogue
          if (FA3B_FWD_QEARLY && j + 2 == w.n_max) ptx::mma_commit(qe(itl));
        }
        if (!FA3B_FWD_QEARLY) ptx::mma_commit(qe(itl));  // once every MMA of this item has read Q
        kvi += 2 * w.n_max;
      }
    }
  } else if (warp < T::NSOFT) {
    // ------------------------------------------------------------ softmax
    if constexpr (T::SOFT_REGS > 0) ptx::setmaxnreg_inc<T::SOFT_REGS>();
    const uint32_t tmem = FA3B_TMEM_BASE;
    const int t = warp / T::WPT;         // query tile
    const int hh = (warp >> 2) % NQ;     // column split of S / O
    const int r = ((warp & 3) << 5) | static_cast<int>(ptx::lane_id());  // row == TMEM lane
    const uint32_t lane_base = static_cast<uint32_t>(32 * (warp & 3)) << 16;
    const uint32_t tS0 = tmem + lane_base + T::s_col(t);
    const uint32_t tO = tmem + lane_base + T::o_col(t);
    float* xch = reinterpret_cast<float*>(smem + T::OFF_XCH) + t * (2 * NQ * 128);  // [2 buf][NQ][128]
    const uint32_t bar_id = 1 + t;
    // exp-phase token (FA3B_FWD_PPBAR): tile t waits on barrier 3 + t, hands over on 3 + (1 - t)
    constexpr bool PPB = FA3B_FWD_PPBAR && NT == 2 && CPS == 1 && !T::S3 && !T::P2 && !T::NOWS;
    auto pp_sync = [&]() {
      if constexpr (PPB) ptx::named_bar_sync(3 + t, 2 * NQ * 128);
    };
    auto pp_arrive = [&]() {
      if constexpr (PPB) ptx::named_bar_arrive(3 + (1 - t), 2 * NQ * 128);
    };
    if (t == 1) pp_arrive();  // tile 0 goes first
    int sc = 0, xc = 0, oc = 0;  // s_full / exchange-buffer / o_full uses so far
    int gbase = 0;               // S3: 2 x (KV blocks of this CTA's previous items)
    int itl = 0;
    // no warp specialization (SCHED_NOWS): thread 0 of the softmax warps is also the
    // TMA producer and the MMA issuer, at fixed points of its own softmax loop
    const bool leader = T::NOWS && threadIdx.x == 0;
    NowsLeader<T, FP8> nows(smem, tmem, &tmQ, &tmK, &tmV, bars, idesc_qk, idesc_pv);
    for (int lin = item_of(0); lin < num_items; lin = item_of(++itl)) {
    const Item w = decode(lin);
    const int b = w.b, h = w.h, hkv = w.hkv, q_base = w.q_base;
    const int q_row = q_base + t * 128 + r;
    if constexpr (T::NOWS)
      if (leader) nows.item_start(w.h, w.hkv, w.b, w.q_base, w.n_t[0], itl);
    const int nt = (t == 0) ? w.n_t[0] : w.n_t[NT - 1];
    constexpr int HC = T::BN / NQ;       // S columns per thread
    constexpr int DH = D / NQ;           // O columns per thread
    constexpr int CW = DH < 32 ? DH : 32;  // O columns per TMEM load / store
    auto tmem_ldw = [](uint32_t a, uint32_t (&v)[CW]) {
      if constexpr (CW == 32) ptx::tmem_ld32(a, v); else ptx::tmem_ld16(a, v);
    };
    auto tmem_stw = [](uint32_t a, const uint32_t (&v)[CW]) {
      if constexpr (CW == 32) ptx::tmem_st32(a, v); else ptx::tmem_st16(a, v);
    };
    auto rescale_o = [&](float f) {
      constexpr int NC = DH / CW;
      constexpr int G = NC < 4 ? NC : 4;
#pragma unroll
      for (int c0 = 0; c0 < NC; c0 += G) {
        uint32_t ov[G][CW];
#pragma unroll
        for (int c = 0; c < G; ++c) tmem_ldw(tO + DH * hh + (c0 + c) * CW, ov[c]);
        ptx::tmem_wait_ld();
#pragma unroll
        for (int c = 0; c < G; ++c) {
#pragma unroll
          for (int i = 0; i < CW; ++i) ov[c][i] = __float_as_uint(__uint_as_float(ov[c][i]) * f);
          tmem_stw(tO + DH * hh + (c0 + c) * CW, ov[c]);
        }
      }
    };
    float sl2 = args.scale_log2;
    const float thr = FP8 ? args.fp8_thr : 8.f;
    float out_scale = 1.f;
    int ks_base = 0;  // FP8: index of this (batch, kv head)'s first K / V block scale
    if constexpr (FP8) {
      const size_t hq = static_cast<size_t>(b) * args.H + h;
      const size_t hk = static_cast<size_t>(b) * args.Hkv + hkv;
      const int nqb_all = (N + 127) / 128;
      // a tile past N (nt == 0, odd block count in the pair path) has no scale
      if (nt > 0)
        sl2 *= args.q_blocked ? args.q_scale[hq * nqb_all + q_base / 128 + t] : args.q_scale[hq];
      ks_base = static_cast<int>(args.kv_blocked ? hk * nqb_all : hk);  // 128-row scale blocks
    }
    float v_cur = 0.f;  // V scale the O accumulator is expressed in (FP8)
    float m_use = -INFINITY;  // running max in use, scaled log2 units (same in both halves)
    float l = 0.f;            // this half's share of the row sum
    // FP8: e4m3 codes of P are P * 448 / 2^thr; exp2(x + log2 pmul) produces them directly
    const float inv_pmul = FP8 ? args.fp8_inv_pmul : 1.f;
    const float lpm = FP8 ? args.fp8_lpm : 0.f;
    // per-block K / V scales of the next block are fetched one iteration ahead
    float ks_next = 1.f, vs_next = 1.f;
    const float* ksp = FP8 ? args.k_scale + ks_base : nullptr;
    const float* vsp = FP8 ? args.v_scale + ks_base : nullptr;
    if constexpr (FP8) {
      if (nt > 0) {
        ks_next = ksp[0];
        vs_next = vsp[0];
      }
    }
    // the block loop body; SPEC (compile time) = exps may start before the max
    // exchange (blocks j >= 1 with FA3B_FWD_SPEC), block 0 never speculates
    auto block = [&](const int j, auto spec_c) {
      constexpr bool SPEC = decltype(spec_c)::value;
      float slj = sl2;
      float vfac = 1.f;  // O rescale for a new V block scale (uniform across the CTA)
      float lrho = 0.f, inv_rho = 1.f;  // FP8: V-scale ratio folded into this block's P
      if constexpr (FP8) {
        slj = sl2 * ks_next;
        const float vs = vs_next;
        if (args.kv_blocked && j + 1 < nt) {  // scales are per 128-key block
          ks_next = ksp[((j + 1) * T::BN) >> 7];
          vs_next = vsp[((j + 1) * T::BN) >> 7];
        }
        if (vs != v_cur) {
          // O stays in units of v_cur while rho = s_v[j] / v_cur is an exact power of
          // two in [2^-8, 1] (equal mantissas): rho then scales this block's P codes
          // exactly (an exponent shift), so O is rescaled only at a new maximum of the
          // V scales. Per-block V scales that are powers of two (fa3b_fp8_prepare with
          // scale_pow2, as the FP8 forward quantizes V) fold at every other block; any
          // other ratio rescales O to s_v[j], the reference's exact per-block
          // s_v (fp8_attention.cpp:158-164).
          const uint32_t ub = __float_as_uint(vs), uc = __float_as_uint(v_cur);
          const int de = static_cast<int>(ub >> 23) - static_cast<int>(uc >> 23);
          if (((ub ^ uc) & 0x807FFFFFu) == 0 && de <= 0 && de >= -8 && v_cur != 0.f) {
            lrho = static_cast<float>(de);
            inv_rho = __uint_as_float(static_cast<uint32_t>(127 - de) << 23);
          } else {
            vfac = v_cur == 0.f ? 0.f : __fdividef(v_cur, vs);  // 0 on the first block: O is empty
            v_cur = vs;
          }
        }
      }
      const bool tr = itl == 0 && (warp % T::WPT) == 0 && ptx::lane_id() == 0;
      if (tr) FA3B_TP(t, j, 0);
      // 2-stage order (flash_fwd.cpp:148-169): softmax_j begins once PV_{j-1} is done
      if constexpr (T::TWO_STAGE)
        if (j > 0) ptx::mbar_wait(&pv_done[t], (sc - 1) & 1);
      if constexpr (T::S2 || T::S3 || T::P2)
        ptx::mbar_wait(&s_full[2 * t + (sc & 1)], (sc >> 1) & 1);
      else
        ptx::mbar_wait(&s_full[2 * t], sc & 1);
      ++sc;
      // S2: S / P of this block live in buffer (sc - 1) & 1
      // S3: S(t, j) lives in buffer (item base + 2 j + t) % 3
      // P2: S(t, j) lives in tile t's buffer (sc - 1) & 1
      const uint32_t tS = T::S2   ? tmem + lane_base + T::s2_col((sc - 1) & 1)
                          : T::S3 ? tmem + lane_base + 128 * ((gbase + 2 * j + t) % 3)
                          : T::P2 ? tmem + lane_base + T::p2_col(t, (sc - 1) & 1)
                                  : tS0;
      if (tr) FA3B_TP(t, j, 1);
#ifdef FA3B_TRACE
      if (itl == 0 && j == 0 && threadIdx.x == 0) FA3B_CTA(3, fa3b_gtime());
      if (j == 0 && (warp % T::WPT) == 0 && ptx::lane_id() == 0) FA3B_IT(itl, 2 + 3 * t);
#endif
      ptx::tc_fence_after();
      float s[HC];
      const int kv0 = j * T::BN + HC * hh;
      const bool need_mask = (j * T::BN + T::BN > N) || (CAUSAL && j * T::BN + T::BN - 1 > q_base + t * 128);
      auto load_s = [&]() {
        uint32_t sr[HC];
#pragma unroll
        for (int c = 0; c < HC / 32; ++c)
          ptx::tmem_ld32(tS + HC * hh + 32 * c, *reinterpret_cast<uint32_t(*)[32]>(&sr[32 * c]));
        ptx::tmem_wait_ld();
#pragma unroll
        for (int i = 0; i < HC; ++i) s[i] = __uint_as_float(sr[i]);
        if (need_mask) {
          const int lim = (CAUSAL ? min(q_row + 1, N) : N) - kv0;
#pragma unroll
          for (int i = 0; i < HC; ++i) s[i] = (i < lim) ? s[i] : -INFINITY;
        }
      };
      load_s();
      if (tr) FA3B_TP(t, j, 2);
      // partial row max: FMNMX3 over 4 independent chains, then exchange with the
      // other column splits of the row
      float a0 = s[0], a1 = s[1], a2 = s[2], a3 = s[3];
#pragma unroll
      for (int i = 4; i + 8 <= HC; i += 8) {
        a0 = ptx::max3(a0, s[i], s[i + 1]);
        a1 = ptx::max3(a1, s[i + 2], s[i + 3]);
        a2 = ptx::max3(a2, s[i + 4], s[i + 5]);
        a3 = ptx::max3(a3, s[i + 6], s[i + 7]);
      }
      a0 = ptx::max3(a0, s[HC - 4], s[HC - 3]);
      a1 = ptx::max3(a1, s[HC - 2], s[HC - 1]);
      const float pm = fmaxf(ptx::max3(a0, a1, a2), a3);
      float* xb = xch + (xc & 1) * (NQ * 128);
      ++xc;
      if constexpr (NQ > 1) ptx::sts_f32(xb + hh * 128 + r, pm);
      // P = 2^(s * slj - msub) for this half: FFMA2 pairs; EMU of every 8 pairs go
      // through the FMA-pipe polynomial, the rest through MUFU.EX2; FADD2 sums.
      constexpr int NPK = FP8 ? HC / 4 : HC / 2;
      uint32_t pk[NPK];
      float psum = 0.f;
      auto exp_half = [&](float msub) {
        const float2 sc2 = make_float2(slj, slj),
                     nm2 = make_float2(lpm + lrho - msub, lpm + lrho - msub);
        float2 acc[4] = {make_float2(0.f, 0.f), make_float2(0.f, 0.f), make_float2(0.f, 0.f),
                         make_float2(0.f, 0.f)};
        float2 prev = make_float2(0.f, 0.f);
#pragma unroll
        for (int i = 0; i < HC / 2; ++i) {
          const float2 x = __ffma2_rn(make_float2(s[2 * i], s[2 * i + 1]), sc2, nm2);
          float2 pp;
          if ((i & 7) < EMU) {
            pp = FP8 ? ptx::ex2_poly2_d2(x) : ptx::ex2_poly2(x);
          } else {
            pp.x = ptx::ex2(x.x);
            pp.y = ptx::ex2(x.y);
          }
          acc[i & 3] = __fadd2_rn(acc[i & 3], pp);
          if constexpr (FP8) {
            if (i & 1)
              pk[i >> 1] = ptx::pack_e4m3x4(prev.x, prev.y, pp.x, pp.y);
            else
              prev = pp;
          } else {
            pk[i] = BF16 ? ptx::pack_bf16(pp.x, pp.y) : ptx::pack_f16(pp.x, pp.y);
          }
          // PSPLIT: the first half of P goes to TMEM as soon as it is packed, which
          // frees its registers for the second half (the exchange barrier has already
          // ordered every split's S load before these stores)
          if constexpr (FA3B_FWD_PSPLIT && NPK >= 16) {
            if (i == HC / 4 - 1) {
              if constexpr (NPK == 16)
                ptx::tmem_st8(tS + HC * hh, *reinterpret_cast<uint32_t(*)[8]>(&pk[0]));
              else
                ptx::tmem_st16(tS + HC * hh, *reinterpret_cast<uint32_t(*)[16]>(&pk[0]));
            }
          }
        }
        const float2 a4 = __fadd2_rn(__fadd2_rn(acc[0], acc[1]), __fadd2_rn(acc[2], acc[3]));
        psum = a4.x + a4.y;
      };
      // also: every split's S load of this tile has completed (NQ = 1: a thread's own
      // tcgen05.wait::ld orders its S load before its P store)
      // FA3B_FWD_SPEC: after the first block the exps start with the running max in
      // use, before the half-row max exchange completes (P <= 2^thr unless the block
      // raises the max by more than thr, which is then redone with the new max), so
      // the exchange barrier overlaps the exps instead of preceding them.
      // SPEC: the S values die in the speculative exps; a redo (the block raised the
      // max by more than thr) reloads S from TMEM, which the P store has not touched yet
      if constexpr (SPEC) exp_half(m_use);
      if constexpr (NQ > 1) ptx::named_bar_sync(bar_id, NQ * 128);
      float mx = pm;
#pragma unroll
      for (int q = 1; q < NQ; ++q) mx = fmaxf(mx, ptx::lds_f32(xb + ((hh + q) % NQ) * 128 + r));
      if (tr) FA3B_TP(t, j, 3);
      const float m_new = fmaxf(m_use, mx * slj);
      const bool resc = m_new > m_use + thr;
      const float m_cur = resc ? m_new : m_use;
      const float factor = resc ? ptx::ex2(m_use - m_new) : 1.f;
      pp_sync();
      if constexpr (SPEC) {
        // tcgen05.ld is warp-collective: the whole warp reloads if any row redoes
        if (__any_sync(0xffffffffu, resc)) {
          load_s();
          if (resc) exp_half(m_cur);
        }
      } else {
        exp_half((m_cur == -INFINITY) ? 0.f : m_cur);
      }
      // P (packed, key order) over the first columns of this warpgroup's own S
      // columns (FwdTraits::p_kcol), which only this thread's row has read
      if constexpr (FA3B_FWD_PSPLIT && NPK >= 16) {
        if constexpr (NPK == 16)
          ptx::tmem_st8(tS + HC * hh + 8, *reinterpret_cast<uint32_t(*)[8]>(&pk[8]));
        else
          ptx::tmem_st16(tS + HC * hh + 16, *reinterpret_cast<uint32_t(*)[16]>(&pk[16]));
      } else if constexpr (NPK == 8) {
        ptx::tmem_st8(tS + HC * hh, *reinterpret_cast<uint32_t(*)[8]>(&pk[0]));
      } else if constexpr (NPK == 16) {
        ptx::tmem_st16(tS + HC * hh, *reinterpret_cast<uint32_t(*)[16]>(&pk[0]));
      } else if constexpr (NPK == 32) {
        ptx::tmem_st32(tS + HC * hh, *reinterpret_cast<uint32_t(*)[32]>(&pk[0]));
      } else {  // NPK = 64: a whole 128-key row of 16-bit P (NQ = 1)
        ptx::tmem_st32(tS, *reinterpret_cast<uint32_t(*)[32]>(&pk[0]));
        ptx::tmem_st32(tS + 32, *reinterpret_cast<uint32_t(*)[32]>(&pk[32]));
      }
      pp_arrive();
      l = l * factor + psum * (inv_pmul * inv_rho);
      if (tr) FA3B_TP(t, j, 4);
      const float ofac = factor * vfac;
      // S2: every iteration waits for PV(V_{j-1}) before handing over P_j, so one
      // PV is in flight at a time and the pv_done parity never skips a phase (a
      // wait only when O needs rescaling hung at bf16 d = 256)
      if constexpr ((T::S2 || T::S3 || T::P2) && !T::TWO_STAGE)
        if (j > 0) ptx::mbar_wait(&pv_done[t], (sc - 2) & 1);
      // PV(V_{j-1}) is complete (see header / above); rescale this thread's O_t columns.
      if (j > 0 && __any_sync(0xffffffffu, ofac != 1.f)) rescale_o(ofac);
      if (tr) FA3B_TP(t, j, 7);
      ptx::tmem_wait_st();
      ptx::tc_fence_before();
      __syncwarp();
      if (tr) FA3B_TP(t, j, 5);
      if (ptx::lane_id() == 0) ptx::mbar_arrive(&p_full[t]);  // one arrival per warp
#ifdef FA3B_TRACE
      if (j + 1 == nt && (warp % T::WPT) == 0 && ptx::lane_id() == 0) FA3B_IT(itl, 3 + 3 * t);
#endif
      m_use = m_cur;
      if constexpr (T::NOWS)
        if (leader) nows.after_p(j, nt);
    };
    if (nt > 0) block(0, std::false_type{});
    for (int j = 1; j < nt; ++j) {
      if constexpr (FA3B_FWD_SPEC)
        block(j, std::true_type{});
      else
        block(j, std::false_type{});
    }
    // token slots of the item's blocks this tile does not have (causal: tile 0 has fewer)
    for (int j = nt; j < w.n_max; ++j) {
      pp_sync();
      pp_arrive();
    }
    if (nt > 0) {
      // ---------------------------------------------------------- epilogue
      float* xb = xch + (xc & 1) * (NQ * 128);
      ++xc;
      if constexpr (NQ > 1) {
        ptx::sts_f32(xb + hh * 128 + r, l);
        ptx::named_bar_sync(bar_id, NQ * 128);
      }
      {
        // the row sum in a fixed order of the splits (the same in every thread of the row)
        float lt = 0.f;
#pragma unroll
        for (int q = 0; q < NQ; ++q) lt += q == hh ? l : ptx::lds_f32(xb + q * 128 + r);
        l = lt;
      }
      ptx::mbar_wait(&o_full[t], oc & 1);
      ++oc;
      ptx::tc_fence_after();
      if constexpr (FP8) out_scale = v_cur * inv_pmul;
      const float inv = l > 0.f ? out_scale / l : 0.f;
      const bool row_ok = q_row < N;
      const size_t obase = static_cast<size_t>(b) * args.o_sb +
                           static_cast<size_t>(q_row) * args.o_ss +
                           static_cast<size_t>(h) * args.o_sh + DH * hh;
#pragma unroll
      for (int c = 0; c < DH / CW; ++c) {
        uint32_t ov[CW];
        tmem_ldw(tO + DH * hh + c * CW, ov);
        ptx::tmem_wait_ld();
        if (!row_ok) continue;
        if (args.out_f32) {
          float4* dst = reinterpret_cast<float4*>(static_cast<float*>(args.o) + obase + c * CW);
#pragma unroll
          for (int i = 0; i < CW / 4; ++i)
            dst[i] = make_float4(__uint_as_float(ov[4 * i]) * inv,
                                 __uint_as_float(ov[4 * i + 1]) * inv,
                                 __uint_as_float(ov[4 * i + 2]) * inv,
                                 __uint_as_float(ov[4 * i + 3]) * inv);
        } else {
          uint32_t pk[CW / 2];
#pragma unroll
          for (int i = 0; i < CW / 2; ++i) {
            const float a = __uint_as_float(ov[2 * i]) * inv;
            const float bb = __uint_as_float(ov[2 * i + 1]) * inv;
            pk[i] = (BF16 || FP8) ? ptx::pack_bf16(a, bb) : ptx::pack_f16(a, bb);
          }
          uint16_t* orow = static_cast<uint16_t*>(args.o) + obase + c * CW;
          if (CW % 16 == 0 && args.o_v8) {
            // one sector per lane and instruction (STG.256): half the store wavefronts
#pragma unroll
            for (int i = 0; i < CW / 16; ++i)
              ptx::st_global_v8(orow + 16 * i, &pk[8 * i]);
          } else {
            uint4* dst = reinterpret_cast<uint4*>(orow);
#pragma unroll
            for (int i = 0; i < CW / 8; ++i)
              dst[i] = make_uint4(pk[4 * i], pk[4 * i + 1], pk[4 * i + 2], pk[4 * i + 3]);
          }
        }
      }
      if (hh == 0 && row_ok && args.lse != nullptr) {
        const float lse = l > 0.f ? (m_use + log2f(l)) * 0.69314718055994531f : -INFINITY;
        args.lse[(static_cast<size_t>(b) * args.H + h) * N + q_row] = lse;
      }
    }
#ifdef FA3B_TRACE
    if (nt > 0 && (warp % T::WPT) == 0 && ptx::lane_id() == 0) FA3B_IT(itl, 4 + 3 * t);
#endif
    gbase += 2 * w.n_max;
    }  // work items
    if (t == 0) pp_sync();  // tile 1's last hand-over
  }

  ptx::tc_fence_before();
  __syncthreads();
#ifdef FA3B_TRACE
  if (threadIdx.x == 0) FA3B_CTA(2, fa3b_gtime());
#endif
  if (warp == T::ALLOC_WARP) {
    ptx::tc_fence_after();
    ptx::tmem_dealloc<T::TMEM_COLS>(FA3B_TMEM_BASE);
  }
}

#undef FA3B_TMEM_BASE
#undef N
#undef nqb
#undef HB
#undef num_items
#undef nkv

}  // namespace fa3b
