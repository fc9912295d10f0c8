// Attention backward on sm_100a (reference flash_bwd, core/src/flash_bwd.cpp:29-126).
//
//   K2 fa3b_bwd_prep_kernel   D = rowsum(dO o O) (bwd_preprocess, :29-41), the LSE in
//                             log2 units, both padded to a multiple of 128 rows with
//                             D = 0, LSE2 = +inf (so padded query columns get P = 0)
//   K3 fa3b_bwd_kernel        KV-outer / Q-inner main loop (:58-110), one CTA per
//                             (128-row KV tile, KV head, batch); the Q tiles of every
//                             query head in the GQA group stream through it
//   K4 fa3b_bwd_dq_kernel     dQ = alpha * dQaccum -> 16-bit (the alpha fold, :121-124)
//
// K3 computes the transposed scores so KV rows are TMEM lanes:
//   S^T  = K Q^T      (tcgen05 SS, TMEM cols [0,128))
//   dP^T = V dO^T     (tcgen05 SS, TMEM cols [128,256))
//   P^T  = exp2(S^T * |alpha| log2e - LSE2), dS^T = P^T o (dP^T - D)   (2 warpgroups)
//   dV  += P^T dO     (tcgen05 TS: P^T as 16-bit pairs in TMEM over the S^T columns)
//   dK  += dS^T Q     (tcgen05 TS: dS^T over the dP^T columns)
//   dQ_i = dS K       (tcgen05 SS: dS staged in shared memory, MN-major A)
// dV and dK stay in TMEM for the whole CTA; dQ_i is drained by the softmax
// warpgroups with red.global.add.v4.f32 into an fp32 workspace (the dQ-writer
// role). By default the KV tiles' dQ contributions land in
// any order (results equal the reference within rounding); with
// fa3b_bwd_params.deterministic = 1 every dQ tile takes them in ascending KV
// order behind a per-tile semaphore, the reference's order (flash_bwd.cpp:58-61),
// so reruns are bitwise identical.
#include <cuda.h>
#include <cuda_runtime.h>

#include <cmath>
#include <mutex>

#include "../../include/fa3b.h"
#include "fa3b_internal.cuh"
#include "sm100_ptx.cuh"

namespace fa3b {

// Optional phase tracing (-DFA3B_TRACE): CTA (0,0,0) records clock64() at the
// K3 phase boundaries of each Q-tile iteration; read with fa3b_debug_bwd_trace().
#ifdef FA3B_TRACE
__device__ unsigned long long g_fa3b_bwd_trace[64][16];
#define BWD_TP(it, k)                                                                      \
  do {                                                                                     \
    if (blockIdx.x == 0 && blockIdx.y == 0 && blockIdx.z == 0 && (it) < 64)               \
      g_fa3b_bwd_trace[it][k] = clock64();                                                 \
  } while (0)
// per-item timeline of CTA 0 (items < 32): [0] producer issues K/V, [1] MMA sees
// K/V, [2] MMA issues the first S, [3] MMA issues the item's last dQ, [4] epilogue
// starts (dK/dV ready), [5] epilogue done; read with fa3b_debug_bwd_items()
__device__ unsigned long long g_fa3b_bwd_items[32][8];
#define BWD_IT(itl, k)                                                                     \
  do {                                                                                     \
    if (blockIdx.x == 0 && (itl) < 32) g_fa3b_bwd_items[itl][k] = clock64();               \
  } while (0)
#else
#define BWD_IT(itl, k) \
  do {                 \
  } while (0)
#define BWD_TP(it, k) \
  do {                \
  } while (0)
#endif

namespace {

constexpr float kLog2e = 1.4426950408889634f;

__device__ __forceinline__ float load_elem(const void* p, size_t i, int dtype) {
  if (dtype == FA3B_DTYPE_BF16) return __bfloat162float(static_cast<const __nv_bfloat16*>(p)[i]);
  if (dtype == FA3B_DTYPE_F16) return __half2float(static_cast<const __half*>(p)[i]);
  return static_cast<const float*>(p)[i];
}

// One warp per row: D_i = sum_j dO_ij O_ij (fp32 accumulate), optional LSE2.
__global__ void fa3b_bwd_prep_kernel(const void* __restrict__ o, long long o_sb, long long o_ss,
                                     long long o_sh, const void* __restrict__ dout,
                                     long long d_sb, long long d_ss, long long d_sh, int dtype,
                                     int N, int H, int D, int n_out, float* __restrict__ delta,
                                     const float* __restrict__ lse, float* __restrict__ lse2) {
  const int row = blockIdx.x * (blockDim.x / 32) + (threadIdx.x >> 5);
  const int h = blockIdx.y, b = blockIdx.z;
  const int lane = threadIdx.x & 31;
  if (row >= n_out) return;
  float acc = 0.f;
  if (row < N) {
    const size_t ob = b * o_sb + static_cast<size_t>(row) * o_ss + h * o_sh;
    const size_t db = b * d_sb + static_cast<size_t>(row) * d_ss + h * d_sh;
    for (int c = lane; c < D; c += 32) acc += load_elem(dout, db + c, dtype) * load_elem(o, ob + c, dtype);
  }
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, off);
  if (lane == 0) {
    const size_t idx = (static_cast<size_t>(b) * H + h) * n_out + row;
    delta[idx] = acc;
    if (lse2 != nullptr) {
      float l = row < N ? lse[(static_cast<size_t>(b) * H + h) * N + row] : -INFINITY;
      // rows that saw no key (L = -inf) and padding rows must get P = 0
      lse2[idx] = (l == -INFINITY) ? INFINITY : l * kLog2e;
    }
  }
}

__global__ void fa3b_bwd_dq_kernel(const float* __restrict__ dq_acc, int Npad, int N, int H,
                                   int D, float alpha, void* __restrict__ dq, long long q_sb,
                                   long long q_ss, long long q_sh, int bf16) {
  // one thread per 8 consecutive elements of a row
  const int per_row = D / 8;
  const long long idx = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (idx >= static_cast<long long>(H) * N * per_row) return;
  const int b = blockIdx.y;
  const int c8 = static_cast<int>(idx % per_row);
  const long long rh = idx / per_row;
  const int row = static_cast<int>(rh % N);
  const int h = static_cast<int>(rh / N);
  const float4* src = reinterpret_cast<const float4*>(
      dq_acc + ((static_cast<size_t>(b) * H + h) * Npad + row) * D + c8 * 8);
  const float4 a = src[0], c = src[1];
  uint4 out;
  if (bf16) {
    out = make_uint4(ptx::pack_bf16(a.x * alpha, a.y * alpha), ptx::pack_bf16(a.z * alpha, a.w * alpha),
                     ptx::pack_bf16(c.x * alpha, c.y * alpha), ptx::pack_bf16(c.z * alpha, c.w * alpha));
  } else {
    out = make_uint4(ptx::pack_f16(a.x * alpha, a.y * alpha), ptx::pack_f16(a.z * alpha, a.w * alpha),
                     ptx::pack_f16(c.x * alpha, c.y * alpha), ptx::pack_f16(c.z * alpha, c.w * alpha));
  }
  *reinterpret_cast<uint4*>(static_cast<uint16_t*>(dq) + b * q_sb + static_cast<size_t>(row) * q_ss +
                            h * q_sh + c8 * 8) = out;
}

struct BwdArgs {
  int B, H, Hkv, N, Npad, group;
  float scale_log2;  // |alpha| log2e
  float alpha;
  const float* lse2;   // [B, H, Npad]
  const float* delta;  // [B, H, Npad]
  float* dq_acc;       // [B, H, Npad, D]
  int* dq_sem;         // deterministic mode: [B, H, Npad / 128] adds done per dQ tile, else null
  void* dk;
  long long dk_sb, dk_ss, dk_sh;
  void* dv;
  long long dv_sb, dv_ss, dv_sh;
  int dkv_v8;  // dK and dV rows 32-byte aligned: 256-bit stores
};

// K3 layout. Warps 0-7: two gradient warpgroups (warpgroup w owns query columns
// [64 w, 64 w + 64) of the S^T / dP^T tile; thread r owns KV row r = TMEM lane r);
// warps 8-11: the dQ-writer warpgroup; warp 12: TMA producer; warp 13: MMA issuer;
// warps 14-15 only complete warpgroup 3, which gives registers to the dQ writer
// (setmaxnreg 128 -> 96 / 128 -> 160 at d = 128) so it can release each dQ tile's
// TMEM columns right after one load of all of them.
//
// TMEM (512 columns): S^T [0,128) (P^T as 16-bit pairs over the first 32 columns of
// each warpgroup half), dP^T [128,256) (dS^T pairs likewise), dV [256, 256+D),
// dK [256+D, 256+2D). dQ_i = dS_i K (M = 128 query rows = TMEM lanes, N = D) goes
// to the dP^T columns at d = 128 (TMEM is full) and to its own columns [384, 448)
// at d = 64. The dQ writer loads it, frees the columns, and sends it to the fp32
// workspace through two 128B-swizzled 128 x 32 fp32 shared-memory boxes and TMA
// reduce-adds (cp.reduce.async.bulk.tensor ... .add), the paper's dQ-writer role
// without per-element atomics on the load/store pipe.
//
// Q_i and dO_i live in tile slots (tile 2i = Q_i, 2i+1 = dO_i): Q double-buffered,
// dO single-buffered at d = 128 (3 slots) or double-buffered at d = 64 (4 slots):
// dO_i is released after dV_i, Q_i after dK_i, which leaves room at d = 128 for
// the dQ staging boxes. LSE2_i and D_i arrive by cp.async.bulk into their own
// double buffer.
//
// Per Q tile i the MMA order is
//   dV += P_i^T dO_i | dK += dS_i^T Q_i | S_{i+1} = K Q_{i+1}^T | dQ_i | dP_{i+1} = V dO_{i+1}^T
// with the softmax split in two phases (P_i after S_i lands, dS_i after dP_i), so
// dV_i starts while dS_i is still being formed and S_{i+1} runs under dQ_i.
#ifndef FA3B_BWD_KV2
#define FA3B_BWD_KV2 0
#endif
// FA3B_BWD_EPI_DQW: the dK / dV epilogue runs on the dQ-writer warpgroup, so the
// gradient warps start the next work item at once (the MMA warp holds the next
// item's first dV / dK MMA until the columns have been read out: dkv_free)
#ifndef FA3B_BWD_EPI_DQW
#define FA3B_BWD_EPI_DQW 1
#endif
template <int D_>
struct BwdTraits {
  static constexpr int D = D_;
  static constexpr int CHUNK_BYTES = 128 * 128;
  static constexpr int TILE_BYTES = (D / 64) * CHUNK_BYTES;  // 128 rows x D 16-bit
  static constexpr bool DQ_IN_DP = (D == 128);
  // d = 128 fits three tile slots next to the dQ staging boxes; d = 64 keeps four
  // (Q and dO each double-buffered: its GEMMs are short, so load latency shows)
  static constexpr int RING = D == 64 ? 4 : 3;
  // with 3 slots the LSE2/D double buffer needs its own release (Q_{i+2} reuses
  // dO_i's slot, freed before phase B of tile i is done); with 4 it rides on Q's
  static constexpr bool VEC_OWN = RING == 3;
  static constexpr int DRAIN_WARP0 = 8;
  static constexpr int LOAD_WARP = 12;
  static constexpr int MMA_WARP = 13;
  static constexpr int NUM_THREADS = 16 * 32;
  // KVB K/V buffers: with two (FA3B_BWD_KV2, d = 64, where shared memory allows)
  // the next work item's K and V load during this item instead of after its last
  // MMA. Measured no gain at N 512-8k (r02be_kv2_ab.log): the item boundary is
  // the gradient warps' dK / dV epilogue (bwd item trace r02bd), not the load. Off.
  static constexpr int KVB = (D == 64 && FA3B_BWD_KV2) ? 2 : 1;
  static constexpr int OFF_K = 0;
  static constexpr int OFF_V = TILE_BYTES;
  static constexpr int KV_STRIDE = 2 * TILE_BYTES;  // buffer b at + b KV_STRIDE
  static constexpr int OFF_RING = KVB * 2 * TILE_BYTES;
  static constexpr int OFF_DS = OFF_RING + RING * TILE_BYTES;  // 128 kv x 128 q 16-bit
  static constexpr int OFF_STG = OFF_DS + 2 * CHUNK_BYTES;      // dQ boxes 2 x (128 x 32 fp32)
  static constexpr int OFF_VEC = OFF_STG + 2 * CHUNK_BYTES;     // LSE2[2][128], Delta[2][128]
  static constexpr int OFF_BAR = OFF_VEC + 4 * 512;
  // kv_full, ring_full[RING], ring_empty[RING], vec_full[2], vec_empty[2], s_full,
  // dp_full, pa_full, pb_full, dq_full, dq_free, dkv_full, kv_empty
  // + the second kv_full / kv_empty, + dkv_free
  static constexpr int NUM_BARS = 13 + 2 * RING + 2 * (KVB - 1) + 1;
  static constexpr int SMEM_BYTES = OFF_BAR + NUM_BARS * 8 + 16;
  static constexpr int COL_S = 0, COL_DP = 128, COL_DV = 256, COL_DK = 256 + D;
  static constexpr int COL_DQ = DQ_IN_DP ? COL_DP : 256 + 2 * D;
#ifndef FA3B_BWD_EMU64
#define FA3B_BWD_EMU64 2
#endif
#ifndef FA3B_BWD_EMU128
#define FA3B_BWD_EMU128 0
#endif
// FA3B_BWD_SPIN: the MMA warp's and the dQ writer's waits (pa/pb_full, dq_full,
// dq_free) poll without the suspend hint: they sit on the iteration's critical
// loop dK_i, dQ_i -> dQ drain -> dP_{i+1} -> phase B_{i+1}. Measured the same
// as the suspend-hint waits (r02bm_spin_ab.log): ~140 cycles per hand-off either
// way. Off.
#ifndef FA3B_BWD_SPIN
#define FA3B_BWD_SPIN 0
#endif
// FA3B_BWD_DK_SS: dK_i = dS_i^T Q_i as an SS-MMA reading dS^T from the shared
// dS tile (K-major view of the tile dQ reads MN-major) instead of a TS-MMA on
// dS^T pairs in the dP^T columns, so dQ_i can be issued first and the dQ drain
// and dP_{i+1} stop waiting behind dK_i. Measured 3-11 % slower (r02bn: the SS
// operand traffic stretches phase A from ~1400 to ~1900 cycles per tile): off
#ifndef FA3B_BWD_DK_SS
#define FA3B_BWD_DK_SS 0
#endif
#ifndef FA3B_BWD_KVPREFETCH
#define FA3B_BWD_KVPREFETCH 0
#endif
#ifndef FA3B_BWD_S_EARLY
#define FA3B_BWD_S_EARLY 1
#endif
  // exp2 pairs (of every 8) evaluated on the FMA-pipe polynomial instead of MUFU.EX2
  static constexpr int EMU = D == 64 ? FA3B_BWD_EMU64 : FA3B_BWD_EMU128;
  static_assert(SMEM_BYTES <= 232448, "shared memory budget");
};

__device__ __forceinline__ void bwait(uint64_t* bar, uint32_t parity) {
  if constexpr (FA3B_BWD_SPIN)
    ptx::mbar_wait_nosleep(bar, parity);
  else
    ptx::mbar_wait(bar, parity);
}

// Deterministic dQ: wait until `want` KV tiles have added into this dQ tile, then
// order the coming TMA reduce-adds after that observation; after issuing them,
// wait for their writes, order them before the release, and count this tile.
__device__ __forceinline__ void sem_wait(const int* sem, int want) {
  while (ptx::ld_acquire_gpu(sem) != want) ptx::nanosleep(64);
  ptx::fence_proxy_async_global();
}
__device__ __forceinline__ void sem_release(int* sem) {
  ptx::bulk_wait_group<0>();
  ptx::fence_proxy_async_global();
  ptx::red_release_add_gpu(sem, 1);
}

// TMEM column of the 16-bit P^T / dS^T pairs for K step t (16 query columns):
// warpgroup w wrote its 64 columns as 32 packed columns at offset 64 w.
__device__ __forceinline__ uint32_t pair_col(int t) { return (t >> 2) * 64 + (t & 3) * 8; }

template <int D, bool CAUSAL, bool BF16>
__global__ void __launch_bounds__(BwdTraits<D>::NUM_THREADS, 1)
    fa3b_bwd_kernel(const __grid_constant__ CUtensorMap tmQ, const __grid_constant__ CUtensorMap tmK,
                    const __grid_constant__ CUtensorMap tmV, const __grid_constant__ CUtensorMap tmdO,
                    const __grid_constant__ CUtensorMap tmDQ, const BwdArgs args,
                    const uint32_t idesc_s, const uint32_t idesc_dp, const uint32_t idesc_acc,
                    const uint32_t idesc_dq) {
  using T = BwdTraits<D>;
  extern __shared__ __align__(1024) uint8_t smem[];
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + T::OFF_BAR);
  uint64_t* kv_full = bars;
  uint64_t* ring_full = bars + 1;
  uint64_t* ring_empty = ring_full + T::RING;
  uint64_t* vec_full = ring_empty + T::RING;
  uint64_t* vec_empty = vec_full + 2;
  uint64_t* s_full = vec_empty + 2;
  uint64_t* dp_full = s_full + 1;
  uint64_t* pa_full = s_full + 2;
  uint64_t* pb_full = s_full + 3;
  uint64_t* dq_full = s_full + 4;
  uint64_t* dq_free = s_full + 5;
  uint64_t* dkv_full = s_full + 6;
  uint64_t* kv_empty = s_full + 7;  // this item's K and V tiles are consumed
  // K/V buffer b's barriers (the second pair after the others)
  auto kvf = [&](int kb) { return kb == 0 ? kv_full : kv_empty + 1; };
  auto kve = [&](int kb) { return kb == 0 ? kv_empty : kv_empty + 2; };
  uint64_t* dkv_free = kv_empty + 1 + 2 * (T::KVB - 1);  // dK / dV columns read out (EPI_DQW)
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + T::NUM_BARS);
  float* lse_s = reinterpret_cast<float*>(smem + T::OFF_VEC);  // [2][128]
  float* del_s = lse_s + 256;                                   // [2][128]

  const int warp = static_cast<int>(ptx::warp_id());
  // Persistent: CTA c walks work items (KV tile j, KV head, batch) c, c + G, ...
  // Causal KV tile j sees nq - j query tiles: items go longest-first across all
  // heads, in boustrophedon rounds so each round's heavy items spread over CTAs.
  const int N = args.N;
  const int nq = args.Npad / 128;
  const int HB = args.Hkv * args.B;
  // recomputed from the kernel parameters at each use (a register-resident copy spills)
#define num_items ((args.Npad / 128) * args.Hkv * args.B)
  auto item_of = [&](int k) {
    const int G = static_cast<int>(gridDim.x), c = static_cast<int>(blockIdx.x);
    return k * G + ((CAUSAL && (k & 1)) ? G - 1 - c : c);
  };
  struct Item {
    int j, hkv, b, i0, per_head, n_iter;
  };
  auto decode = [&](int lin) {
    Item w;
    const int hb = CAUSAL ? lin % HB : lin / nq;
    w.j = CAUSAL ? lin / HB : lin % nq;
    w.hkv = hb % args.Hkv;
    w.b = hb / args.Hkv;
    w.i0 = CAUSAL ? w.j : 0;
    w.per_head = nq - w.i0;
    w.n_iter = w.per_head * args.group;
    return w;
  };
  // ring slot and parity of tile t (t = 2i for Q_i, 2i + 1 for dO_i)
  // Fixed slots: Q_i alternates between slots 0 and 1; dO_i takes slot 2 (3-slot ring,
  // d = 128: dO_{i+1} reloads as soon as dV_i has read dO_i, a full GEMM chain before
  // dP_{i+1} needs it) or alternates between 2 and 3 (4 slots, d = 64).
  auto slot_of = [](int t) {
    const int i = t >> 1;
    return (t & 1) ? (T::RING == 3 ? 2 : 2 + (i & 1)) : (i & 1);
  };
  auto par_of = [](int t) {
    const int i = t >> 1;
    return static_cast<uint32_t>(((t & 1) && T::RING == 3) ? (i & 1) : ((i >> 1) & 1));
  };

  if (warp == T::MMA_WARP) {
    // the tile offsets above assume a 1024-byte aligned dynamic smem base
    if ((ptx::smem_u32(smem) & 1023u) != 0) __trap();
    if (ptx::lane_id() == 0) {
      ptx::mbar_init(kv_full, 1);
      for (int s = 0; s < T::RING; ++s) {
        ptx::mbar_init(&ring_full[s], 1);
        ptx::mbar_init(&ring_empty[s], 1);
      }
      for (int s = 0; s < 2; ++s) {
        ptx::mbar_init(&vec_full[s], 1);
        ptx::mbar_init(&vec_empty[s], 1);
      }
      ptx::mbar_init(s_full, 1);
      ptx::mbar_init(dp_full, 1);
      ptx::mbar_init(pa_full, 8);  // one arrival per gradient warp
      ptx::mbar_init(pb_full, 8);
      ptx::mbar_init(dq_full, 1);
      ptx::mbar_init(dq_free, 4);  // one arrival per dQ-writer warp
      ptx::mbar_init(dkv_full, 1);
      ptx::mbar_init(kv_empty, 1);
      if constexpr (T::KVB == 2) {
        ptx::mbar_init(kvf(1), 1);
        ptx::mbar_init(kve(1), 1);
      }
      ptx::mbar_init(dkv_free, 4);  // one arrival per dQ-writer warp
      ptx::fence_mbar_init();
    }
    __syncwarp();
    ptx::tmem_alloc<512>(tmem_slot);
  }
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  // each setmaxnreg dominates the code of its warpgroup's roles
  if (warp >= 12) {
    if constexpr (D == 128) ptx::setmaxnreg_dec<96>();
    if (warp == T::LOAD_WARP) {
      // ------------------------------------------------ TMA producer
      if (ptx::elect_one()) {
        ptx::prefetch_tmap(&tmQ);
        ptx::prefetch_tmap(&tmK);
        ptx::prefetch_tmap(&tmV);
        ptx::prefetch_tmap(&tmdO);
        int gi = 0;  // Q tiles (iterations) over all items: ring and vector positions
        int itl = 0;
        for (int lin = item_of(0); lin < num_items; lin = item_of(++itl)) {
          const Item w = decode(lin);
          const int kb = itl % T::KVB;
          if (itl >= T::KVB) ptx::mbar_wait(kve(kb), ((itl / T::KVB) - 1) & 1);
          BWD_IT(itl, 0);
          ptx::mbar_arrive_expect_tx(kvf(kb), 2 * T::TILE_BYTES);
          for (int c = 0; c < D / 64; ++c) {
            ptx::tma_load_4d(smem + T::OFF_K + kb * T::KV_STRIDE + c * T::CHUNK_BYTES, &tmK, kvf(kb), c * 64,
                             w.hkv, w.j * 128, w.b, ptx::kEvictFirst);
            ptx::tma_load_4d(smem + T::OFF_V + kb * T::KV_STRIDE + c * T::CHUNK_BYTES, &tmV, kvf(kb), c * 64,
                             w.hkv, w.j * 128, w.b, ptx::kEvictFirst);
          }
#if FA3B_BWD_KVPREFETCH
          // the next item's K / V into L2 now (its TMA load waits for kv_empty, this
          // item's last MMAs): measured 3-7 % slower at d 64 N <= 1k, neutral at d 128
          // (profiles/r02/r02bc_kvpf_ab.log), off
          if (const int nxt = item_of(itl + 1); nxt < num_items) {
            const Item wn = decode(nxt);
            for (int c = 0; c < D / 64; ++c) {
              ptx::tma_prefetch_4d(&tmK, c * 64, wn.hkv, wn.j * 128, wn.b);
              ptx::tma_prefetch_4d(&tmV, c * 64, wn.hkv, wn.j * 128, wn.b);
            }
          }
#endif
          for (int it = 0; it < w.n_iter; ++it, ++gi) {
            const int h = w.hkv * args.group + it / w.per_head;
            const int i = w.i0 + it % w.per_head;
            const size_t vec = (static_cast<size_t>(w.b) * args.H + h) * args.Npad + i * 128;
#pragma unroll
            for (int which = 0; which < 2; ++which) {  // Q_i then dO_i
              const int t = 2 * gi + which;
              const int s = slot_of(t);
              ptx::mbar_wait(&ring_empty[s], par_of(t) ^ 1);
              const bool vec_here = which == 0 && !T::VEC_OWN;
              ptx::mbar_arrive_expect_tx(&ring_full[s], T::TILE_BYTES + (vec_here ? 1024 : 0));
              for (int c = 0; c < D / 64; ++c)
                ptx::tma_load_4d(smem + T::OFF_RING + s * T::TILE_BYTES + c * T::CHUNK_BYTES,
                                 which ? &tmdO : &tmQ, &ring_full[s], c * 64, h, i * 128, w.b,
                                 ptx::kEvictLast);
              if (which == 0) {
                const int vs = gi & 1;
                uint64_t* vbar = &ring_full[s];
                if (T::VEC_OWN) {
                  ptx::mbar_wait(&vec_empty[vs], ((gi >> 1) & 1) ^ 1);
                  ptx::mbar_arrive_expect_tx(&vec_full[vs], 1024);
                  vbar = &vec_full[vs];
                }
                ptx::bulk_load(lse_s + vs * 128, args.lse2 + vec, 512, vbar);
                ptx::bulk_load(del_s + vs * 128, args.delta + vec, 512, vbar);
              }
            }
          }
        }
      }
    } else if (warp == T::MMA_WARP) {
      // ------------------------------------------------ MMA issuer
      if (ptx::elect_one()) {
        uint32_t k_addr = ptx::smem_u32(smem + T::OFF_K);
        uint32_t v_addr = ptx::smem_u32(smem + T::OFF_V);
        const uint32_t ds_addr = ptx::smem_u32(smem + T::OFF_DS);
        auto tile_addr = [&](int t) { return ptx::smem_u32(smem + T::OFF_RING + slot_of(t) * T::TILE_BYTES); };
        auto wait_tile = [&](int t) {
          ptx::mbar_wait(&ring_full[slot_of(t)], par_of(t));
          ptx::tc_fence_after();
        };
        // S^T = K Q^T and dP^T = V dO^T (both operands K-major, 128B swizzle)
        auto issue_s = [&](int it) {
          const uint32_t q_addr = tile_addr(2 * it);
#pragma unroll
          for (int k = 0; k < D / 16; ++k) {
            const uint32_t off = (k >> 2) * T::CHUNK_BYTES + (k & 3) * 32;
            ptx::mma_f16_ss(tmem + T::COL_S, ptx::sw128_desc(k_addr + off, 16, 1024),
                            ptx::sw128_desc(q_addr + off, 16, 1024), idesc_s, k > 0);
          }
        };
        auto issue_dp = [&](int it) {
          const uint32_t do_addr = tile_addr(2 * it + 1);
#pragma unroll
          for (int k = 0; k < D / 16; ++k) {
            const uint32_t off = (k >> 2) * T::CHUNK_BYTES + (k & 3) * 32;
            ptx::mma_f16_ss(tmem + T::COL_DP, ptx::sw128_desc(v_addr + off, 16, 1024),
                            ptx::sw128_desc(do_addr + off, 16, 1024), idesc_dp, k > 0);
          }
        };
        int gi = 0;  // global iteration (Q tile) index: ring tiles and barrier phases
        int itl = 0;
        for (int lin = item_of(0); lin < num_items; lin = item_of(++itl)) {
          const Item w = decode(lin);
          const int kb = itl % T::KVB;
          ptx::mbar_wait(kvf(kb), (itl / T::KVB) & 1);
          BWD_IT(itl, 1);
          k_addr = ptx::smem_u32(smem + T::OFF_K + kb * T::KV_STRIDE);
          v_addr = ptx::smem_u32(smem + T::OFF_V + kb * T::KV_STRIDE);
          if (T::DQ_IN_DP && gi > 0) {  // the previous item's last dQ still sits in the dP^T columns
            bwait(dq_free, (gi - 1) & 1);
          }
          wait_tile(2 * gi);
          issue_s(gi);
          BWD_IT(itl, 2);
          ptx::mma_commit(s_full);
          wait_tile(2 * gi + 1);
          issue_dp(gi);
          ptx::mma_commit(dp_full);
          for (int it = 0; it < w.n_iter; ++it) {
            const int g = gi + it;  // global iteration
            const bool more = it + 1 < w.n_iter;
            // dV += P^T dO (A = P^T pairs in TMEM, B = dO MN-major); then dO_i is free
            bwait(pa_full, g & 1);
            if (itl == 0) BWD_TP(it, 0);
            if (FA3B_BWD_EPI_DQW && it == 0 && itl > 0)  // the previous item's dK / dV read out
              ptx::mbar_wait(dkv_free, (itl - 1) & 1);
            ptx::tc_fence_after();
            const uint32_t do_addr = tile_addr(2 * g + 1);
#pragma unroll
            for (int t = 0; t < 8; ++t)
              ptx::mma_f16_ts(tmem + T::COL_DV, tmem + T::COL_S + pair_col(t),
                              ptx::sw128_desc(do_addr + t * 16 * 128, T::CHUNK_BYTES, 1024), idesc_acc,
                              (it > 0 || t > 0));
            if (T::VEC_OWN) ptx::mma_commit(&ring_empty[slot_of(2 * g + 1)]);  // dO_i free early
#if FA3B_BWD_S_EARLY
            // S_{i+1} may overwrite the S^T columns as soon as dV_i (the last reader of
            // P_i^T) is issued: phase A of tile i+1 then overlaps phase B of tile i
            if (more) {
              wait_tile(2 * g + 2);
              issue_s(g + 1);
              ptx::mma_commit(s_full);
            }
#endif
            bwait(pb_full, g & 1);
            if (itl == 0) BWD_TP(it, 1);
            ptx::tc_fence_after();
            const uint32_t q_addr = tile_addr(2 * g);
            auto issue_dk = [&]() {
#if FA3B_BWD_DK_SS
              // dK += dS^T Q, A = dS^T K-major from the shared dS tile (the one dQ reads)
#pragma unroll
              for (int t = 0; t < 8; ++t)
                ptx::mma_f16_ss(tmem + T::COL_DK,
                                ptx::sw128_desc(ds_addr + (t >> 2) * T::CHUNK_BYTES + (t & 3) * 32, 16, 1024),
                                ptx::sw128_desc(q_addr + t * 16 * 128, T::CHUNK_BYTES, 1024), idesc_acc,
                                (it > 0 || t > 0));
#else
              // dK += dS^T Q (A = dS^T pairs in TMEM, B = Q MN-major)
#pragma unroll
              for (int t = 0; t < 8; ++t)
                ptx::mma_f16_ts(tmem + T::COL_DK, tmem + T::COL_DP + pair_col(t),
                                ptx::sw128_desc(q_addr + t * 16 * 128, T::CHUNK_BYTES, 1024), idesc_acc,
                                (it > 0 || t > 0));
#endif
              // then Q_i, LSE2_i, D_i are free
              ptx::mma_commit(&ring_empty[slot_of(2 * g)]);
              if (T::VEC_OWN)
                ptx::mma_commit(&vec_empty[g & 1]);
              else
                ptx::mma_commit(&ring_empty[slot_of(2 * g + 1)]);
            };
            auto issue_dq = [&]() {
              if (!T::DQ_IN_DP && g > 0) {  // own columns: the previous dQ must have been read out
                bwait(dq_free, (g - 1) & 1);
                ptx::tc_fence_after();
              }
#pragma unroll
              for (int t = 0; t < 8; ++t) {  // dQ = dS K: 16 KV rows per step, both operands MN-major
                const uint32_t off = t * 16 * 128;
                ptx::mma_f16_ss(tmem + T::COL_DQ, ptx::sw128_desc(ds_addr + off, T::CHUNK_BYTES, 1024),
                                ptx::sw128_desc(k_addr + off, T::CHUNK_BYTES, 1024), idesc_dq, t > 0);
              }
              ptx::mma_commit(dq_full);
            };
#if FA3B_BWD_DK_SS
            // dQ_i first: its drain (and, at d = 128, the dP_{i+1} that reuses its
            // columns) then overlaps dK_i instead of following it
            issue_dq();
            issue_dk();
#else
            issue_dk();
#endif
#if !FA3B_BWD_S_EARLY
            if (more) {
              wait_tile(2 * g + 2);
              issue_s(g + 1);
              ptx::mma_commit(s_full);
            }
#endif
#if !FA3B_BWD_DK_SS
            issue_dq();
#endif
            if (more) {
              if (T::DQ_IN_DP) {  // dP_{i+1} overwrites the dQ_i columns once they are read out
                bwait(dq_free, g & 1);
                ptx::tc_fence_after();
              }
              if (itl == 0) BWD_TP(it, 2);
              wait_tile(2 * g + 3);
              issue_dp(g + 1);
              ptx::mma_commit(dp_full);
            }
          }
          BWD_IT(itl, 3);
          ptx::mma_commit(dkv_full);
          ptx::mma_commit(kve(kb));  // K and V of this item are no longer read
          gi += w.n_iter;
        }
      }
    }
  } else if (warp >= T::DRAIN_WARP0) {
    if constexpr (D == 128) ptx::setmaxnreg_inc<160>();
    // ------------------------------------------------ dQ writer (the paper's dQ-writer role)
    const int dw = warp - T::DRAIN_WARP0;  // TMEM lane quarter
    const uint32_t lane_base = static_cast<uint32_t>(32 * dw) << 16;
    const int lane = static_cast<int>(ptx::lane_id());
    const bool leader = dw == 0 && lane == 0;
    const int r = 32 * dw + lane;  // query row of the tile = TMEM lane
    constexpr int NB = D / 32;     // 128 x 32 fp32 boxes per dQ tile
    int gi = 0, itl = 0;
    for (int lin = item_of(0); lin < num_items; lin = item_of(++itl)) {
    const Item w = decode(lin);
    const int b = w.b;
    for (int it = 0; it < w.n_iter; ++it, ++gi) {
      const int h = w.hkv * args.group + it / w.per_head;
      const int i = w.i0 + it % w.per_head;
      // deterministic mode: dQ tile (b, h, i) takes the KV tiles' contributions in
      // ascending j, the reference's order (flash_bwd.cpp:58-61): KV tile j adds
      // once the semaphore shows the j tiles before it have landed
      int* sem = args.dq_sem == nullptr
                     ? nullptr
                     : args.dq_sem + (static_cast<size_t>(b) * args.H + h) * (args.Npad / 128) + i;
      bwait(dq_full, gi & 1);
      if (itl == 0 && dw == 0 && lane == 0) BWD_TP(it, 12);
      ptx::tc_fence_after();
      uint32_t v[NB][32];
#pragma unroll
      for (int c = 0; c < NB; ++c) ptx::tmem_ld32(tmem + lane_base + T::COL_DQ + c * 32, v[c]);
      ptx::tmem_wait_ld();
      ptx::tc_fence_before();
      __syncwarp();
      if (lane == 0) ptx::mbar_arrive(dq_free);
      if (itl == 0 && dw == 0 && lane == 0) BWD_TP(it, 13);
      if constexpr (D == 128) {
        // four boxes through two staging buffers: each buffer is refilled once the
        // reduce-add issued two boxes earlier has finished reading it
#pragma unroll
        for (int c = 0; c < NB; ++c) {
          if (leader && (gi > 0 || c >= 2)) ptx::bulk_wait_group_read<1>();
          ptx::named_bar_sync(3, 128);
          uint8_t* stg = smem + T::OFF_STG + (c & 1) * T::CHUNK_BYTES + r * 128;
#pragma unroll
          for (int u = 0; u < 8; ++u)
            *reinterpret_cast<uint4*>(stg + ((u ^ (r & 7)) << 4)) =
                make_uint4(v[c][4 * u], v[c][4 * u + 1], v[c][4 * u + 2], v[c][4 * u + 3]);
          ptx::fence_proxy_async_smem();
          ptx::named_bar_sync(3, 128);
          if (leader) {
            if (c == 0 && sem != nullptr) sem_wait(sem, w.j);
            ptx::tma_reduce_add_4d(&tmDQ, smem + T::OFF_STG + (c & 1) * T::CHUNK_BYTES, 32 * c, h, i * 128, b);
            ptx::bulk_commit_group();
            if (c == NB - 1 && sem != nullptr) sem_release(sem);
          }
        }
      } else {
        // both boxes at once, after the previous tile's reduce-adds have read them
        if (leader) ptx::bulk_wait_group_read<0>();
        ptx::named_bar_sync(3, 128);
#pragma unroll
        for (int c = 0; c < NB; ++c) {
          uint8_t* stg = smem + T::OFF_STG + c * T::CHUNK_BYTES + r * 128;
#pragma unroll
          for (int u = 0; u < 8; ++u)
            *reinterpret_cast<uint4*>(stg + ((u ^ (r & 7)) << 4)) =
                make_uint4(v[c][4 * u], v[c][4 * u + 1], v[c][4 * u + 2], v[c][4 * u + 3]);
        }
        ptx::fence_proxy_async_smem();
        ptx::named_bar_sync(3, 128);
        if (leader) {
          if (sem != nullptr) sem_wait(sem, w.j);
#pragma unroll
          for (int c = 0; c < NB; ++c)
            ptx::tma_reduce_add_4d(&tmDQ, smem + T::OFF_STG + c * T::CHUNK_BYTES, 32 * c, h, i * 128, b);
          ptx::bulk_commit_group();
          if (sem != nullptr) sem_release(sem);
        }
      }
    }
#if FA3B_BWD_EPI_DQW
    // dK, dV of this item: TMEM -> bf16 rows (alpha folded into dK), then dkv_free
    {
      ptx::mbar_wait(dkv_full, itl & 1);
      if (dw == 0 && lane == 0) BWD_IT(itl, 4);
      ptx::tc_fence_after();
      const int kv_row = w.j * 128 + r;
      const bool row_ok = kv_row < N;
#pragma unroll
      for (int which = 0; which < 2; ++which) {
        const float scale = which ? args.alpha : 1.f;
        uint16_t* base = static_cast<uint16_t*>(which ? args.dk : args.dv);
        const size_t off = which ? (b * args.dk_sb + static_cast<size_t>(kv_row) * args.dk_ss + w.hkv * args.dk_sh)
                                 : (b * args.dv_sb + static_cast<size_t>(kv_row) * args.dv_ss + w.hkv * args.dv_sh);
#pragma unroll
        for (int c = 0; c < D / 32; ++c) {
          uint32_t ev[32];
          ptx::tmem_ld32(tmem + lane_base + (which ? T::COL_DK : T::COL_DV) + c * 32, ev);
          ptx::tmem_wait_ld();
          if (!row_ok) continue;
          uint32_t pk2[16];
#pragma unroll
          for (int e = 0; e < 16; ++e) {
            const float a0 = __uint_as_float(ev[2 * e]) * scale, a1 = __uint_as_float(ev[2 * e + 1]) * scale;
            pk2[e] = BF16 ? ptx::pack_bf16(a0, a1) : ptx::pack_f16(a0, a1);
          }
          uint16_t* orow = base + off + c * 32;
          if (args.dkv_v8) {
            ptx::st_global_v8(orow, &pk2[0]);
            ptx::st_global_v8(orow + 16, &pk2[8]);
          } else {
            uint4* dst = reinterpret_cast<uint4*>(orow);
#pragma unroll
            for (int e = 0; e < 4; ++e) dst[e] = make_uint4(pk2[4 * e], pk2[4 * e + 1], pk2[4 * e + 2], pk2[4 * e + 3]);
          }
        }
      }
      ptx::tc_fence_before();
      __syncwarp();
      if (lane == 0) ptx::mbar_arrive(dkv_free);
      if (dw == 0 && lane == 0) BWD_IT(itl, 5);
    }
#endif
    }  // work items
    if (leader) ptx::bulk_wait_group<0>();
  } else {
    // ------------------------------------------------ 2 gradient warpgroups
    const int w = warp >> 2;          // which 64-column half of the query tile
    const int r = threadIdx.x & 127;  // KV row in the tile == TMEM lane
    const uint32_t lane_base = static_cast<uint32_t>(32 * (warp & 3)) << 16;
    const float sl2 = args.scale_log2;
    uint8_t* ds_row = smem + T::OFF_DS + w * T::CHUNK_BYTES + r * 128;
    int gi = 0, itl = 0;
    for (int lin = item_of(0); lin < num_items; lin = item_of(++itl)) {
    const Item wk = decode(lin);
    const int j = wk.j, b = wk.b, hkv = wk.hkv;
    const int kv_row = j * 128 + r;
    for (int it = 0; it < wk.n_iter; ++it, ++gi) {
      const int s = gi & 1;
      const int i = wk.i0 + it % wk.per_head;
      const float* lse_v = lse_s + s * 128 + 64 * w;
      const float* del_v = del_s + s * 128 + 64 * w;
      // phase A: P^T = exp2(S^T |alpha| log2e - LSE2) -> TMEM pairs, feeds dV
      const bool trc = itl == 0 && (warp & 3) == 0 && ptx::lane_id() == 0;
      ptx::mbar_wait(s_full, gi & 1);
      if (trc) BWD_TP(it, 4 + 4 * w);
      ptx::tc_fence_after();
      uint32_t sr[64];
      ptx::tmem_ld32(tmem + lane_base + T::COL_S + 64 * w, *reinterpret_cast<uint32_t(*)[32]>(&sr[0]));
      ptx::tmem_ld32(tmem + lane_base + T::COL_S + 64 * w + 32, *reinterpret_cast<uint32_t(*)[32]>(&sr[32]));
      // LSE2_i / D_i arrived by cp.async.bulk on their own barrier (d = 128) or on
      // Q_i's ring barrier (d = 64): wait on it here so the async-proxy writes are
      // acquired by these threads directly (not only through the MMA warp's
      // s_full commit; compute-sanitizer racecheck flagged that chain at d = 64)
      if (T::VEC_OWN)
        ptx::mbar_wait(&vec_full[s], (gi >> 1) & 1);
      else
        ptx::mbar_wait(&ring_full[slot_of(2 * gi)], par_of(2 * gi));
      ptx::tmem_wait_ld();
      const bool diag = CAUSAL && i == j;
      const int lim = kv_row - (i * 128 + 64 * w);  // causal: query column c is visible iff c >= lim
      float p[64];
      uint32_t pk[32];
      const float2 sc2 = make_float2(sl2, sl2);
#pragma unroll
      for (int c4 = 0; c4 < 16; ++c4) {
        const float4 l4 = *reinterpret_cast<const float4*>(lse_v + 4 * c4);
#pragma unroll
        for (int hp = 0; hp < 2; ++hp) {
          const int c = 4 * c4 + 2 * hp;
          const float2 x = __ffma2_rn(make_float2(__uint_as_float(sr[c]), __uint_as_float(sr[c + 1])), sc2,
                                      hp ? make_float2(-l4.z, -l4.w) : make_float2(-l4.x, -l4.y));
          float2 pp;
          if (((c >> 1) & 7) < T::EMU) {
            pp = ptx::ex2_poly2(x);
          } else {
            pp.x = ptx::ex2(x.x);
            pp.y = ptx::ex2(x.y);
          }
          if (diag) {
            pp.x = c < lim ? 0.f : pp.x;
            pp.y = c + 1 < lim ? 0.f : pp.y;
          }
          p[c] = pp.x;
          p[c + 1] = pp.y;
          pk[c >> 1] = BF16 ? ptx::pack_bf16(pp.x, pp.y) : ptx::pack_f16(pp.x, pp.y);
        }
      }
      ptx::tmem_st32(tmem + lane_base + T::COL_S + 64 * w, pk);
      ptx::tmem_wait_st();
      ptx::tc_fence_before();
      __syncwarp();
      if (ptx::lane_id() == 0) ptx::mbar_arrive(pa_full);
      if (trc) BWD_TP(it, 5 + 4 * w);
      // phase B: dS^T = P^T o (dP^T - D) -> TMEM pairs (feeds dK) and the swizzled
      // shared tile (feeds dQ), in two 32-column halves
      ptx::mbar_wait(dp_full, gi & 1);
      if (trc) BWD_TP(it, 6 + 4 * w);
      ptx::tc_fence_after();
#pragma unroll
      for (int hf = 0; hf < 2; ++hf) {
        uint32_t dpr[32];
        ptx::tmem_ld32(tmem + lane_base + T::COL_DP + 64 * w + 32 * hf, dpr);
        ptx::tmem_wait_ld();
        uint32_t dk2[16];
#pragma unroll
        for (int c4 = 0; c4 < 8; ++c4) {
          const float4 d4 = *reinterpret_cast<const float4*>(del_v + 32 * hf + 4 * c4);
          const int c = 32 * hf + 4 * c4;
          const float2 a = __fmul2_rn(make_float2(p[c], p[c + 1]),
                                      __fadd2_rn(make_float2(__uint_as_float(dpr[4 * c4]),
                                                             __uint_as_float(dpr[4 * c4 + 1])),
                                                 make_float2(-d4.x, -d4.y)));
          const float2 bq = __fmul2_rn(make_float2(p[c + 2], p[c + 3]),
                                       __fadd2_rn(make_float2(__uint_as_float(dpr[4 * c4 + 2]),
                                                              __uint_as_float(dpr[4 * c4 + 3])),
                                                  make_float2(-d4.z, -d4.w)));
          dk2[2 * c4] = BF16 ? ptx::pack_bf16(a.x, a.y) : ptx::pack_f16(a.x, a.y);
          dk2[2 * c4 + 1] = BF16 ? ptx::pack_bf16(bq.x, bq.y) : ptx::pack_f16(bq.x, bq.y);
        }
        if constexpr (!FA3B_BWD_DK_SS)  // dK reads dS^T from TMEM (else from the shared tile)
          ptx::tmem_st16(tmem + lane_base + T::COL_DP + 64 * w + 16 * hf, dk2);
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const int uu = 4 * hf + u;
          *reinterpret_cast<uint4*>(ds_row + ((uu ^ (r & 7)) << 4)) =
              make_uint4(dk2[4 * u], dk2[4 * u + 1], dk2[4 * u + 2], dk2[4 * u + 3]);
        }
      }
      ptx::fence_proxy_async_smem();
      ptx::tmem_wait_st();
      ptx::tc_fence_before();
      __syncwarp();
      if (ptx::lane_id() == 0) ptx::mbar_arrive(pb_full);
      if (trc) BWD_TP(it, 7 + 4 * w);
    }
    // ------------------------------------------------ epilogue: dK, dV
    if constexpr (!FA3B_BWD_EPI_DQW) {
    ptx::mbar_wait(dkv_full, itl & 1);
    if (threadIdx.x == 0) BWD_IT(itl, 4);
    ptx::tc_fence_after();
    const bool row_ok = kv_row < N;
#pragma unroll
    for (int which = 0; which < 2; ++which) {
      const uint32_t col = (which ? T::COL_DK : T::COL_DV) + w * (D / 2);
      const float scale = which ? args.alpha : 1.f;
      uint16_t* base = static_cast<uint16_t*>(which ? args.dk : args.dv);
      const size_t off = which ? (b * args.dk_sb + static_cast<size_t>(kv_row) * args.dk_ss + hkv * args.dk_sh)
                               : (b * args.dv_sb + static_cast<size_t>(kv_row) * args.dv_ss + hkv * args.dv_sh);
#pragma unroll
      for (int c = 0; c < D / 64; ++c) {
        uint32_t v[32];
        ptx::tmem_ld32(tmem + lane_base + col + c * 32, v);
        ptx::tmem_wait_ld();
        if (!row_ok) continue;
        uint32_t pk2[16];
#pragma unroll
        for (int e = 0; e < 16; ++e) {
          const float a0 = __uint_as_float(v[2 * e]) * scale, a1 = __uint_as_float(v[2 * e + 1]) * scale;
          pk2[e] = BF16 ? ptx::pack_bf16(a0, a1) : ptx::pack_f16(a0, a1);
        }
        uint16_t* orow = base + off + w * (D / 2) + c * 32;
        if (args.dkv_v8) {
          ptx::st_global_v8(orow, &pk2[0]);
          ptx::st_global_v8(orow + 16, &pk2[8]);
        } else {
          uint4* dst = reinterpret_cast<uint4*>(orow);
#pragma unroll
          for (int e = 0; e < 4; ++e) dst[e] = make_uint4(pk2[4 * e], pk2[4 * e + 1], pk2[4 * e + 2], pk2[4 * e + 3]);
        }
      }
    }
    if (threadIdx.x == 0) BWD_IT(itl, 5);
    }  // !FA3B_BWD_EPI_DQW
    }  // work items
  }

  ptx::tc_fence_before();
  __syncthreads();
  if (warp == T::MMA_WARP) {
    ptx::tc_fence_after();
    ptx::tmem_dealloc<512>(tmem);
  }
}
#undef num_items

size_t align256(size_t x) { return (x + 255) & ~static_cast<size_t>(255); }

// dQaccum fp32 [B, H, Npad, D] | dQ semaphores int32 [B, H, Npad / 128] (zeroed with
// dQaccum by one memset) | LSE2 [B, H, Npad] | D [B, H, Npad]
struct Workspace {
  float* dq_acc;
  int* dq_sem;
  float* lse2;
  float* delta;
  size_t zero_bytes;  // dQaccum + semaphores
  size_t bytes;
};

Workspace carve(void* base, int B, int H, int Npad, int D) {
  Workspace w{};
  const size_t dq = align256(static_cast<size_t>(B) * H * Npad * D * 4);
  const size_t sem = align256(static_cast<size_t>(B) * H * (Npad / 128) * 4);
  const size_t vec = align256(static_cast<size_t>(B) * H * Npad * 4);
  uint8_t* p = static_cast<uint8_t*>(base);
  w.dq_acc = reinterpret_cast<float*>(p);
  w.dq_sem = reinterpret_cast<int*>(p + dq);
  w.lse2 = reinterpret_cast<float*>(p + dq + sem);
  w.delta = reinterpret_cast<float*>(p + dq + sem + vec);
  w.zero_bytes = dq + sem;
  w.bytes = dq + sem + 2 * vec;
  return w;
}

template <int D, bool CAUSAL, bool BF16>
int launch_bwd_main(const fa3b_bwd_params& p, const Workspace& ws, int Npad, cudaStream_t st) {
  using Tr = BwdTraits<D>;
  auto kern = fa3b_bwd_kernel<D, CAUSAL, BF16>;
  int rc = ensure_smem_attr(reinterpret_cast<const void*>(kern), Tr::SMEM_BYTES);
  if (rc != FA3B_OK) return rc;
  CUtensorMap tq, tk, tv, tdo;
  if ((rc = make_tmap_4d(&tq, p.q, 2, D, p.heads_q, p.seqlen, p.batch, 64, 128)) != FA3B_OK) return rc;
  if ((rc = make_tmap_4d(&tk, p.k, 2, D, p.heads_kv, p.seqlen, p.batch, 64, 128)) != FA3B_OK) return rc;
  if ((rc = make_tmap_4d(&tv, p.v, 2, D, p.heads_kv, p.seqlen, p.batch, 64, 128)) != FA3B_OK) return rc;
  if ((rc = make_tmap_4d(&tdo, p.dout, 2, D, p.heads_q, p.seqlen, p.batch, 64, 128)) != FA3B_OK) return rc;
  // dQaccum [B, H, Npad, D] fp32 as a 4-D map with 128 x 32-float (128 B, swizzled) boxes
  const fa3b_tensor4 acc{ws.dq_acc, static_cast<int64_t>(p.heads_q) * Npad * D, D, static_cast<int64_t>(Npad) * D};
  CUtensorMap tdq;
  if ((rc = make_tmap_4d(&tdq, acc, 4, D, p.heads_q, Npad, p.batch, 32, 128)) != FA3B_OK) return rc;
  BwdArgs a;
  a.B = p.batch;
  a.H = p.heads_q;
  a.Hkv = p.heads_kv;
  a.N = p.seqlen;
  a.Npad = Npad;
  a.group = p.heads_q / p.heads_kv;
  a.scale_log2 = static_cast<float>(std::fabs(p.alpha) * 1.4426950408889634);
  a.alpha = static_cast<float>(p.alpha);
  a.lse2 = ws.lse2;
  a.delta = ws.delta;
  a.dq_acc = ws.dq_acc;
  a.dq_sem = p.deterministic ? ws.dq_sem : nullptr;
  a.dk = p.dk.ptr;
  a.dk_sb = p.dk.stride_batch;
  a.dk_ss = p.dk.stride_seq;
  a.dk_sh = p.dk.stride_head;
  a.dv = p.dv.ptr;
  a.dv_sb = p.dv.stride_batch;
  a.dv_ss = p.dv.stride_seq;
  a.dv_sh = p.dv.stride_head;
  {
    auto ok32 = [&](const fa3b_tensor4& t) {
      auto st = [](long long x, int extent) { return extent <= 1 || x % 16 == 0; };
      return (reinterpret_cast<uintptr_t>(t.ptr) & 31u) == 0 && st(t.stride_batch, p.batch) &&
             st(t.stride_seq, p.seqlen) && st(t.stride_head, p.heads_kv);
    };
    a.dkv_v8 = ok32(p.dk) && ok32(p.dv);
  }
  const uint32_t fmt = BF16 ? 1u : 0u;
  const uint32_t idesc_s = ptx::make_idesc(128, 128, fmt, fmt, false, false, p.alpha < 0);
  const uint32_t idesc_dp = ptx::make_idesc(128, 128, fmt, fmt, false, false, false);
  const uint32_t idesc_acc = ptx::make_idesc(128, D, fmt, fmt, false, true, false);
  // dQ = dS K (M = 128 query rows, N = D), both operands MN-major
  const uint32_t idesc_dq = ptx::make_idesc(128, D, fmt, fmt, true, true, false);
  // persistent: one CTA per SM over (KV tile, KV head, batch) work items
  const long long items = static_cast<long long>(Npad / 128) * p.heads_kv * p.batch;
  const int grid = static_cast<int>(items < num_sms() ? items : num_sms());
  kern<<<grid, Tr::NUM_THREADS, Tr::SMEM_BYTES, st>>>(tq, tk, tv, tdo, tdq, a, idesc_s, idesc_dp, idesc_acc,
                                                      idesc_dq);
  cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? FA3B_OK : cuda_fail(e);
}

template <int D>
int launch_bwd_main_dt(const fa3b_bwd_params& p, const Workspace& ws, int Npad, cudaStream_t st) {
  const bool bf16 = p.dtype == FA3B_DTYPE_BF16;
  if (p.causal) return bf16 ? launch_bwd_main<D, true, true>(p, ws, Npad, st) : launch_bwd_main<D, true, false>(p, ws, Npad, st);
  return bf16 ? launch_bwd_main<D, false, true>(p, ws, Npad, st) : launch_bwd_main<D, false, false>(p, ws, Npad, st);
}

int launch_prep(const fa3b_tensor4& o, const fa3b_tensor4& dout, int dtype, int B, int H, int N, int D,
                int n_out, float* delta, const float* lse, float* lse2, cudaStream_t st) {
  dim3 grid((n_out + 7) / 8, H, B);
  fa3b_bwd_prep_kernel<<<grid, 256, 0, st>>>(o.ptr, o.stride_batch, o.stride_seq, o.stride_head, dout.ptr,
                                            dout.stride_batch, dout.stride_seq, dout.stride_head, dtype, N,
                                            H, D, n_out, delta, lse, lse2);
  cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? FA3B_OK : cuda_fail(e);
}

}  // namespace
}  // namespace fa3b

using namespace fa3b;

extern "C" {

#ifdef FA3B_TRACE
__attribute__((visibility("default"))) int fa3b_debug_bwd_trace(unsigned long long* out, int n) {
  const size_t bytes = sizeof(unsigned long long) * static_cast<size_t>(n);
  return cudaMemcpyFromSymbol(out, g_fa3b_bwd_trace, bytes) == cudaSuccess ? 0 : -1;
}
__attribute__((visibility("default"))) int fa3b_debug_bwd_items(unsigned long long* out, int n) {
  const size_t bytes = sizeof(unsigned long long) * static_cast<size_t>(n);
  return cudaMemcpyFromSymbol(out, g_fa3b_bwd_items, bytes) == cudaSuccess ? 0 : -1;
}
#endif

size_t fa3b_bwd_workspace_bytes(int32_t batch, int32_t heads_q, int32_t heads_kv, int32_t seqlen,
                                int32_t head_dim) {
  (void)heads_kv;
  if (batch <= 0 || heads_q <= 0 || seqlen <= 0 || head_dim <= 0) return 0;
  const int Npad = (seqlen + 127) / 128 * 128;
  return carve(nullptr, batch, heads_q, Npad, head_dim).bytes;
}

int fa3b_bwd_preprocess(const fa3b_bwd_preprocess_params* pp) {
  g_last_launch_count = 0;
  if (pp == nullptr) return FA3B_ERR_NULL;
  if (pp->struct_size != sizeof(fa3b_bwd_preprocess_params)) return FA3B_ERR_STRUCT;
  const auto& p = *pp;
  if (p.batch <= 0 || p.heads <= 0 || p.seqlen <= 0 || p.head_dim <= 0) return FA3B_ERR_EMPTY;
  if (!p.o.ptr || !p.dout.ptr || !p.delta) return FA3B_ERR_NULL;
  if (p.dtype != FA3B_DTYPE_BF16 && p.dtype != FA3B_DTYPE_F16 && p.dtype != FA3B_DTYPE_F32)
    return FA3B_ERR_DTYPE;
  int rc = check_device();
  if (rc != FA3B_OK) return rc;
  rc = launch_prep(p.o, p.dout, p.dtype, p.batch, p.heads, p.seqlen, p.head_dim, p.seqlen, p.delta,
                       nullptr, nullptr, static_cast<cudaStream_t>(p.stream));
  if (rc == FA3B_OK) g_last_launch_count = 1;
  return rc;
}

int fa3b_bwd(const fa3b_bwd_params* pp) {
  g_last_launch_count = 0;
  if (pp == nullptr) return FA3B_ERR_NULL;
  if (pp->struct_size != sizeof(fa3b_bwd_params)) return FA3B_ERR_STRUCT;
  const auto& p = *pp;
  int rc = validate_problem(p.batch, p.heads_q, p.heads_kv, p.seqlen, p.head_dim, p.alpha);
  if (rc != FA3B_OK) return rc;
  if (p.head_dim == 256) return FA3B_ERR_HEAD_DIM;  // dK + dV alone fill TMEM
  if (p.dtype != FA3B_DTYPE_BF16 && p.dtype != FA3B_DTYPE_F16) return FA3B_ERR_DTYPE;
  if (!p.q.ptr || !p.k.ptr || !p.v.ptr || !p.o.ptr || !p.dout.ptr || !p.dq.ptr || !p.dk.ptr ||
      !p.dv.ptr || !p.lse)
    return FA3B_ERR_NULL;
  const int B = p.batch, H = p.heads_q, Hkv = p.heads_kv, N = p.seqlen, D = p.head_dim;
  if (!strides_ok(p.q, 2, B, N, H) || !strides_ok(p.k, 2, B, N, Hkv) || !strides_ok(p.v, 2, B, N, Hkv) ||
      !strides_ok(p.o, 2, B, N, H) || !strides_ok(p.dout, 2, B, N, H) || !strides_ok(p.dq, 2, B, N, H) ||
      !strides_ok(p.dk, 2, B, N, Hkv) || !strides_ok(p.dv, 2, B, N, Hkv))
    return FA3B_ERR_ALIGNMENT;
  const int Npad = (N + 127) / 128 * 128;
  const Workspace ws = carve(p.workspace, B, H, Npad, D);
  if (p.workspace == nullptr || p.workspace_bytes < ws.bytes || !aligned16(p.workspace))
    return FA3B_ERR_WORKSPACE;
  if ((rc = check_device()) != FA3B_OK) return rc;
  cudaStream_t st = static_cast<cudaStream_t>(p.stream);
  if (p.deterministic != 0 && p.deterministic != 1) return FA3B_ERR_DTYPE;
  cudaError_t e = cudaMemsetAsync(ws.dq_acc, 0, p.deterministic ? ws.zero_bytes : static_cast<size_t>(B) * H * Npad * D * 4, st);
  if (e != cudaSuccess) return cuda_fail(e);
  if ((rc = launch_prep(p.o, p.dout, p.dtype, B, H, N, D, Npad, ws.delta, p.lse, ws.lse2, st)) != FA3B_OK)
    return rc;
  rc = D == 64 ? launch_bwd_main_dt<64>(p, ws, Npad, st) : launch_bwd_main_dt<128>(p, ws, Npad, st);
  if (rc != FA3B_OK) return rc;
  const long long per_b = static_cast<long long>(H) * N * (D / 8);
  dim3 grid(static_cast<unsigned>((per_b + 255) / 256), B);
  fa3b_bwd_dq_kernel<<<grid, 256, 0, st>>>(ws.dq_acc, Npad, N, H, D, static_cast<float>(p.alpha), p.dq.ptr,
                                           p.dq.stride_batch, p.dq.stride_seq, p.dq.stride_head,
                                           p.dtype == FA3B_DTYPE_BF16);
  e = cudaGetLastError();
  if (e != cudaSuccess) return cuda_fail(e);
  g_last_launch_count = 4;  // memset + prep + main + dq convert
  return FA3B_OK;
}

}  // extern "C"
